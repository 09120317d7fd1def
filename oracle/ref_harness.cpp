// TEST INFRASTRUCTURE ONLY: extern "C" harness of the reference library
// compiled unmodified from /root/reference/proj/src (see harness_impl.hpp).
#define NCL_HARNESS_PREFIX ref_
#include "../integration/harness_impl.hpp"
