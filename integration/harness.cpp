// extern "C" harness of the drop-in build (reference driver + B200 KktContext).
#define NCL_HARNESS_PREFIX drop_
#include "harness_impl.hpp"
