// Storage layout shared by host (symbolic.cpp) and device code.
#pragma once

#ifdef __CUDACC__
#define NCLB_HD __host__ __device__
#else
#define NCLB_HD
#endif

namespace nclb {

// Leading dimension of a wide front (f x f column-major in the L buffer):
// rounded up to even so that every column starts on a 16-byte boundary and
// blocks can be staged into shared memory with 16-byte cp.async copies.
NCLB_HD inline int wide_ld(int f) { return (f + 1) & ~1; }

}  // namespace nclb
