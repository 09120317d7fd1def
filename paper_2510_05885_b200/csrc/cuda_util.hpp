// Host-side CUDA helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ncl_b200.h"

namespace nclb {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string& last_error();  // thread-local message behind ncl_last_error()

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess)                                                      \
      throw ::nclb::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t k) {
    if (p) cudaFree(p);
    p = nullptr;
    n = k;
    if (k) CK(cudaMalloc(&p, k * sizeof(T)));
  }
  void upload(const std::vector<T>& v) {
    alloc(v.size());
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  void zero(cudaStream_t st) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), st));
  }
};

// Runs f once per current device for one call site (kernel attributes such as
// the dynamic shared-memory opt-in are set per device); safe when contexts are
// created from several threads at once.
struct PerDeviceOnce {
  std::mutex mu;
  std::atomic<unsigned long long> done{0};  // bit d: device d
  template <class F>
  void operator()(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    std::lock_guard<std::mutex> g(mu);
    if (done.load(std::memory_order_relaxed) & bit) return;
    f();
    done.fetch_or(bit, std::memory_order_release);
  }
};

// exception -> C-ABI return code (include/ncl_b200.h)
template <class F>
int guard(F&& f) {
  try {
    f();
    return NCL_OK;
  } catch (const std::invalid_argument& e) {
    last_error() = e.what();
    return NCL_EINVAL;
  } catch (const CudaError& e) {
    last_error() = e.what();
    return NCL_ECUDA;
  } catch (const std::logic_error& e) {
    last_error() = e.what();
    return NCL_ELOGIC;
  } catch (const std::bad_alloc&) {
    last_error() = "out of memory";
    return NCL_ENOMEM;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return NCL_ECUDA;
  }
}

}  // namespace nclb
