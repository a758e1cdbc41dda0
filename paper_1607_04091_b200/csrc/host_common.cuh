// host_common.cuh -- host-side plumbing shared by the library's translation
// units: error classes (include/gs_b200.h codes), CUDA checks, device
// buffers, the launch counter / per-kernel profiler and the C-ABI guard.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <functional>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gs_b200.h"

namespace gsb {

inline thread_local std::string g_err;  // gs_last_error()

struct GsError {
  int code;
  std::string msg;
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw GsError{code, m}; }

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) ::gsb::fail(GS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define CKL()                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess) ::gsb::fail(GS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
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
  void alloc(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (count == 0) return;
    CK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void upload(const T* h, size_t count, cudaStream_t st) {
    alloc(count);
    if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st));
  }
  size_t bytes() const { return n * sizeof(T); }
};

inline int ilog2(long long v) {
  int l = 0;
  while ((1LL << l) < v) ++l;
  return l;
}
inline bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }
inline unsigned nblk(long long n, int t) { return (unsigned)((n + t - 1) / t); }

// When armed by gs_profile_pair, every launch is followed by an event on the
// launching stream; consecutive events bracket exactly one kernel.
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<std::string> names;
};
inline Prof g_prof;
inline std::atomic<long long> g_launches{0};  // kernels this library has launched (gs_launch_count)

inline void pmark(const char* name, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof.on) return;
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  CK(cudaEventRecord(e, st));
  g_prof.ev.push_back(e);
  g_prof.names.push_back(name);
}

inline bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

inline int guard_call(const std::function<void()>& f) {
  try {
    f();
    return GS_OK;
  } catch (const GsError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return GS_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GS_ERR_CUDA;
  }
}

}  // namespace gsb
