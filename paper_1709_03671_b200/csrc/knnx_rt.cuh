// Error plumbing shared by the C-ABI translation units (runtime.cu, comm.cu):
// every entry point runs its body in guard(), which maps knnx::error (the
// reference's errc), CUDA failures and bad_alloc to the integer status of
// include/knnx.h and records the message for knnx_last_error().
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "knnx_internal.cuh"

namespace knnx_rt {

inline thread_local std::string g_last_error;

inline int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

struct CudaError {
  cudaError_t err;
  const char* what;
};

inline void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError{e, what};
}

template <typename Fn>
int guard(Fn&& fn) {
  try {
    return fn();
  } catch (const knnx::error& e) {
    return fail(1 + static_cast<int>(e.code()), e.what());
  } catch (const CudaError& e) {
    return fail(KNNX_ERR_CUDA, std::string("CudaError: ") + e.what + ": " + cudaGetErrorString(e.err));
  } catch (const std::bad_alloc&) {
    return fail(1 + static_cast<int>(knnx::errc::too_large), "TooLarge: host allocation failed");
  } catch (const std::exception& e) {
    return fail(1 + static_cast<int>(knnx::errc::invalid_argument), e.what());
  }
}

inline void require(bool cond, knnx::errc code, const std::string& msg) {
  if (!cond) throw knnx::error(code, msg);
}
// literal messages: no std::string is built unless the check fails (some
// checks run once per matrix entry)
inline void require(bool cond, knnx::errc code, const char* msg) {
  if (!cond) throw knnx::error(code, msg);
}

inline void launched(knnx_ctx_t ctx, const char* what, int n = 1) {
  check(cudaGetLastError(), what);
  ctx->launches += n;
}

// Makes ctx's device current for the duration of an entry point and restores
// the caller's device afterwards (several contexts may live in one process).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != device) check(cudaSetDevice(device), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace knnx_rt
