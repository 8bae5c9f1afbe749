// common.cuh -- shared helpers for the B200 tilekit kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include <string>

#include "tk_b200.h"

namespace tkb {

// ---------------------------------------------------------------------------
// Error plumbing (host).  Every C-ABI entry point converts a tkb::Failure into
// a status code + thread-local message.
// ---------------------------------------------------------------------------
struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure{code, msg}; }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define TKB_CUDA(x) ::tkb::cuda_check((x), #x)

// Checked builds (`make checked` -> libtilekit_b200_checked.so, built with
// -DTKB_CHECKED=1): device-side invariants of the hand-written indexing --
// shared-memory layout, staging / TMEM / tail / split slots, gather and pad
// source ranges -- as the stand-in for compute-sanitizer, which this GPU
// pool does not allow.  A violated check prints its site and traps, so the
// launch fails and the C ABI reports TK_ERR_CUDA.  Free in release builds.
#ifndef TKB_CHECKED
#define TKB_CHECKED 0
#endif
#if TKB_CHECKED
#define TKB_DCHECK(cond)                                                                   \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      printf("TKB_DCHECK failed: %s (%s:%d, block %d thread %d)\n", #cond, __FILE__,      \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                 \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define TKB_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// Counts kernel launches (tk_launch_count); bumped by every launcher.
void note_launch(int n = 1);

inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
#if defined(__CUDACC__)

// Exact FP32 multiply-accumulate of the reference: one rounding for the
// product, one for the sum, never contracted into FFMA.
__device__ __forceinline__ float mac_exact(float acc, float a, float b) {
  return __fadd_rn(acc, __fmul_rn(a, b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill: copies `bytes` (0 => all zeros) of `size` bytes.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const int src = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const int src = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const int src = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
               "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  // wait_group needs an immediate; the pipelines here use at most 3 stages.
  if (n <= 0) cp_async_wait<0>();
  else if (n == 1) cp_async_wait<1>();
  else cp_async_wait<2>();
}

#endif  // __CUDACC__

}  // namespace tkb
