// Host cost of one C-ABI GEMM call (SGEMM 1024^3 nn, device buffers):
// wall time per call over many back-to-back calls vs. an empty-kernel
// launch, and the split of the C-ABI call into its host stages is read
// from the difference.  nvcc -O2 -o host_call_probe host_call_probe.cu
//   -I../../include -L../../paper_1904_05347_b200 -ltilekit_b200
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
#include "tk_b200.h"

__global__ void empty_kernel() {}

int main() {
  const size_t n = 1024;
  float *a, *b, *c;
  cudaMalloc(&a, n * n * 4);
  cudaMalloc(&b, n * n * 4);
  cudaMalloc(&c, n * n * 4);
  cudaMemset(a, 0, n * n * 4);
  cudaMemset(b, 0, n * n * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  tk_gemm_shape s{n, n, n, 1.0f, 0.0f, 0, 0};
  for (int prec : {TK_PREC_TF32, TK_PREC_BF16, TK_PREC_FP32_EXACT}) {
    tk_exec_options o{};
    o.precision = prec;
    for (int i = 0; i < 20; ++i) tk_gemm_dev(&s, nullptr, &o, a, b, nullptr, c, st);
    cudaStreamSynchronize(st);
    const int reps = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i)
      if (tk_gemm_dev(&s, nullptr, &o, a, b, nullptr, c, st) != 0) { std::printf("err %s\n", tk_last_error()); return 1; }
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::steady_clock::now();
    std::printf("precision %d: host %.2f us/call (enqueue), %.2f us/call incl. drain\n", prec,
                std::chrono::duration<double, std::micro>(t1 - t0).count() / reps,
                std::chrono::duration<double, std::micro>(t2 - t0).count() / reps);
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 2000; ++i) empty_kernel<<<1, 32, 0, st>>>();
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  std::printf("empty kernel launch: %.2f us/call\n",
              std::chrono::duration<double, std::micro>(t1 - t0).count() / 2000);
  return 0;
}
