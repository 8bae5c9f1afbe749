// Throughput of scalar FP32 add/mul vs the packed f32x2 forms (sm_100a):
// does add.rn.f32x2 / mul.rn.f32x2 issue two IEEE-rn FP32 ops per lane per
// instruction slot?  (The exact SIMT path is FMUL+FADD issue-bound.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f32x2_probe f32x2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kAcc = 8;

__global__ void scalar_mac(float* out, float a, float b) {
  float acc[kAcc];
  for (int i = 0; i < kAcc; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) acc[i] = __fadd_rn(acc[i], __fmul_rn(acc[i], a));
  }
  float s = 0;
  for (int i = 0; i < kAcc; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}

__global__ void packed_mac(float* out, float a, float b, float one_f, float nz_f) {
  unsigned long long acc[kAcc];
  for (int i = 0; i < kAcc; ++i) acc[i] = pk(threadIdx.x * 1e-3f + i, i + 0.5f);
  const unsigned long long aa = pk(a, a);
  // runtime 1.0 / -0.0: ptxas cannot see through them, so the two
  // single-rounding FMAs stay separate (no contraction into one FFMA2)
  const unsigned long long nz = pk(nz_f, nz_f), one = pk(one_f, one_f);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kAcc; ++i) {
      unsigned long long prod;
      // exact product: a*b + (-0) rounds once, as mul.rn
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(prod) : "l"(acc[i]), "l"(aa), "l"(nz));
      // exact sum: x*1 + y rounds once, as add.rn
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc[i]) : "l"(prod), "l"(one), "l"(acc[i]));
    }
  }
  float s = 0;
  for (int i = 0; i < kAcc; ++i) {
    float x, y;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(acc[i]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 16 * 256 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int k = 0; k < 2; ++k) {
      cudaEventRecord(e0);
      if (k == 0) scalar_mac<<<148 * 16, 256>>>(out, 0.999f, 1.0f);
      else packed_mac<<<148 * 16, 256>>>(out, 0.999f, 1.0f, 1.0f, -0.0f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 148.0 * 16 * 256 * kIters * kAcc * 2 * (k == 0 ? 1 : 2);  // fp32 ops
      printf("%s: %.3f ms, %.1f T fp32-op/s (mul+add, ieee rn)\n", k == 0 ? "scalar FMUL+FADD" : "packed f32x2  ",
             ms, ops / ms / 1e9);
    }
  }
  return 0;
}
