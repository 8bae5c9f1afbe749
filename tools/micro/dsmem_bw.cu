// DSMEM bandwidth between the two CTAs of a cluster (B200): CTA 1 moves a
// buffer into CTA 0's shared memory (a) with one cp.async.bulk
// shared::cta -> shared::cluster copy completing on CTA 0's mbarrier, (b)
// with st.shared::cluster.v4 from 128 threads; CTA 0 times arrival with
// clock64.  Many clusters run at once (all SMs busy) or one alone.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o dsmem_bw dsmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned; barrier.cluster.wait.aligned;" ::: "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) dsmem_kernel(int bytes, long long* out) {
  extern __shared__ __align__(1024) uint8_t buf[];
  __shared__ uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(MODE == 0 ? 1 : 128));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x * 16; i < bytes; i += 128 * 16) *reinterpret_cast<float4*>(buf + i) = make_float4(rank, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cluster_sync();
  long long t0 = clock64();
  if (rank == 0) {
    if (MODE == 0 && threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
  }
  cluster_sync();  // expect_tx posted before the copy starts
  t0 = clock64();
  if (rank == 1) {
    const uint32_t dst = mapa(smem_u32(buf), 0), rb = mapa(smem_u32(&bar), 0);
    if (MODE == 0) {
      if (threadIdx.x == 0)
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "r"(smem_u32(buf)), "r"(bytes), "r"(rb) : "memory");
    } else {
      for (int i = threadIdx.x * 16; i < bytes; i += 128 * 16) {
        float4 v = *reinterpret_cast<float4*>(buf + i);
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + i), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
      }
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
    }
  } else {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
    if (threadIdx.x == 0) out[blockIdx.x / 2] = clock64() - t0;
  }
  cluster_sync();
}

int main() {
  long long* d;
  cudaMalloc(&d, 1024 * 8);
  long long h[1024];
  for (int mode = 0; mode < 2; ++mode) {
    for (int bytes : {16384, 65536, 131072}) {
      for (int clusters : {1, 74}) {
        auto k = mode == 0 ? dsmem_kernel<0> : dsmem_kernel<1>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        for (int rep = 0; rep < 3; ++rep) k<<<2 * clusters, 128, bytes>>>(bytes, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { std::printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, clusters * 8, cudaMemcpyDeviceToHost);
        long long mx = 0, sum = 0;
        for (int i = 0; i < clusters; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
        std::printf("%s %6d B, %2d clusters: mean %7.0f clk (%.1f B/clk), max %lld clk\n",
                    mode == 0 ? "bulk copy    " : "st.cluster.v4", bytes, clusters,
                    (double)sum / clusters, bytes / ((double)sum / clusters), mx);
      }
    }
  }
  return 0;
}
