// launch_cache.cuh -- host-side caches that keep per-call launch overhead
// off the device timeline: kernel attributes and the dynamic shared-memory
// opt-in (once per kernel and device), and stream-ordered scratch arenas
// (once per stream and slot, grown on demand) instead of a
// cudaMallocAsync / cudaFreeAsync pair on every call.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace tkb {

// cudaFuncGetAttributes of `fn` on the current device, cached.
const cudaFuncAttributes& func_attrs(const void* fn);
// Raise fn's dynamic shared-memory limit to at least `smem` bytes (a no-op
// once it is there).
void func_smem(const void* fn, size_t smem);

// Scratch slots (one arena per stream and slot).
enum ScratchSlot : int {
  kScratchConvWs = 0,  // conv workspace when the caller passes none
  kScratchTail = 1,    // stream-K tail partials of a GEMM
  kScratchPackA = 2,   // packed / converted GEMM operands
  kScratchPackB = 3,
  kScratchSplitA = 4,  // 3xTF32 operand triples
  kScratchSplitB = 5,
  kScratchPart = 6,    // split-K partial outputs of a GEMM
  kScratchSlots = 7
};
// `bytes` of device memory usable in stream order on `st` until the next
// request of the same (stream, slot).  While `st` is being captured into a
// CUDA graph the arena is not touched: the request is served by a graph
// allocation (cudaMallocAsync) that the returned guard frees in stream order.
class Scratch {
 public:
  Scratch(cudaStream_t st, int slot, size_t bytes);
  ~Scratch();
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  void* get() const { return p_; }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void* p_ = nullptr;
  cudaStream_t st_ = nullptr;
  bool owned_ = false;
};

}  // namespace tkb
