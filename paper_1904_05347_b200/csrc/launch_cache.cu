// launch_cache.cu -- see launch_cache.cuh.
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "launch_cache.cuh"

namespace tkb {

namespace {
std::mutex g_mu;

int current_device() {
  int dev = 0;
  TKB_CUDA(cudaGetDevice(&dev));
  return dev;
}

struct FuncInfo {
  cudaFuncAttributes attr{};
  size_t smem_set = 0;
};

FuncInfo& func_info(const void* fn, int dev) {
  static std::map<std::pair<const void*, int>, FuncInfo> infos;
  auto it = infos.find({fn, dev});
  if (it == infos.end()) {
    FuncInfo fi;
    TKB_CUDA(cudaFuncGetAttributes(&fi.attr, fn));
    it = infos.emplace(std::make_pair(fn, dev), fi).first;
  }
  return it->second;
}

struct Arena {
  void* p = nullptr;
  size_t bytes = 0;
};
}  // namespace

const cudaFuncAttributes& func_attrs(const void* fn) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  return func_info(fn, dev).attr;
}

void func_smem(const void* fn, size_t smem) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  FuncInfo& fi = func_info(fn, dev);
  if (smem > fi.smem_set) {
    TKB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fi.smem_set = smem;
  }
}

Scratch::Scratch(cudaStream_t st, int slot, size_t bytes) : st_(st) {
  if (bytes == 0) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  TKB_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    TKB_CUDA(cudaMallocAsync(&p_, bytes, st));
    owned_ = true;
    return;
  }
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  static std::map<std::tuple<int, cudaStream_t, int>, Arena> arenas;
  Arena& a = arenas[{dev, st, slot}];
  if (a.bytes < bytes) {
    // Stream-ordered: work queued on `st` that still uses the old block
    // runs before the free.
    if (a.p) TKB_CUDA(cudaFreeAsync(a.p, st));
    a.p = nullptr;
    a.bytes = 0;
    const size_t grow = bytes + bytes / 4;
    TKB_CUDA(cudaMallocAsync(&a.p, grow, st));
    a.bytes = grow;
  }
  p_ = a.p;
}

Scratch::~Scratch() {
  if (owned_ && p_) cudaFreeAsync(p_, st_);
}

}  // namespace tkb
