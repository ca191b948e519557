// Programmatic dependent launch (PDL). Kernels are launched with programmatic
// stream serialization, so a kernel's blocks can be scheduled while its stream
// predecessor drains (also inside captured graphs); every kernel starts with
// pdl_wait() -- griddepcontrol.wait, a no-op when launched without the
// attribute -- which returns once the predecessor grid has completed and its
// memory is visible, so no kernel touches memory before its inputs exist.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace pmklc_b200 {

__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// The attribute is used only on the stream registered here (the engine's
// critical chain): on a side stream that runs concurrently with other work,
// early-scheduled blocks idle at the wait while holding SM slots.
inline cudaStream_t& pdl_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
struct PdlScope {  // registers `s` as the PDL stream for the scope
  cudaStream_t prev;
  explicit PdlScope(cudaStream_t s) : prev(pdl_stream()) { pdl_stream() = s; }
  ~PdlScope() { pdl_stream() = prev; }
};

// cached cudaStreamGetPriority (launches repeat on a handful of streams)
inline int stream_priority(cudaStream_t st) {
  thread_local cudaStream_t last = nullptr;
  thread_local int prio = 0;
  if (st != last || st == nullptr) {
    int p = 0;
    if (st != nullptr && cudaStreamGetPriority(st, &p) != cudaSuccess) p = 0;
    last = st;
    prio = p;
  }
  return prio;
}

// Opt-in dynamic shared memory above 48 KB. The attribute belongs to the
// current device's context, so it is raised once per (kernel, device) -- a
// process that drives a second device gets its own opt-in -- under a lock
// (entry points are reentrant across threads). A failed call is not cached
// and leaves the error for the launch check to report.
inline void ensure_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (bytes <= have) return;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) ==
      cudaSuccess)
    have = bytes;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (st != nullptr && st == pdl_stream()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  // the stream's scheduling priority, stamped on the launch so that it also
  // holds inside captured graphs (the DM chain of a tick outranks the next
  // tick's static predictions running beside it)
  attr[na].id = cudaLaunchAttributePriority;
  attr[na].val.priority = stream_priority(st);
  ++na;
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  // PMKLC_DEBUG_SYNC=1: every launch synchronised and checked, naming the
  // kernel that failed (a fault otherwise surfaces at the next checked call)
  static const bool dbg = std::getenv("PMKLC_DEBUG_SYNC") != nullptr;
  if (dbg) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    const cudaError_t e = cs == cudaStreamCaptureStatusNone ? cudaStreamSynchronize(st) : cudaGetLastError();
    if (e != cudaSuccess) {
      const char* name = nullptr;
      cudaFuncGetName(&name, reinterpret_cast<const void*>(kernel));
      std::fprintf(stderr, "PMKLC_DEBUG_SYNC: %s after %s\n", cudaGetErrorString(e), name ? name : "?");
      std::abort();
    }
  }
}

}  // namespace pmklc_b200
