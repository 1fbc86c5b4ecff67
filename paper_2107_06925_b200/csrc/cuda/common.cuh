// Shared CUDA helpers for the Chimera-B200 kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "capi_util.hpp"

#define CK_CUDA(expr)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw chimera::capi::InternalError(std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                         " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

namespace chimera::cuda {

// SM count of the current device (148 on a full B200), queried once per device: the
// persistent grids (GEMM tiles, attention items, LayerNorm backward, dQ pass) are sized
// from it, so a part with fewer SMs or a MIG slice is neither over- nor under-subscribed.
inline int num_sms() {
  static int cache[64] = {};
  int dev = 0;
  CK_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) CK_CUDA(cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev));
  return cache[dev];
}

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }

// The product path refuses to run anywhere but on an sm_100 device.
inline void require_sm100() {
  int dev = 0;
  CK_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p{};
  CK_CUDA(cudaGetDeviceProperties(&p, dev));
  if (p.major != 10)
    throw chimera::capi::InternalError("Chimera-B200 kernels require an sm_100 (B200) device, got sm_" +
                                       std::to_string(p.major * 10 + p.minor));
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum for blockDim.x a multiple of 32 (<= 1024); `scratch` >= 32 floats.
__device__ __forceinline__ float block_sum(float v, float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  v = lane < nwarps ? scratch[lane] : 0.f;
  return warp_sum(v);
}
__device__ __forceinline__ float block_max(float v, float* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  v = lane < nwarps ? scratch[lane] : -INFINITY;
  return warp_max(v);
}

// Programmatic dependent launch.  Every kernel of the stage executor is launched with
// programmatic stream serialisation, so it is scheduled while its predecessor in the
// stream is still running (on SMs that predecessor leaves free) and overlaps its
// prologue (barrier init, TMEM allocation, tensor-map prefetch) with the predecessor's
// tail.  Each such kernel calls pdl_wait() before its first global-memory access (read
// or write): griddepcontrol.wait returns once every prerequisite grid has completed and
// flushed.  Persistent kernels (grid <= resident capacity) call pdl_trigger() right after
// their prologue so their successors may be scheduled early.  CK_PDL=0 disables it.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CK_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// Stream priorities (CK_STREAM_PRIO, see gpt.cu): when on, every launch carries its
// stream's priority as a launch attribute so graph kernel nodes keep it (graphs are then
// instantiated with cudaGraphInstantiateFlagUseNodePriority).
inline bool& node_priority_flag() {
  static bool on = false;
  return on;
}
template <typename... KArgs, typename... Args>
inline void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (node_priority_flag()) {
    int prio = 0;
    if (cudaStreamGetPriority(st, &prio) == cudaSuccess) {
      at[n].id = cudaLaunchAttributePriority;
      at[n++].val.priority = prio;
    }
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  CK_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace chimera::cuda
