// Stage-to-stage links of the GPT executor (activation and gradient messages).
//
// A message (replica r, micro-batch m, boundary s, direction) has one producer rank
// and one consumer rank.  Its receive buffer always lives in the CONSUMER's HBM
// ("inbox"); the producer's last kernel of the task (GEMM epilogue / LayerNorm
// backward) stores straight into it -- over NVLink through a CUDA-IPC mapping when
// the consumer is another process -- so no copy engine or staging buffer is
// involved.  Completion is signalled without the host:
//   same process : cudaEventRecord / cudaStreamWaitEvent;
//   cross process: stream memory operations on 32-bit flags, graph-capturable:
//     producer  wait ack==1 (own outbox), ack=0, produce, flag=1 (consumer inbox)
//     consumer  wait flag==1 (own inbox), flag=0, consume ..., ack=1 (producer outbox)
// ack starts at 1, flag at 0, so the protocol needs no per-iteration epoch and the
// whole iteration can be captured once into a CUDA graph and replayed.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "common.cuh"

namespace chimera::gpt {

struct MemOps {
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  WaitFn wait32 = nullptr;
  WriteFn write32 = nullptr;
  unsigned wait_flags = CU_STREAM_WAIT_VALUE_EQ;

  static const MemOps& get() {
    static MemOps m;
    static std::once_flag once;
    std::call_once(once, [] {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
        throw capi::InternalError("cuStreamWaitValue32 unavailable");
      m.wait32 = reinterpret_cast<WaitFn>(p);
      if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
        throw capi::InternalError("cuStreamWriteValue32 unavailable");
      m.write32 = reinterpret_cast<WriteFn>(p);
      int dev = 0, flush = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, dev);
      if (flush) m.wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
    });
    return m;
  }
  void wait(cudaStream_t st, const uint32_t* addr, uint32_t v) const {
    if (wait32(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, wait_flags) != CUDA_SUCCESS)
      throw capi::InternalError("cuStreamWaitValue32 failed");
  }
  // Default flags: the write is preceded by a system-wide memory fence, so every store
  // issued earlier on the stream (including peer stores) is visible before the flag.
  void write(cudaStream_t st, uint32_t* addr, uint32_t v) const {
    if (write32(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, 0) != CUDA_SUCCESS)
      throw capi::InternalError("cuStreamWriteValue32 failed");
  }
};

struct Msg {
  int producer = -1, consumer = -1;  // logical ranks
  bool prod_local = false, cons_local = false;
  __nv_bfloat16* buf = nullptr;  // consumer inbox buffer (peer mapping if consumer is remote)
  cudaEvent_t ev = nullptr;      // both local
  uint32_t* flag = nullptr;      // in the consumer inbox (local or peer pointer)
  uint32_t* ack = nullptr;       // in the producer outbox (local or peer pointer)

  void before_produce(cudaStream_t st) const {
    if (!cons_local) {
      MemOps::get().wait(st, ack, 1);
      MemOps::get().write(st, ack, 0);
    }
  }
  void after_produce(cudaStream_t st) const {
    if (cons_local) CK_CUDA(cudaEventRecord(ev, st));
    else MemOps::get().write(st, flag, 1);
  }
  void before_consume(cudaStream_t st) const {
    if (prod_local) {
      CK_CUDA(cudaStreamWaitEvent(st, ev, 0));
    } else {
      MemOps::get().wait(st, flag, 1);
      MemOps::get().write(st, flag, 0);
    }
  }
  void after_last_use(cudaStream_t st) const {
    if (!prod_local) MemOps::get().write(st, ack, 1);
  }
};

}  // namespace chimera::gpt
