// Private to the runtime (runtime.cpp, runtime_multi.cpp): per-domain device
// context and small CUDA helpers.
//
// A "domain" is a set of co-located instances that share one stream, one set
// of activation buffers and direct access to each other's KV slabs: normally
// all instances of one physical GPU. With ESP_DOMAIN_PER_INSTANCE=1 every
// instance is its own domain even on a shared GPU, which routes ring
// prefill and multi-master decode through the cross-device transport (peer
// copies + events) so that path runs, and is tested, on a single B200.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../kernels/kernels.h"
#include <cstdlib>

#include <nvtx3/nvToolsExt.h>

#include "errors.hpp"
#include "runtime.hpp"

namespace esp {

using k::bf16;

// Split-KV chunk: slots of one request on one instance per decode CTA.
// ESP_DECODE_CHUNK overrides (tuning; 32..1024).
constexpr int kDecodeChunkDefault = 512;
inline int decode_chunk() {
  static const int c = [] {
    const char* e = std::getenv("ESP_DECODE_CHUNK");
    const int v = e ? std::atoi(e) : kDecodeChunkDefault;
    return v < 32 ? 32 : (v > 1024 ? 1024 : v);
  }();
  return c;
}

struct LayerW {
  bf16 *wqkv = nullptr, *wo = nullptr, *wgu = nullptr, *wd = nullptr;
  bf16 *norm1 = nullptr, *norm2 = nullptr;
};

struct DeviceCtx {
  int device = -1;  // physical CUDA ordinal
  int domain = -1;  // index in Runtime::devices_
  cudaStream_t stream = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  bf16* embed = nullptr;
  bf16* lm_head = nullptr;
  bf16* final_norm = nullptr;
  std::vector<LayerW> layers;
  bool owns_weights = true;
  float2* rope = nullptr;
  int rope_max = 0;
  std::vector<InstanceId> slabs;  // slab index -> instance id
  // activations / scratch
  DevBuf x, xn, q, kb, vb, attn, h, logits, tok, pos, rinst, rslot, segs, work, last_rows,
      out_tok, chunks, row_start, part_o, part_ml, counts, result, kvrow, ret_rows, ret_slab,
      ret_slot, qin, chunk_ids, row_list, ss1, ss2, carry_o, carry_ml;
  // Tensor parallelism (runtime_tp.cpp): this plane's fp32 partials of the
  // row-parallel O / down projections, read by every plane's all-reduce, and
  // the events marking them written.
  DevBuf tp_po, tp_pd;
  cudaEvent_t tp_ev_o = nullptr, tp_ev_d = nullptr, tp_ev_r = nullptr;
  // Side stream of the windowed ring: peer copies of the next round's block
  // run here while K1 of the current round runs on `stream`.
  cudaStream_t comm = nullptr;
  std::vector<void*> weight_allocs;
  std::vector<cudaEvent_t> sync_events;  // cross-domain event pool
  size_t sync_used = 0;
  // Ring-transport arrival counters of this domain (one slot per source
  // domain, incremented by the sources' QKV epilogues over NVLink) and the
  // running totals the host expects in each (monotonic across layers and
  // prefills, so no reset races with a source that runs ahead).
  unsigned long long* arrive = nullptr;
  unsigned long long arrive_expect[k::kMaxWaitSrc] = {};
};

// Work list of K1 (items = (segment, query-tile pair, head)) for `segs`, in
// the order the persistent CTAs take it (runtime_multi.cpp).
void build_attention_work(const std::vector<k::RingSegment>& segs, int heads,
                          std::vector<int32_t>& work_sorted);
// Number of work items in a list built by build_attention_work.
int attention_n_work(const std::vector<int32_t>& work);

inline void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

// NVTX range for the duration of a scope (header-only NVTX v3: a no-op
// unless a profiler injects itself). One range per ABI call and per layer.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    cuda_ok(cudaSetDevice(d), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// A fresh event on dc's device (pooled, reset by release_sync_events).
inline cudaEvent_t sync_event(DeviceCtx& dc) {
  if (dc.sync_used == dc.sync_events.size()) {
    DeviceGuard g(dc.device);
    cudaEvent_t e;
    cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    dc.sync_events.push_back(e);
  }
  return dc.sync_events[dc.sync_used++];
}

template <typename T>
T* Runtime::scratch(DevBuf& b, size_t n) {
  const size_t bytes = std::max<size_t>(n * sizeof(T), 256);
  if (b.bytes < bytes) {
    if (b.ptr) cuda_ok(cudaFree(b.ptr), "cudaFree");
    b.ptr = nullptr;
    size_t want = std::max(bytes, b.bytes * 3 / 2);
    cuda_ok(cudaMalloc(&b.ptr, want), "cudaMalloc(scratch)");
    b.bytes = want;
  }
  return static_cast<T*>(b.ptr);
}

template <typename F>
void Runtime::timed(int phase, cudaStream_t s, F&& f) {
  if (!profiling_) {
    f();
    return;
  }
  // Created on the current device (the caller's DeviceGuard), destroyed by
  // collect_phase_events: events may not cross devices.
  auto get = [&]() {
    cudaEvent_t e;
    cuda_ok(cudaEventCreate(&e), "event");
    return e;
  };
  PhaseEvent pe{phase, get(), get()};
  cuda_ok(cudaEventRecord(pe.a, s), "event");
  f();
  cuda_ok(cudaEventRecord(pe.b, s), "event");
  pending_.push_back(pe);
}

}  // namespace esp
