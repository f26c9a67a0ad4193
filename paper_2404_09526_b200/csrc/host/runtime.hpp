// The ESP runtime: elastic instances as GPU-resident slices of one
// token-granular paged KV pool, plus the executor that realizes the
// reference scheduler's PrefillPlan / DecodeStepPlan / KvMove decisions with
// the sm_100a kernels. See include/esp_abi.h for the contract.
#pragma once

#include <cuda_runtime.h>

#include <chrono>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_bf16.h>

#include "esp_abi.h"
#include "planner.hpp"
#include "slab.hpp"

namespace esp {

using k_bf16 = __nv_bfloat16;

namespace k {
struct RingSegment;
}

// One request's slots on one instance, in token order, with a lazily
// synchronized device mirror the kernels read.
struct PageList {
  std::vector<int32_t> slots;
  std::vector<int32_t> pos;  // token position of each slot (parity readback only)
  int32_t* dev = nullptr;
  int64_t dev_cap = 0;
  int64_t dev_n = 0;  // prefix of `slots` already on the device
};

struct RequestRec {
  RequestId id = -1;
  int64_t input_len = 0;
  std::vector<int32_t> tokens;  // prompt, then generated tokens
  std::map<InstanceId, PageList> pages;
  int64_t kv_tokens() const {
    int64_t n = 0;
    for (const auto& kv : pages) n += static_cast<int64_t>(kv.second.slots.size());
    return n;
  }
};

struct InstanceRec {
  InstanceId id = -1;
  int device = -1;
  int domain = -1;  // index of the DeviceCtx (co-location domain) owning the slab
  int slab = -1;    // index among the instances of that domain
  int64_t capacity = 0;
  int64_t used = 0;
  std::vector<int32_t> free_stack;  // back() is the next slot handed out
  // [layers][capacity][hidden] bf16, lazily backed (slab.hpp)
  std::unique_ptr<LazySlab> k_slab, v_slab;
  int64_t high_water = 0;  // slots [0, high_water) are physically backed
  k_bf16* layer_k(int l) const {
    return static_cast<k_bf16*>(k_slab->base()) + static_cast<int64_t>(l) * k_slab->layer_stride_elems();
  }
  k_bf16* layer_v(int l) const {
    return static_cast<k_bf16*>(v_slab->base()) + static_cast<int64_t>(l) * v_slab->layer_stride_elems();
  }
  // Tensor-parallel runtimes (tp > 1): the head shards of planes 1..tp-1
  // (plane 0's shard is k_slab / v_slab); same slot ids on every plane.
  std::vector<std::unique_ptr<LazySlab>> tp_k, tp_v;
  k_bf16* plane_k(int plane, int l) const {
    const LazySlab& sl = plane == 0 ? *k_slab : *tp_k[static_cast<size_t>(plane - 1)];
    return static_cast<k_bf16*>(sl.base()) + static_cast<int64_t>(l) * sl.layer_stride_elems();
  }
  k_bf16* plane_v(int plane, int l) const {
    const LazySlab& sl = plane == 0 ? *v_slab : *tp_v[static_cast<size_t>(plane - 1)];
    return static_cast<k_bf16*>(sl.base()) + static_cast<int64_t>(l) * sl.layer_stride_elems();
  }
};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct DeviceCtx;

struct ProfileRec {
  int dop;
  std::vector<int64_t> lengths;
  double ms;
};

// One measured decode step (no chunk riding on it): the arguments of
// Sib::decode_time (cost_model.cpp:175-187) as the engine computes them
// (engine.cpp:420-425: resident = KV of the batch after the append).
struct DecodeProfileRec {
  int dop, batch, masters;
  int64_t resident;
  double ms;
};

class Runtime {
 public:
  Runtime(const esp_model_config& cfg, int n_instances, const int32_t* devices,
          int64_t kv_capacity);
  // Tensor-parallel instances: every instance spans the `tp`
  // planes (plane r on GPU plane_devices[r]) — heads [r H/tp, (r+1) H/tp)
  // of its KV and the matching Megatron shards of the weights live on plane
  // r; ESP rings run co-located inside each plane (runtime_tp.cpp).
  Runtime(const esp_model_config& cfg, int n_instances, int tp, const int32_t* plane_devices,
          int64_t kv_capacity);
  ~Runtime();
  int tp() const { return tp_; }

  void prefill(const esp_prefill_args& a);
  void decode_step(const esp_decode_args& a);
  void move_kv(RequestId r, InstanceId from, InstanceId to, int64_t tokens);
  void free_request(RequestId r);
  void query_placement(RequestId r, int32_t* inst, int64_t* tok, int32_t cap, int32_t* n) const;
  void instance_info(InstanceId i, int64_t* cap, int64_t* used) const;
  void check_conservation();
  void request_tokens(RequestId r, int32_t* out, int32_t cap, int32_t* n) const;
  const esp_prefill_stats& last_prefill_stats() const { return last_prefill_; }
  // Parity readback: the request's K/V rows of one layer in token order
  // (host bf16 [n x hidden]); *n = the request's KV token count.
  void read_kv(RequestId r, int layer, void* k_out, void* v_out, int64_t cap, int64_t* n);
  // Arms the next prefill (single-request plan) to capture its attention
  // outputs at token positions `pos` in every layer; captured() copies them
  // out as host bf16 [layers x n x hidden].
  void capture_attention(const int64_t* pos, int64_t n);
  void captured_attention(void* out, int64_t cap_rows, int64_t* n);
  // Devices whose access to every mapped chunk of the instance's K and V
  // slabs is read/write (cuMemGetAccess).
  bool slab_accessible(InstanceId i, int device) const;
  void dump_profiles(const std::string& path) const;
  const std::vector<DecodeProfileRec>& decode_profiles() const { return decode_profiles_; }
  bool placement_only() const { return devices_.empty(); }
  void set_profiling(bool on) { profiling_ = on; }
  void phase_times(double* ms, int64_t* launches, int n);

  // Phases of the data path timed with CUDA events when profiling is on.
  enum Phase {
    kPhEmbed = 0, kPhNorm, kPhQkv, kPhAttention, kPhOProj, kPhGateUp, kPhDown, kPhLmHead,
    kPhArgmax, kPhDecodeAttn, kPhCombine, kPhHostEnqueue, kPhCount
  };

 private:
  InstanceRec& inst(InstanceId i);
  const InstanceRec& inst(InstanceId i) const;
  RequestRec& req(RequestId r);
  const RequestRec& req(RequestId r) const;
  std::vector<int32_t> take_slots(InstanceRec& in, int64_t n);
  void release_slots(InstanceRec& in, const std::vector<int32_t>& s);
  void sync_pages(PageList& pl, cudaStream_t s);
  DeviceCtx& device_of(const std::vector<InstanceId>& ids, const char* what);
  // The single domain holding all `ids`, or nullptr when they span domains.
  DeviceCtx* single_domain(const std::vector<InstanceId>& ids);
  void init_device(DeviceCtx& dc, const DeviceCtx* share_weights);
  void read_options();  // environment, once per runtime
  // Tensor parallelism (runtime_tp.cpp): plane `rank`'s weight shards.
  void init_device_tp(DeviceCtx& dc, int rank);
  // Stripe layout of a single-domain ESP prefill: rows ring-position-major,
  // then request, then stripe index; the K1 ring segments over them.
  struct StripePlan {
    std::vector<std::vector<int32_t>> row0;  // [ring position][request] first row
    std::vector<int32_t> tok, pos, inst, slot;  // per row: token, position, resting slab / slot
    std::vector<k::RingSegment> segs;
    int rows = 0;
  };
  StripePlan plan_stripes(const esp_prefill_args& a,
                          const std::vector<std::vector<int32_t>>& tok_inst,
                          const std::vector<std::vector<int32_t>>& tok_slot,
                          const std::vector<int64_t>& tok_base) const;
  void prefill_tp(const esp_prefill_args& a, const std::vector<std::vector<int32_t>>& tok_inst,
                  const std::vector<std::vector<int32_t>>& tok_slot,
                  const std::vector<int64_t>& tok_base);
  void ensure_rope(DeviceCtx& dc, int64_t max_pos);
  // Cross-domain executors (runtime_multi.cpp): ring transport by peer
  // copies + events, retention on pass, query broadcast / partial gather.
  void prefill_multi(const esp_prefill_args& a, const std::vector<InstanceId>& ring,
                     const std::vector<std::vector<int32_t>>& tok_inst,
                     const std::vector<std::vector<int32_t>>& tok_slot,
                     const std::vector<int64_t>& tok_base);
  struct DecodeRow {
    RequestId r;
    InstanceId master;
    int32_t token, pos, slot;
  };
  // A chunked-prefill chunk whose request's KV spans transport domains: the
  // chunk rows run in the domain of the chunk's first instance; K/V go to
  // their page slots by (peer) stores, earlier KV is gathered by (peer) loads.
  void chunk_multi(const esp_decode_args& a, int64_t p_prev,
                   const std::vector<std::pair<InstanceId, int32_t>>& prev,
                   const std::vector<std::pair<InstanceId, int32_t>>& chunk_slots, double* ms);
  void decode_multi(const esp_decode_args& a, const std::vector<DecodeRow>& rows,
                    const std::vector<RequestId>& batch);
  // A chunked-prefill chunk riding on a tp decode step: earlier KV (slab,
  // slot) in any order, then the chunk's own slots in token order.
  struct TpChunk {
    int c = 0;
    int64_t p_prev = 0;
    std::vector<int32_t> kv_slab, kv_slot;  // p_prev + c entries
    std::vector<int32_t> ch_slab, ch_slot;  // c entries
  };
  double decode_tp(const esp_decode_args& a, const std::vector<DecodeRow>& rows,
                   const TpChunk& chunk);
  // The second half of a layer after attention: O projection (+ residual),
  // RMSNorm, gate_up (SiLU·up), down projection (+ residual), on `rows` rows
  // of dc's x / attn / xn / h buffers. Norm handling:
  //   ss_o == null            — unit-gain norm kernel between O and gate_up;
  //   ss_o / ss_d given       — fused: O accumulates row sums of squares into
  //                             ss_o, gate_up scales by them, down accumulates
  //                             into ss_d (the next layer's norm1);
  //   zero_in_kernel          — the skinny kernels clear the next buffer
  //                             (decode, PDL-friendly); otherwise memsets.
  struct NormFuse {
    float* ss_o = nullptr;
    float* ss_d = nullptr;
    bool zero_in_kernel = false;
  };
  void o_and_mlp(DeviceCtx& dc, int l, int rows, k_bf16* x, const k_bf16* attn, k_bf16* xn,
                 k_bf16* hbuf, const NormFuse& nf, cudaStream_t s);
  // Data-path options, read ONCE from the environment when the runtime is
  // created (never per launch):
  //   ESP_DOMAIN_PER_INSTANCE  every instance its own co-location domain
  //                            (the cross-GPU transport on one GPU);
  //   ESP_RING_COPY            prefill ring by peer copies in the reference's
  //                            round order instead of the fused push;
  //   ESP_RING_WINDOW=1 / =0   prefill ring over an O(S/d) window (own block +
  //                            two receive slots, one K1 launch per round with
  //                            the softmax state carried) always / never;
  //                            default: when the all-gather buffers would
  //                            exceed kWindowAutoBytes;
  //   ESP_DECODE_COPY          decode query broadcast / partial gather by peer
  //                            copies instead of fused peer stores;
  //   ESP_PREFILL_NORM_KERNEL / ESP_DECODE_NORM_KERNEL  RMSNorm as kernels
  //                            instead of fused into the GEMMs;
  //   ESP_RING_ARRIVAL         (tests) arrival counters also between domains
  //                            of one GPU, IN ADDITION to the event wait there
  //                            (so the counting is checked where a spinning
  //                            K1 could otherwise starve the source's GEMM).
  struct Options {
    bool domain_per_instance = false;
    bool force_arrival = false;
    bool ring_copy = false;
    int ring_window = -1;  // 1 always, 0 never, -1 when the all-gather would not fit
    bool decode_copy = false;
    bool fuse_norm_prefill = true;
    bool fuse_norm_decode = true;
  };
  Options opts_;
  bool fuse_norm_prefill() const { return opts_.fuse_norm_prefill; }
  void forward_layers_prefill(DeviceCtx& dc, int rows, const std::vector<k::RingSegment>& segs,
                              const std::vector<int32_t>& work);
  template <typename T>
  T* scratch(DevBuf& b, size_t n);
  template <typename F>
  void timed(int phase, cudaStream_t s, F&& f);
  void collect_phase_events();
  // Host wall ms from a call's entry to its last stream operation (phase
  // kPhHostEnqueue, recorded whether or not profiling is on).
  void note_host_enqueue(std::chrono::steady_clock::time_point t0) {
    phase_ms_[kPhHostEnqueue] +=
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    phase_n_[kPhHostEnqueue] += 1;
  }
  void* upload(DeviceCtx& dc, const void* src, size_t bytes);
  void check_cuda(const char* what);

  esp_model_config cfg_;
  int tp_ = 1;  // tensor-parallel degree of every instance (planes = devices_)
  std::vector<InstanceRec> instances_;
  std::map<RequestId, RequestRec> requests_;
  std::vector<std::unique_ptr<DeviceCtx>> devices_;  // empty: placement-only
  std::vector<ProfileRec> profiles_;
  std::vector<DecodeProfileRec> decode_profiles_;
  void record_decode_profile(const std::vector<InstanceId>& members,
                             const std::vector<RequestId>& batch, int n_masters, double ms);
  bool profiling_ = false;
  esp_prefill_stats last_prefill_{};
  // Attention capture of the next prefill (parity tests): positions, and per
  // co-location domain the local stripe rows holding them, the capture
  // index of each, and a device buffer [layers x rows x hidden] bf16.
  std::vector<int64_t> cap_pos_;
  bool cap_armed_ = false;
  std::vector<uint16_t> cap_host_;  // [layers x cap_pos_ x hidden]
  int64_t cap_rows_ = 0;
  struct CapDomain {
    std::vector<int32_t> rows, idx;
    int32_t* d_rows = nullptr;
    k_bf16* d_buf = nullptr;
  };
  std::map<int, CapDomain> cap_dom_;
  // During an armed prefill: local stripe row `row` of domain `dom` holds
  // captured position number `idx`.
  void cap_add(int dom, int32_t row, int32_t idx);
  // After layer l's attention of domain dc: copy its captured rows.
  void cap_layer(DeviceCtx& dc, int l, const k_bf16* attn, cudaStream_t s);
  // After the prefill synchronized: gather the rows to the host and disarm.
  void cap_finish();
  struct PhaseEvent {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<PhaseEvent> pending_;
  std::vector<cudaEvent_t> event_pool_;
  double phase_ms_[kPhCount] = {};
  int64_t phase_n_[kPhCount] = {};
};

}  // namespace esp
