// ESP runtime / executor. See runtime.hpp and include/esp_abi.h.
//
// Data layout in HBM (per device):
//   weights  : embed [V x H], per layer Wqkv [3H x H] (q|k|v rows), Wo [H x H],
//              Wgu [2F x H] (128-row blocks: 64 gate rows, 64 up rows),
//              Wd [H x F], RMSNorm gammas [H]; final norm; LM head [V x H].
//   KV slabs : per instance K and V, [layers][capacity][H] bf16 — one token
//              slot is one page (token-granular PagedAttention),
//              8 KiB per layer per K/V row at LWM-7B shape.
//   prefill  : ring stripe buffers Q/K/V/attn [S x H] in ring-position-major,
//              request-major, stripe order (the O(bsh/d) circulating buffer of
//              PAPER.md:264 for all co-located ring positions).
#include "runtime.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <numeric>
#include <set>
#include <sstream>

#include "../kernels/kernels.h"
#include "../kernels/synthetic.h"
#include "device_ctx.hpp"

namespace esp {

void Runtime::check_cuda(const char* what) { cuda_ok(cudaGetLastError(), what); }

// Call after the stream synchronized: folds recorded event pairs into totals.
void Runtime::collect_phase_events() {
  for (const PhaseEvent& pe : pending_) {
    float ms = 0;
    cuda_ok(cudaEventElapsedTime(&ms, pe.a, pe.b), "elapsed");
    phase_ms_[pe.phase] += ms;
    phase_n_[pe.phase] += 1;
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  pending_.clear();
}

void Runtime::phase_times(double* ms, int64_t* launches, int n) {
  for (int i = 0; i < n && i < kPhCount; ++i) {
    if (ms) ms[i] = phase_ms_[i];
    if (launches) launches[i] = phase_n_[i];
  }
  for (int i = 0; i < kPhCount; ++i) {
    phase_ms_[i] = 0;
    phase_n_[i] = 0;
  }
}

Runtime::Runtime(const esp_model_config& cfg, int n_instances, const int32_t* devices,
                 int64_t kv_capacity)
    : cfg_(cfg) {
  read_options();
  if (n_instances <= 0) throw ConfigError("need at least one instance");
  if (cfg.layers <= 0 || cfg.hidden <= 0 || cfg.heads <= 0 || cfg.head_dim <= 0 ||
      cfg.ffn <= 0 || cfg.vocab <= 0) {
    throw ConfigError("model config fields must be positive");
  }
  if (cfg.heads * cfg.head_dim != cfg.hidden) throw ConfigError("hidden != heads * head_dim");
  instances_.resize(static_cast<size_t>(n_instances));
  for (int i = 0; i < n_instances; ++i) instances_[i].id = i;

  if (devices == nullptr) {  // placement-only runtime: counters and page tables
    if (kv_capacity <= 0) throw ConfigError("placement-only runtime needs kv_capacity > 0");
    for (auto& in : instances_) in.capacity = kv_capacity;
  } else {
    if (cfg.head_dim != 64 && cfg.head_dim != 128) throw ConfigError("head_dim must be 64 or 128");
    if (cfg.hidden % 256 != 0 || cfg.ffn % 64 != 0 || cfg.vocab % 128 != 0) {
      throw ConfigError("hidden % 256, ffn % 64 and vocab % 128 must be 0");
    }
    int ndev = 0;
    cuda_ok(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    // Co-location domains: one per physical GPU, or one per instance when
    // ESP_DOMAIN_PER_INSTANCE is set (exercises the cross-device transport
    // on a single GPU).
    const bool per_instance = opts_.domain_per_instance;
    std::map<int, DeviceCtx*> by_key;
    for (int i = 0; i < n_instances; ++i) {
      const int d = devices[i];
      if (d < 0 || d >= ndev) throw ConfigError("instance device ordinal out of range");
      const int key = per_instance ? i : d;
      if (!by_key.count(key)) {
        devices_.push_back(std::make_unique<DeviceCtx>());
        devices_.back()->device = d;
        devices_.back()->domain = static_cast<int>(devices_.size()) - 1;
        by_key[key] = devices_.back().get();
      }
      DeviceCtx* dc = by_key[key];
      if (static_cast<int>(dc->slabs.size()) >= k::kMaxSlabs) {
        throw ConfigError("too many instances on one device");
      }
      instances_[i].device = d;
      instances_[i].domain = dc->domain;
      instances_[i].slab = static_cast<int>(dc->slabs.size());
      dc->slabs.push_back(i);
    }
    // Peer access between distinct GPUs (NVLink / NVSwitch): ring blocks,
    // broadcast queries and partial outputs move by peer copies.
    std::set<int> phys;
    for (auto& dcp : devices_) phys.insert(dcp->device);
    for (int a : phys) {
      for (int b : phys) {
        if (a == b) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (!can) {
          // The cross-GPU executors store into and load from peer memory
          // (push transport, retention into a remote survivor, K8 moves):
          // refuse GPUs that cannot reach each other instead of faulting.
          throw ConfigError("GPU " + std::to_string(a) + " cannot access GPU " +
                            std::to_string(b) + " (no peer access): one runtime needs "
                            "NVLink/NVSwitch (or PCIe P2P) between all of its GPUs");
        }
        DeviceGuard g(a);
        const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_ok(e, "peer access");
        cudaGetLastError();
      }
    }
    const int64_t bpt = kv_bytes_per_token(cfg.layers, cfg.hidden, cfg.heads, 2);
    std::map<int, const DeviceCtx*> weights_of;
    for (auto& dcp : devices_) {
      DeviceCtx& dc = *dcp;
      auto wit = weights_of.find(dc.device);
      init_device(dc, wit == weights_of.end() ? nullptr : wit->second);
      if (wit == weights_of.end()) weights_of[dc.device] = &dc;
      DeviceGuard g(dc.device);
      int64_t cap = kv_capacity;
      if (cap <= 0) {
        size_t free_b = 0, total_b = 0;
        cuda_ok(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        const int64_t reserve = static_cast<int64_t>(12) << 30;  // prefill activations
        const int64_t avail = static_cast<int64_t>(free_b) - reserve;
        int64_t on_device = 0;
        for (const auto& in : instances_) on_device += in.device == dc.device ? 1 : 0;
        cap = avail / (on_device * bpt);
        if (cap <= 0) throw ConfigError("no HBM left for KV slabs");
      }
      // Slabs reserve the full logical capacity as virtual address space and
      // are backed on demand (slot high-water mark), so co-located instances
      // only consume HBM for resident tokens.
      const size_t row_bytes = static_cast<size_t>(cfg.hidden) * 2;
      for (InstanceId id : dc.slabs) {
        InstanceRec& in = instances_[id];
        in.capacity = cap;
        in.k_slab = std::make_unique<LazySlab>();
        in.v_slab = std::make_unique<LazySlab>();
        in.k_slab->reserve(dc.device, cfg.layers, cap, row_bytes);
        in.v_slab->reserve(dc.device, cfg.layers, cap, row_bytes);
      }
      (void)bpt;
    }
  }
  for (auto& in : instances_) {
    if (in.capacity > INT32_MAX) throw ConfigError("kv_capacity exceeds int32 slot ids");
    in.free_stack.resize(static_cast<size_t>(in.capacity));
    // back() is slot 0: fresh slots come out in ascending order.
    for (int64_t s = 0; s < in.capacity; ++s) {
      in.free_stack[static_cast<size_t>(s)] = static_cast<int32_t>(in.capacity - 1 - s);
    }
  }
}

void Runtime::read_options() {
  opts_.domain_per_instance = std::getenv("ESP_DOMAIN_PER_INSTANCE") != nullptr;
  opts_.ring_copy = std::getenv("ESP_RING_COPY") != nullptr;
  if (const char* w = std::getenv("ESP_RING_WINDOW")) opts_.ring_window = std::atoi(w);
  opts_.force_arrival = std::getenv("ESP_RING_ARRIVAL") != nullptr;
  opts_.decode_copy = std::getenv("ESP_DECODE_COPY") != nullptr;
  opts_.fuse_norm_prefill = std::getenv("ESP_PREFILL_NORM_KERNEL") == nullptr;
  opts_.fuse_norm_decode = std::getenv("ESP_DECODE_NORM_KERNEL") == nullptr;
}

Runtime::~Runtime() {
  for (cudaEvent_t e : event_pool_) cudaEventDestroy(e);
  for (const PhaseEvent& pe : pending_) {
    cudaEventDestroy(pe.a);
    cudaEventDestroy(pe.b);
  }
  for (auto& [id, r] : requests_) {
    for (auto& [i, pl] : r.pages) {
      if (pl.dev) cudaFree(pl.dev);
    }
  }
  for (auto& in : instances_) {
    in.k_slab.reset();
    in.v_slab.reset();
    in.tp_k.clear();
    in.tp_v.clear();
  }
  for (auto& dcp : devices_) {
    DeviceCtx& dc = *dcp;
    cudaSetDevice(dc.device);
    for (void* p : dc.weight_allocs) cudaFree(p);
    DevBuf* bufs[] = {&dc.x, &dc.xn, &dc.q, &dc.kb, &dc.vb, &dc.attn, &dc.h, &dc.logits,
                      &dc.tok, &dc.pos, &dc.rinst, &dc.rslot, &dc.segs, &dc.work,
                      &dc.last_rows, &dc.out_tok, &dc.chunks, &dc.row_start, &dc.part_o,
                      &dc.part_ml, &dc.counts, &dc.result, &dc.kvrow, &dc.ret_rows,
                      &dc.ret_slab, &dc.ret_slot, &dc.qin, &dc.chunk_ids, &dc.row_list,
                      &dc.ss1, &dc.ss2, &dc.tp_po, &dc.tp_pd};
    for (DevBuf* b : bufs) {
      if (b->ptr) cudaFree(b->ptr);
    }
    if (dc.rope) cudaFree(dc.rope);
    if (dc.arrive) cudaFree(dc.arrive);
    for (cudaEvent_t e : dc.sync_events) cudaEventDestroy(e);
    if (dc.tp_ev_o) cudaEventDestroy(dc.tp_ev_o);
    if (dc.tp_ev_d) cudaEventDestroy(dc.tp_ev_d);
    if (dc.tp_ev_r) cudaEventDestroy(dc.tp_ev_r);
    if (dc.e0) cudaEventDestroy(dc.e0);
    if (dc.e1) cudaEventDestroy(dc.e1);
    if (dc.stream) cudaStreamDestroy(dc.stream);
    if (dc.comm) cudaStreamDestroy(dc.comm);
  }
}

void Runtime::ensure_rope(DeviceCtx& dc, int64_t max_pos) {
  if (dc.rope_max >= max_pos) return;
  int want = 4096;
  while (want < max_pos) want *= 2;
  if (dc.rope) {
    cuda_ok(cudaStreamSynchronize(dc.stream), "sync");
    cudaFree(dc.rope);
  }
  cuda_ok(cudaMalloc(&dc.rope, static_cast<size_t>(want) * cfg_.head_dim / 2 * sizeof(float2)),
          "cudaMalloc(rope)");
  k::rope_table(dc.rope, want, cfg_.head_dim, cfg_.rope_theta, dc.stream);
  dc.rope_max = want;
}

void Runtime::init_device(DeviceCtx& dc, const DeviceCtx* share) {
  DeviceGuard g(dc.device);
  cuda_ok(cudaStreamCreateWithFlags(&dc.stream, cudaStreamNonBlocking), "stream");
  cuda_ok(cudaEventCreate(&dc.e0), "event");
  cuda_ok(cudaEventCreate(&dc.e1), "event");
  if (share != nullptr) {  // another domain on the same GPU owns the weights
    dc.embed = share->embed;
    dc.lm_head = share->lm_head;
    dc.final_norm = share->final_norm;
    dc.layers = share->layers;
    dc.owns_weights = false;
    return;
  }
  const int64_t H = cfg_.hidden, F = cfg_.ffn, V = cfg_.vocab;
  auto alloc = [&](int64_t n) {
    void* p = nullptr;
    cuda_ok(cudaMalloc(&p, static_cast<size_t>(n) * sizeof(bf16)), "cudaMalloc(weights)");
    dc.weight_allocs.push_back(p);
    return static_cast<bf16*>(p);
  };
  const uint64_t seed = cfg_.weight_seed;
  cudaStream_t s = dc.stream;
  dc.embed = alloc(V * H);
  k::init_weight(dc.embed, V, H, seed, k::kTensorEmbed, 0, 0, s);
  dc.lm_head = alloc(V * H);
  k::init_weight(dc.lm_head, V, H, seed, k::kTensorLmHead, 0, 0, s);
  dc.final_norm = alloc(H);
  k::fill_bf16(dc.final_norm, H, 1.0f, s);
  dc.layers.resize(static_cast<size_t>(cfg_.layers));
  for (int l = 0; l < cfg_.layers; ++l) {
    LayerW& w = dc.layers[l];
    w.wqkv = alloc(3 * H * H);
    k::init_weight(w.wqkv, 3 * H, H, seed, k::kTensorQ, l, 1, s);
    w.wo = alloc(H * H);
    k::init_weight(w.wo, H, H, seed, k::kTensorO, l, 0, s);
    w.wgu = alloc(2 * F * H);
    k::init_weight(w.wgu, 2 * F, H, seed, k::kTensorGate, l, 2, s);
    w.wd = alloc(H * F);
    k::init_weight(w.wd, H, F, seed, k::kTensorDown, l, 0, s);
    w.norm1 = alloc(H);
    k::fill_bf16(w.norm1, H, 1.0f, s);
    w.norm2 = alloc(H);
    k::fill_bf16(w.norm2, H, 1.0f, s);
    // The two layer RMSNorm gains are folded into the projections that
    // consume them (Wqkv·diag(γ1), Wgu·diag(γ2)); the layer norms then run
    // with unit gain — as a kernel (prefill) or fused into the decode GEMMs.
    k::scale_cols(w.wqkv, 3 * H, H, w.norm1, s);
    k::scale_cols(w.wgu, 2 * F, H, w.norm2, s);
  }
  check_cuda("init weights");
  cuda_ok(cudaStreamSynchronize(s), "init weights sync");
}

InstanceRec& Runtime::inst(InstanceId i) {
  if (i < 0 || i >= static_cast<int>(instances_.size())) {
    throw InternalError("placement names unknown instance");
  }
  return instances_[static_cast<size_t>(i)];
}
const InstanceRec& Runtime::inst(InstanceId i) const {
  return const_cast<Runtime*>(this)->inst(i);
}
RequestRec& Runtime::req(RequestId r) {
  auto it = requests_.find(r);
  if (it == requests_.end()) throw InternalError("unknown request " + std::to_string(r));
  return it->second;
}
const RequestRec& Runtime::req(RequestId r) const { return const_cast<Runtime*>(this)->req(r); }

std::vector<int32_t> Runtime::take_slots(InstanceRec& in, int64_t n) {
  if (in.used + n > in.capacity || static_cast<int64_t>(in.free_stack.size()) < n) {
    throw CapacityError(in.id, "instance " + std::to_string(in.id) + " lacks free slots");
  }
  std::vector<int32_t> out(in.free_stack.end() - n, in.free_stack.end());
  std::reverse(out.begin(), out.end());
  if (in.k_slab && n > 0) {
    // Back the slab up to the highest slot handed out (before any counter
    // moves, so an out-of-memory here leaves the pool untouched).
    const int64_t top = *std::max_element(out.begin(), out.end()) + 1;
    if (top > in.high_water) {
      DeviceGuard g(in.device);
      in.k_slab->ensure(top);
      in.v_slab->ensure(top);
      for (size_t p = 0; p < in.tp_k.size(); ++p) {  // the other planes' head shards
        DeviceGuard gp(devices_[p + 1]->device);
        in.tp_k[p]->ensure(top);
        in.tp_v[p]->ensure(top);
      }
      in.high_water = top;
    }
  }
  in.free_stack.resize(in.free_stack.size() - static_cast<size_t>(n));
  in.used += n;
  return out;
}

void Runtime::release_slots(InstanceRec& in, const std::vector<int32_t>& s) {
  if (in.used < static_cast<int64_t>(s.size())) {
    throw InternalError("freeing more KV than instance " + std::to_string(in.id) + " holds");
  }
  for (auto it = s.rbegin(); it != s.rend(); ++it) in.free_stack.push_back(*it);
  in.used -= static_cast<int64_t>(s.size());
}

void Runtime::sync_pages(PageList& pl, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(pl.slots.size());
  if (pl.dev_n == n && pl.dev) return;
  if (pl.dev_cap < n || !pl.dev) {
    int64_t cap = std::max<int64_t>({n, 64, pl.dev_cap * 2});
    int32_t* p = nullptr;
    cuda_ok(cudaMalloc(&p, static_cast<size_t>(cap) * sizeof(int32_t)), "cudaMalloc(pages)");
    if (pl.dev) {
      cuda_ok(cudaStreamSynchronize(s), "sync pages");
      cudaFree(pl.dev);
    }
    pl.dev = p;
    pl.dev_cap = cap;
    pl.dev_n = 0;
  }
  if (pl.dev_n > n) pl.dev_n = 0;  // shrunk: rewrite
  cuda_ok(cudaMemcpyAsync(pl.dev + pl.dev_n, pl.slots.data() + pl.dev_n,
                          static_cast<size_t>(n - pl.dev_n) * sizeof(int32_t),
                          cudaMemcpyHostToDevice, s),
          "upload pages");
  pl.dev_n = n;
}

DeviceCtx* Runtime::single_domain(const std::vector<InstanceId>& ids) {
  if (devices_.empty()) return nullptr;
  int dom = -1;
  for (InstanceId i : ids) {
    const int d = inst(i).domain;
    if (dom >= 0 && d != dom) return nullptr;
    dom = d;
  }
  return dom < 0 ? nullptr : devices_[static_cast<size_t>(dom)].get();
}

DeviceCtx& Runtime::device_of(const std::vector<InstanceId>& ids, const char* what) {
  if (devices_.empty()) {
    throw NoDeviceError(std::string(what) + " needs a device runtime (placement-only)");
  }
  DeviceCtx* dc = single_domain(ids);
  if (!dc) {
    throw ConfigError(std::string(what) + ": instances span co-location domains");
  }
  return *dc;
}

// ---- prefill -------------------------------------------------------------------
Runtime::StripePlan Runtime::plan_stripes(const esp_prefill_args& a,
                                          const std::vector<std::vector<int32_t>>& tok_slab,
                                          const std::vector<std::vector<int32_t>>& tok_slot,
                                          const std::vector<int64_t>& tok_base) const {
  const int n = a.n_requests, d = a.dop;
  StripePlan sp;
  // Stripe rows: ring-position-major, then request, then stripe index
  // (token t of request r lives at position t mod d, stripe index t / d).
  sp.row0.assign(static_cast<size_t>(d), std::vector<int32_t>(static_cast<size_t>(n)));
  for (int i = 0; i < d; ++i) {
    for (int r = 0; r < n; ++r) {
      sp.row0[i][r] = sp.rows;
      const int64_t len = a.input_lens[r];
      for (int64_t t = i; t < len; t += d) {
        sp.tok.push_back(a.tokens[tok_base[r] + t]);
        sp.pos.push_back(static_cast<int32_t>(t));
        sp.inst.push_back(inst(tok_slab[r][static_cast<size_t>(t)]).slab);
        sp.slot.push_back(tok_slot[r][static_cast<size_t>(t)]);
        ++sp.rows;
      }
    }
  }
  auto stripe_len = [&](int i, int r) -> int32_t {
    const int64_t len = a.input_lens[r];
    return len > i ? static_cast<int32_t>((len - i + d - 1) / d) : 0;
  };
  // Ring segments: position i meets, in round rd, the block of origin
  // (i - rd) mod d (build_ring_schedule, esp_mechanics.cpp:59-68).
  for (int i = 0; i < d; ++i) {
    for (int r = 0; r < n; ++r) {
      const int32_t ql = stripe_len(i, r);
      if (ql == 0) continue;
      k::RingSegment sg{};
      sg.q_row0 = sp.row0[i][r];
      sg.q_len = ql;
      sg.n_rounds = d;
      for (int rd = 0; rd < d; ++rd) {
        const int o = RingSchedule::origin(i, rd, d);
        sg.kv_row0[rd] = sp.row0[o][r];
        sg.kv_len[rd] = stripe_len(o, r);
        sg.shift[rd] = o > i ? 1 : 0;
      }
      sp.segs.push_back(sg);
    }
  }
  return sp;
}

void Runtime::prefill(const esp_prefill_args& a) {
  NvtxRange nvtx("esp_prefill");
  const auto host_t0 = std::chrono::steady_clock::now();
  const int n = a.n_requests, d = a.dop;
  if (n <= 0 || d <= 0) throw InternalError("prefill plan without requests or instances");
  if (!a.request_ids || !a.input_lens || !a.ring || !a.retain_n || !a.retain_instance ||
      !a.retain_tokens) {
    throw ConfigError("prefill: null argument");
  }
  std::vector<InstanceId> ring(a.ring, a.ring + d);
  {
    std::set<InstanceId> seen;
    for (InstanceId i : ring) {
      inst(i);
      if (!seen.insert(i).second) throw InternalError("ring repeats an instance");
    }
  }
  // Validate the resting placement (engine.cpp:327-345) before touching any
  // counter: the allocation is atomic like KvPool::allocate (cluster.cpp:88-99).
  std::map<InstanceId, int64_t> need;
  int64_t off = 0;
  for (int r = 0; r < n; ++r) {
    const RequestId rid = a.request_ids[r];
    if (requests_.count(rid) && requests_.at(rid).kv_tokens() > 0) {
      throw InternalError("prefill plan names a request that already holds KV");
    }
    if (a.input_lens[r] <= 0) throw InternalError("prefill of an empty request");
    int64_t tot = 0;
    for (int p = 0; p < a.retain_n[r]; ++p) {
      const int64_t t = a.retain_tokens[off + p];
      if (t < 0) throw InternalError("negative placement entry");
      inst(a.retain_instance[off + p]);
      need[a.retain_instance[off + p]] += t;
      tot += t;
    }
    off += a.retain_n[r];
    if (tot != a.input_lens[r]) throw InternalError("prefill placement does not cover the input");
  }
  for (const auto& [i, t] : need) {
    if (inst(i).used + t > inst(i).capacity) {
      throw CapacityError(i, "prefill placement overflows instance " + std::to_string(i));
    }
  }
  // The ring the kernels walk and the scale-down its retention realises,
  // through the planner's restatements of the reference mechanics
  // (build_ring_schedule esp_mechanics.cpp:45-70, proactive_scale_down
  // :78-136): ring volume, the part of it that crosses GPUs, and zero extra
  // migration whenever the resting instances are ring members.
  {
    std::vector<Tokens> seg(static_cast<size_t>(d), 0);
    for (int r = 0; r < n; ++r) {
      for (int i = 0; i < d; ++i) {
        seg[static_cast<size_t>(i)] += a.input_lens[r] > i ? (a.input_lens[r] - i + d - 1) / d : 0;
      }
    }
    const RingSchedule rs = build_ring_schedule(ring, seg);
    esp_prefill_stats st{};
    st.ring_volume_tokens = rs.total_comm_volume();
    for (const auto& round : rs.rounds) {
      for (const RingTransfer& t : round) {
        if (!devices_.empty() && inst(t.from).domain != inst(t.to).domain) st.cross_domain_tokens += t.volume;
      }
    }
    st.nvlink_bytes = st.cross_domain_tokens * 2 * cfg_.hidden * 2 * cfg_.layers;
    const std::set<InstanceId> ring_set(ring.begin(), ring.end());
    FillOrder rest;
    std::vector<InstanceId> targets;
    bool inside = true;
    for (const auto& [i, t] : need) {
      if (t == 0) continue;
      inside = inside && ring_set.count(i) > 0;
      rest.emplace_back(i, t);
      targets.push_back(i);
    }
    st.extra_migration_tokens = -1;
    if (inside && !targets.empty()) {
      std::map<InstanceId, Tokens> free;
      for (InstanceId i : ring) free[i] = inst(i).capacity - inst(i).used;
      const ScaleDownResult sd = proactive_scale_down(rs, ring, targets, rest, free);
      st.extra_migration_tokens = sd.extra_migration_volume;
      st.transient_buffer_tokens = sd.transient_buffer_tokens;
    }
    last_prefill_ = st;
  }
  if (!devices_.empty() && !a.tokens) throw ConfigError("prefill: tokens required on a device runtime");
  // The ring kernel keeps all d rounds of a segment in one work item; a
  // placement-only runtime has no kernel and accepts any ring the reference
  // plans (its ring tests go to d = 16).
  if (!devices_.empty() && d > k::kMaxRounds) {
    throw ConfigError("prefill: ESP degree " + std::to_string(d) + " exceeds the kernel's " +
                      std::to_string(k::kMaxRounds) + " rounds");
  }
  // One co-location domain: the batched single-domain pass. Several: ring
  // transport between domains (runtime_multi.cpp), where a token can only
  // be retained by a domain the ring passes through (proactive_scale_down's
  // targets-within-the-group rule, esp_mechanics.cpp:96-108).
  std::vector<InstanceId> all_ids = ring;
  for (const auto& kv : need) all_ids.push_back(kv.first);
  DeviceCtx* dcp = devices_.empty() ? nullptr : single_domain(all_ids);
  const bool multi = !devices_.empty() && dcp == nullptr;
  if (multi) {
    std::set<int> ring_domains;
    for (InstanceId i : ring) ring_domains.insert(inst(i).domain);
    for (const auto& [i, t] : need) {
      if (t > 0 && !ring_domains.count(inst(i).domain)) {
        throw InfeasiblePlanError("resting instance " + std::to_string(i) +
                                  " is outside the prefill ring's devices");
      }
    }
  }

  // Allocate resting slots; tok_inst/tok_slot give each prompt token's page.
  std::vector<std::vector<int32_t>> tok_slab(static_cast<size_t>(n)), tok_slot(static_cast<size_t>(n));
  off = 0;
  int64_t tok_off = 0;
  std::vector<int64_t> tok_base(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) {
    const RequestId rid = a.request_ids[r];
    RequestRec& rr = requests_[rid];
    rr.id = rid;
    rr.input_len = a.input_lens[r];
    rr.tokens.clear();
    if (a.tokens) rr.tokens.assign(a.tokens + tok_off, a.tokens + tok_off + a.input_lens[r]);
    tok_base[r] = tok_off;
    tok_off += a.input_lens[r];
    auto& ts = tok_slab[r];
    auto& tl = tok_slot[r];
    ts.reserve(static_cast<size_t>(rr.input_len));
    tl.reserve(static_cast<size_t>(rr.input_len));
    for (int p = 0; p < a.retain_n[r]; ++p) {
      const InstanceId i = a.retain_instance[off + p];
      const int64_t t = a.retain_tokens[off + p];
      if (t == 0) continue;
      InstanceRec& in = inst(i);
      std::vector<int32_t> slots = take_slots(in, t);
      PageList& pl = rr.pages[i];
      pl.slots.insert(pl.slots.end(), slots.begin(), slots.end());
      for (int32_t s : slots) {
        pl.pos.push_back(static_cast<int32_t>(ts.size()));
        ts.push_back(i);  // resting instance id of the token
        tl.push_back(s);
      }
    }
    off += a.retain_n[r];
  }
  if (devices_.empty()) return;  // placement-only: page tables are the whole effect
  if (tp_ > 1) {
    prefill_tp(a, tok_slab, tok_slot, tok_base);
    return;
  }
  if (multi) {
    prefill_multi(a, ring, tok_slab, tok_slot, tok_base);
    return;
  }

  DeviceCtx& dc = *dcp;
  DeviceGuard g(dc.device);
  cudaStream_t s = dc.stream;
  const int H = cfg_.hidden;

  const StripePlan sp = plan_stripes(a, tok_slab, tok_slot, tok_base);
  const std::vector<std::vector<int32_t>>& row0 = sp.row0;
  const std::vector<k::RingSegment>& segs = sp.segs;
  const int rows = sp.rows;
  std::vector<int32_t> work_sorted;
  build_attention_work(segs, cfg_.heads, work_sorted);
  if (cap_armed_) {  // parity capture: stripe row of each captured position
    if (n != 1) throw ConfigError("attention capture needs a single-request prefill");
    for (size_t c = 0; c < cap_pos_.size(); ++c) {
      const int64_t t = cap_pos_[c];
      if (t < 0 || t >= a.input_lens[0]) throw ConfigError("capture position outside the prompt");
      cap_add(dc.domain, row0[t % d][0] + static_cast<int32_t>(t / d), static_cast<int32_t>(c));
    }
  }

  // RoPE table covering every position of the batch.
  int64_t max_len = 0;
  for (int r = 0; r < n; ++r) max_len = std::max(max_len, a.input_lens[r]);
  ensure_rope(dc, max_len);

  int32_t* d_tok = scratch<int32_t>(dc.tok, rows);
  int32_t* d_pos = scratch<int32_t>(dc.pos, rows);
  int32_t* d_inst = scratch<int32_t>(dc.rinst, rows);
  int32_t* d_slot = scratch<int32_t>(dc.rslot, rows);
  k::RingSegment* d_segs = scratch<k::RingSegment>(dc.segs, segs.size());
  int32_t* d_work = scratch<int32_t>(dc.work, work_sorted.size());
  cuda_ok(cudaMemcpyAsync(d_tok, sp.tok.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_pos, sp.pos.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_inst, sp.inst.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_slot, sp.slot.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * sizeof(k::RingSegment),
                          cudaMemcpyHostToDevice, s),
          "h2d");
  cuda_ok(cudaMemcpyAsync(d_work, work_sorted.data(), work_sorted.size() * 4,
                          cudaMemcpyHostToDevice, s),
          "h2d");

  bf16* x = scratch<bf16>(dc.x, static_cast<size_t>(rows) * H);
  float* ss1 = fuse_norm_prefill() ? scratch<float>(dc.ss1, rows) : nullptr;
  cuda_ok(cudaEventRecord(dc.e0, s), "event");
  timed(kPhEmbed, s, [&] { k::embed(d_tok, dc.embed, x, rows, H, s, ss1); });
  forward_layers_prefill(dc, rows, segs, work_sorted);

  // Last prompt token of each request: position len-1 lives at ring position
  // (len-1) mod d, stripe index (len-1) / d.
  std::vector<int32_t> last(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) {
    const int64_t t = a.input_lens[r] - 1;
    last[r] = row0[t % d][r] + static_cast<int32_t>(t / d);
  }
  int32_t* d_last = scratch<int32_t>(dc.last_rows, n);
  cuda_ok(cudaMemcpyAsync(d_last, last.data(), n * 4, cudaMemcpyHostToDevice, s), "h2d");
  bf16* xn = scratch<bf16>(dc.xn, static_cast<size_t>(std::max(rows, n)) * H);
  timed(kPhNorm, s, [&] { k::rmsnorm(x, d_last, dc.final_norm, xn, n, H, cfg_.rms_eps, s); });
  float* logits = scratch<float>(dc.logits, static_cast<size_t>(n) * cfg_.vocab);
  k::GemmEpilogue ep;
  ep.kind = k::kEpiStoreF32;
  ep.out = logits;
  ep.ldo = cfg_.vocab;
  timed(kPhLmHead, s, [&] { k::gemm(xn, H, dc.lm_head, H, n, cfg_.vocab, H, ep, s); });
  int32_t* d_out = scratch<int32_t>(dc.out_tok, n);
  timed(kPhArgmax, s, [&] { k::argmax_rows(logits, n, cfg_.vocab, d_out, s); });
  cuda_ok(cudaEventRecord(dc.e1, s), "event");
  note_host_enqueue(host_t0);
  check_cuda("prefill launch");
  std::vector<int32_t> first(static_cast<size_t>(n));
  cuda_ok(cudaMemcpyAsync(first.data(), d_out, n * 4, cudaMemcpyDeviceToHost, s), "d2h");
  if (a.logits_out) {
    cuda_ok(cudaMemcpyAsync(a.logits_out, logits, static_cast<size_t>(n) * cfg_.vocab * 4,
                            cudaMemcpyDeviceToHost, s),
            "d2h");
  }
  cuda_ok(cudaStreamSynchronize(s), "prefill");
  if (cap_armed_) cap_finish();
  collect_phase_events();
  float ms = 0;
  cuda_ok(cudaEventElapsedTime(&ms, dc.e0, dc.e1), "elapsed");
  if (a.device_ms_out) *a.device_ms_out = ms;
  last_prefill_.device_ms = ms;
  last_prefill_.kv_ring_rows = rows;
  for (int r = 0; r < n; ++r) {
    requests_[a.request_ids[r]].tokens.push_back(first[r]);
    if (a.first_token_out) a.first_token_out[r] = first[r];
  }
  ProfileRec pr{d, std::vector<int64_t>(a.input_lens, a.input_lens + n), ms};
  profiles_.push_back(std::move(pr));
}

void Runtime::o_and_mlp(DeviceCtx& dc, int l, int rows, bf16* x, const bf16* attn, bf16* xn,
                        bf16* hbuf, const NormFuse& nf, cudaStream_t s) {
  const int H = cfg_.hidden, F = cfg_.ffn;
  const LayerW& w = dc.layers[l];
  const bool fuse = nf.ss_o != nullptr;
  k::GemmEpilogue eo;
  eo.kind = k::kEpiResidual;
  eo.out = x;
  eo.ldo = H;
  if (fuse) {
    eo.ss_out = nf.ss_o;
    if (!nf.zero_in_kernel) {
      cuda_ok(cudaMemsetAsync(nf.ss_o, 0, static_cast<size_t>(rows) * sizeof(float), s), "memset");
    }
  }
  timed(kPhOProj, s, [&] { k::gemm(attn, H, w.wo, H, rows, H, H, eo, s); });
  if (!fuse) {
    timed(kPhNorm, s, [&] { k::rmsnorm(x, nullptr, nullptr, xn, rows, H, cfg_.rms_eps, s); });
  }
  k::GemmEpilogue eg;
  eg.kind = k::kEpiSiluMul;
  eg.out = hbuf;
  eg.ldo = F;
  if (fuse) {
    eg.ss_in = nf.ss_o;
    if (nf.zero_in_kernel) eg.ss_zero = nf.ss_d;
    eg.norm_dim = H;
    eg.norm_eps = cfg_.rms_eps;
  }
  timed(kPhGateUp, s, [&] { k::gemm(fuse ? x : xn, H, w.wgu, H, rows, 2 * F, H, eg, s); });
  k::GemmEpilogue ed;
  ed.kind = k::kEpiResidual;
  ed.out = x;
  ed.ldo = H;
  if (fuse) {
    ed.ss_out = nf.ss_d;
    if (!nf.zero_in_kernel) {
      cuda_ok(cudaMemsetAsync(nf.ss_d, 0, static_cast<size_t>(rows) * sizeof(float), s), "memset");
    }
  }
  timed(kPhDown, s, [&] { k::gemm(hbuf, F, w.wd, F, rows, H, F, ed, s); });
}

void Runtime::forward_layers_prefill(DeviceCtx& dc, int rows,
                                     const std::vector<k::RingSegment>& segs,
                                     const std::vector<int32_t>& work) {
  cudaStream_t s = dc.stream;
  const int H = cfg_.hidden, F = cfg_.ffn;
  bf16* x = static_cast<bf16*>(dc.x.ptr);
  bf16* xn = scratch<bf16>(dc.xn, static_cast<size_t>(rows) * H);
  bf16* q = scratch<bf16>(dc.q, static_cast<size_t>(rows) * H);
  bf16* kb = scratch<bf16>(dc.kb, static_cast<size_t>(rows) * H);
  bf16* vb = scratch<bf16>(dc.vb, static_cast<size_t>(rows) * H);
  bf16* attn = scratch<bf16>(dc.attn, static_cast<size_t>(rows) * H);
  bf16* hbuf = scratch<bf16>(dc.h, static_cast<size_t>(rows) * F);
  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  const int n_work = attention_n_work(work);
  // RMSNorm fused into the GEMMs (gains folded into the weights): the
  // residual epilogues (and embed) accumulate each row's sum of squares, the
  // consuming GEMM scales its accumulator rows. ss2 / ss1 are cleared before
  // the residual GEMM that fills them (their readers have completed).
  const bool fuse = fuse_norm_prefill();
  float* ss1 = fuse ? scratch<float>(dc.ss1, rows) : nullptr;
  float* ss2 = fuse ? scratch<float>(dc.ss2, rows) : nullptr;
  const bf16* a_in = fuse ? x : xn;
  for (int l = 0; l < cfg_.layers; ++l) {
    NvtxRange nvtx_layer("prefill layer");
    const LayerW& w = dc.layers[l];
    if (!fuse) {
      timed(kPhNorm, s, [&] { k::rmsnorm(x, nullptr, nullptr, xn, rows, H, cfg_.rms_eps, s); });
    }
    // QKV projection; epilogue: RoPE, ring stripe write, and the proactive
    // retention write of every token's K/V into its resting page slot.
    k::GemmEpilogue ep;
    ep.kind = k::kEpiQkvRope;
    ep.q_out = q;
    ep.k_out = kb;
    ep.v_out = vb;
    ep.pos = static_cast<const int32_t*>(dc.pos.ptr);
    ep.rope = dc.rope;
    ep.hidden = H;
    ep.head_dim = cfg_.head_dim;
    ep.row_inst = static_cast<const int32_t*>(dc.rinst.ptr);
    ep.row_slot = static_cast<const int32_t*>(dc.rslot.ptr);
    for (size_t j = 0; j < dc.slabs.size(); ++j) {
      const InstanceRec& in = instances_[dc.slabs[j]];
      ep.slab_k[j] = in.layer_k(l);
      ep.slab_v[j] = in.layer_v(l);
    }
    if (fuse) {
      ep.ss_in = ss1;
      ep.norm_dim = H;
      ep.norm_eps = cfg_.rms_eps;
    }
    timed(kPhQkv, s, [&] { k::gemm(a_in, H, w.wqkv, H, rows, 3 * H, H, ep, s); });
    // Striped ring attention over all d rounds.
    timed(kPhAttention, s, [&] {
      k::ring_attention(q, kb, vb, attn, rows, rows, cfg_.heads, cfg_.head_dim, static_cast<const k::RingSegment*>(dc.segs.ptr), static_cast<const int32_t*>(dc.work.ptr), n_work, scale, s);
    });
    if (cap_armed_) cap_layer(dc, l, attn, s);
    NormFuse nf;
    if (fuse) {
      nf.ss_o = ss2;
      nf.ss_d = ss1;
    }
    o_and_mlp(dc, l, rows, x, attn, xn, hbuf, nf, s);
  }
}

// ---- decode ----------------------------------------------------------------------
void Runtime::decode_step(const esp_decode_args& a) {
  NvtxRange nvtx("esp_decode_step");
  const auto host_t0 = std::chrono::steady_clock::now();
  const int b = a.batch_size;
  const bool has_chunk = a.chunk_tokens > 0;
  if (b <= 0 && !has_chunk) throw InternalError("decode step with neither batch nor chunk");
  if (b > 0 && (a.n_masters <= 0 || !a.masters)) throw InternalError("decode step without masters");
  std::vector<InstanceId> members(a.members, a.members + a.n_members);
  std::vector<InstanceId> masters;
  if (a.masters) masters.assign(a.masters, a.masters + a.n_masters);
  for (InstanceId m : masters) inst(m);
  for (InstanceId m : members) inst(m);
  std::vector<RequestId> batch(a.batch, a.batch + b);
  for (RequestId r : batch) {
    if (req(r).kv_tokens() == 0) throw InternalError("decode of a request without KV");
  }
  // Chunked prefill riding on the step (engine.cpp:432-462): validate before
  // any slot is taken.
  std::vector<std::pair<InstanceId, int64_t>> chunk_place;
  if (has_chunk) {
    if (a.chunk_n <= 0 || !a.chunk_instance || !a.chunk_tokens_on) {
      throw InternalError("chunk without a placement");
    }
    int64_t tot = 0;
    for (int i = 0; i < a.chunk_n; ++i) {
      inst(a.chunk_instance[i]);
      if (a.chunk_tokens_on[i] < 0) throw InternalError("negative chunk placement entry");
      chunk_place.emplace_back(a.chunk_instance[i], a.chunk_tokens_on[i]);
      tot += a.chunk_tokens_on[i];
    }
    if (tot != a.chunk_tokens) throw InternalError("chunk size inconsistent with its placement");
    for (RequestId r : batch) {
      if (r == a.chunk_request) throw InternalError("chunk names a request of the decode batch");
    }
    if (!devices_.empty() && !a.chunk_token_ids) {
      throw ConfigError("decode_step: chunk token ids required on a device runtime");
    }
  }
  // Masters exactly as the engine assigns them (engine.cpp:401,
  // esp_mechanics.cpp:220-238), then the append feasibility of
  // decode_step_comm (esp_mechanics.cpp:240-264).
  std::map<InstanceId, std::vector<RequestId>> assign;
  if (b > 0) {
    assign = assign_masters(batch, masters);
    std::map<InstanceId, Tokens> free;
    for (const auto& in : instances_) free[in.id] = in.capacity - in.used;
    decode_step_comm(static_cast<int>(members.size()), assign, free);
  }
  if (has_chunk) {
    // The appends are committed first, then the chunk (engine.cpp:408-462).
    std::map<InstanceId, int64_t> need;
    for (const auto& [m, reqs] : assign) need[m] += static_cast<int64_t>(reqs.size());
    for (const auto& [i, t] : chunk_place) need[i] += t;
    for (const auto& [i, t] : need) {
      if (inst(i).used + t > inst(i).capacity) {
        throw CapacityError(i, "chunk placement overflows instance " + std::to_string(i));
      }
    }
  }

  std::map<RequestId, int32_t> in_tok;
  for (int i = 0; i < b; ++i) {
    RequestRec& rr = req(batch[i]);
    if (a.in_tokens) {
      in_tok[batch[i]] = a.in_tokens[i];
    } else if (!rr.tokens.empty()) {
      in_tok[batch[i]] = rr.tokens.back();
    } else if (!devices_.empty()) {
      throw ConfigError("decode: no token history for request");
    }
  }
  // Rows ordered by master, then request id (the assignment order).
  using Row = DecodeRow;
  std::vector<Row> rows_v;
  std::vector<InstanceId> involved = members;
  for (const auto& [m, reqs] : assign) {
    for (RequestId r : reqs) {
      RequestRec& rr = req(r);
      const int32_t pos = static_cast<int32_t>(rr.kv_tokens());
      std::vector<int32_t> slot = take_slots(inst(m), 1);
      rr.pages[m].slots.push_back(slot[0]);
      rr.pages[m].pos.push_back(pos);
      rows_v.push_back({r, m, in_tok[r], pos, slot[0]});
      for (const auto& kv : rr.pages) involved.push_back(kv.first);
    }
  }
  // Chunk: earlier tokens of the request (any order: all precede the chunk),
  // then the chunk's own slots in token order (ascending instance).
  const int c = has_chunk ? static_cast<int>(a.chunk_tokens) : 0;
  std::vector<int32_t> prev_slab, prev_slot, ch_slab, ch_slot, ch_inst;
  int64_t p_prev = 0;
  if (has_chunk) {
    RequestRec& rr = requests_[a.chunk_request];
    rr.id = a.chunk_request;
    p_prev = rr.kv_tokens();
    for (const auto& [i, pl] : rr.pages) {
      for (int32_t sl : pl.slots) {
        prev_slab.push_back(inst(i).slab);
        prev_slot.push_back(sl);
      }
      involved.push_back(i);
    }
    for (const auto& [i, t] : chunk_place) {
      if (t == 0) continue;
      std::vector<int32_t> sl = take_slots(inst(i), t);
      PageList& pl = rr.pages[i];
      pl.slots.insert(pl.slots.end(), sl.begin(), sl.end());
      for (int32_t x : sl) {
        pl.pos.push_back(static_cast<int32_t>(p_prev + static_cast<int64_t>(ch_slot.size())));
        ch_slab.push_back(inst(i).slab);
        ch_slot.push_back(x);
        ch_inst.push_back(i);
      }
      involved.push_back(i);
    }
    if (a.chunk_token_ids) rr.tokens.insert(rr.tokens.end(), a.chunk_token_ids, a.chunk_token_ids + c);
    rr.input_len = p_prev + c;
  }
  if (devices_.empty()) {
    for (const Row& rw : rows_v) {
      if (a.in_tokens) req(rw.r).tokens.push_back(rw.token);
    }
    if (a.chunk_first_token_out) *a.chunk_first_token_out = -1;
    return;
  }
  if (tp_ > 1) {
    TpChunk tc;
    if (has_chunk) {
      tc.c = c;
      tc.p_prev = p_prev;
      tc.kv_slab = prev_slab;
      tc.kv_slot = prev_slot;
      tc.kv_slab.insert(tc.kv_slab.end(), ch_slab.begin(), ch_slab.end());
      tc.kv_slot.insert(tc.kv_slot.end(), ch_slot.begin(), ch_slot.end());
      tc.ch_slab = ch_slab;
      tc.ch_slot = ch_slot;
    }
    const double ms = decode_tp(a, rows_v, tc);
    if (b > 0 && !has_chunk) record_decode_profile(members, batch, a.n_masters, ms);
    return;
  }
  if (single_domain(involved) == nullptr) {
    double ms_dec = 0, ms_chunk = 0;
    if (b > 0) {
      esp_decode_args da = a;
      da.device_ms_out = &ms_dec;
      decode_multi(da, rows_v, batch);
    }
    if (has_chunk) {
      if (instances_.size() > static_cast<size_t>(k::kMaxSlabs)) {
        throw ConfigError("chunked prefill across domains needs <= 16 instances");
      }
      std::vector<std::pair<InstanceId, int32_t>> prev, cur;
      const RequestRec& rr = requests_[a.chunk_request];
      // earlier tokens: every slot of the request except the chunk's own
      std::map<InstanceId, size_t> own;
      for (size_t i = 0; i < ch_inst.size(); ++i) own[ch_inst[i]]++;
      for (const auto& [iid, pl] : rr.pages) {
        const size_t keep = pl.slots.size() - (own.count(iid) ? own[iid] : 0);
        for (size_t j = 0; j < keep; ++j) prev.emplace_back(iid, pl.slots[j]);
      }
      for (size_t i = 0; i < ch_inst.size(); ++i) cur.emplace_back(ch_inst[i], ch_slot[i]);
      chunk_multi(a, p_prev, prev, cur, &ms_chunk);
    }
    if (a.device_ms_out) *a.device_ms_out = ms_dec + ms_chunk;
    if (b > 0 && !has_chunk) record_decode_profile(members, batch, a.n_masters, ms_dec);
    return;
  }
  DeviceCtx& dc = device_of(involved, "decode_step");
  DeviceGuard g(dc.device);
  cudaStream_t s = dc.stream;
  const int H = cfg_.hidden, F = cfg_.ffn;
  const int rows = b + c;

  std::vector<int32_t> h_tok, h_pos, h_inst, h_slot, h_row_start;
  std::vector<k::DecodeChunk> chunks;
  for (int i = 0; i < b; ++i) {
    const Row& rw = rows_v[i];
    h_tok.push_back(rw.token);
    h_pos.push_back(rw.pos);
    h_inst.push_back(inst(rw.master).slab);
    h_slot.push_back(rw.slot);
    h_row_start.push_back(static_cast<int32_t>(chunks.size()));
    RequestRec& rr = req(rw.r);
    // Split-KV work: every instance holding the request's KV contributes a
    // partial over its own slots (multi-master distributed decoding).
    for (auto& [iid, pl] : rr.pages) {
      if (pl.slots.empty()) continue;
      sync_pages(pl, s);
      const int64_t nsl = static_cast<int64_t>(pl.slots.size());
      for (int64_t c0 = 0; c0 < nsl; c0 += decode_chunk()) {
        k::DecodeChunk ch{};
        ch.slots = pl.dev + c0;
        ch.n = static_cast<int32_t>(std::min<int64_t>(decode_chunk(), nsl - c0));
        ch.row = i;
        ch.slab = inst(iid).slab;
        ch.out = static_cast<int32_t>(chunks.size());
        chunks.push_back(ch);
      }
    }
  }
  h_row_start.push_back(static_cast<int32_t>(chunks.size()));
  for (int i = 0; i < c; ++i) {
    h_tok.push_back(a.chunk_token_ids[i]);
    h_pos.push_back(static_cast<int32_t>(p_prev + i));
    h_inst.push_back(ch_slab[i]);
    h_slot.push_back(ch_slot[i]);
  }
  const int n_chunks = static_cast<int>(chunks.size());
  int max_chunk = 0;
  for (const k::DecodeChunk& ch : chunks) max_chunk = std::max(max_chunk, static_cast<int>(ch.n));
  int64_t max_pos = p_prev + c;
  for (const Row& rw : rows_v) max_pos = std::max<int64_t>(max_pos, rw.pos + 1);
  ensure_rope(dc, max_pos);
  int32_t* d_tok = scratch<int32_t>(dc.tok, rows);
  int32_t* d_pos = scratch<int32_t>(dc.pos, rows);
  int32_t* d_inst = scratch<int32_t>(dc.rinst, rows);
  int32_t* d_slot = scratch<int32_t>(dc.rslot, rows);
  int32_t* d_rs = scratch<int32_t>(dc.row_start, b + 1);
  k::DecodeChunk* d_chunks = scratch<k::DecodeChunk>(dc.chunks, std::max<size_t>(chunks.size(), 1));
  cuda_ok(cudaMemcpyAsync(d_tok, h_tok.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_pos, h_pos.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_inst, h_inst.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_slot, h_slot.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
  cuda_ok(cudaMemcpyAsync(d_rs, h_row_start.data(), (b + 1) * 4, cudaMemcpyHostToDevice, s), "h2d");
  if (!chunks.empty()) {
    cuda_ok(cudaMemcpyAsync(d_chunks, chunks.data(), chunks.size() * sizeof(k::DecodeChunk),
                            cudaMemcpyHostToDevice, s),
            "h2d");
  }
  // Chunk attention: gather list (earlier tokens, then the chunk) and one
  // ring segment of d = 1 whose causal offset is the chunk's start:
  // query a (position p_prev + a) sees key b iff b <= a + p_prev.
  const int kv_n = static_cast<int>(p_prev) + c;
  int32_t* d_gslab = nullptr;
  int32_t* d_gslot = nullptr;
  std::vector<int32_t> work_sorted;
  // The request's slots in token order are often one ascending run on one
  // slab (one instance, a fresh free list): K1 then reads K/V straight from
  // the slab rows — no per-layer gather into contiguous buffers.
  int run_slab = -1, run_slot0 = 0;
  if (has_chunk) {
    std::vector<int32_t> gslab = prev_slab, gslot = prev_slot;
    gslab.insert(gslab.end(), ch_slab.begin(), ch_slab.end());
    gslot.insert(gslot.end(), ch_slot.begin(), ch_slot.end());
    // (earlier tokens may sit in any order — every one precedes the chunk;
    // the chunk's own rows must follow at kv rows p_prev + j)
    bool run = !gslot.empty();
    for (size_t i = 0; run && i < gslot.size(); ++i) {
      run = gslab[i] == gslab[0] && gslot[i] == gslot[0] + static_cast<int32_t>(i);
    }
    if (run) {
      run_slab = gslab[0];
      run_slot0 = gslot[0];
    }
    d_gslab = scratch<int32_t>(dc.ret_slab, kv_n);
    d_gslot = scratch<int32_t>(dc.ret_slot, kv_n);
    cuda_ok(cudaMemcpyAsync(d_gslab, gslab.data(), kv_n * 4, cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(d_gslot, gslot.data(), kv_n * 4, cudaMemcpyHostToDevice, s), "h2d");
    k::RingSegment sg{};
    sg.q_row0 = b;
    sg.q_len = c;
    sg.n_rounds = 1;
    sg.kv_row0[0] = 0;
    sg.kv_len[0] = kv_n;
    sg.shift[0] = -static_cast<int32_t>(p_prev);
    std::vector<k::RingSegment> segs{sg};
    build_attention_work(segs, cfg_.heads, work_sorted);
    k::RingSegment* d_segs = scratch<k::RingSegment>(dc.segs, 1);
    int32_t* d_work = scratch<int32_t>(dc.work, work_sorted.size());
    cuda_ok(cudaMemcpyAsync(d_segs, &sg, sizeof(sg), cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(d_work, work_sorted.data(), work_sorted.size() * 4,
                            cudaMemcpyHostToDevice, s),
            "h2d");
  }
  bf16* x = scratch<bf16>(dc.x, static_cast<size_t>(rows) * H);
  bf16* xn = scratch<bf16>(dc.xn, static_cast<size_t>(rows) * H);
  bf16* q = scratch<bf16>(dc.q, static_cast<size_t>(rows) * H);
  bf16* attn = scratch<bf16>(dc.attn, static_cast<size_t>(rows) * H);
  bf16* hbuf = scratch<bf16>(dc.h, static_cast<size_t>(rows) * F);
  bf16* kg = has_chunk ? scratch<bf16>(dc.kb, static_cast<size_t>(kv_n) * H) : nullptr;
  bf16* vg = has_chunk ? scratch<bf16>(dc.vb, static_cast<size_t>(kv_n) * H) : nullptr;
  float* part_o = scratch<float>(dc.part_o, static_cast<size_t>(std::max(n_chunks, 1)) * cfg_.heads * cfg_.head_dim);
  float* part_ml = scratch<float>(dc.part_ml, static_cast<size_t>(std::max(n_chunks, 1)) * cfg_.heads * 2);
  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  const int n_work = attention_n_work(work_sorted);
  // Decode-shaped steps (<= 32 rows): each layer RMSNorm is fused into the
  // skinny GEMMs — the residual epilogues accumulate row sums of squares
  // (ss1 before QKV, ss2 before gate_up) and the consuming GEMM scales its
  // accumulator rows (gains folded into the weights); no norm kernels.
  // Output buffers sized before the timed region: growing them after the
  // layers are enqueued (the final chunk adds a row) would put a
  // synchronising cudaFree / cudaMalloc inside the step.
  {
    const size_t n_out_max = static_cast<size_t>(b + (has_chunk ? 1 : 0));
    scratch<int32_t>(dc.last_rows, std::max<size_t>(n_out_max, 1));
    scratch<float>(dc.logits, std::max<size_t>(n_out_max, 1) * cfg_.vocab);
    scratch<int32_t>(dc.out_tok, std::max<size_t>(n_out_max, 1));
  }
  const bool fuse_norm = rows <= 32 && opts_.fuse_norm_decode;
  float* ss1 = scratch<float>(dc.ss1, 32);
  float* ss2 = scratch<float>(dc.ss2, 32);
  if (fuse_norm) cuda_ok(cudaMemsetAsync(ss2, 0, 32 * sizeof(float), s), "memset");
  const bf16* a_in = fuse_norm ? x : xn;  // the GEMMs' A operand after a norm

  cuda_ok(cudaEventRecord(dc.e0, s), "event");
  timed(kPhEmbed, s, [&] { k::embed(d_tok, dc.embed, x, rows, H, s, fuse_norm ? ss1 : nullptr); });
  for (int l = 0; l < cfg_.layers; ++l) {
    const LayerW& w = dc.layers[l];
    if (!fuse_norm) {
      timed(kPhNorm, s, [&] { k::rmsnorm(x, nullptr, nullptr, xn, rows, H, cfg_.rms_eps, s); });
    }
    k::GemmEpilogue ep;
    ep.kind = k::kEpiQkvRope;
    if (fuse_norm) {
      ep.ss_in = ss1;
      ep.ss_zero = ss2;
      ep.norm_dim = H;
      ep.norm_eps = cfg_.rms_eps;
    }
    ep.q_out = q;
    ep.pos = d_pos;
    ep.rope = dc.rope;
    ep.hidden = H;
    ep.head_dim = cfg_.head_dim;
    ep.row_inst = d_inst;  // append: the new tokens' K/V go to their page slots
    ep.row_slot = d_slot;
    k::DecodeSlabs slabs{};
    for (size_t j = 0; j < dc.slabs.size(); ++j) {
      const InstanceRec& in = instances_[dc.slabs[j]];
      ep.slab_k[j] = in.layer_k(l);
      ep.slab_v[j] = in.layer_v(l);
      slabs.k[j] = ep.slab_k[j];
      slabs.v[j] = ep.slab_v[j];
    }
    timed(kPhQkv, s, [&] { k::gemm(a_in, H, w.wqkv, H, rows, 3 * H, H, ep, s); });
    if (b > 0) {
      // One chunk per row (every request's KV <= decode_chunk() slots on one
      // instance): K3 normalises its partial in place, no K4 launch.
      const bool direct = n_chunks == b;
      timed(kPhDecodeAttn, s, [&] {
        k::decode_attention(q, d_chunks, n_chunks, slabs, cfg_.heads, cfg_.head_dim, scale,
                            part_o, part_ml, s, nullptr, direct ? attn : nullptr, max_chunk);
      });
      if (!direct) {
        timed(kPhCombine, s, [&] {
          k::decode_combine(part_o, part_ml, d_rs, b, cfg_.heads, cfg_.head_dim, attn, s);
        });
      }
    }
    if (has_chunk) {
      timed(kPhAttention, s, [&] {
        const bf16* kr = kg;
        const bf16* vr = vg;
        if (run_slab >= 0) {
          kr = slabs.k[run_slab] + static_cast<int64_t>(run_slot0) * H;
          vr = slabs.v[run_slab] + static_cast<int64_t>(run_slot0) * H;
        } else {
          k::gather_rows(slabs, d_gslab, d_gslot, kv_n, kg, vg, H, s);
        }
        k::ring_attention(q, kr, vr, attn, rows, kv_n, cfg_.heads, cfg_.head_dim,
                          static_cast<const k::RingSegment*>(dc.segs.ptr),
                          static_cast<const int32_t*>(dc.work.ptr), n_work, scale, s);
      });
    }
    NormFuse nf;
    if (fuse_norm) {
      nf.ss_o = ss2;
      nf.ss_d = ss1;
      nf.zero_in_kernel = true;
    }
    o_and_mlp(dc, l, rows, x, attn, xn, hbuf, nf, s);
  }
  // Output rows: the decode rows, then the chunk's last token when the chunk
  // completes the prompt (its first generated token, engine.cpp:570-579).
  const bool chunk_out = has_chunk && a.chunk_final != 0;
  const int n_out = b + (chunk_out ? 1 : 0);
  std::vector<int32_t> out_rows(static_cast<size_t>(b));
  for (int i = 0; i < b; ++i) out_rows[i] = i;
  if (chunk_out) out_rows.push_back(rows - 1);
  int32_t* d_out_rows = scratch<int32_t>(dc.last_rows, n_out);
  cuda_ok(cudaMemcpyAsync(d_out_rows, out_rows.data(), n_out * 4, cudaMemcpyHostToDevice, s), "h2d");
  timed(kPhNorm, s, [&] {
    k::rmsnorm(x, (n_out == rows) ? nullptr : d_out_rows, dc.final_norm, xn, n_out, H,
               cfg_.rms_eps, s);
  });
  float* logits = scratch<float>(dc.logits, static_cast<size_t>(std::max(n_out, 1)) * cfg_.vocab);
  int32_t* d_out = scratch<int32_t>(dc.out_tok, std::max(n_out, 1));
  if (n_out > 0) {
    k::GemmEpilogue ef;
    ef.kind = k::kEpiStoreF32;
    ef.out = logits;
    ef.ldo = cfg_.vocab;
    timed(kPhLmHead, s, [&] { k::gemm(xn, H, dc.lm_head, H, n_out, cfg_.vocab, H, ef, s); });
    timed(kPhArgmax, s, [&] { k::argmax_rows(logits, n_out, cfg_.vocab, d_out, s); });
  }
  cuda_ok(cudaEventRecord(dc.e1, s), "event");
  note_host_enqueue(host_t0);
  check_cuda("decode launch");
  std::vector<int32_t> out(static_cast<size_t>(std::max(n_out, 1)));
  if (n_out > 0) {
    cuda_ok(cudaMemcpyAsync(out.data(), d_out, n_out * 4, cudaMemcpyDeviceToHost, s), "d2h");
  }
  std::vector<float> lg;
  if ((a.logits_out && b > 0) || (chunk_out && a.chunk_logits_out)) {
    lg.resize(static_cast<size_t>(n_out) * cfg_.vocab);
    cuda_ok(cudaMemcpyAsync(lg.data(), logits, lg.size() * 4, cudaMemcpyDeviceToHost, s), "d2h");
  }
  cuda_ok(cudaStreamSynchronize(s), "decode");
  collect_phase_events();
  float ms = 0;
  cuda_ok(cudaEventElapsedTime(&ms, dc.e0, dc.e1), "elapsed");
  if (a.device_ms_out) *a.device_ms_out = ms;
  if (b > 0 && !has_chunk) record_decode_profile(members, batch, a.n_masters, ms);
  // Results back in the caller's batch order.
  std::map<RequestId, int> row_of;
  for (int i = 0; i < b; ++i) row_of[rows_v[i].r] = i;
  for (int i = 0; i < b; ++i) {
    const int ri = row_of[batch[i]];
    RequestRec& rr = req(batch[i]);
    if (a.in_tokens) rr.tokens.push_back(a.in_tokens[i]);
    rr.tokens.push_back(out[ri]);
    if (a.out_tokens) a.out_tokens[i] = out[ri];
    if (a.logits_out) {
      std::memcpy(a.logits_out + static_cast<size_t>(i) * cfg_.vocab,
                  lg.data() + static_cast<size_t>(ri) * cfg_.vocab, cfg_.vocab * sizeof(float));
    }
  }
  if (has_chunk) {
    if (chunk_out) {
      requests_[a.chunk_request].tokens.push_back(out[b]);
      if (a.chunk_first_token_out) *a.chunk_first_token_out = out[b];
      if (a.chunk_logits_out) {
        std::memcpy(a.chunk_logits_out, lg.data() + static_cast<size_t>(b) * cfg_.vocab,
                    cfg_.vocab * sizeof(float));
      }
    } else if (a.chunk_first_token_out) {
      *a.chunk_first_token_out = -1;
    }
  }
}

// ---- KV moves, frees, readback -------------------------------------------------------
void Runtime::move_kv(RequestId r, InstanceId from, InstanceId to, int64_t tokens) {
  NvtxRange nvtx("esp_move_kv");
  RequestRec& rr = req(r);
  InstanceRec& src = inst(from);
  InstanceRec& dst = inst(to);
  auto it = rr.pages.find(from);
  if (tokens < 0 || it == rr.pages.end() ||
      static_cast<int64_t>(it->second.slots.size()) < tokens) {
    throw InternalError("migration moves KV the request does not hold");
  }
  if (tokens == 0 || from == to) return;
  if (dst.used + tokens > dst.capacity) throw CapacityError(to, "migration target lacks room");
  PageList& spl = it->second;
  std::vector<int32_t> moving(spl.slots.end() - tokens, spl.slots.end());
  std::vector<int32_t> dslots = take_slots(dst, tokens);
  if (tp_ > 1) {
    // Tensor-parallel instances: every plane moves its own head shard.
    for (auto& pc : devices_) {
      DeviceCtx& dc = *pc;
      const int r = dc.domain;
      DeviceGuard g(dc.device);
      int32_t* d_a = scratch<int32_t>(dc.tok, static_cast<size_t>(tokens));
      int32_t* d_b = scratch<int32_t>(dc.pos, static_cast<size_t>(tokens));
      cuda_ok(cudaMemcpyAsync(d_a, moving.data(), tokens * 4, cudaMemcpyHostToDevice, dc.stream), "h2d");
      cuda_ok(cudaMemcpyAsync(d_b, dslots.data(), tokens * 4, cudaMemcpyHostToDevice, dc.stream), "h2d");
      const LazySlab& ss = r == 0 ? *src.k_slab : *src.tp_k[static_cast<size_t>(r - 1)];
      const LazySlab& ds = r == 0 ? *dst.k_slab : *dst.tp_k[static_cast<size_t>(r - 1)];
      k::copy_slots(src.plane_k(r, 0), src.plane_v(r, 0), d_a, dst.plane_k(r, 0),
                    dst.plane_v(r, 0), d_b, static_cast<int>(tokens), cfg_.layers,
                    ss.layer_stride_elems(), ds.layer_stride_elems(), cfg_.hidden / tp_, dc.stream);
    }
    check_cuda("move_kv");
    for (auto& pc : devices_) {
      DeviceGuard g(pc->device);
      cuda_ok(cudaStreamSynchronize(pc->stream), "move_kv");
    }
  } else if (!devices_.empty()) {
    // The copy runs on the destination domain's stream and reads the source
    // slab directly (same GPU, or a peer over NVLink with peer access on).
    DeviceCtx& sdc = *devices_[static_cast<size_t>(src.domain)];
    DeviceCtx& dc = *devices_[static_cast<size_t>(dst.domain)];
    if (&sdc != &dc) {
      DeviceGuard gs(sdc.device);
      cuda_ok(cudaStreamSynchronize(sdc.stream), "move_kv source");
    }
    DeviceGuard g(dc.device);
    int32_t* d_a = scratch<int32_t>(dc.tok, static_cast<size_t>(tokens));
    int32_t* d_b = scratch<int32_t>(dc.pos, static_cast<size_t>(tokens));
    cuda_ok(cudaMemcpyAsync(d_a, moving.data(), tokens * 4, cudaMemcpyHostToDevice, dc.stream), "h2d");
    cuda_ok(cudaMemcpyAsync(d_b, dslots.data(), tokens * 4, cudaMemcpyHostToDevice, dc.stream), "h2d");
    k::copy_slots(src.layer_k(0), src.layer_v(0), d_a, dst.layer_k(0), dst.layer_v(0), d_b,
                  static_cast<int>(tokens), cfg_.layers, src.k_slab->layer_stride_elems(),
                  dst.k_slab->layer_stride_elems(), cfg_.hidden, dc.stream);
    check_cuda("move_kv");
    cuda_ok(cudaStreamSynchronize(dc.stream), "move_kv");
  }
  const std::vector<int32_t> moving_pos(spl.pos.end() - tokens, spl.pos.end());
  spl.slots.resize(spl.slots.size() - static_cast<size_t>(tokens));
  spl.pos.resize(spl.slots.size());
  if (spl.dev_n > static_cast<int64_t>(spl.slots.size())) spl.dev_n = static_cast<int64_t>(spl.slots.size());
  release_slots(src, moving);
  PageList& dpl = rr.pages[to];
  dpl.slots.insert(dpl.slots.end(), dslots.begin(), dslots.end());
  dpl.pos.insert(dpl.pos.end(), moving_pos.begin(), moving_pos.end());
  if (spl.slots.empty()) {
    if (spl.dev) cudaFree(spl.dev);
    rr.pages.erase(from);
  }
}

void Runtime::free_request(RequestId r) {
  auto it = requests_.find(r);
  if (it == requests_.end()) return;
  for (auto& [i, pl] : it->second.pages) {
    release_slots(inst(i), pl.slots);
    if (pl.dev) cudaFree(pl.dev);
  }
  requests_.erase(it);
}

void Runtime::query_placement(RequestId r, int32_t* out_inst, int64_t* out_tok, int32_t cap,
                              int32_t* n) const {
  auto it = requests_.find(r);
  int32_t cnt = 0;
  if (it != requests_.end()) {
    for (const auto& [i, pl] : it->second.pages) {
      if (pl.slots.empty()) continue;
      if (cnt < cap) {
        out_inst[cnt] = i;
        out_tok[cnt] = static_cast<int64_t>(pl.slots.size());
      }
      ++cnt;
    }
  }
  *n = cnt;
}

void Runtime::instance_info(InstanceId i, int64_t* cap, int64_t* used) const {
  const InstanceRec& in = inst(i);
  if (cap) *cap = in.capacity;
  if (used) *used = in.used;
}

void Runtime::request_tokens(RequestId r, int32_t* out, int32_t cap, int32_t* n) const {
  const RequestRec& rr = req(r);
  const int32_t cnt = static_cast<int32_t>(rr.tokens.size());
  for (int32_t i = 0; i < std::min(cap, cnt); ++i) out[i] = rr.tokens[i];
  *n = cnt;
}

void Runtime::check_conservation() {
  // Host counters vs page tables (KvPool::check_conservation, cluster.cpp:113-132).
  std::map<InstanceId, int64_t> held;
  for (const auto& [rid, rr] : requests_) {
    for (const auto& [i, pl] : rr.pages) held[i] += static_cast<int64_t>(pl.slots.size());
  }
  for (const auto& in : instances_) {
    if (in.used != held[in.id]) {
      throw InternalError("instance " + std::to_string(in.id) +
                          " used counter drifted from placements");
    }
    if (in.used > in.capacity) {
      throw InternalError("instance " + std::to_string(in.id) + " holds more KV than its capacity");
    }
    if (in.used + static_cast<int64_t>(in.free_stack.size()) != in.capacity) {
      throw InternalError("instance " + std::to_string(in.id) + " free list drifted");
    }
  }
  if (devices_.empty()) return;
  // Device page tables: recount every slot on the device.
  for (auto& in : instances_) {
    DeviceCtx& dc = device_of({in.id}, "check_conservation");
    DeviceGuard g(dc.device);
    cudaStream_t s = dc.stream;
    int32_t* counts = scratch<int32_t>(dc.counts, static_cast<size_t>(in.capacity) + 1);
    int32_t* res = scratch<int32_t>(dc.result, 2);
    cuda_ok(cudaMemsetAsync(counts, 0, (static_cast<size_t>(in.capacity) + 1) * 4, s), "memset");
    cuda_ok(cudaMemsetAsync(res, 0, 8, s), "memset");
    for (auto& [rid, rr] : requests_) {
      auto it = rr.pages.find(in.id);
      if (it == rr.pages.end() || it->second.slots.empty()) continue;
      sync_pages(it->second, s);
      k::count_slots(it->second.dev, static_cast<int64_t>(it->second.slots.size()), counts,
                     static_cast<int>(in.capacity), s);
    }
    k::check_counts(counts, static_cast<int>(in.capacity), res, s);
    int32_t h[2] = {0, 0};
    cuda_ok(cudaMemcpyAsync(h, res, 8, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_ok(cudaStreamSynchronize(s), "conservation");
    if (h[0] != in.used || h[1] != 0) {
      throw InternalError("device page tables of instance " + std::to_string(in.id) +
                          " disagree: " + std::to_string(h[0]) + " slots mapped, " +
                          std::to_string(h[1]) + " conflicts, host used " +
                          std::to_string(in.used));
    }
  }
}

void Runtime::record_decode_profile(const std::vector<InstanceId>& members,
                                    const std::vector<RequestId>& batch, int n_masters,
                                    double ms) {
  int64_t resident = 0;
  for (RequestId r : batch) resident += req(r).kv_tokens();
  decode_profiles_.push_back(DecodeProfileRec{static_cast<int>(members.size()),
                                              static_cast<int>(batch.size()), n_masters,
                                              resident, ms});
}

void Runtime::dump_profiles(const std::string& path) const {
  std::ofstream out(path, std::ios::app);
  if (!out) throw ConfigError("cannot write profile file: " + path);
  for (const ProfileRec& p : profiles_) {
    out << "{\"dop\": " << p.dop << ", \"tp\": 1, \"kind\": \"profile\", \"lengths\": [";
    for (size_t i = 0; i < p.lengths.size(); ++i) out << (i ? ", " : "") << p.lengths[i];
    out << "], \"measured_ms\": " << std::setprecision(9) << p.ms << "}\n";
  }
}

// ---- parity readback -----------------------------------------------------------------
void Runtime::read_kv(RequestId r, int layer, void* k_out, void* v_out, int64_t cap, int64_t* n) {
  RequestRec& rr = req(r);
  const int64_t total = rr.kv_tokens();
  if (n) *n = total;
  if (layer < 0 || layer >= cfg_.layers) throw ConfigError("read_kv: layer out of range");
  if (devices_.empty()) throw NoDeviceError("read_kv needs a device runtime");
  if (cap < total) return;  // size query
  // tp > 1: plane p holds columns [p H/tp, (p+1) H/tp) of every slot (same
  // slot ids on every plane); the page list lives on plane 0's GPU.
  const size_t H = static_cast<size_t>(cfg_.hidden);
  const size_t Hc = H / static_cast<size_t>(tp_);
  std::vector<uint16_t> kh, vh;
  for (auto& [iid, pl] : rr.pages) {
    const int64_t m = static_cast<int64_t>(pl.slots.size());
    if (m == 0) continue;
    InstanceRec& in = inst(iid);
    {
      DeviceCtx& home = *devices_[static_cast<size_t>(tp_ > 1 ? 0 : in.domain)];
      DeviceGuard g(home.device);
      sync_pages(pl, home.stream);
      cuda_ok(cudaStreamSynchronize(home.stream), "read_kv pages");
    }
    for (int p = 0; p < tp_; ++p) {
      DeviceCtx& dc = *devices_[static_cast<size_t>(tp_ > 1 ? p : in.domain)];
      DeviceGuard g(dc.device);
      cudaStream_t s = dc.stream;
      std::vector<int32_t> zero(static_cast<size_t>(m), 0);
      int32_t* d_slab = scratch<int32_t>(dc.ret_slab, static_cast<size_t>(m));
      cuda_ok(cudaMemcpyAsync(d_slab, zero.data(), m * 4, cudaMemcpyHostToDevice, s), "h2d");
      k::DecodeSlabs src{};
      src.k[0] = in.plane_k(p, layer);
      src.v[0] = in.plane_v(p, layer);
      bf16* ko = scratch<bf16>(dc.kb, static_cast<size_t>(m) * Hc);
      bf16* vo = scratch<bf16>(dc.vb, static_cast<size_t>(m) * Hc);
      k::gather_rows(src, d_slab, pl.dev, static_cast<int>(m), ko, vo, static_cast<int>(Hc), s);
      kh.resize(static_cast<size_t>(m) * Hc);
      vh.resize(static_cast<size_t>(m) * Hc);
      cuda_ok(cudaMemcpyAsync(kh.data(), ko, kh.size() * 2, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_ok(cudaMemcpyAsync(vh.data(), vo, vh.size() * 2, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_ok(cudaStreamSynchronize(s), "read_kv");
      for (int64_t j = 0; j < m; ++j) {
        const int64_t q = pl.pos[static_cast<size_t>(j)];
        if (q < 0 || q >= total) throw InternalError("read_kv: token position out of range");
        const size_t off = static_cast<size_t>(q) * H + static_cast<size_t>(p) * Hc;
        std::memcpy(static_cast<uint16_t*>(k_out) + off, kh.data() + j * Hc, Hc * 2);
        std::memcpy(static_cast<uint16_t*>(v_out) + off, vh.data() + j * Hc, Hc * 2);
      }
    }
  }
}

void Runtime::capture_attention(const int64_t* pos, int64_t n) {
  if (devices_.empty()) throw NoDeviceError("capture_attention needs a device runtime");
  cap_pos_.assign(pos, pos + n);
  cap_armed_ = n > 0;
  cap_host_.clear();
  cap_rows_ = 0;
}

void Runtime::captured_attention(void* out, int64_t cap_rows, int64_t* n) {
  if (n) *n = cap_rows_;
  if (!out || cap_rows < cap_rows_) return;
  std::memcpy(out, cap_host_.data(), cap_host_.size() * 2);
}

void Runtime::cap_add(int dom, int32_t row, int32_t idx) {
  CapDomain& c = cap_dom_[dom];
  c.rows.push_back(row);
  c.idx.push_back(idx);
}

void Runtime::cap_layer(DeviceCtx& dc, int l, const bf16* attn, cudaStream_t s) {
  auto it = cap_dom_.find(dc.domain);
  if (it == cap_dom_.end() || it->second.rows.empty()) return;
  CapDomain& c = it->second;
  const int m = static_cast<int>(c.rows.size());
  const size_t H = static_cast<size_t>(cfg_.hidden / tp_);  // tp > 1: this plane's head columns
  if (!c.d_rows) {
    cuda_ok(cudaMalloc(&c.d_rows, static_cast<size_t>(m) * 4), "cudaMalloc(capture)");
    cuda_ok(cudaMalloc(&c.d_buf, static_cast<size_t>(cfg_.layers) * m * H * 2), "cudaMalloc(capture)");
    cuda_ok(cudaMemcpyAsync(c.d_rows, c.rows.data(), static_cast<size_t>(m) * 4,
                            cudaMemcpyHostToDevice, s),
            "h2d");
  }
  k::copy_rows(attn, c.d_rows, m, c.d_buf + static_cast<size_t>(l) * m * H, static_cast<int>(H), s);
}

void Runtime::cap_finish() {
  const size_t H = static_cast<size_t>(cfg_.hidden), N = cap_pos_.size();
  const size_t Hc = H / static_cast<size_t>(tp_);  // tp > 1: domain = plane, its head columns
  cap_host_.assign(static_cast<size_t>(cfg_.layers) * N * H, 0);
  for (auto& [dom, c] : cap_dom_) {
    const size_t m = c.rows.size();
    if (m == 0 || !c.d_buf) continue;
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    std::vector<uint16_t> h(static_cast<size_t>(cfg_.layers) * m * Hc);
    cuda_ok(cudaMemcpy(h.data(), c.d_buf, h.size() * 2, cudaMemcpyDeviceToHost), "d2h");
    const size_t col = tp_ > 1 ? static_cast<size_t>(dom) * Hc : 0;
    for (int l = 0; l < cfg_.layers; ++l) {
      for (size_t j = 0; j < m; ++j) {
        std::memcpy(cap_host_.data() + (static_cast<size_t>(l) * N + c.idx[j]) * H + col,
                    h.data() + (static_cast<size_t>(l) * m + j) * Hc, Hc * 2);
      }
    }
    cudaFree(c.d_rows);
    cudaFree(c.d_buf);
  }
  cap_dom_.clear();
  cap_rows_ = static_cast<int64_t>(N) * cfg_.layers;
  cap_armed_ = false;
}

bool Runtime::slab_accessible(InstanceId i, int device) const {
  const InstanceRec& in = inst(i);
  if (!in.k_slab) return false;
  return in.k_slab->readable_writable_by(device) && in.v_slab->readable_writable_by(device);
}

}  // namespace esp
