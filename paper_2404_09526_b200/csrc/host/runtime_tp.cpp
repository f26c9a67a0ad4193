// Tensor-parallel elastic instances (StrategyKey.tp,
// types.hpp:36-41; the paper's TP = 2 x ESP = 4 deployment).
//
// Every instance spans `tp` GPUs ("planes"). Plane r holds heads
// [r H/tp, (r+1) H/tp) of every instance's KV (same slot ids on every plane,
// so page tables, counters and the reference's placement are unchanged) and
// the Megatron shards of the weights: QKV and gate_up column-parallel (the
// plane's heads / FFN columns), O and down row-parallel. Per layer the two
// row-parallel projections write fp32 partials of the full hidden width; each
// plane then adds ALL planes' partials, in plane order, to its replicated
// residual stream (k::tp_reduce_residual_norm, reading the other planes'
// partials over NVLink, fused with the next RMSNorm) — every plane computes the same bits, so no broadcast follows.
// Attention needs no exchange: K1 / K3 run on the plane's own heads. The ESP
// machinery is unchanged inside a plane: the ring prefill (striped rows,
// retention into resting page slots) and multi-master split-KV decode run
// co-located on each plane over its head shard. The LM head runs on plane 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <map>
#include <set>

#include "../kernels/synthetic.h"
#include "device_ctx.hpp"
#include "runtime.hpp"

namespace esp {

Runtime::Runtime(const esp_model_config& cfg, int n_instances, int tp, const int32_t* plane_devices,
                 int64_t kv_capacity)
    : cfg_(cfg) {
  read_options();
  if (n_instances <= 0) throw ConfigError("need at least one instance");
  if (tp < 2 || tp > k::kMaxTp) throw ConfigError("tp must be 2..8");
  if (!plane_devices) throw ConfigError("tensor-parallel runtime needs plane devices");
  if (kv_capacity <= 0) throw ConfigError("tensor-parallel runtime needs kv_capacity > 0");
  if (cfg.layers <= 0 || cfg.hidden <= 0 || cfg.heads <= 0 || cfg.head_dim <= 0 ||
      cfg.ffn <= 0 || cfg.vocab <= 0) {
    throw ConfigError("model config fields must be positive");
  }
  if (cfg.heads * cfg.head_dim != cfg.hidden) throw ConfigError("hidden != heads * head_dim");
  if (cfg.head_dim != 64 && cfg.head_dim != 128) throw ConfigError("head_dim must be 64 or 128");
  if (cfg.hidden % 256 != 0 || cfg.ffn % 64 != 0 || cfg.vocab % 128 != 0) {
    throw ConfigError("hidden % 256, ffn % 64 and vocab % 128 must be 0");
  }
  // Shard shapes the GEMMs take: QKV / O tiles of 128 columns, gate_up in
  // 128-row gate|up blocks, K in 64-wide blocks.
  if (cfg.heads % tp != 0 || (cfg.hidden / tp) % 128 != 0 || cfg.ffn % tp != 0 ||
      (cfg.ffn / tp) % 64 != 0) {
    throw ConfigError("tp must divide heads, hidden / tp % 128 and ffn / tp % 64 must be 0");
  }
  if (opts_.domain_per_instance) {
    throw ConfigError("ESP_DOMAIN_PER_INSTANCE is not supported with tp > 1");
  }
  if (n_instances > k::kMaxSlabs) throw ConfigError("too many instances on one plane");
  int ndev = 0;
  cuda_ok(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  tp_ = tp;
  instances_.resize(static_cast<size_t>(n_instances));
  for (int r = 0; r < tp; ++r) {
    const int d = plane_devices[r];
    if (d < 0 || d >= ndev) throw ConfigError("plane device ordinal out of range");
    devices_.push_back(std::make_unique<DeviceCtx>());
    devices_.back()->device = d;
    devices_.back()->domain = r;
    for (int i = 0; i < n_instances; ++i) devices_.back()->slabs.push_back(i);
  }
  for (int i = 0; i < n_instances; ++i) {
    instances_[i].id = i;
    instances_[i].device = plane_devices[0];
    instances_[i].domain = 0;  // host bookkeeping runs as one co-location domain
    instances_[i].slab = i;
  }
  std::set<int> phys(plane_devices, plane_devices + tp);
  for (int a : phys) {
    for (int b : phys) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can) {
        throw ConfigError("GPU " + std::to_string(a) + " cannot access GPU " + std::to_string(b) +
                          ": the tensor-parallel all-reduce reads peer memory");
      }
      DeviceGuard g(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_ok(e, "peer access");
      cudaGetLastError();
    }
  }
  for (int r = 0; r < tp; ++r) init_device_tp(*devices_[r], r);
  const size_t row_bytes = static_cast<size_t>(cfg.hidden / tp) * 2;
  for (auto& in : instances_) {
    in.capacity = kv_capacity;
    in.k_slab = std::make_unique<LazySlab>();
    in.v_slab = std::make_unique<LazySlab>();
    in.k_slab->reserve(plane_devices[0], cfg.layers, kv_capacity, row_bytes);
    in.v_slab->reserve(plane_devices[0], cfg.layers, kv_capacity, row_bytes);
    for (int r = 1; r < tp; ++r) {
      in.tp_k.push_back(std::make_unique<LazySlab>());
      in.tp_v.push_back(std::make_unique<LazySlab>());
      DeviceGuard g(plane_devices[r]);
      in.tp_k.back()->reserve(plane_devices[r], cfg.layers, kv_capacity, row_bytes);
      in.tp_v.back()->reserve(plane_devices[r], cfg.layers, kv_capacity, row_bytes);
    }
    if (in.capacity > INT32_MAX) throw ConfigError("kv_capacity exceeds int32 slot ids");
    in.free_stack.resize(static_cast<size_t>(in.capacity));
    for (int64_t s = 0; s < in.capacity; ++s) {
      in.free_stack[static_cast<size_t>(s)] = static_cast<int32_t>(in.capacity - 1 - s);
    }
  }
}

void Runtime::init_device_tp(DeviceCtx& dc, int rank) {
  DeviceGuard g(dc.device);
  cuda_ok(cudaStreamCreateWithFlags(&dc.stream, cudaStreamNonBlocking), "stream");
  cuda_ok(cudaEventCreate(&dc.e0), "event");
  cuda_ok(cudaEventCreate(&dc.e1), "event");
  cuda_ok(cudaEventCreateWithFlags(&dc.tp_ev_o, cudaEventDisableTiming), "event");
  cuda_ok(cudaEventCreateWithFlags(&dc.tp_ev_d, cudaEventDisableTiming), "event");
  cuda_ok(cudaEventCreateWithFlags(&dc.tp_ev_r, cudaEventDisableTiming), "event");
  const int64_t H = cfg_.hidden, F = cfg_.ffn, V = cfg_.vocab;
  const int64_t Hs = H / tp_, Fs = F / tp_;
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
    // column-parallel: this plane's q | k | v rows (its heads), its gate|up blocks
    w.wqkv = alloc(3 * Hs * H);
    k::init_weight_shard(w.wqkv, 3 * Hs, H, seed, k::kTensorQ, l, 1, Hs, rank * Hs, 0, H, s);
    w.wgu = alloc(2 * Fs * H);
    k::init_weight_shard(w.wgu, 2 * Fs, H, seed, k::kTensorGate, l, 2, 0, rank * 2 * Fs, 0, H, s);
    // row-parallel: the input columns of this plane's heads / FFN columns
    w.wo = alloc(H * Hs);
    k::init_weight_shard(w.wo, H, Hs, seed, k::kTensorO, l, 0, H, 0, rank * Hs, H, s);
    w.wd = alloc(H * Fs);
    k::init_weight_shard(w.wd, H, Fs, seed, k::kTensorDown, l, 0, H, 0, rank * Fs, F, s);
    w.norm1 = alloc(H);
    k::fill_bf16(w.norm1, H, 1.0f, s);
    w.norm2 = alloc(H);
    k::fill_bf16(w.norm2, H, 1.0f, s);
    k::scale_cols(w.wqkv, 3 * Hs, H, w.norm1, s);  // norm gains folded as on one GPU
    k::scale_cols(w.wgu, 2 * Fs, H, w.norm2, s);
  }
  check_cuda("init tp weights");
  cuda_ok(cudaStreamSynchronize(s), "init weights sync");
}

namespace {

// Every plane's stream waits for `ev` of every other plane.
void wait_planes(std::vector<std::unique_ptr<DeviceCtx>>& planes,
                 cudaEvent_t DeviceCtx::*ev) {
  for (auto& p : planes) {
    for (auto& q : planes) {
      if (p == q) continue;
      DeviceGuard g(p->device);
      cuda_ok(cudaStreamWaitEvent(p->stream, (*q).*ev, 0), "tp wait");
    }
  }
}

}  // namespace

// One layer's dense half on every plane, split around the two all-reduces:
// O partial -> reduce -> norm -> gate_up -> down partial -> reduce.
// x / xn / attn / h are each plane's buffers (rows x H, rows x H, rows x Hs,
// rows x Fs); norm kernels with unit gain (gains folded into the weights).
static void tp_dense_half(Runtime* self, std::vector<std::unique_ptr<DeviceCtx>>& planes, int l,
                          int rows, int H, int F, int tp, float eps);

void Runtime::prefill_tp(const esp_prefill_args& a,
                         const std::vector<std::vector<int32_t>>& tok_slab,
                         const std::vector<std::vector<int32_t>>& tok_slot,
                         const std::vector<int64_t>& tok_base) {
  const int n = a.n_requests, d = a.dop, t = tp_;
  const int H = cfg_.hidden, F = cfg_.ffn, Hs = H / t, Fs = F / t, hs = cfg_.heads / t;
  const StripePlan sp = plan_stripes(a, tok_slab, tok_slot, tok_base);
  const int rows = sp.rows;
  if (cap_armed_) {  // parity capture: the same stripe rows on every plane (its head columns)
    if (n != 1) throw ConfigError("attention capture needs a single-request prefill");
    for (size_t c = 0; c < cap_pos_.size(); ++c) {
      const int64_t tt = cap_pos_[c];
      if (tt < 0 || tt >= a.input_lens[0]) throw ConfigError("capture position outside the prompt");
      for (int p = 0; p < t; ++p) {
        cap_add(p, sp.row0[tt % d][0] + static_cast<int32_t>(tt / d), static_cast<int32_t>(c));
      }
    }
  }
  std::vector<int32_t> work_sorted;
  build_attention_work(sp.segs, hs, work_sorted);
  const int n_work = attention_n_work(work_sorted);
  int64_t max_len = 0;
  for (int r = 0; r < n; ++r) max_len = std::max(max_len, a.input_lens[r]);
  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  DeviceCtx& d0 = *devices_[0];
  {
    DeviceGuard g(d0.device);
    cuda_ok(cudaEventRecord(d0.e0, d0.stream), "event");
  }
  for (auto& pc : devices_) {
    DeviceCtx& dc = *pc;
    DeviceGuard g(dc.device);
    cudaStream_t s = dc.stream;
    if (&dc != &d0) cuda_ok(cudaStreamWaitEvent(s, d0.e0, 0), "tp start");
    ensure_rope(dc, max_len);
    int32_t* d_tok = scratch<int32_t>(dc.tok, rows);
    cuda_ok(cudaMemcpyAsync(d_tok, sp.tok.data(), rows * 4, cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(scratch<int32_t>(dc.pos, rows), sp.pos.data(), rows * 4,
                            cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(scratch<int32_t>(dc.rinst, rows), sp.inst.data(), rows * 4,
                            cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(scratch<int32_t>(dc.rslot, rows), sp.slot.data(), rows * 4,
                            cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(scratch<k::RingSegment>(dc.segs, sp.segs.size()), sp.segs.data(),
                            sp.segs.size() * sizeof(k::RingSegment), cudaMemcpyHostToDevice, s),
            "h2d");
    cuda_ok(cudaMemcpyAsync(scratch<int32_t>(dc.work, work_sorted.size()), work_sorted.data(),
                            work_sorted.size() * 4, cudaMemcpyHostToDevice, s), "h2d");
    bf16* x = scratch<bf16>(dc.x, static_cast<size_t>(rows) * H);
    scratch<bf16>(dc.xn, static_cast<size_t>(std::max(rows, n)) * H);
    scratch<bf16>(dc.q, static_cast<size_t>(rows) * Hs);
    scratch<bf16>(dc.kb, static_cast<size_t>(rows) * Hs);
    scratch<bf16>(dc.vb, static_cast<size_t>(rows) * Hs);
    scratch<bf16>(dc.attn, static_cast<size_t>(rows) * Hs);
    scratch<bf16>(dc.h, static_cast<size_t>(rows) * Fs);
    // reduce-scatter layout: tp blocks of ceil(rows / tp) rows
    const size_t part_rows = static_cast<size_t>((rows + t - 1) / t) * t;
    scratch<float>(dc.tp_po, part_rows * H);
    scratch<float>(dc.tp_pd, part_rows * H);
    k::embed(d_tok, dc.embed, x, rows, H, s, nullptr);
  }
  for (int l = 0; l < cfg_.layers; ++l) {
    NvtxRange nvtx_layer("tp prefill layer");
    for (auto& pc : devices_) {
      DeviceCtx& dc = *pc;
      DeviceGuard g(dc.device);
      cudaStream_t s = dc.stream;
      bf16* x = static_cast<bf16*>(dc.x.ptr);
      bf16* xn = static_cast<bf16*>(dc.xn.ptr);
      // layer 0 normalises the embeddings; later layers' xn came with the
      // previous layer's down all-reduce
      if (l == 0) k::rmsnorm(x, nullptr, nullptr, xn, rows, H, cfg_.rms_eps, s);
      k::GemmEpilogue ep;
      ep.kind = k::kEpiQkvRope;
      ep.q_out = static_cast<bf16*>(dc.q.ptr);
      ep.k_out = static_cast<bf16*>(dc.kb.ptr);
      ep.v_out = static_cast<bf16*>(dc.vb.ptr);
      ep.pos = static_cast<const int32_t*>(dc.pos.ptr);
      ep.rope = dc.rope;
      ep.hidden = Hs;  // this plane's heads: q | k | v regions of Hs columns
      ep.head_dim = cfg_.head_dim;
      ep.row_inst = static_cast<const int32_t*>(dc.rinst.ptr);
      ep.row_slot = static_cast<const int32_t*>(dc.rslot.ptr);
      for (size_t j = 0; j < dc.slabs.size(); ++j) {
        const InstanceRec& in = instances_[dc.slabs[j]];
        ep.slab_k[j] = in.plane_k(dc.domain, l);
        ep.slab_v[j] = in.plane_v(dc.domain, l);
      }
      const LayerW& w = dc.layers[l];
      k::gemm(xn, H, w.wqkv, H, rows, 3 * Hs, H, ep, s);
      k::ring_attention(static_cast<bf16*>(dc.q.ptr), static_cast<bf16*>(dc.kb.ptr),
                        static_cast<bf16*>(dc.vb.ptr), static_cast<bf16*>(dc.attn.ptr), rows, rows,
                        hs, cfg_.head_dim, static_cast<const k::RingSegment*>(dc.segs.ptr),
                        static_cast<const int32_t*>(dc.work.ptr), n_work, scale, s);
      if (cap_armed_) cap_layer(dc, l, static_cast<bf16*>(dc.attn.ptr), s);
    }
    tp_dense_half(this, devices_, l, rows, H, F, t, cfg_.rms_eps);
  }
  // Last prompt token of each request: position len-1 lives at ring position
  // (len-1) mod d, stripe index (len-1) / d. LM head on plane 0.
  std::vector<int32_t> last(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) {
    const int64_t tt = a.input_lens[r] - 1;
    last[r] = sp.row0[tt % d][r] + static_cast<int32_t>(tt / d);
  }
  for (auto& pc : devices_) {  // plane 0 finishes after every plane's last reduce
    if (pc.get() == &d0) continue;
    DeviceGuard g(pc->device);
    cuda_ok(cudaEventRecord(pc->tp_ev_d, pc->stream), "event");
    DeviceGuard g0(d0.device);
    cuda_ok(cudaStreamWaitEvent(d0.stream, pc->tp_ev_d, 0), "tp end");
  }
  DeviceGuard g(d0.device);
  cudaStream_t s = d0.stream;
  int32_t* d_last = scratch<int32_t>(d0.last_rows, n);
  cuda_ok(cudaMemcpyAsync(d_last, last.data(), n * 4, cudaMemcpyHostToDevice, s), "h2d");
  bf16* xn = static_cast<bf16*>(d0.xn.ptr);
  k::rmsnorm(static_cast<bf16*>(d0.x.ptr), d_last, d0.final_norm, xn, n, H, cfg_.rms_eps, s);
  float* logits = scratch<float>(d0.logits, static_cast<size_t>(n) * cfg_.vocab);
  k::GemmEpilogue ef;
  ef.kind = k::kEpiStoreF32;
  ef.out = logits;
  ef.ldo = cfg_.vocab;
  k::gemm(xn, H, d0.lm_head, H, n, cfg_.vocab, H, ef, s);
  int32_t* d_out = scratch<int32_t>(d0.out_tok, n);
  k::argmax_rows(logits, n, cfg_.vocab, d_out, s);
  cuda_ok(cudaEventRecord(d0.e1, s), "event");
  check_cuda("tp prefill launch");
  std::vector<int32_t> first(static_cast<size_t>(n));
  cuda_ok(cudaMemcpyAsync(first.data(), d_out, n * 4, cudaMemcpyDeviceToHost, s), "d2h");
  if (a.logits_out) {
    cuda_ok(cudaMemcpyAsync(a.logits_out, logits, static_cast<size_t>(n) * cfg_.vocab * 4,
                            cudaMemcpyDeviceToHost, s), "d2h");
  }
  for (auto& pc : devices_) {
    DeviceGuard gp(pc->device);
    cuda_ok(cudaStreamSynchronize(pc->stream), "tp prefill");
  }
  if (cap_armed_) cap_finish();
  float ms = 0;
  cuda_ok(cudaEventElapsedTime(&ms, d0.e0, d0.e1), "elapsed");
  if (a.device_ms_out) *a.device_ms_out = ms;
  last_prefill_.device_ms = ms;
  last_prefill_.kv_ring_rows = rows;
  for (int r = 0; r < n; ++r) {
    requests_[a.request_ids[r]].tokens.push_back(first[r]);
    if (a.first_token_out) a.first_token_out[r] = first[r];
  }
  profiles_.push_back(ProfileRec{d, std::vector<int64_t>(a.input_lens, a.input_lens + n), ms});
}

// Rows per plane from which the all-reduces run as a reduce-scatter + all-
// gather (prefill) instead of every plane reducing every row (decode).
constexpr int kTpScatterRows = 128;

static void tp_dense_half(Runtime* /*self*/, std::vector<std::unique_ptr<DeviceCtx>>& planes,
                          int l, int rows, int H, int F, int tp, float eps) {
  const int Hs = H / tp, Fs = F / tp;
  // Reduce-scatter mode: row block q (R rows) of every plane's partial is
  // stored by the GEMM epilogue straight into plane q's receive buffer, at
  // block p for source plane p (peer stores while the GEMM runs); plane q
  // then reduces its block locally and stores x to itself and plane 0 (the
  // LM head's plane) and xn to every plane. All-reduce mode: each plane
  // stores its own partial and every plane reduces every row, reading the
  // others' partials.
  // ESP_TP_ALLREDUCE=1: all-reduce mode at every row count (the bit-identity
  // check of tests/test_tp_gpu.py — both modes sum in plane order)
  const bool rs = rows >= kTpScatterRows * tp && std::getenv("ESP_TP_ALLREDUCE") == nullptr;
  const int R = (rows + tp - 1) / tp;
  auto partial = [&](int p, const bf16* a, int K, const bf16* w, DevBuf DeviceCtx::*buf) {
    DeviceCtx& dc = *planes[p];
    k::GemmEpilogue e;
    e.kind = k::kEpiStoreF32;
    e.ldo = H;
    if (rs) {
      e.route_rows = R;
      for (int q = 0; q < tp; ++q) {
        e.route[q] = static_cast<float*>(((*planes[q]).*buf).ptr) + static_cast<int64_t>(p) * R * H;
      }
    } else {
      e.out = (dc.*buf).ptr;
    }
    k::gemm(a, K, w, K, rows, H, K, e, dc.stream);
  };
  auto reduce = [&](int p, DevBuf DeviceCtx::*buf) {
    DeviceCtx& dc = *planes[p];
    k::TpParts parts;
    bf16* xo[k::kMaxTp];
    bf16* xno[k::kMaxTp];
    bf16* x = static_cast<bf16*>(dc.x.ptr);
    if (rs) {
      const int r0 = p * R, n = std::min(rows, r0 + R) - r0;
      if (n <= 0) return;
      const int64_t off = static_cast<int64_t>(r0) * H;
      for (int q = 0; q < tp; ++q) {
        parts.p[parts.n++] = static_cast<const float*>((dc.*buf).ptr) + static_cast<int64_t>(q) * R * H;
        xno[q] = static_cast<bf16*>(planes[q]->xn.ptr) + off;
      }
      xo[0] = x + off;
      int nx = 1;
      if (p != 0) xo[nx++] = static_cast<bf16*>(planes[0]->x.ptr) + off;
      k::tp_reduce_residual_norm(x + off, parts, xo, nx, xno, tp, n, H, eps, dc.stream);
    } else {
      for (auto& pc : planes) parts.p[parts.n++] = static_cast<const float*>(((*pc).*buf).ptr);
      xo[0] = x;
      xno[0] = static_cast<bf16*>(dc.xn.ptr);
      k::tp_reduce_residual_norm(x, parts, xo, 1, xno, 1, rows, H, eps, dc.stream);
    }
    if (rs) cuda_ok(cudaEventRecord(dc.tp_ev_r, dc.stream), "event");
  };
  auto reduce_all = [&](DevBuf DeviceCtx::*buf) {
    for (int p = 0; p < tp; ++p) {
      DeviceGuard g(planes[p]->device);
      reduce(p, buf);
    }
    if (rs) wait_planes(planes, &DeviceCtx::tp_ev_r);  // the all-gather has landed
  };
  // O: attn (rows x Hs) . Wo_shard (H x Hs)^T -> fp32 partial (rows x H)
  for (int p = 0; p < tp; ++p) {
    DeviceCtx& dc = *planes[p];
    DeviceGuard g(dc.device);
    partial(p, static_cast<bf16*>(dc.attn.ptr), Hs, dc.layers[l].wo, &DeviceCtx::tp_po);
    cuda_ok(cudaEventRecord(dc.tp_ev_o, dc.stream), "event");
  }
  wait_planes(planes, &DeviceCtx::tp_ev_o);
  reduce_all(&DeviceCtx::tp_po);  // + the gate_up input norm
  for (int p = 0; p < tp; ++p) {
    DeviceCtx& dc = *planes[p];
    DeviceGuard g(dc.device);
    k::GemmEpilogue eg;
    eg.kind = k::kEpiSiluMul;
    eg.out = dc.h.ptr;
    eg.ldo = Fs;
    k::gemm(static_cast<bf16*>(dc.xn.ptr), H, dc.layers[l].wgu, H, rows, 2 * Fs, H, eg, dc.stream);
    partial(p, static_cast<bf16*>(dc.h.ptr), Fs, dc.layers[l].wd, &DeviceCtx::tp_pd);
    cuda_ok(cudaEventRecord(dc.tp_ev_d, dc.stream), "event");
  }
  wait_planes(planes, &DeviceCtx::tp_ev_d);
  reduce_all(&DeviceCtx::tp_pd);  // + the next layer's QKV input norm
}

double Runtime::decode_tp(const esp_decode_args& a, const std::vector<DecodeRow>& rows_v,
                          const TpChunk& ck) {
  const int b = static_cast<int>(rows_v.size()), t = tp_, c = ck.c, rows = b + c;
  const int H = cfg_.hidden, F = cfg_.ffn, Hs = H / t, Fs = F / t, hs = cfg_.heads / t;
  DeviceCtx& d0 = *devices_[0];
  // Split-KV work (as on one GPU): every instance holding a request's KV
  // contributes chunks of its slots; the page-table mirror lives on plane 0's
  // GPU and the other planes read it over NVLink.
  std::vector<int32_t> h_tok, h_pos, h_inst, h_slot, h_row_start;
  std::vector<k::DecodeChunk> chunks;
  {
    DeviceGuard g(d0.device);
    for (int i = 0; i < b; ++i) {
      const DecodeRow& rw = rows_v[i];
      h_tok.push_back(rw.token);
      h_pos.push_back(rw.pos);
      h_inst.push_back(inst(rw.master).slab);
      h_slot.push_back(rw.slot);
      h_row_start.push_back(static_cast<int32_t>(chunks.size()));
      RequestRec& rr = req(rw.r);
      for (auto& [iid, pl] : rr.pages) {
        if (pl.slots.empty()) continue;
        sync_pages(pl, d0.stream);
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
    cuda_ok(cudaEventRecord(d0.e0, d0.stream), "event");
  }
  // Chunk rows (a chunked prefill riding on the step): their K/V go to the
  // chunk's slots from the QKV epilogue; attention over the gathered earlier
  // KV + the chunk as one causal segment offset by p_prev (as on tp = 1).
  for (int i = 0; i < c; ++i) {
    h_tok.push_back(a.chunk_token_ids[i]);
    h_pos.push_back(static_cast<int32_t>(ck.p_prev + i));
    h_inst.push_back(ck.ch_slab[static_cast<size_t>(i)]);
    h_slot.push_back(ck.ch_slot[static_cast<size_t>(i)]);
  }
  const int kv_n = static_cast<int>(ck.p_prev) + c;
  // one ascending slot run on one slab: K1 reads the slab rows directly
  bool run = c > 0;
  for (size_t i = 0; run && i < ck.kv_slot.size(); ++i) {
    run = ck.kv_slab[i] == ck.kv_slab[0] && ck.kv_slot[i] == ck.kv_slot[0] + static_cast<int32_t>(i);
  }
  std::vector<int32_t> work_sorted;
  k::RingSegment sg{};
  if (c > 0) {
    sg.q_row0 = b;
    sg.q_len = c;
    sg.n_rounds = 1;
    sg.kv_row0[0] = 0;
    sg.kv_len[0] = kv_n;
    sg.shift[0] = -static_cast<int32_t>(ck.p_prev);
    std::vector<k::RingSegment> segs{sg};
    build_attention_work(segs, hs, work_sorted);
  }
  const int n_work = attention_n_work(work_sorted);
  const int n_chunks = static_cast<int>(chunks.size());
  int max_chunk = 0;
  for (const k::DecodeChunk& ch : chunks) max_chunk = std::max(max_chunk, static_cast<int>(ch.n));
  int64_t max_pos = std::max<int64_t>(1, ck.p_prev + c);
  for (const DecodeRow& rw : rows_v) max_pos = std::max<int64_t>(max_pos, rw.pos + 1);
  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  for (auto& pc : devices_) {
    DeviceCtx& dc = *pc;
    DeviceGuard g(dc.device);
    cudaStream_t s = dc.stream;
    if (&dc != &d0) cuda_ok(cudaStreamWaitEvent(s, d0.e0, 0), "tp start");  // page uploads
    ensure_rope(dc, max_pos);
    auto up = [&](DevBuf& buf, const std::vector<int32_t>& v) {
      cuda_ok(cudaMemcpyAsync(scratch<int32_t>(buf, std::max<size_t>(v.size(), 1)), v.data(),
                              v.size() * 4, cudaMemcpyHostToDevice, s), "h2d");
    };
    up(dc.tok, h_tok);
    up(dc.pos, h_pos);
    up(dc.rinst, h_inst);
    up(dc.rslot, h_slot);
    up(dc.row_start, h_row_start);
    cuda_ok(cudaMemcpyAsync(scratch<k::DecodeChunk>(dc.chunks, std::max(n_chunks, 1)), chunks.data(),
                            chunks.size() * sizeof(k::DecodeChunk), cudaMemcpyHostToDevice, s),
            "h2d");
    if (c > 0) {
      up(dc.ret_slab, ck.kv_slab);
      up(dc.ret_slot, ck.kv_slot);
      cuda_ok(cudaMemcpyAsync(scratch<k::RingSegment>(dc.segs, 1), &sg, sizeof(sg),
                              cudaMemcpyHostToDevice, s), "h2d");
      up(dc.work, work_sorted);
      scratch<bf16>(dc.kb, static_cast<size_t>(kv_n) * Hs);
      scratch<bf16>(dc.vb, static_cast<size_t>(kv_n) * Hs);
    }
    bf16* x = scratch<bf16>(dc.x, static_cast<size_t>(rows) * H);
    scratch<bf16>(dc.xn, static_cast<size_t>(rows) * H);
    scratch<bf16>(dc.q, static_cast<size_t>(rows) * Hs);
    scratch<bf16>(dc.attn, static_cast<size_t>(rows) * Hs);
    scratch<bf16>(dc.h, static_cast<size_t>(rows) * Fs);
    scratch<float>(dc.part_o, static_cast<size_t>(std::max(n_chunks, 1)) * hs * cfg_.head_dim);
    scratch<float>(dc.part_ml, static_cast<size_t>(std::max(n_chunks, 1)) * hs * 2);
    const size_t part_rows = static_cast<size_t>((rows + t - 1) / t) * t;  // reduce-scatter layout
    scratch<float>(dc.tp_po, part_rows * H);
    scratch<float>(dc.tp_pd, part_rows * H);
    if (&dc == &d0) {  // output buffers sized before the layers (no cudaFree mid-step)
      const size_t n_out_max = static_cast<size_t>(b + (c > 0 ? 1 : 0));
      scratch<int32_t>(dc.last_rows, std::max<size_t>(n_out_max, 1));
      scratch<float>(dc.logits, std::max<size_t>(n_out_max, 1) * cfg_.vocab);
      scratch<int32_t>(dc.out_tok, std::max<size_t>(n_out_max, 1));
    }
    k::embed(static_cast<const int32_t*>(dc.tok.ptr), dc.embed, x, rows, H, s, nullptr);
  }
  for (int l = 0; l < cfg_.layers; ++l) {
    for (auto& pc : devices_) {
      DeviceCtx& dc = *pc;
      DeviceGuard g(dc.device);
      cudaStream_t s = dc.stream;
      bf16* x = static_cast<bf16*>(dc.x.ptr);
      bf16* xn = static_cast<bf16*>(dc.xn.ptr);
      bf16* q = static_cast<bf16*>(dc.q.ptr);
      if (l == 0) k::rmsnorm(x, nullptr, nullptr, xn, rows, H, cfg_.rms_eps, s);
      k::GemmEpilogue ep;
      ep.kind = k::kEpiQkvRope;
      ep.q_out = q;
      ep.pos = static_cast<const int32_t*>(dc.pos.ptr);
      ep.rope = dc.rope;
      ep.hidden = Hs;
      ep.head_dim = cfg_.head_dim;
      ep.row_inst = static_cast<const int32_t*>(dc.rinst.ptr);  // append at the masters' slots
      ep.row_slot = static_cast<const int32_t*>(dc.rslot.ptr);
      k::DecodeSlabs slabs{};
      for (size_t j = 0; j < dc.slabs.size(); ++j) {
        const InstanceRec& in = instances_[dc.slabs[j]];
        ep.slab_k[j] = in.plane_k(dc.domain, l);
        ep.slab_v[j] = in.plane_v(dc.domain, l);
        slabs.k[j] = ep.slab_k[j];
        slabs.v[j] = ep.slab_v[j];
      }
      k::gemm(xn, H, dc.layers[l].wqkv, H, rows, 3 * Hs, H, ep, s);
      bf16* attn = static_cast<bf16*>(dc.attn.ptr);
      if (b > 0) {
        const bool direct = n_chunks == b;  // one chunk per row: K3 normalises in place
        k::decode_attention(q, static_cast<const k::DecodeChunk*>(dc.chunks.ptr), n_chunks, slabs,
                            hs, cfg_.head_dim, scale, static_cast<float*>(dc.part_o.ptr),
                            static_cast<float*>(dc.part_ml.ptr), s, nullptr,
                            direct ? attn : nullptr, max_chunk);
        if (!direct) {
          k::decode_combine(static_cast<float*>(dc.part_o.ptr),
                            static_cast<float*>(dc.part_ml.ptr),
                            static_cast<const int32_t*>(dc.row_start.ptr), b, hs, cfg_.head_dim,
                            attn, s);
        }
      }
      if (c > 0) {
        const bf16* kg = static_cast<bf16*>(dc.kb.ptr);
        const bf16* vg = static_cast<bf16*>(dc.vb.ptr);
        if (run) {
          kg = slabs.k[ck.kv_slab[0]] + static_cast<int64_t>(ck.kv_slot[0]) * Hs;
          vg = slabs.v[ck.kv_slab[0]] + static_cast<int64_t>(ck.kv_slot[0]) * Hs;
        } else {
          k::gather_rows(slabs, static_cast<const int32_t*>(dc.ret_slab.ptr),
                         static_cast<const int32_t*>(dc.ret_slot.ptr), kv_n,
                         static_cast<bf16*>(dc.kb.ptr), static_cast<bf16*>(dc.vb.ptr), Hs, s);
        }
        k::ring_attention(q, kg, vg, attn, rows, kv_n, hs, cfg_.head_dim,
                          static_cast<const k::RingSegment*>(dc.segs.ptr),
                          static_cast<const int32_t*>(dc.work.ptr), n_work, scale, s);
      }
    }
    tp_dense_half(this, devices_, l, rows, H, F, t, cfg_.rms_eps);
  }
  for (auto& pc : devices_) {
    if (pc.get() == &d0) continue;
    DeviceGuard g(pc->device);
    cuda_ok(cudaEventRecord(pc->tp_ev_d, pc->stream), "event");
    DeviceGuard g0(d0.device);
    cuda_ok(cudaStreamWaitEvent(d0.stream, pc->tp_ev_d, 0), "tp end");
  }
  // Output rows: the decode rows, then the chunk's last token when the chunk
  // completes the prompt (its first generated token, engine.cpp:570-579).
  const bool chunk_out = c > 0 && a.chunk_final != 0;
  const int n_out = b + (chunk_out ? 1 : 0);
  std::vector<int32_t> out_rows(static_cast<size_t>(b));
  for (int i = 0; i < b; ++i) out_rows[i] = i;
  if (chunk_out) out_rows.push_back(rows - 1);
  DeviceGuard g(d0.device);
  cudaStream_t s = d0.stream;
  int32_t* d_out_rows = scratch<int32_t>(d0.last_rows, std::max(n_out, 1));
  cuda_ok(cudaMemcpyAsync(d_out_rows, out_rows.data(), n_out * 4, cudaMemcpyHostToDevice, s), "h2d");
  bf16* xn = static_cast<bf16*>(d0.xn.ptr);
  float* logits = scratch<float>(d0.logits, static_cast<size_t>(std::max(n_out, 1)) * cfg_.vocab);
  int32_t* d_out = scratch<int32_t>(d0.out_tok, std::max(n_out, 1));
  if (n_out > 0) {
    k::rmsnorm(static_cast<bf16*>(d0.x.ptr), n_out == rows ? nullptr : d_out_rows, d0.final_norm,
               xn, n_out, H, cfg_.rms_eps, s);
    k::GemmEpilogue ef;
    ef.kind = k::kEpiStoreF32;
    ef.out = logits;
    ef.ldo = cfg_.vocab;
    k::gemm(xn, H, d0.lm_head, H, n_out, cfg_.vocab, H, ef, s);
    k::argmax_rows(logits, n_out, cfg_.vocab, d_out, s);
  }
  cuda_ok(cudaEventRecord(d0.e1, s), "event");
  check_cuda("tp decode launch");
  std::vector<int32_t> out(static_cast<size_t>(std::max(n_out, 1)));
  if (n_out > 0) {
    cuda_ok(cudaMemcpyAsync(out.data(), d_out, n_out * 4, cudaMemcpyDeviceToHost, s), "d2h");
  }
  std::vector<float> lg;
  if ((a.logits_out && b > 0) || (chunk_out && a.chunk_logits_out)) {
    lg.resize(static_cast<size_t>(n_out) * cfg_.vocab);
    cuda_ok(cudaMemcpyAsync(lg.data(), logits, lg.size() * 4, cudaMemcpyDeviceToHost, s), "d2h");
  }
  for (auto& pc : devices_) {
    DeviceGuard gp(pc->device);
    cuda_ok(cudaStreamSynchronize(pc->stream), "tp decode");
  }
  float ms = 0;
  cuda_ok(cudaEventElapsedTime(&ms, d0.e0, d0.e1), "elapsed");
  if (a.device_ms_out) *a.device_ms_out = ms;
  // Results back in the caller's batch order (rows are ordered by master).
  std::map<RequestId, int> row_of;
  for (int i = 0; i < b; ++i) row_of[rows_v[i].r] = i;
  for (int i = 0; i < b; ++i) {
    const int ri = row_of[a.batch[i]];
    RequestRec& rr = req(a.batch[i]);
    if (a.in_tokens) rr.tokens.push_back(a.in_tokens[i]);
    rr.tokens.push_back(out[ri]);
    if (a.out_tokens) a.out_tokens[i] = out[ri];
    if (a.logits_out) {
      std::copy(lg.begin() + static_cast<int64_t>(ri) * cfg_.vocab,
                lg.begin() + static_cast<int64_t>(ri + 1) * cfg_.vocab,
                a.logits_out + static_cast<int64_t>(i) * cfg_.vocab);
    }
  }
  if (c > 0) {
    if (chunk_out) {
      requests_[a.chunk_request].tokens.push_back(out[b]);
      if (a.chunk_first_token_out) *a.chunk_first_token_out = out[b];
      if (a.chunk_logits_out) {
        std::copy(lg.begin() + static_cast<int64_t>(b) * cfg_.vocab,
                  lg.begin() + static_cast<int64_t>(b + 1) * cfg_.vocab, a.chunk_logits_out);
      }
    } else if (a.chunk_first_token_out) {
      *a.chunk_first_token_out = -1;
    }
  }
  return ms;
}

}  // namespace esp
