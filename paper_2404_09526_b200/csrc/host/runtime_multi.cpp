// Cross-domain ESP executors: a prefill ring or a decode group whose
// instances live in different co-location domains (different GPUs, or —
// with ESP_DOMAIN_PER_INSTANCE — different domains of one GPU).
//
// Prefill (build_ring_schedule esp_mechanics.cpp:45-70)
//   Every domain computes embed / QKV / O / MLP for the stripe rows of its own
//   ring positions. K/V blocks then travel the ring exactly as the reference
//   schedules them: in round r position i forwards the block of origin
//   (i - r) mod d to position i+1. A hop between domains is one peer copy per
//   block into the receiver's gather buffer, ordered by CUDA events. A hop
//   inside a domain is free, because co-located positions share the buffer.
//   Proactive scale-down without extra traffic: a token whose resting
//   instance lives in another domain is written into its page slot by THAT
//   domain when the block passes through it (retain_rows), never migrated.
//
// Decode (multi-master)
//   Masters run their requests' dense layers. Each layer:
//   - every master domain's query rows are broadcast to the domains holding
//     the requests' KV;
//   - each of those domains computes split-KV partials over its own slots;
//   - the partials are gathered back to the master domain and LSE-combined.
//
// Everything is stream-ordered with events. Write-after-read hazards on the
// gather, query and partial buffers across layers are fenced with events
// recorded after each peer copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <set>

#include "device_ctx.hpp"
#include "runtime.hpp"

namespace esp {

void build_attention_work(const std::vector<k::RingSegment>& segs, int heads,
                          std::vector<int32_t>& work_sorted) {
  struct ItemC {
    int32_t seg, packed;
    int64_t cost;
  };
  std::vector<std::vector<ItemC>> per_sh;  // items of one (segment, head)
  constexpr int span = 2;  // a work item is a pair of 128-row query tiles
  for (size_t si = 0; si < segs.size(); ++si) {
    const k::RingSegment& sg = segs[si];
    const int n_items = (k::q_tiles(sg.q_len) + span - 1) / span;
    std::vector<int64_t> cost(static_cast<size_t>(n_items), 0);
    for (int qi = 0; qi < n_items; ++qi) {
      for (int qt = qi * span; qt < std::min(k::q_tiles(sg.q_len), (qi + 1) * span); ++qt) {
        for (int rd = 0; rd < sg.n_rounds; ++rd) {
          const int64_t vis = std::min<int64_t>(
              sg.kv_len[rd], std::min(qt * 128 + 127, sg.q_len - 1) - sg.shift[rd] + 1);
          cost[qi] += vis > 0 ? (vis + 127) / 128 : 0;
        }
      }
    }
    for (int hd = 0; hd < heads; ++hd) {
      std::vector<ItemC> v;
      for (int qi = 0; qi < n_items; ++qi) {
        // An item that sees no KV tile (a one-row stripe against a later
        // origin's block, windowed ring) has no work: K1 would wait for a
        // tile that never comes. Its rows keep their carried state.
        if (cost[qi] == 0) continue;
        v.push_back({static_cast<int32_t>(si), (qi << 8) | hd, cost[qi]});
      }
      per_sh.push_back(std::move(v));
    }
  }
  // Units of near-equal cost: within one (segment, head), the cheapest
  // causal item rides with the dearest (q tiles i and n-1-i see i+1 and n-i
  // KV tiles). Units are dealt head-major to the persistent CTAs by least
  // load (LPT), so the CTAs advance through the heads together and the K/V of
  // only ~2-3 heads is live in L2 at a time (the previous round-robin over a
  // cost-sorted list let CTAs drift across head groups: 5.6x the algorithmic
  // DRAM traffic).
  struct Unit {
    int head;
    int64_t cost;
    std::vector<ItemC> items;
  };
  std::vector<Unit> units;
  for (auto& v : per_sh) {
    std::stable_sort(v.begin(), v.end(),
                     [](const ItemC& x, const ItemC& y) { return x.cost > y.cost; });
    size_t lo = 0, hi = v.size();
    while (lo < hi) {
      Unit u;
      u.head = v[lo].packed & 0xFF;
      u.items.push_back(v[lo]);
      u.cost = v[lo].cost;
      if (hi - 1 > lo) {
        u.items.push_back(v[hi - 1]);
        u.cost += v[hi - 1].cost;
      }
      units.push_back(std::move(u));
      ++lo;
      --hi;
    }
  }
  std::stable_sort(units.begin(), units.end(), [](const Unit& x, const Unit& y) {
    return x.head != y.head ? x.head < y.head : x.cost > y.cost;
  });
  static const int n_sm = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    return v;
  }();
  const int G = static_cast<int>(std::max<size_t>(1, std::min<size_t>(units.size(), n_sm)));
  std::vector<std::vector<const Unit*>> per_cta(static_cast<size_t>(G));
  std::vector<int64_t> load(static_cast<size_t>(G), 0);
  for (const Unit& u : units) {
    int best = 0;
    for (int c = 1; c < G; ++c) {
      if (load[c] < load[best]) best = c;
    }
    per_cta[best].push_back(&u);
    load[best] += u.cost;
  }
  // Layout: [items: 2 ints each, CTA-contiguous][G][offsets 0..G][n_items];
  // CTA c of K1 takes items offsets[c] .. offsets[c+1].
  work_sorted.clear();
  std::vector<int32_t> offsets{0};
  int n_items = 0;
  for (const auto& lst : per_cta) {
    for (const Unit* u : lst) {
      for (const ItemC& it : u->items) {
        work_sorted.push_back(it.seg);
        work_sorted.push_back(it.packed);
        ++n_items;
      }
    }
    offsets.push_back(n_items);
  }
  work_sorted.push_back(G);
  work_sorted.insert(work_sorted.end(), offsets.begin(), offsets.end());
  work_sorted.push_back(n_items);
}

int attention_n_work(const std::vector<int32_t>& work) {
  return work.empty() ? 0 : work.back();
}

namespace {

template <typename T>
void h2d(T* dst, const std::vector<T>& src, cudaStream_t s) {
  if (src.empty()) return;
  cuda_ok(cudaMemcpyAsync(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, s),
          "h2d");
}

void peer_copy(void* dst, int dst_dev, const void* src, int src_dev, size_t bytes,
               cudaStream_t s) {
  if (bytes == 0) return;
  cuda_ok(cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes, s), "peer copy");
}

}  // namespace

// ---- prefill -------------------------------------------------------------------
void Runtime::prefill_multi(const esp_prefill_args& a, const std::vector<InstanceId>& ring,
                            const std::vector<std::vector<int32_t>>& tok_inst,
                            const std::vector<std::vector<int32_t>>& tok_slot,
                            const std::vector<int64_t>& tok_base) {
  const int n = a.n_requests, d = a.dop, H = cfg_.hidden, F = cfg_.ffn;
  auto stripe_len = [&](int i, int r) -> int32_t {
    const int64_t len = a.input_lens[r];
    return len > i ? static_cast<int32_t>((len - i + d - 1) / d) : 0;
  };
  // Global rows in ring-position-major order, as the single-domain pass.
  std::vector<std::vector<int32_t>> row0(static_cast<size_t>(d), std::vector<int32_t>(static_cast<size_t>(n)));
  std::vector<int32_t> blk0(static_cast<size_t>(d) + 1);
  int rows = 0;
  for (int i = 0; i < d; ++i) {
    blk0[i] = rows;
    for (int r = 0; r < n; ++r) {
      row0[i][r] = rows;
      rows += stripe_len(i, r);
    }
  }
  blk0[d] = rows;
  std::vector<int> dom_of(static_cast<size_t>(d));
  std::set<int> dom_set;
  for (int i = 0; i < d; ++i) {
    dom_of[i] = inst(ring[i]).domain;
    dom_set.insert(dom_of[i]);
  }
  struct Part {
    std::vector<int> positions;
    std::map<int, int32_t> local_row0;  // ring position -> first local row
    int rows = 0;
    std::vector<int32_t> tok, pos, rinst, rslot, kvrow, ret_rows, ret_slab, ret_slot;
    std::vector<k::RingSegment> segs;
    std::vector<int32_t> work;
    std::vector<std::pair<int, int32_t>> last;  // (request index, local row)
    // windowed ring: per round, the segments / work of that round's launch
    std::vector<std::vector<k::RingSegment>> wsegs;
    std::vector<std::vector<int32_t>> wwork;
    std::vector<size_t> seg_off, work_off;
  };
  std::map<int, Part> parts;
  for (int dom : dom_set) parts[dom];
  // Transport: fused push (default) — the QKV epilogue of each domain stores
  // its K/V rows into every domain's gather buffer and each token's K/V into
  // its resting page slot wherever that is (peer stores), so the ring's
  // all-gather and the retention ride inside the GEMM; or the copy-engine
  // ring in the reference's round order (ESP_RING_COPY=1).
  // Windowed ring (O(S/d) per GPU): every domain holds one
  // ring position, its own K/V block and two receive slots. In round r the
  // block of origin (i - r) mod d arrives from position i-1 (a peer copy on
  // a side stream, the reference's round order, esp_mechanics.cpp:59-68)
  // while K1 runs round r-1 on the other slot; K1 runs once per round and
  // carries its online-softmax state (O, max, sum) between rounds in HBM.
  // Chosen when the all-gather buffers (two layer parities of every block)
  // would exceed kWindowAutoBytes, or forced by ESP_RING_WINDOW.
  constexpr size_t kWindowAutoBytes = static_cast<size_t>(8) << 30;
  const size_t gather_bytes = static_cast<size_t>(2) * 2 * rows * H * sizeof(bf16);
  const bool window = d > 1 && dom_set.size() == static_cast<size_t>(d) && !opts_.ring_copy &&
                      instances_.size() <= static_cast<size_t>(k::kMaxSlabs) &&
                      (opts_.ring_window == 1 ||
                       (opts_.ring_window < 0 && gather_bytes > kWindowAutoBytes));
  const bool push = !window && !opts_.ring_copy &&
                    instances_.size() <= static_cast<size_t>(k::kMaxSlabs) &&
                    dom_set.size() <= static_cast<size_t>(k::kMaxPeers) + 1;
  for (int i = 0; i < d; ++i) {
    Part& p = parts[dom_of[i]];
    p.positions.push_back(i);
    p.local_row0[i] = p.rows;
    for (int r = 0; r < n; ++r) {
      const int64_t len = a.input_lens[r];
      for (int64_t t = i; t < len; t += d) {
        const int32_t g = row0[i][r] + static_cast<int32_t>(t / d);
        const InstanceRec& rest = inst(tok_inst[r][static_cast<size_t>(t)]);
        const int32_t slot = tok_slot[r][static_cast<size_t>(t)];
        p.tok.push_back(a.tokens[tok_base[r] + t]);
        p.pos.push_back(static_cast<int32_t>(t));
        p.kvrow.push_back(g);
        if (push || window) {  // retained by the origin's QKV epilogue, local or peer store
          p.rinst.push_back(static_cast<int32_t>(tok_inst[r][static_cast<size_t>(t)]));
          p.rslot.push_back(slot);
        } else if (rest.domain == dom_of[i]) {  // retained at the origin, in the QKV epilogue
          p.rinst.push_back(rest.slab);
          p.rslot.push_back(slot);
        } else {  // retained on pass by the resting domain
          p.rinst.push_back(-1);
          p.rslot.push_back(0);
          Part& q = parts[rest.domain];
          q.ret_rows.push_back(g);
          q.ret_slab.push_back(rest.slab);
          q.ret_slot.push_back(slot);
        }
      }
      const int64_t t_last = len - 1;
      if (t_last % d == i) {
        p.last.emplace_back(r, p.rows + (row0[i][r] - blk0[i]) + static_cast<int32_t>(t_last / d));
      }
    }
    p.rows += blk0[i + 1] - blk0[i];
  }
  // Cross-GPU arrivals: destination `dst` waits for source `src`'s K/V
  // blocks on the device (arrival counter polled by K1's producer) when they
  // sit on different GPUs and the source's QKV runs the tcgen05 kernels that
  // signal (> 32 rows). Otherwise — same GPU (ESP_DOMAIN_PER_INSTANCE: a
  // spinning K1 could starve the source's GEMM of SMs), skinny sources or
  // the copy ring — the stream waits for the source's QKV event instead.
  auto same_gpu = [&](int a, int b) {
    return devices_[static_cast<size_t>(a)]->device == devices_[static_cast<size_t>(b)]->device;
  };
  auto use_ctr = [&](int src, int dst) {
    return push && src != dst && src < k::kMaxWaitSrc && parts[src].rows > 32 &&
           (!same_gpu(src, dst) || opts_.force_arrival);
  };
  int32_t max_blk = 0;
  for (int o = 0; o < d; ++o) max_blk = std::max(max_blk, blk0[o + 1] - blk0[o]);
  for (auto& [dom, p] : parts) {
    if (window) {  // one launch per round: round rd meets the block of origin (i - rd) mod d
      const int i = p.positions[0];
      p.wsegs.assign(static_cast<size_t>(d), {});
      p.wwork.assign(static_cast<size_t>(d), {});
      for (int rd = 0; rd < d; ++rd) {
        const int o = RingSchedule::origin(i, rd, d);
        for (int r = 0; r < n; ++r) {
          const int32_t ql = stripe_len(i, r), kl = stripe_len(o, r);
          if (ql == 0 || kl == 0) continue;
          k::RingSegment sg{};
          sg.q_row0 = row0[i][r] - blk0[i];
          sg.q_len = ql;
          sg.n_rounds = 1;
          sg.kv_row0[0] = row0[o][r] - blk0[o];
          sg.kv_len[0] = kl;
          sg.shift[0] = o > i ? 1 : 0;
          p.wsegs[rd].push_back(sg);
        }
        build_attention_work(p.wsegs[rd], cfg_.heads, p.wwork[rd]);
        p.seg_off.push_back(p.segs.size());
        p.segs.insert(p.segs.end(), p.wsegs[rd].begin(), p.wsegs[rd].end());
        p.work_off.push_back(p.work.size());
        p.work.insert(p.work.end(), p.wwork[rd].begin(), p.wwork[rd].end());
      }
      continue;
    }
    for (int i : p.positions) {
      for (int r = 0; r < n; ++r) {
        const int32_t ql = stripe_len(i, r);
        if (ql == 0) continue;
        k::RingSegment sg{};
        sg.q_row0 = p.local_row0[i] + (row0[i][r] - blk0[i]);
        sg.q_len = ql;
        sg.n_rounds = d;
        for (int rd = 0; rd < d; ++rd) {
          const int o = RingSchedule::origin(i, rd, d);
          sg.kv_row0[rd] = row0[o][r];
          sg.kv_len[rd] = stripe_len(o, r);
          sg.shift[rd] = o > i ? 1 : 0;
          sg.wait_src[rd] = use_ctr(dom_of[o], dom) ? dom_of[o] + 1 : 0;
        }
        p.segs.push_back(sg);
      }
    }
    build_attention_work(p.segs, cfg_.heads, p.work);
  }
  if (cap_armed_) {  // parity capture: (domain, local stripe row) of each position
    if (n != 1) throw ConfigError("attention capture needs a single-request prefill");
    for (size_t c = 0; c < cap_pos_.size(); ++c) {
      const int64_t t = cap_pos_[c];
      if (t < 0 || t >= a.input_lens[0]) throw ConfigError("capture position outside the prompt");
      const int i = static_cast<int>(t % d);
      Part& p = parts[dom_of[i]];
      cap_add(dom_of[i], p.local_row0[i] + (row0[i][0] - blk0[i]) + static_cast<int32_t>(t / d),
              static_cast<int32_t>(c));
    }
  }

  int64_t max_len = 0;
  for (int r = 0; r < n; ++r) max_len = std::max(max_len, a.input_lens[r]);
  int64_t ring_rows_max = 0;
  // Per-domain setup: uploads, embedding.
  for (auto& [dom, p] : parts) {
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cudaStream_t s = dc.stream;
    dc.sync_used = 0;
    ensure_rope(dc, max_len);
    const size_t lr = static_cast<size_t>(std::max(p.rows, 1));
    h2d(scratch<int32_t>(dc.tok, lr), p.tok, s);
    h2d(scratch<int32_t>(dc.pos, lr), p.pos, s);
    h2d(scratch<int32_t>(dc.rinst, lr), p.rinst, s);
    h2d(scratch<int32_t>(dc.rslot, lr), p.rslot, s);
    h2d(scratch<int32_t>(dc.kvrow, lr), p.kvrow, s);
    h2d(scratch<int32_t>(dc.ret_rows, p.ret_rows.size() + 1), p.ret_rows, s);
    h2d(scratch<int32_t>(dc.ret_slab, p.ret_slab.size() + 1), p.ret_slab, s);
    h2d(scratch<int32_t>(dc.ret_slot, p.ret_slot.size() + 1), p.ret_slot, s);
    h2d(scratch<k::RingSegment>(dc.segs, p.segs.size() + 1), p.segs, s);
    h2d(scratch<int32_t>(dc.work, p.work.size() + 1), p.work, s);
    scratch<bf16>(dc.x, lr * H);
    scratch<bf16>(dc.xn, lr * H);
    scratch<bf16>(dc.q, lr * H);
    scratch<bf16>(dc.attn, lr * H);
    scratch<bf16>(dc.h, lr * F);
    // Gather buffers hold every block of the layer; the push transport
    // double-buffers them by layer parity, so a source may store layer l+1
    // while this domain's K1 still reads layer l.
    // The windowed ring holds its own block and two receive slots instead.
    const size_t nbuf = push ? 2 : 1;
    const size_t kv_rows_buf = window ? lr + 2 * static_cast<size_t>(std::max(max_blk, 1))
                                      : nbuf * static_cast<size_t>(rows);
    scratch<bf16>(dc.kb, kv_rows_buf * H);
    ring_rows_max = std::max<int64_t>(ring_rows_max, static_cast<int64_t>(kv_rows_buf));
    scratch<bf16>(dc.vb, kv_rows_buf * H);
    if (window) {
      scratch<float>(dc.carry_o, lr * H);
      scratch<float2>(dc.carry_ml, lr * cfg_.heads);
      if (!dc.comm) cuda_ok(cudaStreamCreateWithFlags(&dc.comm, cudaStreamNonBlocking), "stream");
    }
    if (fuse_norm_prefill()) {
      scratch<float>(dc.ss1, lr);
      scratch<float>(dc.ss2, lr);
    }
    if (push && !dc.arrive) {
      cuda_ok(cudaMalloc(&dc.arrive, k::kMaxWaitSrc * sizeof(unsigned long long)), "cudaMalloc(arrive)");
      cuda_ok(cudaMemsetAsync(dc.arrive, 0, k::kMaxWaitSrc * sizeof(unsigned long long), s), "memset");
      std::fill(std::begin(dc.arrive_expect), std::end(dc.arrive_expect), 0ull);
    }
    cuda_ok(cudaEventRecord(dc.e0, s), "event");
    if (p.rows > 0) {
      timed(kPhEmbed, s, [&] {
        k::embed(static_cast<int32_t*>(dc.tok.ptr), dc.embed, static_cast<bf16*>(dc.x.ptr),
                 p.rows, H, s, fuse_norm_prefill() ? static_cast<float*>(dc.ss1.ptr) : nullptr);
      });
    }
  }
  // Source domains' arrival counters must exist before any epilogue
  // signals them (allocation above is stream-ordered per domain).
  if (push) {
    for (auto& [dom, p] : parts) {
      DeviceGuard g(devices_[static_cast<size_t>(dom)]->device);
      cuda_ok(cudaStreamSynchronize(devices_[static_cast<size_t>(dom)]->stream), "arrive init");
    }
  }
  const bool fuse = fuse_norm_prefill();

  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  std::map<int, std::vector<cudaEvent_t>> readers;  // copies reading a domain's gather buffer
  // push: attn_done[dom][parity] = dom's K1 of the last layer that read that
  // gather-buffer parity (peers may overwrite it once it has completed)
  std::map<int, std::array<cudaEvent_t, 2>> attn_done;
  // windowed ring, per domain and receive slot: the K1 round that last read
  // the slot, and the copy that last forwarded from it (the next receive
  // into the slot waits for both, across layers)
  std::map<int, std::array<cudaEvent_t, 2>> win_k1, win_fwd;
  for (auto& [dom, p] : parts) {
    win_k1[dom] = {nullptr, nullptr};
    win_fwd[dom] = {nullptr, nullptr};
  }
  for (int l = 0; l < cfg_.layers; ++l) {
    NvtxRange nvtx_layer("prefill layer (cross-domain)");
    const int par = push ? (l & 1) : 0;
    const size_t boff = static_cast<size_t>(par) * rows * H;
    std::map<int, cudaEvent_t> qkv_done;  // push: domain's QKV (and its pushes) of this layer
    std::map<int, std::vector<cudaEvent_t>> ready;  // domain -> block -> event (nullptr: absent)
    for (auto& [dom, p] : parts) ready[dom].assign(static_cast<size_t>(d), nullptr);
    // 1. per-domain QKV (+RoPE, + retention, + the push to every peer's gather buffer).
    for (auto& [dom, p] : parts) {
      DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
      DeviceGuard g(dc.device);
      cudaStream_t s = dc.stream;
      for (cudaEvent_t e : readers[dom]) cuda_ok(cudaStreamWaitEvent(s, e, 0), "wait");
      readers[dom].clear();
      if (push) {  // peers' buffers of this parity are free once their K1 of layer l-2 is done
        for (auto& [od, ev] : attn_done) {
          if (od != dom && ev[par] != nullptr) cuda_ok(cudaStreamWaitEvent(s, ev[par], 0), "wait");
        }
      }
      if (p.rows == 0) {  // empty stripes (prompt shorter than the ring): nothing to send
        cudaEvent_t e = sync_event(dc);
        cuda_ok(cudaEventRecord(e, s), "event");
        for (int i : p.positions) ready[dom][i] = e;
        qkv_done[dom] = e;
        continue;
      }
      const LayerW& w = dc.layers[l];
      bf16* x = static_cast<bf16*>(dc.x.ptr);
      bf16* xn = static_cast<bf16*>(dc.xn.ptr);
      if (!fuse) {
        timed(kPhNorm, s, [&] { k::rmsnorm(x, nullptr, nullptr, xn, p.rows, H, cfg_.rms_eps, s); });
      }
      k::GemmEpilogue ep;
      ep.kind = k::kEpiQkvRope;
      ep.q_out = static_cast<bf16*>(dc.q.ptr);
      ep.k_out = static_cast<bf16*>(dc.kb.ptr) + boff;
      ep.v_out = static_cast<bf16*>(dc.vb.ptr) + boff;
      ep.kv_rows = window ? nullptr : static_cast<int32_t*>(dc.kvrow.ptr);
      ep.pos = static_cast<int32_t*>(dc.pos.ptr);
      ep.rope = dc.rope;
      ep.hidden = H;
      ep.head_dim = cfg_.head_dim;
      ep.row_inst = static_cast<int32_t*>(dc.rinst.ptr);
      ep.row_slot = static_cast<int32_t*>(dc.rslot.ptr);
      if (fuse) {
        ep.ss_in = static_cast<float*>(dc.ss1.ptr);
        ep.norm_dim = H;
        ep.norm_eps = cfg_.rms_eps;
      }
      if (push || window) {
        for (size_t j = 0; j < instances_.size(); ++j) {
          ep.slab_k[j] = instances_[j].layer_k(l);
          ep.slab_v[j] = instances_[j].layer_v(l);
        }
        for (auto& [od, op] : parts) {
          if (window) break;  // blocks travel by the round copies below
          if (od == dom) continue;
          DeviceCtx& pc = *devices_[static_cast<size_t>(od)];
          ep.k_peer[ep.n_peer] = static_cast<bf16*>(pc.kb.ptr) + boff;
          ep.v_peer[ep.n_peer] = static_cast<bf16*>(pc.vb.ptr) + boff;
          ++ep.n_peer;
          if (use_ctr(dom, od)) ep.arrive[ep.n_arrive++] = pc.arrive + dom;
        }
      } else {
        for (size_t j = 0; j < dc.slabs.size(); ++j) {
          ep.slab_k[j] = instances_[dc.slabs[j]].layer_k(l);
          ep.slab_v[j] = instances_[dc.slabs[j]].layer_v(l);
        }
      }
      timed(kPhQkv, s, [&] { k::gemm(fuse ? x : xn, H, w.wqkv, H, p.rows, 3 * H, H, ep, s); });
      cudaEvent_t e = sync_event(dc);
      cuda_ok(cudaEventRecord(e, s), "event");
      for (int i : p.positions) ready[dom][i] = e;
      qkv_done[dom] = e;
    }
    // 2. ring transport in the reference's round order (copy mode only).
    for (int r = 0; !push && !window && r + 1 < d; ++r) {
      for (int i = 0; i < d; ++i) {
        const int o = RingSchedule::origin(i, r, d);
        const int src = dom_of[i], dst = dom_of[(i + 1) % d];
        if (src == dst || ready[dst][o] != nullptr) continue;
        if (ready[src][o] == nullptr) throw InternalError("ring block forwarded before it arrived");
        DeviceCtx& sd = *devices_[static_cast<size_t>(src)];
        DeviceCtx& dd = *devices_[static_cast<size_t>(dst)];
        DeviceGuard g(dd.device);
        cuda_ok(cudaStreamWaitEvent(dd.stream, ready[src][o], 0), "wait");
        const size_t off = static_cast<size_t>(blk0[o]) * H;
        const size_t bytes = static_cast<size_t>(blk0[o + 1] - blk0[o]) * H * sizeof(bf16);
        peer_copy(static_cast<bf16*>(dd.kb.ptr) + off, dd.device,
                  static_cast<bf16*>(sd.kb.ptr) + off, sd.device, bytes, dd.stream);
        peer_copy(static_cast<bf16*>(dd.vb.ptr) + off, dd.device,
                  static_cast<bf16*>(sd.vb.ptr) + off, sd.device, bytes, dd.stream);
        cudaEvent_t e = sync_event(dd);
        cuda_ok(cudaEventRecord(e, dd.stream), "event");
        ready[dst][o] = e;
        readers[src].push_back(e);
      }
    }
    // 2b. windowed ring: round-major across domains, so every event a copy or
    // launch waits on is recorded before the wait is enqueued.
    if (window) {
      auto slot_ptr = [&](DevBuf& b, const Part& pp, int sl) {
        return static_cast<bf16*>(b.ptr) +
               (static_cast<size_t>(std::max(pp.rows, 1)) + static_cast<size_t>(sl) * max_blk) * H;
      };
      auto launch_round = [&](int dom, Part& p, int rd, const bf16* kp, const bf16* vp, int kv_n) {
        if (p.rows == 0 || attention_n_work(p.wwork[rd]) == 0) return;
        DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
        k::RingCarry cy;
        cy.o = static_cast<float*>(dc.carry_o.ptr);
        cy.ml = static_cast<float2*>(dc.carry_ml.ptr);
        cy.carry_in = rd > 0 ? 1 : 0;
        timed(kPhAttention, dc.stream, [&] {
          k::ring_attention(static_cast<bf16*>(dc.q.ptr), kp, vp, static_cast<bf16*>(dc.attn.ptr),
                            p.rows, std::max(kv_n, 1), cfg_.heads, cfg_.head_dim,
                            static_cast<k::RingSegment*>(dc.segs.ptr) + p.seg_off[rd],
                            static_cast<int32_t*>(dc.work.ptr) + p.work_off[rd],
                            attention_n_work(p.wwork[rd]), scale, dc.stream, nullptr, &cy);
        });
      };
      for (auto& [dom, p] : parts) {  // round 0: the own block, as soon as QKV is done
        DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
        DeviceGuard g(dc.device);
        launch_round(dom, p, 0, static_cast<bf16*>(dc.kb.ptr), static_cast<bf16*>(dc.vb.ptr), p.rows);
      }
      std::vector<cudaEvent_t> landed_prev(static_cast<size_t>(d), nullptr);
      for (int r = 1; r < d; ++r) {
        std::vector<cudaEvent_t> landed(static_cast<size_t>(d), nullptr);
        for (auto& [dom, p] : parts) {  // block of origin (i - r) mod d: position i-1 -> i
          const int i = p.positions[0];
          const int sp_i = (i - 1 + d) % d, src = dom_of[sp_i];
          const int o = RingSchedule::origin(i, r, d);
          DeviceCtx& sd = *devices_[static_cast<size_t>(src)];
          DeviceCtx& dd = *devices_[static_cast<size_t>(dom)];
          Part& sp = parts[src];
          DeviceGuard g(dd.device);
          const int sl = r & 1;
          cuda_ok(cudaStreamWaitEvent(dd.comm, r == 1 ? qkv_done[src] : landed_prev[sp_i], 0), "wait");
          for (cudaEvent_t e : {win_k1[dom][sl], win_fwd[dom][sl]}) {
            if (e != nullptr) cuda_ok(cudaStreamWaitEvent(dd.comm, e, 0), "wait");
          }
          const size_t bytes = static_cast<size_t>(blk0[o + 1] - blk0[o]) * H * sizeof(bf16);
          const bf16* sk = r == 1 ? static_cast<bf16*>(sd.kb.ptr) : slot_ptr(sd.kb, sp, (r - 1) & 1);
          const bf16* sv = r == 1 ? static_cast<bf16*>(sd.vb.ptr) : slot_ptr(sd.vb, sp, (r - 1) & 1);
          peer_copy(slot_ptr(dd.kb, p, sl), dd.device, sk, sd.device, bytes, dd.comm);
          peer_copy(slot_ptr(dd.vb, p, sl), dd.device, sv, sd.device, bytes, dd.comm);
          cudaEvent_t e = sync_event(dd);
          cuda_ok(cudaEventRecord(e, dd.comm), "event");
          landed[i] = e;
          if (r == 1) {
            readers[src].push_back(e);  // the source's next QKV overwrites its own block
          } else {
            win_fwd[src][(r - 1) & 1] = e;  // its next receive into that slot waits for this
          }
        }
        for (auto& [dom, p] : parts) {  // round r on the slot that just landed
          const int i = p.positions[0];
          const int o = RingSchedule::origin(i, r, d);
          DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
          DeviceGuard g(dc.device);
          cuda_ok(cudaStreamWaitEvent(dc.stream, landed[i], 0), "wait");
          launch_round(dom, p, r, slot_ptr(dc.kb, p, r & 1), slot_ptr(dc.vb, p, r & 1),
                       blk0[o + 1] - blk0[o]);
          cudaEvent_t e = sync_event(dc);
          cuda_ok(cudaEventRecord(e, dc.stream), "event");
          win_k1[dom][r & 1] = e;
        }
        landed_prev = landed;
      }
    }
    // 3. retention on pass (copy mode), attention, O, MLP — local to each domain.
    for (auto& [dom, p] : parts) {
      DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
      DeviceGuard g(dc.device);
      cudaStream_t s = dc.stream;
      k::RingWait wait;
      bool any_wait = false;
      if (push) {
        // Every other domain's K/V rows must have landed here: by its QKV
        // event, or on the device through its arrival counter (K1 starts on
        // its own block while remote blocks still stream in over NVLink).
        for (auto& [od, e] : qkv_done) {
          if (od == dom) continue;
          if (use_ctr(od, dom)) {
            dc.arrive_expect[od] += static_cast<unsigned long long>(parts[od].rows) * 2 * H;
            wait.target[od] = dc.arrive_expect[od];
            any_wait = true;
          }
          if (!use_ctr(od, dom) || same_gpu(od, dom)) cuda_ok(cudaStreamWaitEvent(s, e, 0), "wait");
        }
        wait.ctr = dc.arrive;
      }
      k::DecodeSlabs slabs{};
      for (size_t j = 0; j < dc.slabs.size(); ++j) {
        slabs.k[j] = instances_[dc.slabs[j]].layer_k(l);
        slabs.v[j] = instances_[dc.slabs[j]].layer_v(l);
      }
      k::retain_rows(static_cast<bf16*>(dc.kb.ptr), static_cast<bf16*>(dc.vb.ptr),
                     static_cast<int32_t*>(dc.ret_rows.ptr), static_cast<int32_t*>(dc.ret_slab.ptr),
                     static_cast<int32_t*>(dc.ret_slot.ptr), static_cast<int>(p.ret_rows.size()),
                     slabs, H, s);
      if (p.rows == 0) continue;
      bf16* x = static_cast<bf16*>(dc.x.ptr);
      bf16* xn = static_cast<bf16*>(dc.xn.ptr);
      bf16* attn = static_cast<bf16*>(dc.attn.ptr);
      bf16* hbuf = static_cast<bf16*>(dc.h.ptr);
      const int n_work = attention_n_work(p.work);
      if (window) {  // every round done (stream order): normalise the carry
        k::RingCarry cy;
        cy.o = static_cast<float*>(dc.carry_o.ptr);
        cy.ml = static_cast<float2*>(dc.carry_ml.ptr);
        timed(kPhAttention, s, [&] {
          k::ring_attention_finalize(cy, attn, p.rows, cfg_.heads, cfg_.head_dim, s);
        });
      } else timed(kPhAttention, s, [&] {
        const bf16* qd = static_cast<bf16*>(dc.q.ptr);
        // Q rows are this domain's local rows, K/V rows are global.
        k::ring_attention(qd, static_cast<bf16*>(dc.kb.ptr) + boff,
                          static_cast<bf16*>(dc.vb.ptr) + boff, attn, p.rows, rows, cfg_.heads,
                          cfg_.head_dim, static_cast<k::RingSegment*>(dc.segs.ptr),
                          static_cast<int32_t*>(dc.work.ptr), n_work, scale, s,
                          any_wait ? &wait : nullptr);
      });
      if (cap_armed_) cap_layer(dc, l, attn, s);
      if (push) {  // peers may overwrite this parity of the gather buffer after this
        cudaEvent_t e = sync_event(dc);
        cuda_ok(cudaEventRecord(e, s), "event");
        auto it = attn_done.find(dom);
        if (it == attn_done.end()) it = attn_done.emplace(dom, std::array<cudaEvent_t, 2>{nullptr, nullptr}).first;
        it->second[par] = e;
      }
      NormFuse nf;
      if (fuse) {
        nf.ss_o = static_cast<float*>(dc.ss2.ptr);
        nf.ss_d = static_cast<float*>(dc.ss1.ptr);
      }
      o_and_mlp(dc, l, p.rows, x, attn, xn, hbuf, nf, s);
    }
  }

  // 4. LM head + greedy token where each request's last prompt token lives.
  std::vector<int32_t> first(static_cast<size_t>(n), -1);
  std::map<int, std::vector<int32_t>> out_tok;
  std::map<int, std::vector<float>> out_lg;
  for (auto& [dom, p] : parts) {
    if (p.last.empty()) continue;
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cudaStream_t s = dc.stream;
    const int nl = static_cast<int>(p.last.size());
    std::vector<int32_t> lrows;
    for (const auto& [r, row] : p.last) lrows.push_back(row);
    int32_t* d_last = scratch<int32_t>(dc.last_rows, lrows.size());
    h2d(d_last, lrows, s);
    bf16* xn = static_cast<bf16*>(dc.xn.ptr);
    timed(kPhNorm, s, [&] {
      k::rmsnorm(static_cast<bf16*>(dc.x.ptr), d_last, dc.final_norm, xn, nl, H, cfg_.rms_eps, s);
    });
    float* logits = scratch<float>(dc.logits, static_cast<size_t>(nl) * cfg_.vocab);
    k::GemmEpilogue ep;
    ep.kind = k::kEpiStoreF32;
    ep.out = logits;
    ep.ldo = cfg_.vocab;
    timed(kPhLmHead, s, [&] { k::gemm(xn, H, dc.lm_head, H, nl, cfg_.vocab, H, ep, s); });
    int32_t* d_out = scratch<int32_t>(dc.out_tok, nl);
    timed(kPhArgmax, s, [&] { k::argmax_rows(logits, nl, cfg_.vocab, d_out, s); });
    out_tok[dom].resize(static_cast<size_t>(nl));
    cuda_ok(cudaMemcpyAsync(out_tok[dom].data(), d_out, nl * 4, cudaMemcpyDeviceToHost, s), "d2h");
    if (a.logits_out) {
      out_lg[dom].resize(static_cast<size_t>(nl) * cfg_.vocab);
      cuda_ok(cudaMemcpyAsync(out_lg[dom].data(), logits, out_lg[dom].size() * 4,
                              cudaMemcpyDeviceToHost, s),
              "d2h");
    }
  }
  double ms_max = 0;
  for (auto& [dom, p] : parts) {
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cuda_ok(cudaEventRecord(dc.e1, dc.stream), "event");
    check_cuda("prefill (multi-domain) launch");
  }
  for (auto& [dom, p] : parts) {
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cuda_ok(cudaStreamSynchronize(dc.stream), "prefill (multi-domain)");
    float ms = 0;
    cuda_ok(cudaEventElapsedTime(&ms, dc.e0, dc.e1), "elapsed");
    ms_max = std::max<double>(ms_max, ms);
  }
  if (cap_armed_) cap_finish();
  collect_phase_events();
  for (auto& [dom, p] : parts) {
    for (size_t j = 0; j < p.last.size(); ++j) {
      const int r = p.last[j].first;
      first[r] = out_tok[dom][j];
      if (a.logits_out) {
        std::memcpy(a.logits_out + static_cast<size_t>(r) * cfg_.vocab,
                    out_lg[dom].data() + j * cfg_.vocab, cfg_.vocab * sizeof(float));
      }
    }
  }
  if (a.device_ms_out) *a.device_ms_out = ms_max;
  last_prefill_.device_ms = ms_max;
  last_prefill_.kv_ring_rows = ring_rows_max;
  for (int r = 0; r < n; ++r) {
    requests_[a.request_ids[r]].tokens.push_back(first[r]);
    if (a.first_token_out) a.first_token_out[r] = first[r];
  }
  profiles_.push_back(ProfileRec{d, std::vector<int64_t>(a.input_lens, a.input_lens + n), ms_max});
}

// ---- decode ------------------------------------------------------------------------
void Runtime::chunk_multi(const esp_decode_args& a, int64_t p_prev,
                          const std::vector<std::pair<InstanceId, int32_t>>& prev,
                          const std::vector<std::pair<InstanceId, int32_t>>& chunk_slots,
                          double* ms_out) {
  const int c = static_cast<int>(a.chunk_tokens);
  const int H = cfg_.hidden, F = cfg_.ffn;
  DeviceCtx& dc = *devices_[static_cast<size_t>(inst(chunk_slots.front().first).domain)];
  DeviceGuard g(dc.device);
  cudaStream_t s = dc.stream;
  const int kv_n = static_cast<int>(p_prev) + c;
  // Rows: the chunk's tokens. K/V rest in page slots addressed by GLOBAL
  // instance id (slab pointers of every instance; remote ones are peer
  // memory over NVLink). Gather list: earlier tokens, then the chunk's own.
  std::vector<int32_t> tok(a.chunk_token_ids, a.chunk_token_ids + c), pos, rinst, rslot, gi, gs;
  for (int i = 0; i < c; ++i) {
    pos.push_back(static_cast<int32_t>(p_prev + i));
    rinst.push_back(chunk_slots[static_cast<size_t>(i)].first);
    rslot.push_back(chunk_slots[static_cast<size_t>(i)].second);
  }
  for (const auto& [i, sl] : prev) {
    gi.push_back(i);
    gs.push_back(sl);
  }
  gi.insert(gi.end(), rinst.begin(), rinst.end());
  gs.insert(gs.end(), rslot.begin(), rslot.end());
  ensure_rope(dc, p_prev + c);
  h2d(scratch<int32_t>(dc.tok, c), tok, s);
  h2d(scratch<int32_t>(dc.pos, c), pos, s);
  h2d(scratch<int32_t>(dc.rinst, c), rinst, s);
  h2d(scratch<int32_t>(dc.rslot, c), rslot, s);
  int32_t* d_gi = scratch<int32_t>(dc.ret_slab, kv_n);
  int32_t* d_gs = scratch<int32_t>(dc.ret_slot, kv_n);
  h2d(d_gi, gi, s);
  h2d(d_gs, gs, s);
  k::RingSegment sg{};
  sg.q_row0 = 0;
  sg.q_len = c;
  sg.n_rounds = 1;
  sg.kv_row0[0] = 0;
  sg.kv_len[0] = kv_n;
  sg.shift[0] = -static_cast<int32_t>(p_prev);
  std::vector<int32_t> work;
  build_attention_work({sg}, cfg_.heads, work);
  k::RingSegment* d_seg = scratch<k::RingSegment>(dc.segs, 1);
  cuda_ok(cudaMemcpyAsync(d_seg, &sg, sizeof(sg), cudaMemcpyHostToDevice, s), "h2d");
  h2d(scratch<int32_t>(dc.work, work.size()), work, s);
  const int n_work = attention_n_work(work);
  bf16* x = scratch<bf16>(dc.x, static_cast<size_t>(c) * H);
  bf16* xn = scratch<bf16>(dc.xn, static_cast<size_t>(c) * H);
  bf16* q = scratch<bf16>(dc.q, static_cast<size_t>(c) * H);
  bf16* attn = scratch<bf16>(dc.attn, static_cast<size_t>(c) * H);
  bf16* hbuf = scratch<bf16>(dc.h, static_cast<size_t>(c) * F);
  bf16* kg = scratch<bf16>(dc.kb, static_cast<size_t>(kv_n) * H);
  bf16* vg = scratch<bf16>(dc.vb, static_cast<size_t>(kv_n) * H);
  const float scale = 1.0f / std::sqrt(static_cast<float>(cfg_.head_dim));
  cudaEvent_t t0, t1;
  cuda_ok(cudaEventCreate(&t0), "event");
  cuda_ok(cudaEventCreate(&t1), "event");
  cuda_ok(cudaEventRecord(t0, s), "event");
  k::embed(static_cast<int32_t*>(dc.tok.ptr), dc.embed, x, c, H, s);
  for (int l = 0; l < cfg_.layers; ++l) {
    const LayerW& w = dc.layers[l];
    k::rmsnorm(x, nullptr, nullptr, xn, c, H, cfg_.rms_eps, s);
    k::GemmEpilogue ep;
    ep.kind = k::kEpiQkvRope;
    ep.q_out = q;
    ep.pos = static_cast<int32_t*>(dc.pos.ptr);
    ep.rope = dc.rope;
    ep.hidden = H;
    ep.head_dim = cfg_.head_dim;
    ep.row_inst = static_cast<int32_t*>(dc.rinst.ptr);  // global instance ids
    ep.row_slot = static_cast<int32_t*>(dc.rslot.ptr);
    k::DecodeSlabs slabs{};
    for (size_t j = 0; j < instances_.size(); ++j) {
      ep.slab_k[j] = instances_[j].layer_k(l);
      ep.slab_v[j] = instances_[j].layer_v(l);
      slabs.k[j] = ep.slab_k[j];
      slabs.v[j] = ep.slab_v[j];
    }
    k::gemm(xn, H, w.wqkv, H, c, 3 * H, H, ep, s);
    k::gather_rows(slabs, d_gi, d_gs, kv_n, kg, vg, H, s);
    k::ring_attention(q, kg, vg, attn, c, kv_n, cfg_.heads, cfg_.head_dim, d_seg, static_cast<int32_t*>(dc.work.ptr), n_work, scale, s);
    o_and_mlp(dc, l, c, x, attn, xn, hbuf, NormFuse{}, s);
  }
  int32_t first = -1;
  std::vector<float> lg;
  if (a.chunk_final) {
    const int32_t last = c - 1;
    int32_t* d_last = scratch<int32_t>(dc.last_rows, 1);
    cuda_ok(cudaMemcpyAsync(d_last, &last, 4, cudaMemcpyHostToDevice, s), "h2d");
    k::rmsnorm(x, d_last, dc.final_norm, xn, 1, H, cfg_.rms_eps, s);
    float* logits = scratch<float>(dc.logits, cfg_.vocab);
    k::GemmEpilogue ef;
    ef.kind = k::kEpiStoreF32;
    ef.out = logits;
    ef.ldo = cfg_.vocab;
    k::gemm(xn, H, dc.lm_head, H, 1, cfg_.vocab, H, ef, s);
    int32_t* d_out = scratch<int32_t>(dc.out_tok, 1);
    k::argmax_rows(logits, 1, cfg_.vocab, d_out, s);
    cuda_ok(cudaMemcpyAsync(&first, d_out, 4, cudaMemcpyDeviceToHost, s), "d2h");
    if (a.chunk_logits_out) {
      lg.resize(static_cast<size_t>(cfg_.vocab));
      cuda_ok(cudaMemcpyAsync(lg.data(), logits, lg.size() * 4, cudaMemcpyDeviceToHost, s), "d2h");
    }
  }
  cuda_ok(cudaEventRecord(t1, s), "event");
  check_cuda("chunk (multi-domain) launch");
  cuda_ok(cudaStreamSynchronize(s), "chunk");
  float ms = 0;
  cuda_ok(cudaEventElapsedTime(&ms, t0, t1), "elapsed");
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (ms_out) *ms_out = ms;
  if (a.chunk_final) {
    requests_[a.chunk_request].tokens.push_back(first);
    if (a.chunk_first_token_out) *a.chunk_first_token_out = first;
    if (a.chunk_logits_out) std::memcpy(a.chunk_logits_out, lg.data(), lg.size() * sizeof(float));
  } else if (a.chunk_first_token_out) {
    *a.chunk_first_token_out = -1;
  }
}

void Runtime::decode_multi(const esp_decode_args& a, const std::vector<DecodeRow>& rows_v,
                           const std::vector<RequestId>& batch) {
  const int b = static_cast<int>(rows_v.size());
  const int H = cfg_.hidden, F = cfg_.ffn, heads = cfg_.heads, hd = cfg_.head_dim;
  // Row g's master domain; per master domain its rows (ascending g).
  std::vector<int> mdom(static_cast<size_t>(b));
  std::map<int, std::vector<int32_t>> mrows;
  for (int g = 0; g < b; ++g) {
    mdom[g] = inst(rows_v[g].master).domain;
    mrows[mdom[g]].push_back(g);
  }
  std::map<int, std::map<int32_t, int32_t>> local_of;  // domain -> global row -> local
  for (auto& [dom, rs] : mrows) {
    for (size_t j = 0; j < rs.size(); ++j) local_of[dom][rs[j]] = static_cast<int32_t>(j);
  }
  // Chunks ordered by (master domain, KV domain, row, instance): the partials
  // one KV domain owes one master domain form one contiguous range.
  struct Ch {
    int md, xd;
    int32_t row;
    InstanceId inst;
    const int32_t* slots;
    int32_t n;
  };
  std::vector<Ch> all;
  for (int g = 0; g < b; ++g) {
    RequestRec& rr = req(rows_v[g].r);
    for (auto& [iid, pl] : rr.pages) {
      if (pl.slots.empty()) continue;
      DeviceCtx& xc = *devices_[static_cast<size_t>(inst(iid).domain)];
      DeviceGuard gd(xc.device);
      sync_pages(pl, xc.stream);
      const int64_t nsl = static_cast<int64_t>(pl.slots.size());
      for (int64_t c0 = 0; c0 < nsl; c0 += decode_chunk()) {
        all.push_back({mdom[g], inst(iid).domain, g, iid, pl.dev + c0,
                       static_cast<int32_t>(std::min<int64_t>(decode_chunk(), nsl - c0))});
      }
    }
  }
  std::stable_sort(all.begin(), all.end(), [](const Ch& x, const Ch& y) {
    return x.md != y.md ? x.md < y.md : (x.xd != y.xd ? x.xd < y.xd : x.row < y.row);
  });
  const int n_chunks = static_cast<int>(all.size());
  std::map<int, std::vector<k::DecodeChunk>> xchunks;              // per KV domain
  std::map<std::pair<int, int>, std::pair<int, int>> range_of;     // (md, xd) -> [c0, c1)
  std::map<int, std::set<int32_t>> q_need;                          // xd -> rows it needs
  std::vector<std::vector<int32_t>> chunks_of_row(static_cast<size_t>(b));
  for (int c = 0; c < n_chunks; ++c) {
    const Ch& ch = all[static_cast<size_t>(c)];
    xchunks[ch.xd].push_back({ch.slots, ch.n, ch.row, inst(ch.inst).slab, c});
    auto key = std::make_pair(ch.md, ch.xd);
    auto it = range_of.find(key);
    if (it == range_of.end()) range_of[key] = {c, c + 1};
    else it->second.second = c + 1;
    q_need[ch.xd].insert(ch.row);
    chunks_of_row[ch.row].push_back(c);
  }
  std::vector<int32_t> row_start(static_cast<size_t>(b) + 1, 0), chunk_ids;
  for (int g = 0; g < b; ++g) {
    row_start[g] = static_cast<int32_t>(chunk_ids.size());
    chunk_ids.insert(chunk_ids.end(), chunks_of_row[g].begin(), chunks_of_row[g].end());
  }
  row_start[b] = static_cast<int32_t>(chunk_ids.size());
  std::set<int> doms;
  for (auto& kv : mrows) doms.insert(kv.first);
  for (auto& kv : xchunks) doms.insert(kv.first);

  int64_t max_pos = 0;
  for (const DecodeRow& rw : rows_v) max_pos = std::max<int64_t>(max_pos, rw.pos + 1);
  for (int dom : doms) {
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cudaStream_t s = dc.stream;
    dc.sync_used = 0;
    ensure_rope(dc, max_pos);
    scratch<bf16>(dc.qin, static_cast<size_t>(b) * H);
    scratch<float>(dc.part_o, static_cast<size_t>(std::max(n_chunks, 1)) * heads * hd);
    scratch<float>(dc.part_ml, static_cast<size_t>(std::max(n_chunks, 1)) * heads * 2);
    if (xchunks.count(dom)) {
      h2d(scratch<k::DecodeChunk>(dc.chunks, xchunks[dom].size()), xchunks[dom], s);
    }
    cuda_ok(cudaEventRecord(dc.e0, s), "event");
    if (!mrows.count(dom)) continue;
    const std::vector<int32_t>& rs = mrows[dom];
    std::vector<int32_t> tok, pos, rinst, rslot;
    for (int32_t gr : rs) {
      tok.push_back(rows_v[gr].token);
      pos.push_back(rows_v[gr].pos);
      rinst.push_back(inst(rows_v[gr].master).slab);
      rslot.push_back(rows_v[gr].slot);
    }
    const size_t nl = rs.size();
    h2d(scratch<int32_t>(dc.tok, nl), tok, s);
    h2d(scratch<int32_t>(dc.pos, nl), pos, s);
    h2d(scratch<int32_t>(dc.rinst, nl), rinst, s);
    h2d(scratch<int32_t>(dc.rslot, nl), rslot, s);
    h2d(scratch<int32_t>(dc.row_start, row_start.size()), row_start, s);
    h2d(scratch<int32_t>(dc.chunk_ids, chunk_ids.size() + 1), chunk_ids, s);
    h2d(scratch<int32_t>(dc.row_list, nl), rs, s);
    scratch<bf16>(dc.x, nl * H);
    scratch<bf16>(dc.xn, nl * H);
    scratch<bf16>(dc.q, nl * H);
    scratch<bf16>(dc.attn, nl * H);
    scratch<bf16>(dc.h, nl * F);
    // sums of squares for the fused RMSNorm (used when fuse_dec below holds)
    float* ss1 = nullptr;
    if (opts_.fuse_norm_decode && !opts_.decode_copy && nl <= 32) {
      ss1 = scratch<float>(dc.ss1, 32);
      cuda_ok(cudaMemsetAsync(scratch<float>(dc.ss2, 32), 0, 32 * sizeof(float), s), "memset");
    }
    timed(kPhEmbed, s, [&] {
      k::embed(static_cast<int32_t*>(dc.tok.ptr), dc.embed, static_cast<bf16*>(dc.x.ptr),
               static_cast<int>(nl), H, s, ss1);
    });
  }
  const float scale = 1.0f / std::sqrt(static_cast<float>(hd));
  // Fused transport (default): the masters' QKV epilogues store their q rows
  // straight into every KV domain's query buffer (the broadcast as peer
  // stores), and each KV domain's attention kernel stores its split-KV
  // partials straight into the master domains' partial buffers (the gather as
  // peer stores). Only events order the domains. ESP_DECODE_COPY=1 keeps the
  // copy-engine transport (peer copies of row runs / chunk ranges).
  const bool copy_transport = opts_.decode_copy;
  // Per master domain: the KV domains its rows need (q destinations); per KV
  // domain: the master domains it owes partials (PartDst entries).
  std::map<int, std::vector<int>> q_dests;
  std::map<int, std::vector<int>> part_dests;
  for (auto& [key, rg] : range_of) {
    q_dests[key.first].push_back(key.second);
    part_dests[key.second].push_back(key.first);
  }
  bool fused = !copy_transport;
  for (auto& [md, v] : q_dests) {
    if (static_cast<int>(v.size()) > k::kMaxPeers + 1) fused = false;
  }
  for (auto& [xd, v] : part_dests) {
    if (static_cast<int>(v.size()) > k::kMaxPartDst) fused = false;
  }
  // Fused transport: a KV domain that is also a master computes the chunks
  // of its OWN rows first, in a launch that needs only its own QKV, while the
  // other masters' queries are still on their way (the query
  // exchange overlapped with local attention); the rest follows once they
  // have landed. own_n[xd] = number of leading own-row chunks.
  std::map<int, int> own_n;
  if (fused) {
    for (auto& [xd, chs] : xchunks) {
      std::stable_partition(chs.begin(), chs.end(),
                            [&](const k::DecodeChunk& ch) { return mdom[ch.row] == xd; });
      int own = 0;
      for (const k::DecodeChunk& ch : chs) own += mdom[ch.row] == xd ? 1 : 0;
      own_n[xd] = own;
      // chunk -> index of its master domain in the KV domain's PartDst table
      const std::vector<int>& pdv = part_dests[xd];
      for (k::DecodeChunk& ch : chs) {
        const int md = mdom[ch.row];
        ch.dst = static_cast<int32_t>(std::find(pdv.begin(), pdv.end(), md) - pdv.begin());
      }
      DeviceCtx& xc = *devices_[static_cast<size_t>(xd)];
      DeviceGuard g(xc.device);
      h2d(static_cast<k::DecodeChunk*>(xc.chunks.ptr), chs, xc.stream);
    }
  }
  // RMSNorm fused into the masters' skinny GEMMs (<= 32 rows per master),
  // exactly as the single-domain decode: sums of squares accumulate in the
  // residual epilogues, the consuming GEMM scales its rows.
  const bool fuse_dec = fused && opts_.fuse_norm_decode && [&] {
    for (auto& [md, rs] : mrows) {
      if (rs.size() > 32) return false;
    }
    return true;
  }();
  // (the masters' embeddings above already stored the sums of squares)
  if (fused) {
    std::map<int, cudaEvent_t> att_done, comb_done;  // previous layer's
    for (int l = 0; l < cfg_.layers; ++l) {
      std::map<int, cudaEvent_t> q_ready;
      // 1. masters: norm + QKV; q rows pushed to the KV domains' qin.
      for (auto& [md, rs] : mrows) {
        DeviceCtx& dc = *devices_[static_cast<size_t>(md)];
        DeviceGuard g(dc.device);
        cudaStream_t s = dc.stream;
        for (int xd : q_dests[md]) {  // qin readers of the previous layer
          if (att_done.count(xd)) cuda_ok(cudaStreamWaitEvent(s, att_done[xd], 0), "wait");
        }
        const int nl = static_cast<int>(rs.size());
        const LayerW& w = dc.layers[l];
        bf16* x = static_cast<bf16*>(dc.x.ptr);
        bf16* xn = static_cast<bf16*>(dc.xn.ptr);
        if (!fuse_dec) {
          timed(kPhNorm, s, [&] { k::rmsnorm(x, nullptr, nullptr, xn, nl, H, cfg_.rms_eps, s); });
        }
        k::GemmEpilogue ep;
        ep.kind = k::kEpiQkvRope;
        if (fuse_dec) {
          ep.ss_in = static_cast<float*>(dc.ss1.ptr);
          ep.ss_zero = static_cast<float*>(dc.ss2.ptr);
          ep.norm_dim = H;
          ep.norm_eps = cfg_.rms_eps;
        }
        ep.q_out = static_cast<bf16*>(dc.q.ptr);
        ep.pos = static_cast<int32_t*>(dc.pos.ptr);
        ep.rope = dc.rope;
        ep.hidden = H;
        ep.head_dim = hd;
        ep.row_inst = static_cast<int32_t*>(dc.rinst.ptr);
        ep.row_slot = static_cast<int32_t*>(dc.rslot.ptr);
        ep.q_rows = static_cast<int32_t*>(dc.row_list.ptr);  // local row -> global row
        bool own = false;
        for (int xd : q_dests[md]) {
          bf16* qin = static_cast<bf16*>(devices_[static_cast<size_t>(xd)]->qin.ptr);
          if (xd == md) {
            ep.q_out = qin;  // this domain's own KV: its qin is the q output
            own = true;
          } else {
            ep.q_peer[ep.n_qpeer++] = qin;
          }
        }
        if (!own) ep.q_out = nullptr;
        if (ep.n_qpeer > k::kMaxPeers) throw InternalError("too many query destinations");
        for (size_t j = 0; j < dc.slabs.size(); ++j) {
          ep.slab_k[j] = instances_[dc.slabs[j]].layer_k(l);
          ep.slab_v[j] = instances_[dc.slabs[j]].layer_v(l);
        }
        timed(kPhQkv, s, [&] { k::gemm(fuse_dec ? x : xn, H, w.wqkv, H, nl, 3 * H, H, ep, s); });
        cudaEvent_t e = sync_event(dc);
        cuda_ok(cudaEventRecord(e, s), "event");
        q_ready[md] = e;
      }
      // 2. KV domains: split-KV partials pushed to the masters' buffers —
      // own rows first (no cross-domain wait), then the other masters' rows.
      std::map<int, cudaEvent_t> att_now;
      for (auto& [xd, chs] : xchunks) {
        DeviceCtx& xc = *devices_[static_cast<size_t>(xd)];
        DeviceGuard g(xc.device);
        cudaStream_t s = xc.stream;
        k::PartDst pd;
        const std::vector<int>& pdv = part_dests[xd];
        for (size_t i = 0; i < pdv.size(); ++i) {
          DeviceCtx& mc = *devices_[static_cast<size_t>(pdv[i])];
          pd.o[i] = static_cast<float*>(mc.part_o.ptr);
          pd.ml[i] = static_cast<float*>(mc.part_ml.ptr);
        }
        k::DecodeSlabs slabs{};
        for (size_t j = 0; j < xc.slabs.size(); ++j) {
          slabs.k[j] = instances_[xc.slabs[j]].layer_k(l);
          slabs.v[j] = instances_[xc.slabs[j]].layer_v(l);
        }
        const int own = own_n[xd], n_ch = static_cast<int>(chs.size());
        auto attend = [&](int c0, int c1) {
          if (c1 <= c0) return;
          int max_n = 0;
          for (int c = c0; c < c1; ++c) max_n = std::max(max_n, static_cast<int>(chs[c].n));
          timed(kPhDecodeAttn, s, [&] {
            k::decode_attention(static_cast<bf16*>(xc.qin.ptr),
                                static_cast<k::DecodeChunk*>(xc.chunks.ptr) + c0, c1 - c0, slabs,
                                heads, hd, scale, static_cast<float*>(xc.part_o.ptr),
                                static_cast<float*>(xc.part_ml.ptr), s, &pd, nullptr, max_n);
          });
        };
        // own rows: this domain's QKV is earlier on its stream; its own
        // combine of the previous layer too (stream order)
        attend(0, own);
        for (int md : pdv) {
          if (md == xd) continue;
          cuda_ok(cudaStreamWaitEvent(s, q_ready[md], 0), "wait");
          // the master's combine of the previous layer has read its partials
          if (comb_done.count(md)) cuda_ok(cudaStreamWaitEvent(s, comb_done[md], 0), "wait");
        }
        attend(own, n_ch);
        cudaEvent_t e = sync_event(xc);
        cuda_ok(cudaEventRecord(e, s), "event");
        att_now[xd] = e;
      }
      att_done = att_now;
      // 3. masters: LSE combine over the pushed partials, then the dense layers.
      std::map<int, cudaEvent_t> comb_now;
      for (auto& [md, rs] : mrows) {
        DeviceCtx& mc = *devices_[static_cast<size_t>(md)];
        DeviceGuard g(mc.device);
        cudaStream_t s = mc.stream;
        for (int xd : q_dests[md]) cuda_ok(cudaStreamWaitEvent(s, att_done[xd], 0), "wait");
        const int nl = static_cast<int>(rs.size());
        const LayerW& w = mc.layers[l];
        bf16* x = static_cast<bf16*>(mc.x.ptr);
        bf16* xn = static_cast<bf16*>(mc.xn.ptr);
        bf16* attn = static_cast<bf16*>(mc.attn.ptr);
        bf16* hbuf = static_cast<bf16*>(mc.h.ptr);
        timed(kPhCombine, s, [&] {
          k::decode_combine_rows(static_cast<float*>(mc.part_o.ptr),
                                 static_cast<float*>(mc.part_ml.ptr),
                                 static_cast<int32_t*>(mc.row_start.ptr),
                                 static_cast<int32_t*>(mc.chunk_ids.ptr),
                                 static_cast<int32_t*>(mc.row_list.ptr), nl, heads, hd, attn, s);
        });
        cudaEvent_t e = sync_event(mc);
        cuda_ok(cudaEventRecord(e, s), "event");
        comb_now[md] = e;
        NormFuse nf;
        if (fuse_dec) {
          nf.ss_o = static_cast<float*>(mc.ss2.ptr);
          nf.ss_d = static_cast<float*>(mc.ss1.ptr);
          nf.zero_in_kernel = true;
        }
        o_and_mlp(mc, l, nl, x, attn, xn, hbuf, nf, s);
      }
      comb_done = comb_now;
    }
  }
  std::map<int, std::vector<cudaEvent_t>> q_readers, part_readers;
  for (int l = 0; !fused && l < cfg_.layers; ++l) {
    std::map<int, cudaEvent_t> q_ready, part_ready;
    // 1. masters: norm + QKV (+RoPE, the new token's K/V appended at the master).
    for (auto& [dom, rs] : mrows) {
      DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
      DeviceGuard g(dc.device);
      cudaStream_t s = dc.stream;
      for (cudaEvent_t e : q_readers[dom]) cuda_ok(cudaStreamWaitEvent(s, e, 0), "wait");
      q_readers[dom].clear();
      const int nl = static_cast<int>(rs.size());
      const LayerW& w = dc.layers[l];
      bf16* x = static_cast<bf16*>(dc.x.ptr);
      bf16* xn = static_cast<bf16*>(dc.xn.ptr);
      timed(kPhNorm, s, [&] { k::rmsnorm(x, nullptr, nullptr, xn, nl, H, cfg_.rms_eps, s); });
      k::GemmEpilogue ep;
      ep.kind = k::kEpiQkvRope;
      ep.q_out = static_cast<bf16*>(dc.q.ptr);
      ep.pos = static_cast<int32_t*>(dc.pos.ptr);
      ep.rope = dc.rope;
      ep.hidden = H;
      ep.head_dim = hd;
      ep.row_inst = static_cast<int32_t*>(dc.rinst.ptr);
      ep.row_slot = static_cast<int32_t*>(dc.rslot.ptr);
      for (size_t j = 0; j < dc.slabs.size(); ++j) {
        ep.slab_k[j] = instances_[dc.slabs[j]].layer_k(l);
        ep.slab_v[j] = instances_[dc.slabs[j]].layer_v(l);
      }
      timed(kPhQkv, s, [&] { k::gemm(xn, H, w.wqkv, H, nl, 3 * H, H, ep, s); });
      cudaEvent_t e = sync_event(dc);
      cuda_ok(cudaEventRecord(e, s), "event");
      q_ready[dom] = e;
    }
    // 2. query broadcast to the KV domains, split-KV partials there.
    for (auto& [xd, chs] : xchunks) {
      DeviceCtx& xc = *devices_[static_cast<size_t>(xd)];
      DeviceGuard g(xc.device);
      cudaStream_t s = xc.stream;
      for (cudaEvent_t e : part_readers[xd]) cuda_ok(cudaStreamWaitEvent(s, e, 0), "wait");
      part_readers[xd].clear();
      for (auto& [md, rs] : mrows) {
        DeviceCtx& mc = *devices_[static_cast<size_t>(md)];
        bool waited = false;
        // maximal runs of this master domain's rows that xd needs
        for (size_t j = 0; j < rs.size();) {
          if (!q_need[xd].count(rs[j])) {
            ++j;
            continue;
          }
          size_t k2 = j + 1;
          while (k2 < rs.size() && q_need[xd].count(rs[k2]) && rs[k2] == rs[k2 - 1] + 1) ++k2;
          if (!waited) {
            cuda_ok(cudaStreamWaitEvent(s, q_ready[md], 0), "wait");
            waited = true;
          }
          peer_copy(static_cast<bf16*>(xc.qin.ptr) + static_cast<size_t>(rs[j]) * H, xc.device,
                    static_cast<bf16*>(mc.q.ptr) + j * H, mc.device, (k2 - j) * H * sizeof(bf16), s);
          j = k2;
        }
        if (waited) {
          cudaEvent_t e = sync_event(xc);
          cuda_ok(cudaEventRecord(e, s), "event");
          q_readers[md].push_back(e);
        }
      }
      k::DecodeSlabs slabs{};
      for (size_t j = 0; j < xc.slabs.size(); ++j) {
        slabs.k[j] = instances_[xc.slabs[j]].layer_k(l);
        slabs.v[j] = instances_[xc.slabs[j]].layer_v(l);
      }
      int max_n = 0;
      for (const k::DecodeChunk& c : chs) max_n = std::max(max_n, static_cast<int>(c.n));
      timed(kPhDecodeAttn, s, [&] {
        k::decode_attention(static_cast<bf16*>(xc.qin.ptr),
                            static_cast<k::DecodeChunk*>(xc.chunks.ptr),
                            static_cast<int>(chs.size()), slabs, heads, hd, scale,
                            static_cast<float*>(xc.part_o.ptr), static_cast<float*>(xc.part_ml.ptr), s,
                            nullptr, nullptr, max_n);
      });
      cudaEvent_t e = sync_event(xc);
      cuda_ok(cudaEventRecord(e, s), "event");
      part_ready[xd] = e;
    }
    // 3. partial gather + LSE combine at the masters, then the dense layers.
    for (auto& [md, rs] : mrows) {
      DeviceCtx& mc = *devices_[static_cast<size_t>(md)];
      DeviceGuard g(mc.device);
      cudaStream_t s = mc.stream;
      for (auto& [key, rg] : range_of) {
        if (key.first != md) continue;
        const int xd = key.second;
        cuda_ok(cudaStreamWaitEvent(s, part_ready[xd], 0), "wait");
        if (xd == md) continue;
        DeviceCtx& xc = *devices_[static_cast<size_t>(xd)];
        const size_t c0 = static_cast<size_t>(rg.first), c1 = static_cast<size_t>(rg.second);
        peer_copy(static_cast<float*>(mc.part_o.ptr) + c0 * heads * hd, mc.device,
                  static_cast<float*>(xc.part_o.ptr) + c0 * heads * hd, xc.device,
                  (c1 - c0) * heads * hd * sizeof(float), s);
        peer_copy(static_cast<float*>(mc.part_ml.ptr) + c0 * heads * 2, mc.device,
                  static_cast<float*>(xc.part_ml.ptr) + c0 * heads * 2, xc.device,
                  (c1 - c0) * heads * 2 * sizeof(float), s);
        cudaEvent_t e = sync_event(mc);
        cuda_ok(cudaEventRecord(e, s), "event");
        part_readers[xd].push_back(e);
      }
      const int nl = static_cast<int>(rs.size());
      const LayerW& w = mc.layers[l];
      bf16* x = static_cast<bf16*>(mc.x.ptr);
      bf16* xn = static_cast<bf16*>(mc.xn.ptr);
      bf16* attn = static_cast<bf16*>(mc.attn.ptr);
      bf16* hbuf = static_cast<bf16*>(mc.h.ptr);
      timed(kPhCombine, s, [&] {
        k::decode_combine_rows(static_cast<float*>(mc.part_o.ptr), static_cast<float*>(mc.part_ml.ptr),
                               static_cast<int32_t*>(mc.row_start.ptr),
                               static_cast<int32_t*>(mc.chunk_ids.ptr),
                               static_cast<int32_t*>(mc.row_list.ptr), nl, heads, hd, attn, s);
      });
      o_and_mlp(mc, l, nl, x, attn, xn, hbuf, NormFuse{}, s);
    }
  }
  // 4. LM head + greedy token at each master.
  std::map<int, std::vector<int32_t>> out_tok;
  std::map<int, std::vector<float>> out_lg;
  for (auto& [md, rs] : mrows) {
    DeviceCtx& mc = *devices_[static_cast<size_t>(md)];
    DeviceGuard g(mc.device);
    cudaStream_t s = mc.stream;
    const int nl = static_cast<int>(rs.size());
    bf16* xn = static_cast<bf16*>(mc.xn.ptr);
    timed(kPhNorm, s, [&] {
      k::rmsnorm(static_cast<bf16*>(mc.x.ptr), nullptr, mc.final_norm, xn, nl, H, cfg_.rms_eps, s);
    });
    float* logits = scratch<float>(mc.logits, static_cast<size_t>(nl) * cfg_.vocab);
    k::GemmEpilogue ef;
    ef.kind = k::kEpiStoreF32;
    ef.out = logits;
    ef.ldo = cfg_.vocab;
    timed(kPhLmHead, s, [&] { k::gemm(xn, H, mc.lm_head, H, nl, cfg_.vocab, H, ef, s); });
    int32_t* d_out = scratch<int32_t>(mc.out_tok, nl);
    timed(kPhArgmax, s, [&] { k::argmax_rows(logits, nl, cfg_.vocab, d_out, s); });
    out_tok[md].resize(static_cast<size_t>(nl));
    cuda_ok(cudaMemcpyAsync(out_tok[md].data(), d_out, nl * 4, cudaMemcpyDeviceToHost, s), "d2h");
    if (a.logits_out) {
      out_lg[md].resize(static_cast<size_t>(nl) * cfg_.vocab);
      cuda_ok(cudaMemcpyAsync(out_lg[md].data(), logits, out_lg[md].size() * 4,
                              cudaMemcpyDeviceToHost, s),
              "d2h");
    }
  }
  double ms_max = 0;
  for (int dom : doms) {
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cuda_ok(cudaEventRecord(dc.e1, dc.stream), "event");
    check_cuda("decode (multi-domain) launch");
  }
  for (int dom : doms) {
    DeviceCtx& dc = *devices_[static_cast<size_t>(dom)];
    DeviceGuard g(dc.device);
    cuda_ok(cudaStreamSynchronize(dc.stream), "decode (multi-domain)");
    float ms = 0;
    cuda_ok(cudaEventElapsedTime(&ms, dc.e0, dc.e1), "elapsed");
    ms_max = std::max<double>(ms_max, ms);
  }
  if (cap_armed_) cap_finish();
  collect_phase_events();
  if (a.device_ms_out) *a.device_ms_out = ms_max;
  std::map<RequestId, std::pair<int, int>> where;  // request -> (domain, local row)
  for (auto& [md, rs] : mrows) {
    for (size_t j = 0; j < rs.size(); ++j) where[rows_v[rs[j]].r] = {md, static_cast<int>(j)};
  }
  for (int i = 0; i < b; ++i) {
    const auto [md, j] = where.at(batch[i]);
    RequestRec& rr = req(batch[i]);
    const int32_t tok = out_tok[md][static_cast<size_t>(j)];
    if (a.in_tokens) rr.tokens.push_back(a.in_tokens[i]);
    rr.tokens.push_back(tok);
    if (a.out_tokens) a.out_tokens[i] = tok;
    if (a.logits_out) {
      std::memcpy(a.logits_out + static_cast<size_t>(i) * cfg_.vocab,
                  out_lg[md].data() + static_cast<size_t>(j) * cfg_.vocab,
                  cfg_.vocab * sizeof(float));
    }
  }
}

}  // namespace esp
