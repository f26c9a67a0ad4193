// K1: striped ring attention, two query tiles per CTA.
//
// Flash attention over the striped causal mask of a ring position (key b of
// origin o is visible to query a of position i iff b <= a - [o > i]),
// structured so the tensor core never waits on one softmax:
//   * a CTA owns 256 query rows = two 128-row tiles (t = 0, 1) of the same
//     (segment, head); both share every K/V tile loaded by TMA;
//   * TMEM = S0 | S1 | O0 | O1 (512 columns). Tile t's softmax reads S_t,
//     writes P_t (bf16, 2 per 32-bit column) back over S_t, and the MMA warp
//     issues O_t += P_t V with A read straight from TMEM (no smem round trip);
//   * the MMA warp interleaves the tiles: PV_0,j  S_0,j+1  PV_1,j  S_1,j+1 —
//     while softmax WG 0 works on S_0,j+1 the tensor core runs tile 1's PV and
//     S, and vice versa;
//   * warp-group register split with setmaxnreg (producer/MMA WG shrinks,
//     the two softmax WGs grow).
// The union of the two tiles' visible KV tiles is streamed once; tile 0
// (earlier queries) skips the causal tail it cannot see.
#include <cuda.h>

#include <cstdlib>
#include <mutex>
#include <stdexcept>

#include "kernels.h"
#include "ptx.cuh"

namespace esp::k {

CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld,
                           int box_rows);

namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int kVStagesDefault = 2;  // V stages
constexpr int kPartsDefault = 4;    // P stored (and P.V issued) in this many key parts:
                                    // in-step A/B 4 vs 2: K1 +2.7 % (r02_k1_parts_study.txt)
#ifndef ESP_K1_KSTAGES
#define ESP_K1_KSTAGES 2
#endif
constexpr int kKStages = ESP_K1_KSTAGES;  // K stages (3 measured: no gain, 6.91-7.01 vs 6.76-6.96 ms)
constexpr int kThreads = 384;
constexpr float kRescaleThreshold = 8.0f;
constexpr int kDefaultPoly8 = 2;  // in-step A/B (profiles/r02_poly_ab.txt): 2 > 0 > 1

template <int HD, int kVSt>
struct Cfg2 {
  static constexpr int kBoxes = HD / 64;
  static constexpr int kQBytes = BM * HD * 2;
  static constexpr int kKvBytes = BN * HD * 2;
  static constexpr int kSmem = 2 * kQBytes + (kKStages + kVSt) * kKvBytes + 1024 + 512;
};

// Packed fp32x2 arithmetic (sm_100a FFMA2 / FADD2): half the FMA-pipe
// instructions of the softmax.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// 2^x for a pair on the FMA/ALU pipes (x <= 2^7): round-to-nearest split
// x = n + f with the 1.5*2^23 trick, a polynomial for 2^f on [-1/2, 1/2]
// (minimax quadratic; Taylor cubic in the study build), 2^n by adding n
// to the exponent field. Used for kPoly8/8 of the softmax exponentials so the
// MUFU (ex2) pipe (16/clk/SM, shared by both softmax warpgroups) stops being
// the co-bottleneck with the tensor core.
template <bool kCubic>
__device__ __forceinline__ void exp2_fma2(float x0, float x1, float& p0, float& p1) {
  const uint64_t x = f2pack(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
  const uint64_t magic = f2pack(12582912.0f, 12582912.0f);
  const uint64_t t = fadd2(x, magic);
  const uint64_t r = fadd2(t, f2pack(-12582912.0f, -12582912.0f));
  const uint64_t f = ffma2(r, f2pack(-1.0f, -1.0f), x);
  uint64_t p;
  if constexpr (kCubic) {  // Taylor cubic, rel. err < 7.9e-4
    p = ffma2(f2pack(0.0555041087f, 0.0555041087f), f, f2pack(0.240226507f, 0.240226507f));
    p = ffma2(p, f, f2pack(0.693147181f, 0.693147181f));
    p = ffma2(p, f, f2pack(1.0f, 1.0f));
  } else {
    // minimax quadratic on [-1/2, 1/2]: rel. err < 1.73e-3, under the bf16
    // half ulp (1.95e-3) P is rounded to anyway; one FFMA2 per pair less
    // (in-step A/B vs the cubic: K1 +1 %, r02_k1_parts_study.txt)
    p = ffma2(f2pack(0.2384257f, 0.2384257f), f, f2pack(0.70344281f, 0.70344281f));
    p = ffma2(p, f, f2pack(1.00044296f, 1.00044296f));
  }
  float t0, t1, q0, q1;
  f2unpack(t, t0, t1);
  f2unpack(p, q0, q1);
  // (n << 23) with n = bits(t) - 0x4B400000 equals bits(t) << 23 mod 2^32.
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ int tiles_visible(const RingSegment& sg, int r, int q0) {
  const int a_max = min(q0 + BM - 1, sg.q_len - 1);
  const int vis = min(sg.kv_len[r], a_max - sg.shift[r] + 1);
  return vis <= 0 ? 0 : (vis + BN - 1) / BN;
}

struct Item {
  int seg, pair, head;
  int q0[2];
  bool act1;  // tile 1 exists (q rows past q_len are not a tile)
};

__device__ __forceinline__ Item load_item(const int32_t* work, int w,
                                          const RingSegment* segs) {
  Item it;
  it.seg = __ldg(&work[2 * w]);
  const int packed = __ldg(&work[2 * w + 1]);
  it.pair = packed >> 8;
  it.head = packed & 0xFF;
  it.q0[0] = it.pair * 2 * BM;
  it.q0[1] = it.q0[0] + BM;
  it.act1 = it.q0[1] < segs[it.seg].q_len;
  return it;
}

// Iterates the union KV-tile sequence of an item: (round r, tile tt) and
// whether each query tile sees it.
struct Steps {
  const RingSegment* sg;
  int q_own;  // q0 of the tile that owns the union (tile 1 if active)
  int q0t0;
  int r = 0, tt = 0, n_r = 0, n0_r = 0;
  __device__ void begin(const RingSegment* s, const Item& it) {
    sg = s;
    q_own = it.act1 ? it.q0[1] : it.q0[0];
    q0t0 = it.q0[0];
    r = -1;
    tt = 0;
    n_r = 0;
    advance_round();
  }
  __device__ void advance_round() {
    do {
      ++r;
      if (r >= sg->n_rounds) return;
      n_r = tiles_visible(*sg, r, q_own);
      n0_r = tiles_visible(*sg, r, q0t0);
      tt = 0;
    } while (n_r == 0);
  }
  __device__ bool valid() const { return r < sg->n_rounds; }
  __device__ void next() {
    if (++tt >= n_r) advance_round();
  }
  __device__ int kv_row() const { return sg->kv_row0[r] + tt * BN; }
  __device__ bool active0() const { return tt < n0_r; }
};

// Opt-in cycle accounting (kProf): per CTA, 4 roles x 8 counters of clock64
// cycles spent waiting on each barrier / computing; see esp_k_ring_attention.
#define ESP_PROF_WAIT(slot, expr)                  \
  do {                                             \
    if constexpr (kProf) {                         \
      const uint64_t _t0 = clock64();              \
      expr;                                        \
      prof_acc[slot] += clock64() - _t0;           \
    } else {                                       \
      expr;                                        \
    }                                              \
  } while (0)

template <int HD, bool kProf, int kPoly8, bool kCarry, int kParts, int kStages, bool kCubic>
__global__ void __launch_bounds__(kThreads, 1)
    ring_attention_tcgen05(const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ out,
                      int hidden, const RingSegment* __restrict__ segs,
                      const int32_t* __restrict__ work, int n_work, float scale_log2,
                      uint64_t* __restrict__ prof, const __grid_constant__ RingWait wait,
                      const __grid_constant__ RingCarry carry) {
  using C = Cfg2<HD, kStages>;
  static_assert(kParts == 2 || kParts == 4 || kParts == 8, "P parts");
  constexpr int kCP = 64 / kParts;  // packed bf16x2 P columns per part (2 keys each)
  uint64_t prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint64_t prof_t_begin = kProf ? clock64() : 0;
  auto prof_store = [&](int role) {
    if constexpr (kProf) {
      prof_acc[7] = clock64() - prof_t_begin;
      for (int i = 0; i < 8; ++i) prof[(blockIdx.x * 4 + role) * 8 + i] = prof_acc[i];
    }
  };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                                 // [2][kQBytes]
  uint8_t* sK = sQ + 2 * C::kQBytes;                  // [kKStages][kKvBytes]
  uint8_t* sV = sK + kKStages * C::kKvBytes;          // [kStages][kKvBytes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kStages * C::kKvBytes);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = k_full + kKStages;
  uint64_t* v_full = k_empty + kKStages;
  uint64_t* v_empty = v_full + kStages;
  uint64_t* s_full = v_empty + kStages;  // [2] per query tile
  uint64_t* p_full = s_full + 2;         // [2 tiles][kParts key parts]
  uint64_t* o_done = p_full + 2 * kParts;  // [2]
  uint64_t* o_free = o_done + 2;         // [2]
  uint64_t* o_init = o_free + 2;         // [2] carried O stored into TMEM (carry_in)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_init + 2);
  const bool cin = kCarry && carry.carry_in != 0;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmQ);
    ptx::tma_prefetch_desc(&tmK);
    ptx::tma_prefetch_desc(&tmV);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < kKStages; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      for (int p = 0; p < kParts; ++p) ptx::mbar_init(&p_full[kParts * t + p], 128);
      ptx::mbar_init(&o_done[t], 1);
      ptx::mbar_init(&o_free[t], 128);
      ptx::mbar_init(&o_init[t], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // This CTA's contiguous slice of the host-built schedule (after the items:
  // G, then G+1 offsets; build_attention_work). CTAs >= G have no work.
  const int n_sched = __ldg(&work[2 * n_work]);
  const int w_begin = static_cast<int>(blockIdx.x) < n_sched ? __ldg(&work[2 * n_work + 1 + blockIdx.x]) : 0;
  const int w_end = static_cast<int>(blockIdx.x) < n_sched ? __ldg(&work[2 * n_work + 2 + blockIdx.x]) : 0;
  const uint32_t t_s[2] = {tmem, tmem + BN};
  const uint32_t t_o[2] = {tmem + 2 * BN, tmem + 2 * BN + HD};

  if (warp < 4) {
    ptx::setmaxnreg_dec<104>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------- producer
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0, items = 0;
      uint32_t arrived = 0;  // source domains whose blocks of this launch have landed
      for (int w = w_begin; w < w_end; ++w, ++items) {
        const Item it = load_item(work, w, segs);
        const RingSegment* sg = &segs[it.seg];
        ESP_PROF_WAIT(0, ptx::mbar_wait(q_empty, (items & 1) ^ 1));
        ptx::mbar_expect_tx(q_full, C::kQBytes * (it.act1 ? 2 : 1));
        for (int t = 0; t < (it.act1 ? 2 : 1); ++t) {
          for (int b = 0; b < C::kBoxes; ++b) {
            ptx::tma_load_2d(sQ + t * C::kQBytes + b * (BM * 128), &tmQ, q_full,
                             it.head * HD + b * 64, sg->q_row0 + it.q0[0] + t * BM);
          }
        }
        Steps st;
        for (st.begin(sg, it); st.valid(); st.next()) {
          const int row = st.kv_row();
          const int src = sg->wait_src[st.r] - 1;
          if (src >= 0 && !(arrived >> src & 1u)) {
            // The round's block comes from another GPU's QKV epilogue (peer
            // stores + system-scope counter): wait for the layer's total,
            // then order those generic-proxy writes before our TMA reads.
            const uint64_t t0 = ptx::globaltimer_ns();
            while (ptx::ld_acquire_sys_u64(wait.ctr + src) < wait.target[src]) {
              __nanosleep(128);
              // a source that never arrives is a bug: fail the launch
              // (an error the host sees) rather than hang the GPU
              if (ptx::globaltimer_ns() - t0 > 20000000000ull) __trap();
            }
            ptx::fence_proxy_async_global();
            arrived |= 1u << src;
          }
          ESP_PROF_WAIT(1, ptx::mbar_wait(&k_empty[ks], kph ^ 1));
          ptx::mbar_expect_tx(&k_full[ks], C::kKvBytes);
          for (int b = 0; b < C::kBoxes; ++b) {
            ptx::tma_load_2d(sK + ks * C::kKvBytes + b * (BN * 128), &tmK, &k_full[ks],
                             it.head * HD + b * 64, row);
          }
          if (++ks == kKStages) { ks = 0; kph ^= 1; }
          ESP_PROF_WAIT(2, ptx::mbar_wait(&v_empty[vs], vph ^ 1));
          ptx::mbar_expect_tx(&v_full[vs], C::kKvBytes);
          for (int b = 0; b < C::kBoxes; ++b) {
            ptx::tma_load_2d(sV + vs * C::kKvBytes + b * (BN * 128), &tmV, &v_full[vs],
                             it.head * HD + b * 64, row);
          }
          if (++vs == kStages) { vs = 0; vph ^= 1; }
        }
      }
      prof_store(0);
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      // The whole warp runs the (warp-uniform) loop so descriptors live in
      // uniform registers; one elected lane issues each tcgen05.mma/commit.
      // (A single-lane loop costs an R2UR per operand per MMA, which made
      // issue — not the tensor core — the bottleneck for 128x128x16 MMAs.)
      const bool leader = ptx::elect_one();
      constexpr uint32_t idesc_s = ptx::make_idesc_bf16(BM, BN, false, false);
      constexpr uint32_t idesc_o = ptx::make_idesc_bf16(BM, HD, false, true);
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0, items = 0;
      uint32_t cnt[2] = {0, 0};    // per-tile global step count (barrier phases)
      uint32_t titems[2] = {0, 0}; // per-tile item count (o_free phases)
      const uint32_t q_addr[2] = {ptx::smem_u32(sQ), ptx::smem_u32(sQ + C::kQBytes)};
      auto commit = [&](uint64_t* bar) {
        if (leader) ptx::tc_commit(bar);
        __syncwarp();
      };
      auto issue_s = [&](int t, uint32_t k_addr) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (BM * 128) + (k & 3) * 32;
          const uint64_t da = ptx::make_sdesc_sw128(q_addr[t] + off, 16, 1024);
          const uint64_t db = ptx::make_sdesc_sw128(k_addr + off, 16, 1024);
          if (leader) ptx::umma_f16_ss(t_s[t], da, db, idesc_s, k != 0);
        }
        commit(&s_full[t]);
      };
      for (int w = w_begin; w < w_end; ++w, ++items) {
        const Item it = load_item(work, w, segs);
        const RingSegment* sg = &segs[it.seg];
        const bool act[2] = {true, it.act1};
        ESP_PROF_WAIT(0, ptx::mbar_wait(q_full, items & 1));
        ptx::tc_fence_after();
        Steps st;
        st.begin(sg, it);
        // Prologue: S_t,0 for every tile that sees the first KV tile.
        {
          ESP_PROF_WAIT(1, ptx::mbar_wait(&k_full[ks], kph));
          ptx::tc_fence_after();
          const uint32_t k_addr = ptx::smem_u32(sK + ks * C::kKvBytes);
          if (st.active0()) issue_s(0, k_addr);
          if (act[1]) issue_s(1, k_addr);
          commit(&k_empty[ks]);
          if (++ks == kKStages) { ks = 0; kph ^= 1; }
        }
        bool first_pv[2] = {true, true};
        while (st.valid()) {
          const bool a_now[2] = {st.active0(), act[1]};
          Steps nx = st;
          nx.next();
          const bool has_next = nx.valid();
          const bool a_next[2] = {has_next && nx.active0(), has_next && act[1]};
          ESP_PROF_WAIT(2, ptx::mbar_wait(&v_full[vs], vph));
          uint32_t k_addr = 0;
          if (has_next) {
            ESP_PROF_WAIT(1, ptx::mbar_wait(&k_full[ks], kph));
            k_addr = ptx::smem_u32(sK + ks * C::kKvBytes);
          }
          const uint32_t v_addr = ptx::smem_u32(sV + vs * C::kKvBytes);
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (a_now[t]) {
              if (first_pv[t]) {
                ESP_PROF_WAIT(5, ptx::mbar_wait(&o_free[t], (titems[t] & 1) ^ 1));
                // windowed ring: the carried O is in TMEM before P.V adds to it
                if (cin) ptx::mbar_wait(&o_init[t], titems[t] & 1);
              }
#pragma unroll
              for (int part = 0; part < kParts; ++part) {
                ESP_PROF_WAIT(3 + t, ptx::mbar_wait(&p_full[kParts * t + part], cnt[t] & 1));
                ptx::tc_fence_after();
#pragma unroll
                for (int k = part * (8 / kParts); k < (part + 1) * (8 / kParts); ++k) {
                  const uint64_t dv = ptx::make_sdesc_sw128(v_addr + k * 2048, BN * 128, 1024);
                  if (leader) {
                    ptx::umma_f16_ts(t_o[t], t_s[t] + k * 8, dv, idesc_o,
                                     (!first_pv[t] || k != 0 || cin) ? 1u : 0u);
                  }
                }
              }
              commit(&o_done[t]);
              first_pv[t] = false;
              ++cnt[t];
            }
            // S_t of the next step overwrites P_t in TMEM: issued after PV_t
            // (tcgen05.mma executes in issue order). A tile idle at this step
            // (tile 0 past its causal limit in this round) may be active again
            // at the next round's first step.
            if (a_next[t]) {
              ptx::tc_fence_after();
              issue_s(t, k_addr);
            }
          }
          commit(&v_empty[vs]);
          if (++vs == kStages) { vs = 0; vph ^= 1; }
          if (has_next) {
            commit(&k_empty[ks]);
            if (++ks == kKStages) { ks = 0; kph ^= 1; }
          }
          st = nx;
        }
        commit(q_empty);
        for (int t = 0; t < 2; ++t) titems[t] += act[t] ? 1 : 0;
      }
      if (lane == 0) prof_store(1);
    }
  } else {
    ptx::setmaxnreg_inc<192>();
    // ------------------------------------------------------------ softmax
    const int t = (warp >= 8) ? 1 : 0;
    // this tile's TMEM columns (runtime t: no array indexing -> no local memory)
    const uint32_t ts_t = tmem + t * BN, to_t = tmem + 2 * BN + t * HD;
    const uint32_t quad = warp & 3;
    const int row = static_cast<int>(quad * 32 + lane);
    const uint32_t lane_off = (quad * 32) << 16;
    uint32_t cnt = 0;
    for (int w = w_begin; w < w_end; ++w) {
      const Item it = load_item(work, w, segs);
      if (t == 1 && !it.act1) continue;
      const RingSegment* sg = &segs[it.seg];
      const int q0 = (it.q0[0] + t * BM);
      const int a = q0 + row;
      float m_run = -INFINITY, l_run = 0.f;
      const int64_t crow = static_cast<int64_t>(sg->q_row0 + a);
      if (cin) {
        // Windowed ring: resume from the state the previous round's launch
        // left (unnormalised O in fp32, running max and sum), O into TMEM.
        const bool ok = a < sg->q_len;
        if (ok) {
          const float2 ml = carry.ml[crow * (hidden / HD) + it.head];
          m_run = ml.x;
          l_run = ml.y;
        }
        const float4* src = reinterpret_cast<const float4*>(carry.o + crow * hidden + it.head * HD);
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t o[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 v4 = ok ? src[c / 4 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
            o[4 * i] = __float_as_uint(v4.x);
            o[4 * i + 1] = __float_as_uint(v4.y);
            o[4 * i + 2] = __float_as_uint(v4.z);
            o[4 * i + 3] = __float_as_uint(v4.w);
          }
          ptx::tmem_st_32x32b_x32(to_t + lane_off + c, o);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&o_init[t]);
      }
      int j = 0;
      Steps st;
      for (st.begin(sg, it); st.valid(); st.next()) {
        if (t == 0 && !st.active0()) continue;
        const int b0 = st.tt * BN;
        const int shift = sg->shift[st.r];
        const int kv_len = sg->kv_len[st.r];
        ESP_PROF_WAIT(0, ptx::mbar_wait(&s_full[t], cnt & 1));
        // Observe every o_done phase (the previous step's P.V): it completed
        // before this S did (tcgen05 ops retire in issue order), so this never
        // blocks, and no barrier phase goes unobserved (compute-sanitizer
        // synccheck; the lazy rescale below relies on the same ordering).
        if (cnt > 0) ptx::mbar_wait(&o_done[t], (cnt - 1) & 1);
        const uint64_t prof_t_step = kProf ? clock64() : 0;
        ptx::tc_fence_after();
        uint32_t s[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t (&chunk)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[32 * c]);
          ptx::tmem_ld_32x32b_x32(ts_t + lane_off + 32 * c, chunk);
        }
        ptx::tmem_wait_ld();
        if constexpr (kProf) prof_acc[2] += clock64() - prof_t_step;  // S readback
        const bool full_tile = (b0 + BN - 1 <= q0 - shift) && (b0 + BN <= kv_len);
        const int lim = min(a - shift - b0, kv_len - 1 - b0);  // visible iff c <= lim
        if (!full_tile) {
#pragma unroll
          for (int c = 0; c < 128; ++c) {
            if (c > lim) s[c] = __float_as_uint(-INFINITY);
          }
        }
        // Row max with 8 independent chains of 3-input max (FMNMX3), then a tree.
        auto row_max = [&]() {
          float mx8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            mx8[k] = fmax3(__uint_as_float(s[k]), __uint_as_float(s[8 + k]),
                           __uint_as_float(s[120 + k]));
          }
#pragma unroll
          for (int c = 16; c < 120; c += 16) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              mx8[k] = fmax3(mx8[k], __uint_as_float(s[c + k]), __uint_as_float(s[c + 8 + k]));
            }
          }
          return fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]),
                       fmaxf(mx8[6], mx8[7]));
        };
        // O *= f in TMEM. O holds PV_{j-1}, complete once o_done of the
        // previous step fired (rare: a row max grew past the threshold).
        auto rescale_o = [&](float f) {
          ptx::mbar_wait(&o_done[t], (cnt - 1) & 1);
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < HD; c += 32) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(to_t + lane_off + c, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * f);
            ptx::tmem_st_32x32b_x32(to_t + lane_off + c, o);
          }
        };
        // P in place: s[c] <- bf16x2(p[2c], p[2c+1]) (reads of s[2c], s[2c+1]
        // precede the write of s[c], c <= 2c), then P over S_t in TMEM, in
        // kParts parts of 128/kParts keys: the MMA warp starts P.V on the
        // first keys while the later ones are still being exponentiated.
        const uint64_t scale2 = f2pack(scale_log2, scale_log2);
        uint64_t sum2a = f2pack(0.f, 0.f), sum2b = f2pack(0.f, 0.f);
        auto exp_part = [&](int part, float m_sub) {
          const uint64_t negm2 = f2pack(-m_sub, -m_sub);
#pragma unroll
          for (int c = kCP * part; c < kCP * part + kCP; ++c) {
            float x0, x1, p0, p1;
            f2unpack(ffma2(f2pack(__uint_as_float(s[2 * c]), __uint_as_float(s[2 * c + 1])),
                           scale2, negm2),
                     x0, x1);
            if (((c * kPoly8) & 7) < kPoly8) {
              exp2_fma2<kCubic>(x0, x1, p0, p1);  // kPoly8 pairs in 8 on the FMA pipe
            } else {
              p0 = ptx::ex2(x0);
              p1 = ptx::ex2(x1);
            }
            if (c & 1) {
              sum2b = fadd2(sum2b, f2pack(p0, p1));
            } else {
              sum2a = fadd2(sum2a, f2pack(p0, p1));
            }
            s[c] = ptx::pack_bf16(p0, p1);
          }
        };
        auto signal_part = [&](int part) {
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&p_full[kParts * t + part]);
        };
        auto issue_part = [&](int part) {
          if constexpr (kCP == 32) {
            ptx::tmem_st_32x32b_x32(ts_t + lane_off + kCP * part,
                                    *reinterpret_cast<uint32_t(*)[32]>(&s[kCP * part]));
          } else if constexpr (kCP == 8) {
            ptx::tmem_st_32x32b_x8(ts_t + lane_off + kCP * part,
                                   *reinterpret_cast<uint32_t(*)[8]>(&s[kCP * part]));
          } else {
            ptx::tmem_st_32x32b_x16(ts_t + lane_off + kCP * part,
                                    *reinterpret_cast<uint32_t(*)[16]>(&s[kCP * part]));
          }
        };
        // The raw scores of the later parts are still in registers; an empty
        // volatile asm that "modifies" them pins their exponentials after the
        // earlier part's P store and arrive.
        auto pin_from = [&](int c0) {
#pragma unroll
          for (int c = c0; c < 128; c += 16) {
            asm volatile(""
                         : "+r"(s[c]), "+r"(s[c + 1]), "+r"(s[c + 2]), "+r"(s[c + 3]),
                           "+r"(s[c + 4]), "+r"(s[c + 5]), "+r"(s[c + 6]), "+r"(s[c + 7]),
                           "+r"(s[c + 8]), "+r"(s[c + 9]), "+r"(s[c + 10]), "+r"(s[c + 11]),
                           "+r"(s[c + 12]), "+r"(s[c + 13]), "+r"(s[c + 14]), "+r"(s[c + 15]));
          }
        };
        {
          const float mx = row_max();
          if constexpr (kProf) prof_acc[3] += clock64() - prof_t_step;  // ..through row max
          const float m_tile = mx * scale_log2;
          const float m_new = fmaxf(m_run, m_tile);
          const bool need = (m_run == -INFINITY) ? (m_new != -INFINITY)
                                                 : (m_new > m_run + kRescaleThreshold);
          float alpha = 1.f;
          if (need) {
            alpha = m_run == -INFINITY ? 0.f : ptx::ex2(m_run - m_new);
            m_run = m_new;
          }
          const float m_sub = m_run == -INFINITY ? 0.f : m_run;
          if ((j > 0 || cin) && __any_sync(0xffffffff, need)) rescale_o(alpha);
#pragma unroll
          for (int part = 0; part < kParts; ++part) {
            exp_part(part, m_sub);
            issue_part(part);
            signal_part(part);
            if (part + 1 < kParts) pin_from(2 * kCP * (part + 1));
          }
          if constexpr (kProf) prof_acc[4] += clock64() - prof_t_step;  // ..through P stored
          float sa0, sa1;
          f2unpack(fadd2(sum2a, sum2b), sa0, sa1);
          l_run = l_run * alpha + (sa0 + sa1);
        }
        if constexpr (kProf) {
          prof_acc[1] += clock64() - prof_t_step;  // softmax step (S ready -> P ready)
          prof_acc[5] += 1;
        }
        ++cnt;
        ++j;
      }
      // Final O / l for this tile's rows.
      ESP_PROF_WAIT(6, ptx::mbar_wait(&o_done[t], (cnt - 1) & 1));
      ptx::tc_fence_after();
      const bool valid = a < sg->q_len;
      const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
      bf16* orow = out + crow * hidden + it.head * HD;
      if (kCarry) {
        // Windowed ring: hand the unnormalised state to the next round.
        float4* dst = reinterpret_cast<float4*>(carry.o + crow * hidden + it.head * HD);
#pragma unroll 1
        for (int c = 0; c < HD; c += 32) {
          uint32_t o[32];
          ptx::tmem_ld_32x32b_x32(to_t + lane_off + c, o);
          ptx::tmem_wait_ld();
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              dst[c / 4 + i] = make_float4(__uint_as_float(o[4 * i]), __uint_as_float(o[4 * i + 1]),
                                           __uint_as_float(o[4 * i + 2]), __uint_as_float(o[4 * i + 3]));
            }
          }
        }
        if (valid) carry.ml[crow * (hidden / HD) + it.head] = make_float2(m_run, l_run);
      }
#pragma unroll 1
      for (int c = 0; c < HD && !kCarry; c += 32) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(to_t + lane_off + c, o);
        ptx::tmem_wait_ld();
        if (valid) {
          uint4* d = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            d[i] = make_uint4(ptx::pack_bf16(__uint_as_float(o[8 * i]) * inv_l,
                                             __uint_as_float(o[8 * i + 1]) * inv_l),
                              ptx::pack_bf16(__uint_as_float(o[8 * i + 2]) * inv_l,
                                             __uint_as_float(o[8 * i + 3]) * inv_l),
                              ptx::pack_bf16(__uint_as_float(o[8 * i + 4]) * inv_l,
                                             __uint_as_float(o[8 * i + 5]) * inv_l),
                              ptx::pack_bf16(__uint_as_float(o[8 * i + 6]) * inv_l,
                                             __uint_as_float(o[8 * i + 7]) * inv_l));
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&o_free[t]);
    }
    if (quad == 0 && lane == 0) prof_store(2 + t);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int sm_count2() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int HD, bool kProf, int kPoly8, bool kCarry = false, int kParts = kPartsDefault,
          int kVSt = kVStagesDefault, bool kCubic = false>
void launch2(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows, int kv_rows,
             int heads, const RingSegment* segs, const int32_t* work, int n_work, float scale,
             cudaStream_t s, uint64_t* prof, const RingWait& wait, const RingCarry& carry) {
  using C = Cfg2<HD, kVSt>;
  auto* kern = ring_attention_tcgen05<HD, kProf, kPoly8, kCarry, kParts, kVSt, kCubic>;
  once_per_device(reinterpret_cast<const void*>(kern), [kern] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  const int hidden = heads * HD;
  const CUtensorMap tq = make_tmap_bf16(q, q_rows, hidden, hidden, BM);
  const CUtensorMap tk = make_tmap_bf16(k, kv_rows, hidden, hidden, BN);
  const CUtensorMap tv = make_tmap_bf16(v, kv_rows, hidden, hidden, BN);
  const int grid = n_work < sm_count2() ? n_work : sm_count2();
  kern<<<grid, kThreads, C::kSmem, s>>>(
      tq, tk, tv, out, hidden, segs, work, n_work, scale * 1.4426950408889634f, prof, wait, carry);
  count_launch();
}

template <bool kProf>
void dispatch2(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows, int kv_rows,
               int heads, int head_dim, const RingSegment* d_segs, const int32_t* d_work,
               int n_work, float scale, cudaStream_t s, uint64_t* prof,
               const RingWait& wait = RingWait{}, const RingCarry& carry = RingCarry{}) {
  if (n_work <= 0) return;
  if (heads > 255) throw std::runtime_error("ring_attention: heads > 255");
  // Exponentials computed on the FMA pipe, in eighths of each row's keys
  // (MUFU/FMA balance: 2 in 8 measured best in the step in round 2, r02_poly_ab.txt).
  if (carry.o != nullptr) {  // windowed ring: the carry variant (kCarry)
    if (kProf) throw std::runtime_error("ring_attention: no profiled carry variant");
    if (head_dim == 128) {
      launch2<128, false, kDefaultPoly8, true>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work,
                                               n_work, scale, s, prof, wait, carry);
    } else if (head_dim == 64) {
      launch2<64, false, kDefaultPoly8, true>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work,
                                              n_work, scale, s, prof, wait, carry);
    } else {
      throw std::runtime_error("ring_attention: head_dim must be 64 or 128");
    }
    return;
  }
  if (head_dim == 128) {
#ifdef ESP_STUDY
    // kernel-study build: ESP_ATTN_POLY = eighths of the exponentials on the FMA pipe
    static const int poly = [] {
      const char* e = std::getenv("ESP_ATTN_POLY");
      return e ? std::atoi(e) : kDefaultPoly8;
    }();
    // ESP_K1_PARTS2 / ESP_K1_PARTS8: P in 2 / 8 key parts; ESP_K1_VST3: three V
    // stages; ESP_K1_CUBIC: the cubic exponential polynomial
    static const int var = (std::getenv("ESP_K1_PARTS2") ? 1 : 0) | (std::getenv("ESP_K1_PARTS8") ? 2 : 0) |
                           (std::getenv("ESP_K1_VST3") ? 4 : 0) | (std::getenv("ESP_K1_CUBIC") ? 8 : 0);
    switch (var) {
      case 1: launch2<128, kProf, kDefaultPoly8, false, 2, 2>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 2: launch2<128, kProf, kDefaultPoly8, false, 8, 2>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 4: launch2<128, kProf, kDefaultPoly8, false, 4, 3>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 6: launch2<128, kProf, kDefaultPoly8, false, 8, 3>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 8: launch2<128, kProf, kDefaultPoly8, false, kPartsDefault, kVStagesDefault, true>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      default: break;
    }
    switch (poly) {
      case 0: launch2<128, kProf, 0>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 2: launch2<128, kProf, 2>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 3: launch2<128, kProf, 3>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      case 4: launch2<128, kProf, 4>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s, prof, wait, carry); return;
      default: break;
    }
#endif
    launch2<128, kProf, kDefaultPoly8>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work,
                                       n_work, scale, s, prof, wait, carry);
  } else if (head_dim == 64) {
    launch2<64, kProf, kDefaultPoly8>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work,
                                      n_work, scale, s, prof, wait, carry);
  } else {
    throw std::runtime_error("ring_attention: head_dim must be 64 or 128");
  }
}

}  // namespace

void ring_attention(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows,
                    int kv_rows, int heads, int head_dim, const RingSegment* d_segs,
                    const int32_t* d_work, int n_work, float scale, cudaStream_t s,
                    const RingWait* wait, const RingCarry* carry) {
  dispatch2<false>(q, k, v, out, q_rows, kv_rows, heads, head_dim, d_segs, d_work, n_work, scale,
                   s, nullptr, wait ? *wait : RingWait{}, carry ? *carry : RingCarry{});
}

namespace {
// One CTA per row, one thread per 4 columns: out = o / l of the row's head.
__global__ void ring_finalize_kernel(const float* __restrict__ o, const float2* __restrict__ ml,
                                     bf16* __restrict__ out, int hidden, int head_dim) {
  const int64_t row = blockIdx.x;
  const int heads = hidden / head_dim;
  for (int c = threadIdx.x * 4; c < hidden; c += blockDim.x * 4) {
    const float l = ml[row * heads + c / head_dim].y;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const float4 v = *reinterpret_cast<const float4*>(o + row * hidden + c);
    uint2 w;
    w.x = ptx::pack_bf16(v.x * inv, v.y * inv);
    w.y = ptx::pack_bf16(v.z * inv, v.w * inv);
    *reinterpret_cast<uint2*>(out + row * hidden + c) = w;
  }
}
}  // namespace

void ring_attention_finalize(const RingCarry& carry, bf16* out, int rows, int heads, int head_dim,
                             cudaStream_t s) {
  if (rows <= 0) return;
  ring_finalize_kernel<<<rows, 256, 0, s>>>(carry.o, carry.ml, out, heads * head_dim, head_dim);
  count_launch();
}

#ifdef ESP_STUDY
void ring_attention_profiled(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows,
                             int kv_rows, int heads, int head_dim, const RingSegment* d_segs,
                             const int32_t* d_work, int n_work, float scale, cudaStream_t s,
                             uint64_t* prof) {
  dispatch2<true>(q, k, v, out, q_rows, kv_rows, heads, head_dim, d_segs, d_work, n_work, scale,
                  s, prof);  // (no carry)
}
#endif

}  // namespace esp::k
