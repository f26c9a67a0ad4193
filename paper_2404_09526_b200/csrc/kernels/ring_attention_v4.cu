// K1 (v4): striped ring attention, one 128-row query tile per CTA, with the
// query tile and a double-buffered score tile in tensor memory.
//
// Same math and striped-causal mask as v1/v2. What changes is what waits on
// what. In v2 each query tile's next S = QK^T could only be issued after that
// tile's PV, so every step paid softmax latency + tensor-core time in series.
// Here:
//   * TMEM = S[0] | S[1] | O | Q[0] | Q[1] (128+128+HD+HD/2+HD/2 <= 512 cols).
//     S of step j+1 (and j+2) is computed into the other S buffer while the
//     softmax warps work on step j: the softmax warps never wait for the
//     tensor core after the first step of an item, only for their own
//     throughput (MUFU / FMA pipes) — the tensor core never waits for them
//     for longer than one softmax step minus one step of MMAs;
//   * Q lives in TMEM (two buffers, by item parity) and S = Q K^T uses the
//     TS form of tcgen05.mma (A from TMEM): shared memory only feeds K and V
//     to the tensor core (62 B/clk each) — with one query tile per CTA the
//     SS form would need ~124 B/clk for S plus the TMA writes, over the 128
//     B/clk shared-memory budget (tools/ubench/umma.cu);
//   * the producer TMA-loads Q (SW128) into shared memory; the softmax warps
//     copy it into TMEM (un-swizzling) before the previous item's epilogue,
//     so the next item's first two S MMAs run during that epilogue;
//   * softmax on two warpgroups, each owning 64 of the 128 key columns of S
//     (row max exchanged through shared memory + a 256-thread named barrier),
//     P written as bf16 over S in TMEM; PV is issued per 64-key half as soon
//     as that half's P is stored; lazy O rescale (threshold 2^8), each
//     warpgroup rescales and finally normalises its half of the O columns.
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
constexpr int kStages = 2;
constexpr int kThreads = 384;  // WG0 (TMA, MMA, TMEM alloc) + 2 softmax WGs
constexpr float kRescaleThreshold = 8.0f;

template <int HD>
struct Cfg4 {
  static constexpr int kBoxes = HD / 64;
  static constexpr int kQBytes = BM * HD * 2;
  static constexpr int kKvBytes = BN * HD * 2;
  static constexpr int kXchgBytes = (2 * 2 * BM + 2 * BM) * 4;  // max [parity][half][row], sum
  static constexpr int kSmem = kQBytes + 2 * kStages * kKvBytes + kXchgBytes + 1024 + 512;
  // TMEM columns
  static constexpr uint32_t kS0 = 0, kS1 = BN, kO = 2 * BN, kQ0 = 2 * BN + HD,
                            kQ1 = 2 * BN + HD + HD / 2;
  static_assert(kQ1 + HD / 2 <= 512, "TMEM budget");
};

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
// 2^x for a pair on the FMA pipe (see ring_attention_v2.cu).
__device__ __forceinline__ void exp2_fma2(float x0, float x1, float& p0, float& p1) {
  const uint64_t x = f2pack(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
  const uint64_t t = fadd2(x, f2pack(12582912.0f, 12582912.0f));
  const uint64_t r = fadd2(t, f2pack(-12582912.0f, -12582912.0f));
  const uint64_t f = ffma2(r, f2pack(-1.0f, -1.0f), x);
  uint64_t p = ffma2(f2pack(0.0555041087f, 0.0555041087f), f, f2pack(0.240226507f, 0.240226507f));
  p = ffma2(p, f, f2pack(0.693147181f, 0.693147181f));
  p = ffma2(p, f, f2pack(1.0f, 1.0f));
  float t0, t1, q0, q1;
  f2unpack(t, t0, t1);
  f2unpack(p, q0, q1);
  p0 = __int_as_float(__float_as_int(q0) + (__float_as_int(t0) << 23));
  p1 = __int_as_float(__float_as_int(q1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ int tiles_visible4(const RingSegment& sg, int r, int q0) {
  const int a_max = min(q0 + BM - 1, sg.q_len - 1);
  const int vis = min(sg.kv_len[r], a_max - sg.shift[r] + 1);
  return vis <= 0 ? 0 : (vis + BN - 1) / BN;
}

struct Item4 {
  int seg, head, q0;
};
__device__ __forceinline__ Item4 load_item4(const int32_t* work, int w) {
  Item4 it;
  it.seg = __ldg(&work[2 * w]);
  const int packed = __ldg(&work[2 * w + 1]);
  it.q0 = (packed >> 8) * BM;
  it.head = packed & 0xFF;
  return it;
}

// The KV-tile sequence (round r, tile tt) a query tile sees.
struct Steps4 {
  const RingSegment* sg;
  int q0;
  int r = 0, tt = 0, n_r = 0;
  __device__ void begin(const RingSegment* s, int q0_) {
    sg = s;
    q0 = q0_;
    r = -1;
    tt = 0;
    n_r = 0;
    advance_round();
  }
  __device__ void advance_round() {
    do {
      ++r;
      if (r >= sg->n_rounds) return;
      n_r = tiles_visible4(*sg, r, q0);
      tt = 0;
    } while (n_r == 0);
  }
  __device__ bool valid() const { return r < sg->n_rounds; }
  __device__ void next() {
    if (++tt >= n_r) advance_round();
  }
  __device__ int kv_row() const { return sg->kv_row0[r] + tt * BN; }
};

template <int HD, int kPoly8>
__global__ void __launch_bounds__(kThreads, 1)
    ring_attention_v4(const __grid_constant__ CUtensorMap tmQ,
                      const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ out,
                      int hidden, const RingSegment* __restrict__ segs,
                      const int32_t* __restrict__ work, int n_work, float scale_log2) {
  using C = Cfg4<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;                        // [kQBytes], SW128 boxes of 64 columns
  uint8_t* sK = sQ + C::kQBytes;             // [kStages][kKvBytes]
  uint8_t* sV = sK + kStages * C::kKvBytes;  // [kStages][kKvBytes]
  float* xchg_max = reinterpret_cast<float*>(sV + kStages * C::kKvBytes);  // [2][2][BM]
  float* xchg_sum = xchg_max + 2 * 2 * BM;                                  // [2][BM]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xchg_sum + 2 * BM);
  uint64_t* q_full = bars;            // Q in shared memory (TMA)
  uint64_t* q_empty = bars + 1;       // Q copied out of shared memory
  uint64_t* qt_full = bars + 2;       // [2] Q in TMEM buffer (by item parity)
  uint64_t* k_full = bars + 4;
  uint64_t* k_empty = k_full + kStages;
  uint64_t* v_full = k_empty + kStages;
  uint64_t* v_empty = v_full + kStages;
  uint64_t* s_full = v_empty + kStages;  // [2] S buffer
  uint64_t* p_full = s_full + 2;         // [2 buffers][2 key halves]
  uint64_t* o_done = p_full + 4;         // PV of a step complete
  uint64_t* o_free = o_done + 1;         // O read out by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmQ);
    ptx::tma_prefetch_desc(&tmK);
    ptx::tma_prefetch_desc(&tmV);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 256);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&qt_full[b], 256);
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&p_full[2 * b], 128);
      ptx::mbar_init(&p_full[2 * b + 1], 128);
    }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    ptx::mbar_init(o_done, 1);
    ptx::mbar_init(o_free, 256);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s[2] = {tmem + C::kS0, tmem + C::kS1};
  const uint32_t t_o = tmem + C::kO;
  const uint32_t t_q[2] = {tmem + C::kQ0, tmem + C::kQ1};

  if (warp < 4) {
    ptx::setmaxnreg_dec<104>();
    if (warp == 0 && lane == 0) {
      // ---------------------------------------------------------- producer
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0, items = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++items) {
        const Item4 it = load_item4(work, w);
        const RingSegment* sg = &segs[it.seg];
        ptx::mbar_wait(q_empty, (items & 1) ^ 1);
        ptx::mbar_expect_tx(q_full, C::kQBytes);
        for (int b = 0; b < C::kBoxes; ++b) {
          ptx::tma_load_2d(sQ + b * (BM * 128), &tmQ, q_full, it.head * HD + b * 64,
                           sg->q_row0 + it.q0);
        }
        Steps4 st;
        for (st.begin(sg, it.q0); st.valid(); st.next()) {
          const int row = st.kv_row();
          ptx::mbar_wait(&k_empty[ks], kph ^ 1);
          ptx::mbar_expect_tx(&k_full[ks], C::kKvBytes);
          for (int b = 0; b < C::kBoxes; ++b) {
            ptx::tma_load_2d(sK + ks * C::kKvBytes + b * (BN * 128), &tmK, &k_full[ks],
                             it.head * HD + b * 64, row);
          }
          if (++ks == kStages) { ks = 0; kph ^= 1; }
          ptx::mbar_wait(&v_empty[vs], vph ^ 1);
          ptx::mbar_expect_tx(&v_full[vs], C::kKvBytes);
          for (int b = 0; b < C::kBoxes; ++b) {
            ptx::tma_load_2d(sV + vs * C::kKvBytes + b * (BN * 128), &tmV, &v_full[vs],
                             it.head * HD + b * 64, row);
          }
          if (++vs == kStages) { vs = 0; vph ^= 1; }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer
      const bool leader = ptx::elect_one();
      constexpr uint32_t idesc_s = ptx::make_idesc_bf16(BM, BN, false, false);
      constexpr uint32_t idesc_o = ptx::make_idesc_bf16(BM, HD, false, true);
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0, items = 0;
      uint32_t gs = 0, gp = 0;  // global S-issue and PV step counters
      auto commit = [&](uint64_t* bar) {
        if (leader) ptx::tc_commit(bar);
        __syncwarp();
      };
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++items) {
        const Item4 it = load_item4(work, w);
        const RingSegment* sg = &segs[it.seg];
        const uint32_t qb = items & 1;
        ptx::mbar_wait(&qt_full[qb], (items >> 1) & 1);
        ptx::tc_fence_after();
        auto issue_s = [&]() {
          ptx::mbar_wait(&k_full[ks], kph);
          ptx::tc_fence_after();
          const uint32_t k_addr = ptx::smem_u32(sK + ks * C::kKvBytes);
          const uint32_t sb = gs & 1;
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * (BN * 128) + (k & 3) * 32;
            const uint64_t db = ptx::make_sdesc_sw128(k_addr + off, 16, 1024);
            if (leader) ptx::umma_f16_ts(t_s[sb], t_q[qb] + k * 8, db, idesc_s, k != 0);
          }
          commit(&s_full[sb]);
          commit(&k_empty[ks]);
          if (++ks == kStages) { ks = 0; kph ^= 1; }
          ++gs;
        };
        Steps4 ahead, st;
        ahead.begin(sg, it.q0);
        for (int j = 0; j < 2 && ahead.valid(); ++j, ahead.next()) issue_s();
        bool first = true;
        for (st.begin(sg, it.q0); st.valid(); st.next()) {
          ptx::mbar_wait(&v_full[vs], vph);
          if (first) ptx::mbar_wait(o_free, (items & 1) ^ 1);
          const uint32_t v_addr = ptx::smem_u32(sV + vs * C::kKvBytes);
          const uint32_t pb = gp & 1;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            ptx::mbar_wait(&p_full[2 * pb + half], (gp >> 1) & 1);
            ptx::tc_fence_after();
#pragma unroll
            for (int k = 4 * half; k < 4 * half + 4; ++k) {
              const uint64_t dv = ptx::make_sdesc_sw128(v_addr + k * 2048, BN * 128, 1024);
              if (leader) {
                ptx::umma_f16_ts(t_o, t_s[pb] + k * 8, dv, idesc_o, (!first || k != 0) ? 1u : 0u);
              }
            }
          }
          commit(o_done);
          commit(&v_empty[vs]);
          if (++vs == kStages) { vs = 0; vph ^= 1; }
          ++gp;
          first = false;
          // S two steps ahead reuses this step's buffer (its P was read by
          // the PV just issued: tcgen05.mma executes in order).
          if (ahead.valid()) {
            issue_s();
            ahead.next();
          }
        }
      }
    }
  } else {
    ptx::setmaxnreg_inc<192>();
    // ------------------------------------------------------------ softmax
    // Warps 4..11: key half h = (warp - 4) / 4 (S columns [64h, 64h+64)),
    // TMEM lane quadrant = warp % 4; thread = one query row.
    const int h = (static_cast<int>(warp) - 4) >> 2;
    const uint32_t quad = warp & 3;
    const int row = static_cast<int>(quad * 32 + lane);
    const uint32_t lane_off = (quad * 32) << 16;
    constexpr int HO = HD / 2;  // O columns owned by this half
    float* my_max = xchg_max;   // [parity][half][row]
    uint32_t g = 0, items = 0;
    // Q (shared memory, SW128 boxes) -> TMEM buffer qb: this half copies
    // the row's columns [HO*h, HO*h + HO) = HO/8 chunks of 16 bytes.
    auto copy_q = [&](uint32_t it_idx) {
      ptx::mbar_wait(q_full, it_idx & 1);
      uint32_t qv[HO / 2];
#pragma unroll
      for (int c = 0; c < HO / 8; ++c) {
        const int col = HO * h + 8 * c;  // first of 8 bf16
        const int box = col >> 6, chunk = (col & 63) >> 3;
        const uint4 v = *reinterpret_cast<const uint4*>(
            sQ + box * (BM * 128) + row * 128 + ((chunk ^ (row & 7)) << 4));
        qv[4 * c] = v.x;
        qv[4 * c + 1] = v.y;
        qv[4 * c + 2] = v.z;
        qv[4 * c + 3] = v.w;
      }
      ptx::mbar_arrive(q_empty);
      if constexpr (HO / 2 == 32) {
        ptx::tmem_st_32x32b_x32(t_q[it_idx & 1] + lane_off + (HO / 2) * h,
                                *reinterpret_cast<uint32_t(*)[32]>(&qv[0]));
      } else {
        ptx::tmem_st_32x32b_x16(t_q[it_idx & 1] + lane_off + (HO / 2) * h,
                                *reinterpret_cast<uint32_t(*)[16]>(&qv[0]));
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&qt_full[it_idx & 1]);
    };
    if (static_cast<int>(blockIdx.x) < n_work) copy_q(0);
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++items) {
      const Item4 it = load_item4(work, w);
      const RingSegment* sg = &segs[it.seg];
      const int q0 = it.q0;
      const int a = q0 + row;
      float m_run = -INFINITY, l_half = 0.f;
      int j = 0;
      Steps4 st;
      for (st.begin(sg, q0); st.valid(); st.next(), ++j, ++g) {
        const int b0 = st.tt * BN + 64 * h;  // first key of this half
        const int shift = sg->shift[st.r];
        const int kv_len = sg->kv_len[st.r];
        const uint32_t sb = g & 1;
        ptx::mbar_wait(&s_full[sb], (g >> 1) & 1);
        ptx::tc_fence_after();
        uint32_t s[64];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          ptx::tmem_ld_32x32b_x32(t_s[sb] + lane_off + 64 * h + 32 * c,
                                  *reinterpret_cast<uint32_t(*)[32]>(&s[32 * c]));
        }
        ptx::tmem_wait_ld();
        const bool full_half = (b0 + 63 <= q0 - shift) && (b0 + 64 <= kv_len);
        if (!full_half) {
          const int lim = min(a - shift - b0, kv_len - 1 - b0);  // visible iff c <= lim
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            if (c > lim) s[c] = __float_as_uint(-INFINITY);
          }
        }
        float mx8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          mx8[k] = fmax3(__uint_as_float(s[k]), __uint_as_float(s[8 + k]),
                         __uint_as_float(s[16 + k]));
        }
#pragma unroll
        for (int c = 24; c < 56; c += 16) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            mx8[k] = fmax3(mx8[k], __uint_as_float(s[c + k]), __uint_as_float(s[c + 8 + k]));
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) mx8[k] = fmaxf(mx8[k], __uint_as_float(s[56 + k]));
        float mx = fmax3(fmax3(mx8[0], mx8[1], mx8[2]), fmax3(mx8[3], mx8[4], mx8[5]),
                         fmaxf(mx8[6], mx8[7]));
        // Row max across the two halves (double-buffered by step parity).
        float* slot = my_max + (g & 1) * 2 * BM;
        slot[h * BM + row] = mx;
        ptx::named_bar_sync(1, 256);
        mx = fmaxf(mx, slot[(h ^ 1) * BM + row]);
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
        if (j > 0 && __any_sync(0xffffffff, need)) {
          // O holds PV_{j-1}: wait for it, rescale this half's O columns.
          ptx::mbar_wait(o_done, (g - 1) & 1);
          ptx::tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < HO; c += 32) {
            uint32_t o[32];
            ptx::tmem_ld_32x32b_x32(t_o + lane_off + HO * h + c, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_32x32b_x32(t_o + lane_off + HO * h + c, o);
          }
        }
        // P in place: s[c] <- bf16x2(p[2c], p[2c+1]), then into this half's
        // 32 P columns of the S buffer.
        const uint64_t scale2 = f2pack(scale_log2, scale_log2);
        const uint64_t negm2 = f2pack(-m_sub, -m_sub);
        uint64_t sum2a = f2pack(0.f, 0.f), sum2b = f2pack(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          float x0, x1, p0, p1;
          f2unpack(ffma2(f2pack(__uint_as_float(s[2 * c]), __uint_as_float(s[2 * c + 1])),
                         scale2, negm2),
                   x0, x1);
          if (((c * kPoly8) & 7) < kPoly8) {
            exp2_fma2(x0, x1, p0, p1);
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
        ptx::tmem_st_32x32b_x32(t_s[sb] + lane_off + 32 * h,
                                *reinterpret_cast<uint32_t(*)[32]>(&s[0]));
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&p_full[2 * sb + h]);
        float sa0, sa1;
        f2unpack(fadd2(sum2a, sum2b), sa0, sa1);
        l_half = l_half * alpha + (sa0 + sa1);
      }
      // The next item's Q into TMEM now, so its first S MMAs overlap this
      // item's epilogue.
      if (w + static_cast<int>(gridDim.x) < n_work) copy_q(items + 1);
      // Final O / l: merge the two halves' row sums, normalise own columns.
      xchg_sum[h * BM + row] = l_half;
      ptx::named_bar_sync(1, 256);
      const float l_run = l_half + xchg_sum[(h ^ 1) * BM + row];
      ptx::mbar_wait(o_done, (g - 1) & 1);
      ptx::tc_fence_after();
      const bool valid = a < sg->q_len;
      const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
      bf16* orow = out + static_cast<int64_t>(sg->q_row0 + a) * hidden + it.head * HD + HO * h;
#pragma unroll 1
      for (int c = 0; c < HO; c += 32) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(t_o + lane_off + HO * h + c, o);
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
      // xchg_sum is rewritten by the next item: both halves must have read it.
      ptx::named_bar_sync(1, 256);
      ptx::tc_fence_before();
      ptx::mbar_arrive(o_free);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int sm_count4() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int HD, int kPoly8>
void launch4(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows, int kv_rows,
             int heads, const RingSegment* segs, const int32_t* work, int n_work, float scale,
             cudaStream_t s) {
  using C = Cfg4<HD>;
  once_per_device(reinterpret_cast<const void*>(ring_attention_v4<HD, kPoly8>), [] {
    cudaFuncSetAttribute(ring_attention_v4<HD, kPoly8>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  const int hidden = heads * HD;
  const CUtensorMap tq = make_tmap_bf16(q, q_rows, hidden, hidden, BM);
  const CUtensorMap tk = make_tmap_bf16(k, kv_rows, hidden, hidden, BN);
  const CUtensorMap tv = make_tmap_bf16(v, kv_rows, hidden, hidden, BN);
  const int grid = n_work < sm_count4() ? n_work : sm_count4();
  ring_attention_v4<HD, kPoly8><<<grid, kThreads, C::kSmem, s>>>(
      tq, tk, tv, out, hidden, segs, work, n_work, scale * 1.4426950408889634f);
  count_launch();
}

}  // namespace

// Work items for v4 are (segment, 128-row query tile, head), as for v1.
void ring_attention_single(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows,
                           int kv_rows, int heads, int head_dim, const RingSegment* d_segs,
                           const int32_t* d_work, int n_work, float scale, cudaStream_t s) {
  if (n_work <= 0) return;
  if (heads > 255) throw std::runtime_error("ring_attention: heads > 255");
  static const int poly = [] {
    const char* e = getenv("ESP_ATTN_POLY");
    return e ? atoi(e) : 2;
  }();
  if (head_dim == 128) {
    if (poly == 3) {
      launch4<128, 3>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s);
    } else {
      launch4<128, 2>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s);
    }
  } else if (head_dim == 64) {
    launch4<64, 2>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s);
  } else {
    throw std::runtime_error("ring_attention: head_dim must be 64 or 128");
  }
}

void ring_attention_variant(int variant, const bf16* q, const bf16* k, const bf16* v, bf16* out,
                            int q_rows, int kv_rows, int heads, int head_dim,
                            const RingSegment* d_segs, int n_segs, const int32_t* d_work,
                            int n_work, float scale, cudaStream_t s) {
  if (variant == 4) {
    ring_attention_single(q, k, v, out, q_rows, kv_rows, heads, head_dim, d_segs, d_work, n_work,
                          scale, s);
  } else if (variant == 2) {
    ring_attention_pairs(q, k, v, out, q_rows, kv_rows, heads, head_dim, d_segs, d_work, n_work,
                         scale, s);
  } else {
    ring_attention(q, k, v, out, q_rows, kv_rows, heads, head_dim, d_segs, n_segs, d_work, n_work,
                   scale, s);
  }
}

}  // namespace esp::k
