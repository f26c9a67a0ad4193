// K1: striped ring attention for ESP prefill on 5th-gen tensor cores.
//
// Ring position i of d holds the query stripe of every request in the batch
// (tokens t = i mod d, LoongServe PAPER.md:179). In round r it meets the KV
// stripe that started at position origin = (i - r) mod d
// (build_ring_schedule, esp_mechanics.cpp:45-70). With stripe index a for a
// local query and b for a visiting key, the causal mask on the original
// positions a*d+i >= b*d+origin reduces to  b <= a - [origin > i].
// The online softmax state (row max m, row sum l, O) persists across all d
// rounds of a work item, so the kernel's output is the exact attention over
// the whole prefix.
//
// Per CTA (one per SM, persistent over (segment, 128-row q tile, head) items):
//   warp 0      TMA producer: Q tile once per item; K_j / V_j 128-row tiles
//               through two mbarrier rings.
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into TMEM (double
//               buffered, S_{j+1} issued before PV_j), O += P_j V_j into TMEM.
//   warps 4..7  softmax: thread == query row == TMEM lane. tcgen05.ld of the
//               S row, striped-causal mask, exp2, P_j (bf16) into smem in the
//               UMMA K-major SW128 layout; lazy O rescale (only when the row
//               max grows by > 2^8) through tcgen05.ld/st; final O / l.
#include <cuda.h>

#include <mutex>
#include <stdexcept>

#include "kernels.h"
#include "ptx.cuh"

namespace esp::k {

CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld,
                           int box_rows);

namespace {

constexpr int BM = 128;  // query rows per tile
constexpr int BN = 128;  // key rows per tile
constexpr int kKvStages = 2;
constexpr int kThreads = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int HD>
struct ACfg {
  static constexpr int kBoxes = HD / 64;                 // 64-wide column boxes
  static constexpr int kQBytes = BM * HD * 2;
  static constexpr int kKvBytes = BN * HD * 2;
  static constexpr int kPBytes = BM * BN * 2;
  static constexpr int kSmemData = kQBytes + 2 * kKvStages * kKvBytes + 2 * kPBytes;
  static constexpr int kSmem = kSmemData + 1024 + 512;
  static constexpr uint32_t kTmemCols = 512;  // S0 | S1 | O
};

struct TileIter {
  // Visible KV tiles of one round for one q tile.
  __device__ static int count(const RingSegment& sg, int r, int q0) {
    const int a_max = min(q0 + BM - 1, sg.q_len - 1);
    const int vis = min(sg.kv_len[r], a_max - sg.shift[r] + 1);
    return vis <= 0 ? 0 : (vis + BN - 1) / BN;
  }
};

__device__ __forceinline__ void decode_work(const int32_t* work, int w, int& seg, int& qt,
                                            int& head) {
  seg = __ldg(&work[2 * w]);
  const int packed = __ldg(&work[2 * w + 1]);
  qt = packed >> 8;
  head = packed & 0xFF;
}

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    ring_attention_tcgen05(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, bf16* __restrict__ out,
                           int hidden, const RingSegment* __restrict__ segs,
                           const int32_t* __restrict__ work, int n_work, float scale_log2) {
  using C = ACfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::kQBytes;
  uint8_t* sV = sK + kKvStages * C::kKvBytes;
  uint8_t* sP = sV + kKvStages * C::kKvBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * C::kPBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;                 // [kKvStages]
  uint64_t* k_empty = k_full + kKvStages;      // [kKvStages]
  uint64_t* v_full = k_empty + kKvStages;      // [kKvStages]
  uint64_t* v_empty = v_full + kKvStages;      // [kKvStages]
  uint64_t* s_full = v_empty + kKvStages;      // [2]
  uint64_t* s_empty = s_full + 2;              // [2]
  uint64_t* p_full = s_empty + 2;              // [2]
  uint64_t* p_free = p_full + 2;               // [2]
  uint64_t* o_done = p_free + 2;
  uint64_t* o_free = o_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmQ);
    ptx::tma_prefetch_desc(&tmK);
    ptx::tma_prefetch_desc(&tmV);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(q_empty, 1);
    for (int s = 0; s < kKvStages; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&s_empty[b], 128);
      ptx::mbar_init(&p_full[b], 128);
      ptx::mbar_init(&p_free[b], 1);
    }
    ptx::mbar_init(o_done, 1);
    ptx::mbar_init(o_free, 128);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_s = tmem_base;          // S buffers at cols [0,128), [128,256)
  const uint32_t tmem_o = tmem_base + 2 * BN; // O at cols [256, 256+HD)

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      uint32_t items = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++items) {
        int seg_i, qt, head;
        decode_work(work, w, seg_i, qt, head);
        const RingSegment& sg = segs[seg_i];
        const int q0 = qt * BM;
        ptx::mbar_wait(q_empty, (items & 1) ^ 1);
        ptx::mbar_expect_tx(q_full, C::kQBytes);
        for (int b = 0; b < C::kBoxes; ++b) {
          ptx::tma_load_2d(sQ + b * (BM * 128), &tmQ, q_full, head * HD + b * 64,
                           sg.q_row0 + q0);
        }
        for (int r = 0; r < sg.n_rounds; ++r) {
          const int nt = TileIter::count(sg, r, q0);
          for (int t = 0; t < nt; ++t) {
            const int row = sg.kv_row0[r] + t * BN;
            ptx::mbar_wait(&k_empty[ks], kph ^ 1);
            ptx::mbar_expect_tx(&k_full[ks], C::kKvBytes);
            for (int b = 0; b < C::kBoxes; ++b) {
              ptx::tma_load_2d(sK + ks * C::kKvBytes + b * (BN * 128), &tmK, &k_full[ks],
                               head * HD + b * 64, row);
            }
            if (++ks == kKvStages) { ks = 0; kph ^= 1; }
            ptx::mbar_wait(&v_empty[vs], vph ^ 1);
            ptx::mbar_expect_tx(&v_full[vs], C::kKvBytes);
            for (int b = 0; b < C::kBoxes; ++b) {
              ptx::tma_load_2d(sV + vs * C::kKvBytes + b * (BN * 128), &tmV, &v_full[vs],
                               head * HD + b * 64, row);
            }
            if (++vs == kKvStages) { vs = 0; vph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = ptx::make_idesc_bf16(BM, BN, false, false);
      constexpr uint32_t idesc_o = ptx::make_idesc_bf16(BM, HD, false, true);
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      uint32_t g = 0;      // global KV-tile counter (S/P buffer = g & 1)
      uint32_t items = 0;
      const uint32_t q_addr = ptx::smem_u32(sQ);
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++items) {
        int seg_i, qt, head;
        decode_work(work, w, seg_i, qt, head);
        const RingSegment& sg = segs[seg_i];
        const int q0 = qt * BM;
        int n = 0;
        for (int r = 0; r < sg.n_rounds; ++r) n += TileIter::count(sg, r, q0);
        ptx::mbar_wait(q_full, items & 1);
        ptx::tc_fence_after();
        auto issue_s = [&](uint32_t gj) {
          const uint32_t b = gj & 1;
          ptx::mbar_wait(&s_empty[b], ((gj >> 1) & 1) ^ 1);
          ptx::mbar_wait(&k_full[ks], kph);
          ptx::tc_fence_after();
          const uint32_t k_addr = ptx::smem_u32(sK + ks * C::kKvBytes);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * (BM * 128) + (k & 3) * 32;
            const uint32_t koff = (k >> 2) * (BN * 128) + (k & 3) * 32;
            ptx::umma_f16_ss(tmem_s + b * BN, ptx::make_sdesc_sw128(q_addr + off, 16, 1024),
                             ptx::make_sdesc_sw128(k_addr + koff, 16, 1024), idesc_s, k != 0);
          }
          ptx::tc_commit(&k_empty[ks]);
          ptx::tc_commit(&s_full[b]);
          if (++ks == kKvStages) { ks = 0; kph ^= 1; }
        };
        issue_s(g);
        for (int j = 0; j < n; ++j) {
          const uint32_t gj = g + j;
          if (j + 1 < n) issue_s(gj + 1);
          if (j + 1 == n) ptx::tc_commit(q_empty);  // last S of the item issued
          const uint32_t b = gj & 1;
          if (j == 0) ptx::mbar_wait(o_free, (items & 1) ^ 1);  // O drained
          ptx::mbar_wait(&p_full[b], (gj >> 1) & 1);
          ptx::mbar_wait(&v_full[vs], vph);
          ptx::tc_fence_after();
          const uint32_t p_addr = ptx::smem_u32(sP + b * C::kPBytes);
          const uint32_t v_addr = ptx::smem_u32(sV + vs * C::kKvBytes);
#pragma unroll
          for (int k = 0; k < BN / 16; ++k) {
            // A = P (K-major, keys along K); B = V (MN-major: dims contiguous).
            const uint32_t poff = (k >> 2) * (BM * 128) + (k & 3) * 32;
            ptx::umma_f16_ss(tmem_o, ptx::make_sdesc_sw128(p_addr + poff, 16, 1024),
                             ptx::make_sdesc_sw128(v_addr + k * 2048, BN * 128, 1024),
                             idesc_o, (j | k) != 0);
          }
          ptx::tc_commit(&v_empty[vs]);
          ptx::tc_commit(&p_free[b]);
          ptx::tc_commit(o_done);
          if (++vs == kKvStages) { vs = 0; vph ^= 1; }
        }
        g += n;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    const uint32_t quad = warp & 3;
    const int row = static_cast<int>(quad * 32 + lane);
    const uint32_t lane_off = (quad * 32) << 16;
    uint32_t g = 0, items = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++items) {
      int seg_i, qt, head;
      decode_work(work, w, seg_i, qt, head);
      const RingSegment& sg = segs[seg_i];
      const int q0 = qt * BM;
      const int a = q0 + row;  // stripe index of this thread's query
      float m_run = -INFINITY, l_run = 0.f;
      int j = 0;
      for (int r = 0; r < sg.n_rounds; ++r) {
        const int nt = TileIter::count(sg, r, q0);
        const int limit = a - sg.shift[r];
        const int kv_len = sg.kv_len[r];
        for (int t = 0; t < nt; ++t, ++j) {
          const uint32_t gj = g + j;
          const uint32_t b = gj & 1;
          const int b0 = t * BN;
          ptx::mbar_wait(&s_full[b], (gj >> 1) & 1);
          ptx::tc_fence_after();
          uint32_t s[128];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t (&chunk)[32] = *reinterpret_cast<uint32_t(*)[32]>(&s[32 * c]);
            ptx::tmem_ld_32x32b_x32(tmem_s + b * BN + lane_off + 32 * c, chunk);
          }
          ptx::tmem_wait_ld();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&s_empty[b]);
          // Striped-causal + tail mask; only diagonal / tail tiles need it.
          const bool full_tile = (b0 + BN - 1 <= q0 - sg.shift[r]) && (b0 + BN <= kv_len);
          float mx = -INFINITY;
          if (full_tile) {
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const float x = __uint_as_float(s[c]) * scale_log2;
              s[c] = __float_as_uint(x);
              mx = fmaxf(mx, x);
            }
          } else {
            const int lim = min(limit - b0, kv_len - 1 - b0);  // visible iff c <= lim
#pragma unroll
            for (int c = 0; c < 128; ++c) {
              const float x = c <= lim ? __uint_as_float(s[c]) * scale_log2 : -INFINITY;
              s[c] = __float_as_uint(x);
              mx = fmaxf(mx, x);
            }
          }
          // Lazy rescale: keep the stale max unless it grew by > 2^8.
          const float m_new = fmaxf(m_run, mx);
          const bool need = m_new > m_run + kRescaleThreshold || (m_run == -INFINITY && m_new != -INFINITY);
          float alpha = 1.f;
          if (need) {
            alpha = m_run == -INFINITY ? 0.f : exp2f(m_run - m_new);
            m_run = m_new;
          }
          if (j > 0 && __any_sync(0xffffffff, need)) {
            // O currently holds PV_{j-1}: wait for it, then scale in TMEM.
            ptx::mbar_wait(o_done, (gj - 1) & 1);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < HD; c += 32) {
              uint32_t o[32];
              ptx::tmem_ld_32x32b_x32(tmem_o + lane_off + c, o);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
              ptx::tmem_st_32x32b_x32(tmem_o + lane_off + c, o);
            }
            ptx::tmem_wait_st();
          }
          const float m_sub = m_run == -INFINITY ? 0.f : m_run;
          // P_j into smem once PV_{j-2} has released this buffer.
          if (j >= 2) ptx::mbar_wait(&p_free[b], ((gj >> 1) & 1) ^ 1);
          uint8_t* prow = sP + b * C::kPBytes + (row >> 3) * 1024 + (row & 7) * 128;
          float sum = 0.f;
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float p[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              p[e] = exp2f(__uint_as_float(s[8 * q + e]) - m_sub);
              sum += p[e];
            }
            const uint4 v = make_uint4(ptx::pack_bf16(p[0], p[1]), ptx::pack_bf16(p[2], p[3]),
                                       ptx::pack_bf16(p[4], p[5]), ptx::pack_bf16(p[6], p[7]));
            const int box = q >> 3, chunk = (q & 7) ^ (row & 7);
            *reinterpret_cast<uint4*>(prow + box * (BM * 128) + chunk * 16) = v;
          }
          l_run = l_run * alpha + sum;
          ptx::fence_async_shared();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&p_full[b]);
        }
      }
      const int n = j;
      // Final: O / l -> bf16 row of the output stripe.
      ptx::mbar_wait(o_done, (g + n - 1) & 1);
      ptx::tc_fence_after();
      const bool valid = a < sg.q_len;
      const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
      bf16* orow = out + static_cast<int64_t>(sg.q_row0 + a) * hidden + head * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t o[32];
        ptx::tmem_ld_32x32b_x32(tmem_o + lane_off + c, o);
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
      ptx::mbar_arrive(o_free);
      g += n;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int HD>
void launch(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows, int kv_rows,
            int heads, const RingSegment* segs, const int32_t* work, int n_work, float scale,
            cudaStream_t s) {
  using C = ACfg<HD>;
  once_per_device(reinterpret_cast<const void*>(ring_attention_tcgen05<HD>), [] {
    cudaFuncSetAttribute(ring_attention_tcgen05<HD>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  const int hidden = heads * HD;
  const CUtensorMap tq = make_tmap_bf16(q, q_rows, hidden, hidden, BM);
  const CUtensorMap tk = make_tmap_bf16(k, kv_rows, hidden, hidden, BN);
  const CUtensorMap tv = make_tmap_bf16(v, kv_rows, hidden, hidden, BN);
  const int grid = n_work < sm_count() ? n_work : sm_count();
  ring_attention_tcgen05<HD><<<grid, kThreads, C::kSmem, s>>>(
      tq, tk, tv, out, hidden, segs, work, n_work, scale * 1.4426950408889634f);
  count_launch();
}

}  // namespace

void ring_attention(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows,
                    int kv_rows, int heads, int head_dim, const RingSegment* d_segs, int n_segs,
                    const int32_t* d_work, int n_work, float scale, cudaStream_t s) {
  (void)n_segs;
  if (n_work <= 0) return;
  if (heads > 255) throw std::runtime_error("ring_attention: heads > 255");
  if (head_dim == 128) {
    launch<128>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s);
  } else if (head_dim == 64) {
    launch<64>(q, k, v, out, q_rows, kv_rows, heads, d_segs, d_work, n_work, scale, s);
  } else {
    throw std::runtime_error("ring_attention: head_dim must be 64 or 128");
  }
}

}  // namespace esp::k
