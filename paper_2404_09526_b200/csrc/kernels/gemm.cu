// K2/K5: persistent warp-specialized bf16 GEMM on 5th-gen tensor cores.
//
//   D[M x N] = A[M x K] . B[N x K]^T      (A activations, B nn.Linear weights)
//
// One CTA per SM. TMA (SWIZZLE_128B) streams 128 x 64 A tiles and BN x 64 B
// tiles through a STAGES-deep mbarrier ring; one elected thread issues
// tcgen05.mma (M=128, N=BN, K=16) into a double-buffered fp32 TMEM
// accumulator; four epilogue warps drain TMEM with tcgen05.ld while the next
// tile's MMAs run, and apply the fused epilogue:
//   store / residual-add (O and down projections) / fp32 (LM head) /
//   SiLU(gate)*up (gate_up projection) / QKV split + RoPE + ring-stripe write +
//   proactive-retention write into the page slot of the token's resting
//   instance (the QKV projection of ESP prefill; the KV append of decode).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "kernels.h"
#include "ptx.cuh"

namespace esp::k {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 256;

// kSkinny (M <= 32: decode, LM head of a few rows): only 32 A rows are loaded
// per stage. The UMMA (M = 128) still reads a 128-row A tile; its rows 32..127
// alias the following stages' A rows (garbage rows of D that are never
// stored), so a stage costs 4 KB of A instead of 16 KB and the pipeline keeps
// 9 weight tiles in flight per SM — these GEMMs are weight-streaming bound.
template <int BN, bool kSkinny>
struct Cfg {
  static constexpr int kARows = kSkinny ? 32 : BM;
  static constexpr int kStages = kSkinny ? 9 : (BN == 256 ? 4 : 6);
  static constexpr int kAStride = kARows * BK * 2;  // A bytes per stage
  static constexpr int kAPad = kSkinny ? (BM - kARows) * BK * 2 : 0;
  static constexpr int kARegion = kStages * kAStride + kAPad;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kTxBytes = kAStride + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = kARegion + kStages * kBBytes + 1024 + 256;
};

// m-blocks per raster group (L2 reuse of B).
constexpr int kRasterGroup = 16;

__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int& mb, int& nb) {
  constexpr int kGroup = kRasterGroup;
  const int per_group = kGroup * num_n;
  const int g = tile / per_group;
  const int first = g * kGroup;
  const int gsize = min(num_m - first, kGroup);
  const int t = tile % per_group;
  mb = first + t % gsize;
  nb = t / gsize;
}

__device__ __forceinline__ void store_row_bf16(bf16* dst, const uint32_t (&r)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d[i] = make_uint4(
        ptx::pack_bf16(__uint_as_float(r[8 * i + 0]), __uint_as_float(r[8 * i + 1])),
        ptx::pack_bf16(__uint_as_float(r[8 * i + 2]), __uint_as_float(r[8 * i + 3])),
        ptx::pack_bf16(__uint_as_float(r[8 * i + 4]), __uint_as_float(r[8 * i + 5])),
        ptx::pack_bf16(__uint_as_float(r[8 * i + 6]), __uint_as_float(r[8 * i + 7])));
  }
}

__device__ __forceinline__ void store_vals_bf16(bf16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    d[i] = make_uint4(ptx::pack_bf16(v[8 * i + 0], v[8 * i + 1]),
                      ptx::pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                      ptx::pack_bf16(v[8 * i + 4], v[8 * i + 5]),
                      ptx::pack_bf16(v[8 * i + 6], v[8 * i + 7]));
  }
}

// Accumulator sources of the epilogue: TMEM (the GEMM kernels) or an fp32
// row in global memory (the stream-K finalize of skinny GEMMs).
struct TmemAcc {
  uint32_t base;
  __device__ __forceinline__ void load(int c, uint32_t (&r)[32]) const {
    ptx::tmem_ld_32x32b_x32(base + c, r);
  }
  __device__ __forceinline__ void wait() const { ptx::tmem_wait_ld(); }
};
// Sum, in segment order (deterministic), of the fp32 partial rows that the
// stream-K segments of one tile left in their workspace slots.
struct SegSumAcc {
  const float* row;  // segment 0's row
  int nseg;
  int64_t stride;    // floats between consecutive segments' slots
  __device__ __forceinline__ void load(int c, uint32_t (&r)[32]) const {
    float4 v[8];  // all loads of a segment in flight together (L2 latency)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __ldcg(reinterpret_cast<const float4*>(row + c) + i);
    for (int sg = 1; sg < nseg; ++sg) {
      float4 w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        w[i] = __ldcg(reinterpret_cast<const float4*>(row + sg * stride + c) + i);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i].x += w[i].x;
        v[i].y += w[i].y;
        v[i].z += w[i].z;
        v[i].w += w[i].w;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      r[4 * i] = __float_as_uint(v[i].x);
      r[4 * i + 1] = __float_as_uint(v[i].y);
      r[4 * i + 2] = __float_as_uint(v[i].z);
      r[4 * i + 3] = __float_as_uint(v[i].w);
    }
  }
  __device__ __forceinline__ void wait() const {}
};

// Fused RMSNorm (GemmEpilogue.ss_in): the accumulator row m is W·diag(γ)·x_m
// and is scaled by rsqrt(mean(x_m²) + ε) as it is read.
__device__ __forceinline__ void scale32(uint32_t (&r)[32], float inv) {
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * inv);
}

template <int BN, typename Acc>
__device__ __forceinline__ void epilogue_tile(const GemmEpilogue& ep, const Acc& acc, int m,
                                              bool valid, int nb, int N) {
  uint32_t r[32];
  const bool norm = ep.ss_in != nullptr && valid;
  const float inv =
      norm ? rsqrtf(__ldcg(ep.ss_in + m) / static_cast<float>(ep.norm_dim) + ep.norm_eps) : 1.f;
  float ss_acc = 0.f;  // kEpiResidual with ss_out: this tile row's sum of squares
  if (ep.kind == kEpiStore || ep.kind == kEpiResidual || ep.kind == kEpiStoreF32 ||
      ep.kind == kEpiAtomicF32) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      acc.load(c, r);
      acc.wait();
      if (!valid) continue;
      if (norm) scale32(r, inv);
      const int64_t off = static_cast<int64_t>(m) * ep.ldo + nb * BN + c;
      if (ep.kind == kEpiAtomicF32) {
        float* d = static_cast<float*>(ep.out) + off;
#pragma unroll
        for (int i = 0; i < 32; ++i) atomicAdd(d + i, __uint_as_float(r[i]));
      } else if (ep.kind == kEpiStoreF32) {
        float* row = ep.route_rows > 0
                         ? ep.route[m / ep.route_rows] +
                               static_cast<int64_t>(m % ep.route_rows) * ep.ldo
                         : static_cast<float*>(ep.out) + static_cast<int64_t>(m) * ep.ldo;
        float4* d = reinterpret_cast<float4*>(row + nb * BN + c);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          d[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                             __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        }
      } else if (ep.kind == kEpiStore) {
        store_row_bf16(static_cast<bf16*>(ep.out) + off, r);
      } else {
        bf16* dst = static_cast<bf16*>(ep.out) + off;
        const uint4* src = reinterpret_cast<const uint4*>(dst);
        float v[32];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 o = src[i];
          const uint32_t w[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = ptx::unpack_bf16(w[j]);
            v[8 * i + 2 * j] = f.x + __uint_as_float(r[8 * i + 2 * j]);
            v[8 * i + 2 * j + 1] = f.y + __uint_as_float(r[8 * i + 2 * j + 1]);
          }
        }
        store_vals_bf16(dst, v);
        if (ep.ss_out) {  // sum of squares of the stored (bf16) row slice
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float b = __bfloat162float(__float2bfloat16_rn(v[i]));
            ss_acc = fmaf(b, b, ss_acc);
          }
        }
      }
    }
    if (ep.ss_out && valid && ep.kind == kEpiResidual) atomicAdd(ep.ss_out + m, ss_acc);
  } else if (ep.kind == kEpiSiluMul) {
    // Physical rows of the gate_up weight come in 128-row blocks: 64 gate
    // rows then the 64 matching up rows.
    uint32_t u[32];
#pragma unroll 1
    for (int p = 0; p < BN / 128; ++p) {
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        acc.load(p * 128 + c, r);
        acc.load(p * 128 + 64 + c, u);
        acc.wait();
        if (!valid) continue;
        if (norm) {
          scale32(r, inv);
          scale32(u, inv);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float g = __uint_as_float(r[i]);
          v[i] = g / (1.0f + __expf(-g)) * __uint_as_float(u[i]);
        }
        const int64_t col = static_cast<int64_t>(nb) * (BN / 2) + p * 64 + c;
        store_vals_bf16(static_cast<bf16*>(ep.out) + static_cast<int64_t>(m) * ep.ldo + col, v);
      }
    }
  } else {  // kEpiQkvRope
    const int n0 = nb * BN;
    const int region = n0 / ep.hidden;  // 0 q, 1 k, 2 v
    const int col0 = n0 - region * ep.hidden;
    const int hd = ep.head_dim, half = hd >> 1;
    int inst = -1, slot = 0, pos = 0;
    if (valid) {
      pos = ep.pos[m];
      if (ep.row_inst) {
        inst = ep.row_inst[m];
        slot = ep.row_slot ? ep.row_slot[m] : 0;
      }
    }
    bf16* dst_main =
        region == 0 ? ep.q_out : (region == 1 ? ep.k_out : ep.v_out);
    bf16* dst_slab = nullptr;
    if (region > 0 && inst >= 0) {
      dst_slab = (region == 1 ? ep.slab_k[inst] : ep.slab_v[inst]) +
                 static_cast<int64_t>(slot) * ep.hidden;
    }
    // q rows follow the GEMM rows (or q_rows); k/v rows may be remapped (ring
    // gather buffers hold every ring position's rows in global order).
    int row_map = m;
    if (valid && region > 0 && ep.kv_rows) row_map = ep.kv_rows[m];
    if (valid && region == 0 && ep.q_rows) row_map = ep.q_rows[m];
    const int64_t row_off = static_cast<int64_t>(row_map) * ep.hidden;
    if (region == 2) {
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        acc.load(c, r);
        acc.wait();
        if (!valid) continue;
        if (norm) scale32(r, inv);
        if (dst_main) store_row_bf16(dst_main + row_off + col0 + c, r);
        if (dst_slab) store_row_bf16(dst_slab + col0 + c, r);
        for (int pr = 0; pr < ep.n_peer; ++pr) store_row_bf16(ep.v_peer[pr] + row_off + col0 + c, r);
      }
    } else {
      uint32_t h[32];
      const float2* cs_row = ep.rope + static_cast<int64_t>(pos) * half;
#pragma unroll 1
      for (int hb = 0; hb < BN; hb += hd) {
#pragma unroll 1
        for (int j = 0; j < half; j += 32) {
          acc.load(hb + j, r);
          acc.load(hb + j + half, h);
          acc.wait();
          if (!valid) continue;
          if (norm) {
            scale32(r, inv);
            scale32(h, inv);
          }
          float lo[32], hi[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float2 cs = cs_row[j + e];
            const float x1 = __uint_as_float(r[e]), x2 = __uint_as_float(h[e]);
            lo[e] = x1 * cs.x - x2 * cs.y;
            hi[e] = x2 * cs.x + x1 * cs.y;
          }
          const int c_lo = col0 + hb + j, c_hi = c_lo + half;
          if (dst_main) {
            store_vals_bf16(dst_main + row_off + c_lo, lo);
            store_vals_bf16(dst_main + row_off + c_hi, hi);
          }
          if (dst_slab) {
            store_vals_bf16(dst_slab + c_lo, lo);
            store_vals_bf16(dst_slab + c_hi, hi);
          }
          if (region == 1) {
            for (int pr = 0; pr < ep.n_peer; ++pr) {
              store_vals_bf16(ep.k_peer[pr] + row_off + c_lo, lo);
              store_vals_bf16(ep.k_peer[pr] + row_off + c_hi, hi);
            }
          } else {
            for (int pr = 0; pr < ep.n_qpeer; ++pr) {
              store_vals_bf16(ep.q_peer[pr] + row_off + c_lo, lo);
              store_vals_bf16(ep.q_peer[pr] + row_off + c_hi, hi);
            }
          }
        }
      }
    }
  }
}

// Arrival signal of the fused ring transport (GemmEpilogue.arrive): called by
// the CTA's 128 epilogue threads after each output tile. When the tile was a
// K or V tile of a QKV epilogue with peers, every thread's peer stores are
// made visible system-wide, the 128 threads meet at a named barrier, and one
// thread adds rows x cols to each peer's counter slot of this source domain.
// Uniform per CTA, so the barrier is reached by all 128 threads or none.
__device__ __forceinline__ void signal_arrival(const GemmEpilogue& ep, int n0, int rows_valid,
                                               int cols) {
  if (ep.kind != kEpiQkvRope || ep.n_arrive == 0 || n0 < ep.hidden) return;
  __threadfence_system();
  ptx::named_bar_sync(2, 128);
  if ((threadIdx.x & 127) == 0 && rows_valid > 0) {
    const unsigned long long add = static_cast<unsigned long long>(rows_valid) * cols;
    for (int p = 0; p < ep.n_arrive; ++p) atomicAdd_system(ep.arrive[p], add);
  }
}

// Work of one persistent CTA: whole output tiles round-robin (kb_per_cta ==
// 0), or stream-K (kb_per_cta > 0): the (tile, K block) space is cut into
// equal contiguous ranges of kb_per_cta K blocks, one per CTA, each range
// split at tile boundaries into segments whose partial sums the epilogue
// (kEpiAtomicF32) adds into an fp32 workspace.
struct WorkRange {
  int next, end, num_k, stride;
  bool stream;
  int sub_lo = -1, sub_hi = -1;  // strided tiles, each over K blocks [sub_lo, sub_hi)
  __device__ WorkRange(int tiles, int num_k_, int kb_per_cta) : num_k(num_k_) {
    stream = kb_per_cta > 0;
    if (stream) {
      next = static_cast<int>(blockIdx.x) * kb_per_cta;
      end = min(tiles * num_k, next + kb_per_cta);
      stride = 0;
    } else {
      next = static_cast<int>(blockIdx.x);
      end = tiles;
      stride = static_cast<int>(gridDim.x);
    }
  }
  __device__ bool get(int& tile, int& kb0, int& kb1) {
    if (next >= end) return false;
    if (stream) {
      tile = next / num_k;
      kb0 = next - tile * num_k;
      kb1 = min(num_k, kb0 + (end - next));
      next += kb1 - kb0;
    } else {
      tile = next;
      kb0 = sub_lo >= 0 ? sub_lo : 0;
      kb1 = sub_lo >= 0 ? sub_hi : num_k;
      next += stride;
    }
    return true;
  }
};

template <int BN, bool kSkinny>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                      int kb_per_cta, const __grid_constant__ GemmEpilogue ep,
                      float* __restrict__ ws, int* __restrict__ tile_kb) {
  using C = Cfg<BN, kSkinny>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kARegion;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::kStages * C::kBBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  volatile uint32_t* last_flag = tmem_slot + 1;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m = (M + BM - 1) / BM, num_n = N / BN, num_k = K / BK;
  const int tiles = num_m * num_n;
  WorkRange work(tiles, num_k, kb_per_cta);
  int tile, kb0, kb1;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t keep = ptx::policy_evict_last();  // B (weights) is re-read by every M tile
      while (work.get(tile, kb0, kb1)) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], C::kTxBytes);
          ptx::tma_load_2d(sA + stage * C::kAStride, &tmA, &full[stage], kb * BK, mb * BM);
          ptx::tma_load_2d_hint(sB + stage * C::kBBytes, &tmB, &full[stage], kb * BK, nb * BN, keep);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // Whole warp runs the uniform loop (descriptors in uniform registers);
    // one elected lane issues each tcgen05.mma / commit.
    const bool leader = ptx::elect_one();
    constexpr uint32_t idesc = ptx::make_idesc_bf16(BM, BN, false, false);
    int stage = 0;
    uint32_t phase = 0;
    int lt = 0;
    for (; work.get(tile, kb0, kb1); ++lt) {
      const int acc = lt & 1;
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint32_t a0 = ptx::smem_u32(sA + stage * C::kAStride);
        const uint32_t b0 = ptx::smem_u32(sB + stage * C::kBBytes);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t da = ptx::make_sdesc_sw128(a0 + k * 32, 16, 1024);
          const uint64_t db = ptx::make_sdesc_sw128(b0 + k * 32, 16, 1024);
          if (leader) ptx::umma_f16_ss(d_tmem, da, db, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
        }
        if (leader) ptx::tc_commit(&empty[stage]);
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (leader) ptx::tc_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const uint32_t quad = warp & 3;
    const int row = static_cast<int>(quad * 32 + lane);
    int lt = 0;
    for (; work.get(tile, kb0, kb1); ++lt) {
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int acc = lt & 1;
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const uint32_t tacc = tmem_base + acc * BN + ((quad * 32) << 16);
      const int m = mb * BM + row;
      if (!work.stream) {
        epilogue_tile<BN>(ep, TmemAcc{tacc}, m, m < M, nb, N);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
        signal_arrival(ep, nb * BN, min(BM, M - mb * BM), BN);
        continue;
      }
      // Stream-K: store this segment's fp32 partial rows in its own
      // workspace slot (no atomics), free the accumulator, and count the
      // tile's K blocks; the CTA that completes the tile sums the slots in
      // segment order and applies the real epilogue.
      const int max_seg = (num_k + kb_per_cta - 1) / kb_per_cta + 1;
      const int first_cta = tile * num_k / kb_per_cta;
      const int last_cta = ((tile + 1) * num_k - 1) / kb_per_cta;
      const int64_t slot_floats = static_cast<int64_t>(M) * BN;
      float* tile_ws = ws + static_cast<int64_t>(tile) * max_seg * slot_floats;
      float* my_row = tile_ws + (static_cast<int>(blockIdx.x) - first_cta) * slot_floats +
                      static_cast<int64_t>(m) * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tacc + c, r);
        ptx::tmem_wait_ld();
        if (m < M) {
          float4* d = reinterpret_cast<float4*>(my_row + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            __stcg(d + i, make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                      __uint_as_float(r[4 * i + 2]),
                                      __uint_as_float(r[4 * i + 3])));
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      __threadfence();
      ptx::named_bar_sync(1, 128);
      if (threadIdx.x == 128) {
        const int done = atomicAdd(&tile_kb[tile], kb1 - kb0) + (kb1 - kb0);
        *last_flag = done == num_k ? 1u : 0u;
      }
      ptx::named_bar_sync(1, 128);
      if (*last_flag) {
        __threadfence();
        if (m < M) {
          const SegSumAcc sum{tile_ws + static_cast<int64_t>(m) * BN, last_cta - first_cta + 1,
                              slot_floats};
          epilogue_tile<BN>(ep, sum, m, true, nb, N);
        }
        if (threadIdx.x == 128) tile_kb[tile] = 0;
      }
      ptx::named_bar_sync(1, 128);  // last_flag is rewritten by the next segment
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

// Decode-shaped GEMM with the operands swapped (D^T = W . X^T): the weight
// tile is the UMMA's M = 128 operand and the <= 32 activation rows are its
// N = NT operand, so the tensor core does 128 x NT x 64 per K block instead
// of 128 x 128 x 64 with 7/8 of the rows wasted (which made the M = 128
// skinny kernel tensor-bound at ~50 GB/s of weights per SM). Weight tiles
// (16 KB) stream through kStages stages with an evict-first L2 hint; the
// NT x 64 activation tile rides along (L2-resident). The accumulator is
// 128 TMEM lanes (output columns) x NT columns (tokens); the epilogue warps
// transpose it through shared memory into NT fp32 rows and then run the same
// fused epilogues as the other GEMMs (thread = output row) — or, under
// stream-K, store the rows as partial sums for the tile's last CTA.
namespace swp {
constexpr int kStages = 10;
template <int NT>
struct Cfg {
  static constexpr int kWBytes = 128 * BK * 2;     // 16 KB
  static constexpr int kXBytes = NT * BK * 2;      // 2 or 4 KB
  static constexpr int kTx = kWBytes + kXBytes;
  static constexpr int kTBytes = NT * 128 * 4;     // transposed accumulator
  static constexpr int kSmem = kStages * (kWBytes + kXBytes) + kTBytes + 1024 + 256;
  static constexpr int kTmemCols = NT * 2 < 32 ? 32 : NT * 2;
};
}  // namespace swp

struct RowAcc {  // one fp32 row in shared memory
  const float* row;
  __device__ __forceinline__ void load(int c, uint32_t (&r)[32]) const {
#pragma unroll
    for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(row[c + i]);
  }
  __device__ __forceinline__ void wait() const {}
};

// Fused epilogue of one 128-column tile from its row-major fp32 image in
// shared memory. Store / residual / fp32 kinds: four threads per row, 32
// columns each (independent global reads in flight); the kinds that pair
// columns 64 apart (SiLU gate/up, RoPE halves) run one thread per row.
__device__ __forceinline__ void swap_epilogue(const GemmEpilogue& ep, float* sT, int M,
                                              int t, int tile, int N) {
  if (ep.kind == kEpiStore || ep.kind == kEpiResidual || ep.kind == kEpiStoreF32) {
    const int m = t >> 2, j = t & 3;
    if (m < M) epilogue_tile<32>(ep, RowAcc{sT + m * 128 + j * 32}, m, true, tile * 4 + j, N);
  } else if (t < M) {
    epilogue_tile<128>(ep, RowAcc{sT + t * 128}, t, true, tile, N);
  }
}

template <int NT, int SPLIT>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_skinny_swap(const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ CUtensorMap tmW, int M, int N, int K,
                     int kb_per_cta, const __grid_constant__ GemmEpilogue ep,
                     float* __restrict__ ws, int* __restrict__ tile_kb,
                     unsigned long long* __restrict__ trace) {
  using C = swp::Cfg<NT>;
  auto gtime = [] {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
  };
  unsigned long long* tr = trace ? trace + blockIdx.x * 8 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtime();
  constexpr int S = swp::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sW = smem;
  uint8_t* sX = sW + S * C::kWBytes;
  float* sT = reinterpret_cast<float*>(sX + S * C::kXBytes);  // [NT][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sT) + C::kTBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* pair_bar = tempty + 2;  // [0] partial ready (rank 0), [1] partial consumed (rank 1)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pair_bar + 2);
  volatile uint32_t* last_flag = tmem_slot + 1;

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0 && lane == 0) {
    ptx::mbar_init(&pair_bar[0], 1);
    ptx::mbar_init(&pair_bar[1], 1);
    ptx::tma_prefetch_desc(&tmX);
    ptx::tma_prefetch_desc(&tmW);
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 128);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (SPLIT == -2) ptx::cluster_sync();  // the peer's barriers are initialised
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  const int num_n = N / 128, num_k = K / BK;
  WorkRange work(num_n, num_k, kb_per_cta);
  if constexpr (SPLIT == -2) {
    // Persistent pair split: cluster c of a 2-CTA grid walks tiles c,
    // c + nclusters, ...; rank r covers K blocks [r, r+1) * num_k / 2 of each.
    // Balances tile counts that do not divide the SM count (gate_up: 172
    // tiles on 148 SMs -> at most 1.5 tiles of weights per SM instead of 2).
    const int r = static_cast<int>(blockIdx.x) & 1;
    work.next = static_cast<int>(blockIdx.x) >> 1;
    work.end = num_n;
    work.stride = static_cast<int>(gridDim.x) >> 1;
    work.stream = false;
    work.sub_lo = r * num_k / 2;
    work.sub_hi = (r + 1) * num_k / 2;
  }
  if constexpr (SPLIT > 1) {
    // Split-K over a cluster of SPLIT CTAs: CTA rank r of cluster c computes
    // tile c over K blocks [r, r+1) * num_k / SPLIT; the partial
    // accumulators are summed through distributed shared memory below.
    const int r = static_cast<int>(blockIdx.x) % SPLIT;
    work.next = static_cast<int>(blockIdx.x) / SPLIT * num_k + r * num_k / SPLIT;
    work.end = static_cast<int>(blockIdx.x) / SPLIT * num_k + (r + 1) * num_k / SPLIT;
    work.stream = true;
    work.stride = 0;
  }
  int tile, kb0, kb1;

  ptx::griddep_launch();
  if (warp == 0) {
    if (lane == 0) {
      // PDL: the first S weight tiles do not depend on the previous kernel
      // and are requested before griddepcontrol.wait (they stream while the
      // previous kernel drains); their activation tiles follow the wait.
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t stream_once = ptx::policy_evict_first();
      int pre_kb[S];
      int n_pre = 0;
      bool waited = false;
      auto release = [&] {
        ptx::griddep_wait();
        for (int i = 0; i < n_pre; ++i) {
          ptx::tma_load_2d(sX + i * C::kXBytes, &tmX, &full[i], pre_kb[i] * BK, 0);
        }
        waited = true;
      };
      while (work.get(tile, kb0, kb1)) {
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], C::kTx);
          ptx::tma_load_2d_hint(sW + stage * C::kWBytes, &tmW, &full[stage], kb * BK, tile * 128,
                                stream_once);
          if (waited) {
            ptx::tma_load_2d(sX + stage * C::kXBytes, &tmX, &full[stage], kb * BK, 0);
          } else {
            pre_kb[n_pre++] = kb;
            if (n_pre == S) release();
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (!waited) release();
    }
  } else if (warp == 1) {
    const bool leader = ptx::elect_one();
    constexpr uint32_t idesc = ptx::make_idesc_bf16(128, NT, false, false);
    int stage = 0;
    uint32_t phase = 0;
    int lt = 0;
    for (; work.get(tile, kb0, kb1); ++lt) {
      const int acc = lt & 1;
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * NT;
      for (int kb = kb0; kb < kb1; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (tr && lt == 0 && kb == kb0 && lane == 0) tr[2] = gtime();
        const uint32_t w0 = ptx::smem_u32(sW + stage * C::kWBytes);
        const uint32_t x0 = ptx::smem_u32(sX + stage * C::kXBytes);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t dw = ptx::make_sdesc_sw128(w0 + k * 32, 16, 1024);
          const uint64_t dx = ptx::make_sdesc_sw128(x0 + k * 32, 16, 1024);
          if (leader) ptx::umma_f16_ss(d_tmem, dw, dx, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
        }
        if (leader) ptx::tc_commit(&empty[stage]);
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (leader) ptx::tc_commit(&tfull[acc]);
      __syncwarp();
    }
    if (tr && lane == 0) tr[3] = gtime();
  } else if (warp >= 4) {
    ptx::griddep_wait();  // residual / outputs are the previous kernels' data
    const uint32_t quad = warp & 3;
    const int t = static_cast<int>(quad * 32 + lane);  // output column of the tile
    if (ep.ss_zero != nullptr && blockIdx.x == 0 && t < 32) ep.ss_zero[t] = 0.f;
    int lt = 0;
    for (; work.get(tile, kb0, kb1); ++lt) {
      const int acc = lt & 1;
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      if (tr && t == 0 && lt == 0) tr[6] = gtime();
      const uint32_t tacc = tmem_base + acc * NT + ((quad * 32) << 16);
      // sT is reused tile after tile: the previous tile's readers are done
      // (barrier at the end of the previous iteration).
      if constexpr (NT == 16) {
        uint32_t r[16];
        ptx::tmem_ld_32x32b_x16(tacc, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) sT[j * 128 + t] = __uint_as_float(r[j]);
      } else {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tacc, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) sT[j * 128 + t] = __uint_as_float(r[j]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      if constexpr (SPLIT > 1) continue;  // reduced across the cluster below
      if constexpr (SPLIT == -2) {
        // rank 1 hands its partial tile to rank 0 through DSMEM; rank 0 adds
        // it to its own, frees the peer's sT and applies the epilogue.
        const uint32_t rank = ptx::cluster_ctarank();
        ptx::named_bar_sync(1, 128);
        if (rank == 1) {
          if (t == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&pair_bar[0]), 0));
          // sT is rewritten for the next tile only after rank 0 has read it
          ptx::mbar_wait_cluster(&pair_bar[1], static_cast<uint32_t>(lt) & 1);
          continue;
        }
        ptx::mbar_wait_cluster(&pair_bar[0], static_cast<uint32_t>(lt) & 1);
        float4* own = reinterpret_cast<float4*>(sT);
        for (int i = t; i < M * 32; i += 128) {
          float4 v = own[i];
          const float4 w = ptx::ld_cluster_f32x4(ptx::mapa(ptx::smem_u32(own + i), 1));
          v.x += w.x;
          v.y += w.y;
          v.z += w.z;
          v.w += w.w;
          own[i] = v;
        }
        ptx::named_bar_sync(1, 128);
        if (t == 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&pair_bar[1]), 1));
        swap_epilogue(ep, sT, M, t, tile, N);
        ptx::named_bar_sync(1, 128);
        continue;
      }
      ptx::named_bar_sync(1, 128);
      if (!work.stream) {
        swap_epilogue(ep, sT, M, t, tile, N);
        ptx::named_bar_sync(1, 128);
        continue;
      }
      const int m = t;
      const float* my = sT + m * 128;
      const int max_seg = (num_k + kb_per_cta - 1) / kb_per_cta + 1;
      const int first_cta = tile * num_k / kb_per_cta;
      const int last_cta = ((tile + 1) * num_k - 1) / kb_per_cta;
      const int64_t slot_floats = static_cast<int64_t>(M) * 128;
      float* tile_ws = ws + static_cast<int64_t>(tile) * max_seg * slot_floats;
      if (m < M) {
        float4* d = reinterpret_cast<float4*>(
            tile_ws + (static_cast<int>(blockIdx.x) - first_cta) * slot_floats +
            static_cast<int64_t>(m) * 128);
        const float4* src = reinterpret_cast<const float4*>(my);
#pragma unroll 4
        for (int i = 0; i < 32; ++i) __stcg(d + i, src[i]);
      }
      __threadfence();
      ptx::named_bar_sync(1, 128);
      if (t == 0) {
        const int done = atomicAdd(&tile_kb[tile], kb1 - kb0) + (kb1 - kb0);
        *last_flag = done == num_k ? 1u : 0u;
      }
      ptx::named_bar_sync(1, 128);
      if (*last_flag) {
        __threadfence();
        // Sum the tile's segment partials cooperatively into sT (all loads
        // of up to 8 segments in flight at once), then the fused epilogue.
        const int nseg = last_cta - first_cta + 1;
        const int n4 = M * 32;  // float4s per slot
        for (int i0 = t; i0 < n4; i0 += 4 * 128) {
          float4 a[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int sg0 = 0; sg0 < nseg; sg0 += 8) {
#pragma unroll
            for (int sg = 0; sg < 8; ++sg) {
              if (sg0 + sg < nseg) {
                const float4* src =
                    reinterpret_cast<const float4*>(tile_ws + (sg0 + sg) * slot_floats);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const int idx = i0 + i * 128;
                  if (idx < n4) {
                    const float4 w = __ldcg(src + idx);
                    a[i].x += w.x;
                    a[i].y += w.y;
                    a[i].z += w.z;
                    a[i].w += w.w;
                  }
                }
              }
            }
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int idx = i0 + i * 128;
            if (idx < n4) reinterpret_cast<float4*>(sT)[idx] = a[i];
          }
        }
        ptx::named_bar_sync(1, 128);
        swap_epilogue(ep, sT, M, t, tile, N);
        if (t == 0) tile_kb[tile] = 0;
      }
      ptx::named_bar_sync(1, 128);
    }
    if (tr && t == 0) tr[4] = gtime();
  }
  if constexpr (SPLIT == -2) ptx::cluster_sync();  // peers' smem alive until read
  if constexpr (SPLIT > 1) {
    // Every CTA's partial tile is in its sT; rank 0 sums the others' over
    // DSMEM (no global workspace, no atomics) and applies the epilogue; the
    // second cluster barrier keeps the peers' shared memory alive until then.
    ptx::cluster_sync();
    if (ptx::cluster_ctarank() == 0 && warp >= 4) {
      const int t = static_cast<int>((warp & 3) * 32 + lane);
      const int tile0 = static_cast<int>(blockIdx.x) / SPLIT;
      const int n4 = M * 32;  // float4s of the M valid rows
      float4* own = reinterpret_cast<float4*>(sT);
      for (int i = t; i < n4; i += 128) {
        float4 v = own[i];
#pragma unroll
        for (int r = 1; r < SPLIT; ++r) {
          const float4 w = ptx::ld_cluster_f32x4(ptx::mapa(ptx::smem_u32(own + i), r));
          v.x += w.x;
          v.y += w.y;
          v.z += w.z;
          v.w += w.w;
        }
        own[i] = v;
      }
      ptx::named_bar_sync(1, 128);
      swap_epilogue(ep, sT, M, t, tile0, N);
    }
    ptx::cluster_sync();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  if (tr && threadIdx.x == 0) tr[5] = gtime();
}

// CTA-pair variant for the large prefill GEMMs: a cluster of two CTAs on one
// TPC owns a 256 x 256 output tile. Each CTA TMA-loads its 128 A rows and its
// 128 B rows (32 KB per K block instead of 48 KB for a 1-CTA 128 x 256 tile),
// the leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256), and each CTA
// drains its own 128 accumulator rows through the same fused epilogue.
namespace pair {
constexpr int kTileM = 256, kTileN = 256, kRows = 128;
constexpr int kStageBytes = 2 * kRows * BK * 2;  // A half + B half
constexpr int kStages = 6;
constexpr int kTmemCols = 512;
constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
}  // namespace pair

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                           const __grid_constant__ GemmEpilogue ep) {
  using namespace pair;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;                        // [stage][128 x 64]
  uint8_t* sB = smem + kStages * kRows * BK * 2;  // [stage][128 x 64]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t rank = ptx::cluster_ctarank();
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tfull[a], 1);
      ptx::mbar_init(&tempty[a], 8);  // one arrival per epilogue warp of both CTAs
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc_pair<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m = (M + kTileM - 1) / kTileM, num_n = N / kTileN, num_k = K / BK;
  const int units = num_m * num_n;
  const int cid = static_cast<int>(ptx::cluster_id_x());
  const int ncl = static_cast<int>(ptx::nclusters_x());

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full_lead = ptx::mapa(ptx::smem_u32(full), 0);
      const uint64_t keep = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < units; u += ncl) {
        int mb, nb;
        tile_coords(u, num_m, num_n, mb, nb);
        const int a_row = mb * kTileM + static_cast<int>(rank) * kRows;
        const int b_row = nb * kTileN + static_cast<int>(rank) * kRows;
        for (int kb = 0; kb < num_k; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) ptx::mbar_expect_tx(&full[stage], 2 * kStageBytes);
          const uint32_t bar = full_lead + stage * 8;
          ptx::tma_load_2d_pair(sA + stage * kRows * BK * 2, &tmA, bar, kb * BK, a_row, keep);
          ptx::tma_load_2d_pair(sB + stage * kRows * BK * 2, &tmB, bar, kb * BK, b_row, keep);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const bool leader = ptx::elect_one();
      constexpr uint32_t idesc = ptx::make_idesc_bf16(kTileM, kTileN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      for (int u = cid; u < units; u += ncl, ++lt) {
        const int acc = lt & 1;
        const uint32_t use = static_cast<uint32_t>(lt >> 1);
        ptx::mbar_wait(&tempty[acc], (use & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kTileN;
        for (int kb = 0; kb < num_k; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a0 = ptx::smem_u32(sA + stage * kRows * BK * 2);
          const uint32_t b0 = ptx::smem_u32(sB + stage * kRows * BK * 2);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t da = ptx::make_sdesc_sw128(a0 + k * 32, 16, 1024);
            const uint64_t db = ptx::make_sdesc_sw128(b0 + k * 32, 16, 1024);
            if (leader) ptx::umma_f16_ss_pair(d_tmem, da, db, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          if (leader) ptx::tc_commit_pair(&empty[stage], 0x3);
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (leader) ptx::tc_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const uint32_t quad = warp & 3;
    const int row = static_cast<int>(quad * 32 + lane);
    const uint32_t tempty_lead = ptx::mapa(ptx::smem_u32(tempty), 0);
    int lt = 0;
    for (int u = cid; u < units; u += ncl, ++lt) {
      int mb, nb;
      tile_coords(u, num_m, num_n, mb, nb);
      const int acc = lt & 1;
      const uint32_t use = static_cast<uint32_t>(lt >> 1);
      ptx::mbar_wait(&tfull[acc], use & 1);
      ptx::tc_fence_after();
      const uint32_t tacc = tmem_base + acc * kTileN + ((quad * 32) << 16);
      const int m = mb * kTileM + static_cast<int>(rank) * kRows + row;
      epilogue_tile<kTileN>(ep, TmemAcc{tacc}, m, m < M, nb, N);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(tempty_lead + acc * 8);
      signal_arrival(ep, nb * kTileN,
                     min(kRows, M - (mb * kTileM + static_cast<int>(rank) * kRows)), kTileN);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_pair<pair::kTmemCols>(tmem_base);
  }
}

// ---- host: tensor maps -----------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        p == nullptr) {
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

}  // namespace

// bf16 [rows x cols] row-major (row pitch ld elements), box box_rows x 64,
// 128-byte swizzle (the UMMA K-major SW128 canonical layout). The encoding
// is a pure function of its arguments, so it is memoised per host thread: a
// decode step launches ~200 GEMMs over the same weight and activation
// buffers, and re-encoding two maps per launch costs host time the PDL
// chain then waits for.
CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld,
                           int box_rows) {
  struct Key {
    const void* base;
    int64_t rows, cols, ld;
    int box;
    bool operator==(const Key& o) const {
      return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      size_t h = std::hash<const void*>()(k.base);
      for (int64_t v : {k.rows, k.cols, k.ld, static_cast<int64_t>(k.box)}) {
        h ^= std::hash<int64_t>()(v) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      }
      return h;
    }
  };
  thread_local std::unordered_map<Key, CUtensorMap, Hash> cache;
  const Key key{base, rows, cols, ld, box_rows};
  if (auto it = cache.find(key); it != cache.end()) return it->second;
  if (cache.size() > 8192) cache.clear();
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                           dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  }
  cache.emplace(key, m);
  return m;
}

template <int BN, bool kSkinny>
static void launch_gemm(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
                        int kb_per_cta, const GemmEpilogue& ep, cudaStream_t s,
                        float* ws = nullptr, int* tile_kb = nullptr) {
  using C = Cfg<BN, kSkinny>;
  once_per_device(reinterpret_cast<const void*>(gemm_bf16_tcgen05<BN, kSkinny>), [] {
    cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, kSkinny>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  });
  const CUtensorMap ta = make_tmap_bf16(A, M, K, lda, C::kARows);
  const CUtensorMap tb = make_tmap_bf16(B, N, K, ldb, BN);
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  const int grid = kb_per_cta > 0 ? (tiles * (K / BK) + kb_per_cta - 1) / kb_per_cta
                                  : std::min(tiles, num_sms());
  gemm_bf16_tcgen05<BN, kSkinny><<<grid, kThreads, C::kSmem, s>>>(ta, tb, M, N, K, kb_per_cta,
                                                                  ep, ws, tile_kb);
  count_launch();
}

template <int NT, int SPLIT>
static void launch_skinny_swap(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
                               int kb_per_cta, const GemmEpilogue& ep, cudaStream_t s,
                               float* ws, int* tile_kb) {
  using C = swp::Cfg<NT>;
  once_per_device(reinterpret_cast<const void*>(gemm_skinny_swap<NT, SPLIT>), [] {
    cudaFuncSetAttribute(gemm_skinny_swap<NT, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         C::kSmem);
    if (SPLIT > 1 || SPLIT == -2) {
      cudaFuncSetAttribute(gemm_skinny_swap<NT, SPLIT>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
  });
  const CUtensorMap tx = make_tmap_bf16(A, M, K, lda, NT);
  const CUtensorMap tw = make_tmap_bf16(B, N, K, ldb, 128);
  const int tiles = N / 128;
  const int grid = SPLIT > 1    ? tiles * SPLIT
                   : SPLIT == -2 ? 2 * std::min(tiles, num_sms() / 2)
                   : kb_per_cta > 0 ? (tiles * (K / BK) + kb_per_cta - 1) / kb_per_cta
                                    : std::min(tiles, num_sms());
  unsigned long long* trace = nullptr;
#ifdef ESP_STUDY
  // Kernel-study build: ESP_GEMM_TRACE=<file> appends per-CTA globaltimer
  // stamps (entry, setup done, first stage landed, last MMA, first tile
  // drained, epilogue done, exit) of every skinny launch to <file>.
  static const char* trace_path = getenv("ESP_GEMM_TRACE");
  if (trace_path) {
    cudaMalloc(&trace, static_cast<size_t>(grid) * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(trace, 0, static_cast<size_t>(grid) * 8 * sizeof(unsigned long long), s);
  }
#endif
  if constexpr (SPLIT > 1 || SPLIT == -2) {
    // Cluster of SPLIT CTAs per output tile (split-K reduced over DSMEM) or a
    // persistent CTA pair (SPLIT == -2), with programmatic dependent launch
    // like the other decode kernels.
    constexpr int kCluster = SPLIT > 1 ? SPLIT : 2;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled(1) ? 2 : 1;
    cudaLaunchKernelEx(&cfg, gemm_skinny_swap<NT, SPLIT>, tx, tw, M, N, K, 0, ep, ws, tile_kb,
                       trace);
  } else {
    launch_pdl(1, gemm_skinny_swap<NT, SPLIT>, dim3(grid), dim3(kThreads), C::kSmem, s, tx, tw,
               M, N, K, kb_per_cta, ep, ws, tile_kb, trace);
  }
  count_launch();
#ifdef ESP_STUDY
  if (trace) {
    std::vector<unsigned long long> h(static_cast<size_t>(grid) * 8);
    cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(trace);
    if (FILE* f = fopen(trace_path, "a")) {
      fprintf(f, "launch N=%d K=%d M=%d per=%d grid=%d\n", N, K, M, kb_per_cta, grid);
      for (int b = 0; b < grid; ++b) {
        fprintf(f, "%d", b);
        for (int i = 0; i < 7; ++i) fprintf(f, " %llu", h[static_cast<size_t>(b) * 8 + i]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
#endif
}

// Co-resident CTA pairs of the current device (normally num_sms / 2).
static int pair_clusters() {
  static std::unordered_map<int, int> cache;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  cudaFuncSetAttribute(gemm_bf16_tcgen05_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       pair::kSmem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * num_sms());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = pair::kSmem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_bf16_tcgen05_pair, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  cache[dev] = n;
  return n;
}

static bool launch_gemm_pair(const bf16* A, int lda, const bf16* B, int ldb, int M, int N,
                             int K, const GemmEpilogue& ep, cudaStream_t s) {
  if (M < pair::kTileM || N % pair::kTileN != 0) return false;
  if (ep.kind == kEpiQkvRope && ep.hidden % pair::kTileN != 0) return false;
  const int clusters = pair_clusters();
  const int units = ((M + pair::kTileM - 1) / pair::kTileM) * (N / pair::kTileN);
  if (clusters <= 0 || units < clusters) return false;
  const CUtensorMap ta = make_tmap_bf16(A, M, K, lda, pair::kRows);
  const CUtensorMap tb = make_tmap_bf16(B, N, K, ldb, pair::kRows);
  gemm_bf16_tcgen05_pair<<<2 * clusters, kThreads, pair::kSmem, s>>>(ta, tb, M, N, K, ep);
  count_launch();
  return true;
}

// Stream-K workspace per (device, stream) — concurrent GEMMs on different
// streams of one device never share it: fp32 partial-row slots [tile][segment]
// [M x 128], and one zero-initialised K-block counter per output tile at the
// end of the buffer (the CTA that completes a tile re-zeroes it).
struct StreamKWs {
  float* sums;
  int* tile_kb;
};
StreamKWs streamk_workspace(size_t elems, size_t tiles, cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<char*, size_t>> ws;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  auto& w = ws[{dev, s}];
  const size_t sum_bytes = (elems * sizeof(float) + 255) & ~static_cast<size_t>(255);
  const size_t need = sum_bytes + tiles * sizeof(int);
  if (w.second < need) {
    if (w.first) {
      cudaStreamSynchronize(s);
      cudaFree(w.first);
    }
    w.second = std::max(need * 2, static_cast<size_t>(8) << 20);
    if (cudaMalloc(&w.first, w.second) != cudaSuccess) {
      throw std::runtime_error("stream-K workspace allocation failed");
    }
    cudaMemsetAsync(w.first, 0, w.second, s);
  }
  // Counters live at the END of the buffer so their offset does not depend
  // on this call's slot layout (all counters are zero between calls).
  return {reinterpret_cast<float*>(w.first),
          reinterpret_cast<int*>(w.first + w.second) - tiles};
}

void gemm(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
          const GemmEpilogue& ep, cudaStream_t s, int path) {
  if (M <= 0) return;
  struct {
    bool no_pair, no_streamk, streamk_all;
  } const paths{path == kGemmNoPair, path == kGemmTilesOnly, path == kGemmStreamKAll};
  if (ep.ss_zero != nullptr && M > 32) {
    throw std::runtime_error("gemm: ss_zero is implemented by the skinny (M <= 32) kernel");
  }
  if (N % 128 != 0 || K % 64 != 0) throw std::runtime_error("gemm: N%128 or K%64 != 0");
  if (M <= 32) {
    // Decode-shaped: weight-streaming bound (swap-AB skinny kernel: the
    // 128-row weight tile is the UMMA M operand, the <= 32 token rows its N).
    const int tiles = N / 128, total = tiles * (K / BK);
    const bool forced = paths.no_streamk || paths.streamk_all;
    // Few wide tiles (O, down: 32 on 148 SMs): split-K over a cluster of 4
    // CTAs reduced through distributed shared memory — 128 SMs stream
    // weights and there is no global fixup (O 15.3 -> 10.1 us, down 37.5 ->
    // 18.2 us; one SM streams ~82 GB/s of weights).
    if (!forced && tiles * 4 <= num_sms() && K / BK >= 16) {
      if (M <= 16) launch_skinny_swap<16, 4>(A, lda, B, ldb, M, N, K, 0, ep, s, nullptr, nullptr);
      else launch_skinny_swap<32, 4>(A, lda, B, ldb, M, N, K, 0, ep, s, nullptr, nullptr);
      return;
    }
    // Tile counts between one and two waves (gate_up: 172 on 148 SMs): a
    // persistent CTA pair per cluster splits every tile's K in two, so the
    // busiest SM streams 1.5 tiles of weights instead of 2.
    const int pairs = num_sms() / 2;
    if (!forced && K / BK >= 32 &&
        2 * ((tiles + num_sms() - 1) / num_sms()) > (tiles + pairs - 1) / pairs) {
      if (M <= 16) launch_skinny_swap<16, -2>(A, lda, B, ldb, M, N, K, 0, ep, s, nullptr, nullptr);
      else launch_skinny_swap<32, -2>(A, lda, B, ldb, M, N, K, 0, ep, s, nullptr, nullptr);
      return;
    }
    // Whole tiles (QKV: 96, LM head: 250), or stream-K over (tile, K block)
    // when whole tiles would leave more than half the SMs idle; the CTA
    // completing a tile applies the fused epilogue to its fp32 partial sums.
    const bool streamk = paths.streamk_all || (!paths.no_streamk && 2 * tiles < num_sms());
    if (!streamk) {
      if (M <= 16) launch_skinny_swap<16, 1>(A, lda, B, ldb, M, N, K, 0, ep, s, nullptr, nullptr);
      else launch_skinny_swap<32, 1>(A, lda, B, ldb, M, N, K, 0, ep, s, nullptr, nullptr);
      return;
    }
    const int per = (total + num_sms() - 1) / num_sms();
    const int max_seg = (K / BK + per - 1) / per + 1;
    const StreamKWs w =
        streamk_workspace(static_cast<size_t>(tiles) * max_seg * M * 128, tiles, s);
    if (M <= 16) launch_skinny_swap<16, 1>(A, lda, B, ldb, M, N, K, per, ep, s, w.sums, w.tile_kb);
    else launch_skinny_swap<32, 1>(A, lda, B, ldb, M, N, K, per, ep, s, w.sums, w.tile_kb);
    return;
  }
  if (!paths.no_pair && launch_gemm_pair(A, lda, B, ldb, M, N, K, ep, s)) return;
  const bool n256 = N % 256 == 0;
  const int tiles256 = ((M + BM - 1) / BM) * (N / 256);
  // Prefer the wide tile unless it would leave SMs idle.
  if (n256 && tiles256 >= num_sms()) {
    launch_gemm<256, false>(A, lda, B, ldb, M, N, K, 0, ep, s);
  } else {
    launch_gemm<128, false>(A, lda, B, ldb, M, N, K, 0, ep, s);
  }
}

}  // namespace esp::k
