// K3 + K4: multi-master distributed decoding (LoongServe PAPER.md:272-284).
//
// K3 (split-KV paged attention): every instance that holds part of a
// request's KV computes a partial attention of the request's new query over
// its own token slots. A request's slots on one instance are split into
// chunks of <= kChunk tokens; one CTA handles one (chunk, head). The slab
// layout is [layer][slot][heads*head_dim] bf16, so one token's K row of one
// head is head_dim*2 contiguous bytes: head_dim/8 lanes each issue one
// 128-bit non-caching load (ld.global.nc.L1::no_allocate.v4) per token, the
// dot product is reduced with warp shuffles, and the online softmax runs per
// token in registers. Output: (o, m, l) per (chunk, head), fp32.
//
// K4 (LSE combine at the master): o = sum_c e^{m_c-M} o_c / sum_c e^{m_c-M} l_c
// over all chunks of the request, on every instance that held its KV.
#include <cfloat>
#include <cstdlib>
#include <stdexcept>

#include "kernels.h"
#include "ptx.cuh"

namespace esp::k {

namespace {

constexpr int kWarps = 4;
constexpr int kUnroll = 4;

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Kernel-parameter arrays indexed by a runtime value are copied to local
// memory (a 256-byte stack frame per thread); an unrolled compare-select
// keeps them in the constant bank.
template <int N, typename T>
__device__ __forceinline__ T pick(const T (&a)[N], int i) {
  T r = a[0];
#pragma unroll
  for (int j = 1; j < N; ++j) r = (i == j) ? a[j] : r;
  return r;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
    const float2 x = __bfloat1622float2(b);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}

// Fused LSE combine (single-domain decode): the last CTA to finish a (row,
// head) merges that row's chunk partials (row_start) into the bf16 output.
struct FusedCombine {
  const int32_t* row_start = nullptr;  // null: partials only (combined elsewhere)
  int* counters = nullptr;             // [rows x heads], zero between launches
  bf16* out = nullptr;
};

template <int HD>
__device__ __forceinline__ void combine_row_head(const float* part_o, const float* part_ml,
                                                 int c0, int c1, int heads, int head, bf16* out) {
  float mm = -INFINITY;
  for (int c = c0; c < c1; ++c) mm = fmaxf(mm, __ldcg(&part_ml[(static_cast<int64_t>(c) * heads + head) * 2]));
  for (int d = threadIdx.x; d < HD; d += blockDim.x) {
    float acc = 0.f, ll = 0.f;
    for (int c = c0; c < c1; ++c) {
      const int64_t p = static_cast<int64_t>(c) * heads + head;
      const float mc = __ldcg(&part_ml[p * 2]);
      const float w = mc == -INFINITY ? 0.f : exp2f(mc - mm);
      acc += w * __ldcg(&part_o[p * HD + d]);
      ll += w * __ldcg(&part_ml[p * 2 + 1]);
    }
    out[d] = __float2bfloat16_rn(ll > 0.f ? acc / ll : 0.f);
  }
}

template <int HD, int UNR = kUnroll, int MINB = 1, int PF = 0, int W = kWarps>
__global__ void __launch_bounds__(W * 32, MINB)
    decode_attention_kernel(const bf16* __restrict__ q, const DecodeChunk* __restrict__ chunks,
                            const DecodeSlabs slabs, int heads, float scale_log2,
                            float* __restrict__ part_o, float* __restrict__ part_ml,
                            const FusedCombine fc, const PartDst dst) {
  constexpr int LPT = HD / 8;     // lanes per token
  constexpr int TPW = 32 / LPT;   // tokens per warp step
  // blockIdx.x = head (fastest): the CTAs resident at a time cover every head
  // of a few chunks, so each token's whole K/V row (all heads, contiguous) is
  // read at about the same time (DRAM page locality).
  ptx::griddep_wait();  // q and the appended K/V come from the QKV GEMM
  ptx::griddep_launch();
  const int head = blockIdx.x, ci = blockIdx.y;
  const DecodeChunk ch = chunks[ci];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPT;          // token group within the warp
  const int dl = lane % LPT;           // dim slice: dims [8*dl, 8*dl+8)
  const int hidden = heads * HD;

  float qf[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(q + static_cast<int64_t>(ch.row) * hidden +
                                                head * HD + dl * 8),
                qf);
#pragma unroll
  for (int e = 0; e < 8; ++e) qf[e] *= scale_log2;

  const bf16* kb = pick(slabs.k, ch.slab) + head * HD + dl * 8;
  const bf16* vb = pick(slabs.v, ch.slab) + head * HD + dl * 8;
  float m = -INFINITY, l = 0.f, o[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  const int step = W * TPW;
  // PF: the next iteration's slot ids are loaded one iteration ahead (no
  // index -> data dependency on the critical path) and, with PF == 2, their
  // K/V lines are prefetched into L2.
  int cur[UNR];
  if constexpr (PF > 0) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = warp * TPW + sub + u * step;
      cur[u] = t < ch.n ? __ldg(&ch.slots[t]) : -1;
    }
  }
  // The loop bound is warp-uniform (full-mask shuffles inside); lanes past
  // the end of the chunk just carry ok[u] = false.
  for (int tw = warp * TPW; tw < ch.n; tw += step * UNR) {
    uint4 kr[UNR], vr[UNR];
    bool ok[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int t = tw + sub + u * step;
      ok[u] = t < ch.n;
      if (ok[u]) {
        const int64_t off =
            static_cast<int64_t>(PF > 0 ? cur[u] : __ldg(&ch.slots[t])) * hidden;
        kr[u] = ld_nc_v4(kb + off);
        vr[u] = ld_nc_v4(vb + off);
      }
    }
    if constexpr (PF > 0) {
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int t = tw + step * UNR + sub + u * step;
        cur[u] = t < ch.n ? __ldg(&ch.slots[t]) : -1;
        if (PF > 1 && cur[u] >= 0) {
          const int64_t off = static_cast<int64_t>(cur[u]) * hidden;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(kb + off));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(vb + off));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      float kf[8];
      float s = 0.f;
      if (ok[u]) {
        bf16x8_to_f32(kr[u], kf);
#pragma unroll
        for (int e = 0; e < 8; ++e) s = fmaf(qf[e], kf[e], s);
      }
#pragma unroll
      for (int w = LPT / 2; w >= 1; w >>= 1) s += __shfl_xor_sync(0xffffffff, s, w);
      if (ok[u]) {
        const float m_new = fmaxf(m, s);
        const float corr = exp2f(m - m_new);
        const float p = exp2f(s - m_new);
        float vf[8];
        bf16x8_to_f32(vr[u], vf);
        l = l * corr + p;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = fmaf(o[e], corr, p * vf[e]);
        m = m_new;
      }
    }
  }
  // Merge the TPW token groups of the warp (lanes with equal dl).
#pragma unroll
  for (int w = LPT; w < 32; w <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffff, m, w);
    const float l2 = __shfl_xor_sync(0xffffffff, l, w);
    const float mm = fmaxf(m, m2);
    const float c1 = m == -INFINITY ? 0.f : exp2f(m - mm);
    const float c2 = m2 == -INFINITY ? 0.f : exp2f(m2 - mm);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float o2 = __shfl_xor_sync(0xffffffff, o[e], w);
      o[e] = o[e] * c1 + o2 * c2;
    }
    l = l * c1 + l2 * c2;
    m = mm;
  }
  // Merge warps through shared memory.
  __shared__ float sm_m[W], sm_l[W];
  __shared__ float sm_o[W][HD];
  if (sub == 0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) sm_o[warp][dl * 8 + e] = o[e];
    if (dl == 0) {
      sm_m[warp] = m;
      sm_l[warp] = l;
    }
  }
  __syncthreads();
  (void)ci;
  const int64_t pidx = static_cast<int64_t>(ch.out) * heads + head;
  if (dst.o[0] != nullptr) {  // fused partial gather: store to the master's buffers
    part_o = pick(dst.o, ch.dst);
    part_ml = pick(dst.ml, ch.dst);
  }
  for (int d = threadIdx.x; d < HD; d += blockDim.x) {
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < W; ++w) mm = fmaxf(mm, sm_m[w]);
    float acc = 0.f, ll = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const float c = sm_m[w] == -INFINITY ? 0.f : exp2f(sm_m[w] - mm);
      acc += c * sm_o[w][d];
      ll += c * sm_l[w];
    }
    part_o[pidx * HD + d] = acc;
    if (d == 0) {
      part_ml[pidx * 2] = mm;
      part_ml[pidx * 2 + 1] = ll;
    }
  }
  if (fc.row_start != nullptr) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    const int c0 = __ldg(&fc.row_start[ch.row]), c1 = __ldg(&fc.row_start[ch.row + 1]);
    int* cnt = &fc.counters[ch.row * heads + head];
    if (threadIdx.x == 0) last = atomicAdd(cnt, 1) == c1 - c0 - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      combine_row_head<HD>(part_o, part_ml, c0, c1, heads, head,
                           fc.out + static_cast<int64_t>(ch.row) * hidden + head * HD);
      if (threadIdx.x == 0) *cnt = 0;
    }
  }
}

// K3 v2: the same (chunk, head) decomposition with the K/V loads decoupled
// from the registers. The chunk's slot ids are staged in shared memory once
// (one coalesced read, no dependent index load per token), then every lane
// streams its own 16-byte K and V pieces through an NS-stage cp.async.cg ring
// in shared memory (L2 only, no L1 allocation). Each lane reads back exactly
// the bytes it copied, so a per-thread cp.async.wait_group is the only
// synchronisation; NS-1 stages (NS-1 x 16 KB per CTA) stay in flight while
// the current stage is reduced, independent of the register budget. U tokens
// per lane share one running-max update (one rescale exp per U tokens).
__device__ __forceinline__ void cp_async_cg16(void* smem, const void* gmem) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kV2MaxChunk = 1024;

template <int HD, int NS>
__global__ void __launch_bounds__(kWarps * 32)
    decode_attention_v2_kernel(const bf16* __restrict__ q, const DecodeChunk* __restrict__ chunks,
                               const DecodeSlabs slabs, int heads, float scale_log2,
                               float* __restrict__ part_o, float* __restrict__ part_ml) {
  constexpr int LPT = HD / 8;         // lanes per token
  constexpr int TPW = 32 / LPT;       // tokens per warp per load instruction
  constexpr int U = kUnroll;          // load instructions per lane per stage
  constexpr int TOK_W = TPW * U;      // tokens per warp per stage
  constexpr int TOK_S = TOK_W * kWarps;  // tokens per CTA per stage
  extern __shared__ uint4 ring[];     // [NS][warp][U][lane][K,V]
  __shared__ int32_t sidx[kV2MaxChunk];
  const int head = blockIdx.x;
  const DecodeChunk ch = chunks[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / LPT, dl = lane % LPT;
  const int hidden = heads * HD;
  for (int i = threadIdx.x; i < ch.n; i += blockDim.x) sidx[i] = __ldg(&ch.slots[i]);

  float qf[8];
  bf16x8_to_f32(*reinterpret_cast<const uint4*>(q + static_cast<int64_t>(ch.row) * hidden +
                                                head * HD + dl * 8),
                qf);
#pragma unroll
  for (int e = 0; e < 8; ++e) qf[e] *= scale_log2;
  const bf16* kb = pick(slabs.k, ch.slab) + head * HD + dl * 8;
  const bf16* vb = pick(slabs.v, ch.slab) + head * HD + dl * 8;
  __syncthreads();

  const int n_stages = (ch.n + TOK_S - 1) / TOK_S;
  auto issue = [&](int st) {
    if (st < n_stages) {
      uint4* buf = ring + ((st % NS) * kWarps + warp) * U * 64;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = st * TOK_S + warp * TOK_W + u * TPW + sub;
        if (t < ch.n) {
          const int64_t off = static_cast<int64_t>(sidx[t]) * hidden;
          cp_async_cg16(&buf[(u * 32 + lane) * 2], kb + off);
          cp_async_cg16(&buf[(u * 32 + lane) * 2 + 1], vb + off);
        }
      }
    }
    cp_async_commit();  // empty groups past the end keep the wait count uniform
  };
#pragma unroll
  for (int st = 0; st < NS - 1; ++st) issue(st);

  float m = -INFINITY, l = 0.f, o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int st = 0; st < n_stages; ++st) {
    issue(st + NS - 1);
    cp_async_wait<NS - 1>();
    const uint4* buf = ring + ((st % NS) * kWarps + warp) * U * 64;
    float sc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = st * TOK_S + warp * TOK_W + u * TPW + sub;
      float kf[8];
      bf16x8_to_f32(buf[(u * 32 + lane) * 2], kf);
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fmaf(qf[e], kf[e], s);
#pragma unroll
      for (int w = LPT / 2; w >= 1; w >>= 1) s += __shfl_xor_sync(0xffffffff, s, w);
      sc[u] = t < ch.n ? s : -INFINITY;
    }
    float mx = m;
#pragma unroll
    for (int u = 0; u < U; ++u) mx = fmaxf(mx, sc[u]);
    if (mx == -INFINITY) continue;  // nothing valid for this token group yet
    const float corr = exp2f(m - mx);
    l *= corr;
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] *= corr;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float p = exp2f(sc[u] - mx);
      if (sc[u] != -INFINITY) {
        float vf[8];
        bf16x8_to_f32(buf[(u * 32 + lane) * 2 + 1], vf);
        l += p;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = fmaf(p, vf[e], o[e]);
      }
    }
    m = mx;
  }
  cp_async_wait<0>();
#pragma unroll
  for (int w = LPT; w < 32; w <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffff, m, w);
    const float l2 = __shfl_xor_sync(0xffffffff, l, w);
    const float mm = fmaxf(m, m2);
    const float c1 = m == -INFINITY ? 0.f : exp2f(m - mm);
    const float c2 = m2 == -INFINITY ? 0.f : exp2f(m2 - mm);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float o2 = __shfl_xor_sync(0xffffffff, o[e], w);
      o[e] = o[e] * c1 + o2 * c2;
    }
    l = l * c1 + l2 * c2;
    m = mm;
  }
  __shared__ float sm_m[kWarps], sm_l[kWarps];
  __shared__ float sm_o[kWarps][HD];
  if (sub == 0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) sm_o[warp][dl * 8 + e] = o[e];
    if (dl == 0) {
      sm_m[warp] = m;
      sm_l[warp] = l;
    }
  }
  __syncthreads();
  const int64_t pidx = static_cast<int64_t>(ch.out) * heads + head;
  for (int d = threadIdx.x; d < HD; d += blockDim.x) {
    float mm = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mm = fmaxf(mm, sm_m[w]);
    float acc = 0.f, ll = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float c = sm_m[w] == -INFINITY ? 0.f : exp2f(sm_m[w] - mm);
      acc += c * sm_o[w][d];
      ll += c * sm_l[w];
    }
    part_o[pidx * HD + d] = acc;
    if (d == 0) {
      part_ml[pidx * 2] = mm;
      part_ml[pidx * 2 + 1] = ll;
    }
  }
}

template <int HD, int NS>
void launch_decode_v2(const dim3& grid, cudaStream_t s, const bf16* q, const DecodeChunk* chunks,
                      const DecodeSlabs& slabs, int heads, float sl2, float* part_o,
                      float* part_ml) {
  constexpr int smem = NS * kWarps * kUnroll * 64 * 16;
  once_per_device(reinterpret_cast<const void*>(decode_attention_v2_kernel<HD, NS>), [] {
    cudaFuncSetAttribute(decode_attention_v2_kernel<HD, NS>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  decode_attention_v2_kernel<HD, NS><<<grid, kWarps * 32, smem, s>>>(q, chunks, slabs, heads, sl2,
                                                                     part_o, part_ml);
}

__global__ void decode_combine_kernel(const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml,
                                      const int32_t* __restrict__ row_start,
                                      const int32_t* __restrict__ chunk_ids,
                                      const int32_t* __restrict__ rows, int heads, int hd,
                                      bf16* __restrict__ out) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  const int orow = blockIdx.x, head = blockIdx.y;
  const int row = rows ? rows[orow] : orow;
  const int c0 = row_start[row], c1 = row_start[row + 1];
  // Chunk weights in shared memory, computed in parallel (one thread per
  // chunk): w_c = e^{m_c - M}, L = sum_c w_c l_c. Then every thread sums its
  // dims over the chunks with independent loads.
  constexpr int kMaxC = 256;
  __shared__ float sw[kMaxC];
  __shared__ int64_t sp[kMaxC];
  __shared__ float red[2][32];
  const int nc = c1 - c0;
  float mloc = -INFINITY;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const int64_t p = static_cast<int64_t>(chunk_ids ? chunk_ids[c0 + c] : c0 + c) * heads + head;
    if (c < kMaxC) sp[c] = p;
    mloc = fmaxf(mloc, part_ml[p * 2]);
  }
  for (int w = 16; w >= 1; w >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffff, mloc, w));
  if ((threadIdx.x & 31) == 0) red[0][threadIdx.x >> 5] = mloc;
  __syncthreads();
  float mm = -INFINITY;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) mm = fmaxf(mm, red[0][i]);
  float lloc = 0.f;
  for (int c = threadIdx.x; c < nc; c += blockDim.x) {
    const int64_t p = c < kMaxC ? sp[c]
                                : static_cast<int64_t>(chunk_ids ? chunk_ids[c0 + c] : c0 + c) * heads + head;
    const float mc = part_ml[p * 2];
    const float wc = mc == -INFINITY ? 0.f : exp2f(mc - mm);
    if (c < kMaxC) sw[c] = wc;
    lloc += wc * part_ml[p * 2 + 1];
  }
  for (int w = 16; w >= 1; w >>= 1) lloc += __shfl_xor_sync(0xffffffff, lloc, w);
  if ((threadIdx.x & 31) == 0) red[1][threadIdx.x >> 5] = lloc;
  __syncthreads();
  float ll = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) ll += red[1][i];
  for (int d = threadIdx.x; d < hd; d += blockDim.x) {
    float acc = 0.f;
    int c = 0;
    for (; c + 4 <= nc && c + 4 <= kMaxC; c += 4) {
      const float o0 = part_o[sp[c] * hd + d], o1 = part_o[sp[c + 1] * hd + d];
      const float o2 = part_o[sp[c + 2] * hd + d], o3 = part_o[sp[c + 3] * hd + d];
      acc += sw[c] * o0 + sw[c + 1] * o1 + sw[c + 2] * o2 + sw[c + 3] * o3;
    }
    for (; c < nc; ++c) {
      const int64_t p = c < kMaxC ? sp[c]
                                  : static_cast<int64_t>(chunk_ids ? chunk_ids[c0 + c] : c0 + c) * heads + head;
      const float mc = part_ml[p * 2];
      const float wc = c < kMaxC ? sw[c] : (mc == -INFINITY ? 0.f : exp2f(mc - mm));
      acc += wc * part_o[p * hd + d];
    }
    out[static_cast<int64_t>(orow) * heads * hd + head * hd + d] =
        __float2bfloat16_rn(ll > 0.f ? acc / ll : 0.f);
  }
}

__global__ void retain_rows_kernel(const bf16* __restrict__ k, const bf16* __restrict__ v,
                                   const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ slab,
                                   const int32_t* __restrict__ slot, const DecodeSlabs dst,
                                   int hidden) {
  const int i = blockIdx.x;
  const int64_t so = static_cast<int64_t>(rows[i]) * hidden;
  const int64_t d = static_cast<int64_t>(slot[i]) * hidden;
  bf16* dk = const_cast<bf16*>(dst.k[slab[i]]) + d;
  bf16* dv = const_cast<bf16*>(dst.v[slab[i]]) + d;
  for (int c = threadIdx.x * 8; c < hidden; c += blockDim.x * 8) {
    *reinterpret_cast<uint4*>(dk + c) = *reinterpret_cast<const uint4*>(k + so + c);
    *reinterpret_cast<uint4*>(dv + c) = *reinterpret_cast<const uint4*>(v + so + c);
  }
}

// Contiguous K/V rows of a request gathered from its page slots (one layer):
// out_k/out_v[i] = slab_{slab[i]}[slot[i]] (the chunked-prefill attention's
// key/value rows).
__global__ void gather_rows_kernel(const DecodeSlabs src, const int32_t* __restrict__ slab,
                                   const int32_t* __restrict__ slot, bf16* __restrict__ out_k,
                                   bf16* __restrict__ out_v, int hidden) {
  const int i = blockIdx.x;
  const int64_t so = static_cast<int64_t>(slot[i]) * hidden;
  const int64_t d = static_cast<int64_t>(i) * hidden;
  const bf16* sk = src.k[slab[i]] + so;
  const bf16* sv = src.v[slab[i]] + so;
  for (int c = threadIdx.x * 8; c < hidden; c += blockDim.x * 8) {
    *reinterpret_cast<uint4*>(out_k + d + c) = *reinterpret_cast<const uint4*>(sk + c);
    *reinterpret_cast<uint4*>(out_v + d + c) = *reinterpret_cast<const uint4*>(sv + c);
  }
}

__global__ void copy_rows_kernel(const bf16* __restrict__ src, const int32_t* __restrict__ rows,
                                 bf16* __restrict__ dst, int hidden) {
  const int64_t so = static_cast<int64_t>(rows[blockIdx.x]) * hidden;
  const int64_t d = static_cast<int64_t>(blockIdx.x) * hidden;
  for (int c = threadIdx.x * 8; c < hidden; c += blockDim.x * 8) {
    *reinterpret_cast<uint4*>(dst + d + c) = *reinterpret_cast<const uint4*>(src + so + c);
  }
}

}  // namespace

void copy_rows(const bf16* src, const int32_t* rows, int n, bf16* dst, int hidden, cudaStream_t s) {
  if (n <= 0) return;
  copy_rows_kernel<<<n, 128, 0, s>>>(src, rows, dst, hidden);
  count_launch();
}

void gather_rows(const DecodeSlabs& src, const int32_t* slab, const int32_t* slot, int n,
                 bf16* out_k, bf16* out_v, int hidden, cudaStream_t s) {
  if (n <= 0) return;
  gather_rows_kernel<<<n, 128, 0, s>>>(src, slab, slot, out_k, out_v, hidden);
  count_launch();
}

void decode_attention(const bf16* q, const DecodeChunk* d_chunks, int n_chunks,
                      const DecodeSlabs& slabs, int heads, int head_dim, float scale,
                      float* part_o, float* part_ml, cudaStream_t s, const int32_t* row_start,
                      int* counters, bf16* out, int rows, const PartDst* dst) {
  if (n_chunks <= 0) return;
  const PartDst pd = dst ? *dst : PartDst{};
  FusedCombine fc;
  fc.row_start = row_start;
  fc.counters = counters;
  fc.out = out;
  if (n_chunks > 65535) throw std::runtime_error("decode_attention: more than 65535 chunks");
  const dim3 grid(heads, n_chunks);
  const float sl2 = scale * 1.4426950408889634f;
  // Default: the register-staged v1 at <= 64 registers (8 CTAs of 4 warps
  // per SM), 3 tokens per lane in flight and the next iteration's slot ids
  // loaded one iteration ahead: 6.81-6.85 TB/s on 16 x 8K (4 in flight
  // without the look-ahead: 6.44-6.47; tools/decode_probe.py sweeps). ESP_DECODE_ATTN=2: the
  // cp.async ring (v2) with ESP_DECODE_STAGES stages — slower on B200
  // (3.3-4.0 TB/s: its shared-memory ring caps resident CTAs per SM).
  const char* var = std::getenv("ESP_DECODE_ATTN");
  if (var != nullptr && std::atoi(var) == 2 && dst == nullptr) {
    const char* st = std::getenv("ESP_DECODE_STAGES");
    const int ns = st ? std::atoi(st) : 4;
    if (head_dim != 128 && head_dim != 64) {
      throw std::runtime_error("decode_attention: head_dim must be 64 or 128");
    }
#define ESP_V2(HD, NS) launch_decode_v2<HD, NS>(grid, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml)
    if (head_dim == 128) {
      if (ns <= 2) ESP_V2(128, 2); else if (ns == 3) ESP_V2(128, 3); else if (ns == 4) ESP_V2(128, 4); else ESP_V2(128, 6);
    } else {
      if (ns <= 2) ESP_V2(64, 2); else if (ns == 3) ESP_V2(64, 3); else if (ns == 4) ESP_V2(64, 4); else ESP_V2(64, 6);
    }
#undef ESP_V2
    count_launch();
    if (row_start != nullptr) decode_combine(part_o, part_ml, row_start, rows, heads, head_dim, out, s);
    return;
  }
  if (head_dim == 128) {
    // ESP_DECODE_V1=<unroll><min blocks per SM> tuning variants of v1
    const char* tv = std::getenv("ESP_DECODE_V1");
    const int tune = tv ? std::atoi(tv) : 0;
#define ESP_V1(U, B) launch_pdl(4, decode_attention_kernel<128, U, B>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd)
    switch (tune) {
      case 481: launch_pdl(4, decode_attention_kernel<128, 4, 8, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 482: launch_pdl(4, decode_attention_kernel<128, 4, 8, 2>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 381: launch_pdl(4, decode_attention_kernel<128, 3, 8, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 3101: launch_pdl(4, decode_attention_kernel<128, 3, 10, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 281: launch_pdl(4, decode_attention_kernel<128, 2, 8, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 2101: launch_pdl(4, decode_attention_kernel<128, 2, 10, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 2121: launch_pdl(4, decode_attention_kernel<128, 2, 12, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 361: launch_pdl(4, decode_attention_kernel<128, 3, 6, 1>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 3418: launch_pdl(4, decode_attention_kernel<128, 3, 4, 1, 8>, grid, dim3(8 * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 2418: launch_pdl(4, decode_attention_kernel<128, 2, 4, 1, 8>, grid, dim3(8 * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 31612: launch_pdl(4, decode_attention_kernel<128, 3, 16, 1, 2>, grid, dim3(2 * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 3518: launch_pdl(4, decode_attention_kernel<128, 3, 5, 1, 8>, grid, dim3(8 * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 282: launch_pdl(4, decode_attention_kernel<128, 2, 8, 2>, grid, dim3(kWarps * 32), 0, s, q, d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd); break;
      case 41: ESP_V1(4, 1); break;
      case 410: ESP_V1(4, 10); break;
      case 38: ESP_V1(3, 8); break;
      case 310: ESP_V1(3, 10); break;
      case 28: ESP_V1(2, 8); break;
      case 210: ESP_V1(2, 10); break;
      case 412: ESP_V1(4, 12); break;
      case 416: ESP_V1(4, 16); break;
      case 216: ESP_V1(2, 16); break;
      case 212: ESP_V1(2, 12); break;
      case 88: ESP_V1(8, 8); break;
      case 86: ESP_V1(8, 6); break;
      case 48: ESP_V1(4, 8); break;
      default:
        launch_pdl(4, decode_attention_kernel<128, 3, 8, 1>, grid, dim3(kWarps * 32), 0, s, q,
                   d_chunks, slabs, heads, sl2, part_o, part_ml, fc, pd);
    }
#undef ESP_V1
  } else if (head_dim == 64) {
    decode_attention_kernel<64, 3, 8, 1><<<grid, kWarps * 32, 0, s>>>(q, d_chunks, slabs, heads,
                                                                     sl2, part_o, part_ml, fc, pd);
  } else {
    throw std::runtime_error("decode_attention: head_dim must be 64 or 128");
  }
  count_launch();
}

void decode_combine(const float* part_o, const float* part_ml, const int32_t* row_start,
                    int rows, int heads, int head_dim, bf16* out, cudaStream_t s) {
  if (rows <= 0) return;
  launch_pdl(8, decode_combine_kernel, dim3(rows, heads), dim3(head_dim), 0, s, part_o, part_ml,
             row_start, static_cast<const int32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
             heads, head_dim, out);
  count_launch();
}

void decode_combine_rows(const float* part_o, const float* part_ml, const int32_t* row_start,
                         const int32_t* chunk_ids, const int32_t* rows, int n, int heads,
                         int head_dim, bf16* out, cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(8, decode_combine_kernel, dim3(n, heads), dim3(head_dim), 0, s, part_o, part_ml, row_start,
                                                            chunk_ids, rows, heads, head_dim, out);
  count_launch();
}

void retain_rows(const bf16* k, const bf16* v, const int32_t* rows, const int32_t* slab,
                 const int32_t* slot, int n, const DecodeSlabs& dst, int hidden, cudaStream_t s) {
  if (n <= 0) return;
  retain_rows_kernel<<<n, 128, 0, s>>>(k, v, rows, slab, slot, dst, hidden);
  count_launch();
}

}  // namespace esp::k
