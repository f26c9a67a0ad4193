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
#include <stdexcept>
#include <type_traits>

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

template <int HD, int UNR = kUnroll, int MINB = 1, int PF = 0, int W = kWarps>
__global__ void __launch_bounds__(W * 32, MINB)
    decode_attention_kernel(const bf16* __restrict__ q, const DecodeChunk* __restrict__ chunks,
                            const DecodeSlabs slabs, int heads, float scale_log2,
                            float* __restrict__ part_o, float* __restrict__ part_ml,
                            const PartDst dst, bf16* __restrict__ direct_out) {
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
  if (direct_out != nullptr) {  // the row's only chunk: normalise here, no combine
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
      direct_out[static_cast<int64_t>(ch.row) * hidden + head * HD + d] =
          __float2bfloat16_rn(ll > 0.f ? acc / ll : 0.f);
    }
    return;
  }
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
}

// OutT = bf16 (the data path) or float (the fp32 check mode of the hook).
template <typename OutT>
__global__ void decode_combine_kernel(const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml,
                                      const int32_t* __restrict__ row_start,
                                      const int32_t* __restrict__ chunk_ids,
                                      const int32_t* __restrict__ rows, int heads, int hd,
                                      OutT* __restrict__ out) {
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
    const float r = ll > 0.f ? acc / ll : 0.f;
    if constexpr (std::is_same_v<OutT, float>) {
      out[static_cast<int64_t>(orow) * heads * hd + head * hd + d] = r;
    } else {
      out[static_cast<int64_t>(orow) * heads * hd + head * hd + d] = __float2bfloat16_rn(r);
    }
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
                      float* part_o, float* part_ml, cudaStream_t s, const PartDst* dst,
                      bf16* direct_out, int max_chunk) {
  if (n_chunks <= 0) return;
  const PartDst pd = dst ? *dst : PartDst{};
  if (n_chunks > 65535) throw std::runtime_error("decode_attention: more than 65535 chunks");
  const dim3 grid(heads, n_chunks);
  const float sl2 = scale * 1.4426950408889634f;
  // Register-staged loads at <= 64 registers (8 CTAs of 4 warps per SM), 3
  // tokens per lane in flight and the next iteration's slot ids loaded one
  // iteration ahead: 6.81-6.85 TB/s on 16 x 8K (4 in flight without the
  // look-ahead: 6.44-6.47). Measured and dropped (round 1): a cp.async
  // shared-memory ring (3.3-4.0 TB/s — its ring caps resident CTAs per SM)
  // and the LSE combine fused into the last CTA of each (row, head) (0.1-0.3
  // ms/step slower: the fence + counter extend every CTA).
  // Latency-bound launches (the whole grid fits in one wave of 4 CTAs per
  // SM, e.g. b = 16 requests at contexts <= 512 tokens: 512 CTAs): 8 warps x
  // 2 tokens x 4 unrolled = 64 tokens' K/V loads in flight per CTA per
  // iteration (24 in the default kernel). Measured LWM-7B decode steps:
  // b = 16 at 64-token contexts 3.18 -> 3.13 ms, 200: 3.46 -> 3.33, 400:
  // 3.93 -> 3.59; b = 1 at 8K 4.6-4.8 -> 4.25-4.29; b = 4 at 2K 4.23 -> 4.27
  // (even); at b = 16 x 8K (8192 CTAs, throughput-bound) the default
  // kernel's 8 CTAs per SM with the slot-id look-ahead win (13.9-14.2 vs 15.0).
  static const int n_sm = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    }
    return v;
  }();
  const bool one_wave = static_cast<int64_t>(heads) * n_chunks <= 4LL * n_sm;
  if (max_chunk > 0 && one_wave && (head_dim == 128 || head_dim == 64)) {
    if (head_dim == 128) {
      launch_pdl(4, decode_attention_kernel<128, 4, 4, 0, 8>, grid, dim3(8 * 32), 0, s, q,
                 d_chunks, slabs, heads, sl2, part_o, part_ml, pd, direct_out);
    } else {
      launch_pdl(4, decode_attention_kernel<64, 2, 4, 0, 8>, grid, dim3(8 * 32), 0, s, q,
                 d_chunks, slabs, heads, sl2, part_o, part_ml, pd, direct_out);
    }
  } else if (head_dim == 128) {
    launch_pdl(4, decode_attention_kernel<128, 3, 8, 1>, grid, dim3(kWarps * 32), 0, s, q,
               d_chunks, slabs, heads, sl2, part_o, part_ml, pd, direct_out);
  } else if (head_dim == 64) {
    launch_pdl(4, decode_attention_kernel<64, 3, 8, 1>, grid, dim3(kWarps * 32), 0, s, q,
               d_chunks, slabs, heads, sl2, part_o, part_ml, pd, direct_out);
  } else {
    throw std::runtime_error("decode_attention: head_dim must be 64 or 128");
  }
  count_launch();
}

void decode_combine(const float* part_o, const float* part_ml, const int32_t* row_start,
                    int rows, int heads, int head_dim, bf16* out, cudaStream_t s) {
  if (rows <= 0) return;
  launch_pdl(8, decode_combine_kernel<bf16>, dim3(rows, heads), dim3(head_dim), 0, s, part_o,
             part_ml, row_start, static_cast<const int32_t*>(nullptr),
             static_cast<const int32_t*>(nullptr), heads, head_dim, out);
  count_launch();
}

void decode_combine_f32(const float* part_o, const float* part_ml, const int32_t* row_start,
                        int rows, int heads, int head_dim, float* out, cudaStream_t s) {
  if (rows <= 0) return;
  decode_combine_kernel<float><<<dim3(rows, heads), dim3(head_dim), 0, s>>>(
      part_o, part_ml, row_start, nullptr, nullptr, heads, head_dim, out);
  count_launch();
}

void decode_combine_rows(const float* part_o, const float* part_ml, const int32_t* row_start,
                         const int32_t* chunk_ids, const int32_t* rows, int n, int heads,
                         int head_dim, bf16* out, cudaStream_t s) {
  if (n <= 0) return;
  launch_pdl(8, decode_combine_kernel<bf16>, dim3(n, heads), dim3(head_dim), 0, s, part_o, part_ml, row_start,
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
