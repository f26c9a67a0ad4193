// K6: small fused ops of the ESP data path (memory-bound, CUDA cores):
// embedding gather, RMSNorm (optionally gathering rows), greedy argmax, RoPE
// table, seeded synthetic weights, and the page-table / KV-slot utilities
// (device-side conservation recount, KV slot moves).
#include <atomic>
#include <algorithm>
#include <cfloat>
#include <stdexcept>
#include <type_traits>

#include "kernels.h"
#include "ptx.cuh"
#include "synthetic.h"

namespace esp::k {

namespace {
std::atomic<int64_t> g_launches{0};
}
int64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1); }
bool pdl_enabled(int cls) {
  static const int mask = [] {
    const char* e = std::getenv("ESP_PDL");
    // Default: GEMMs and norms (decode attention with PDL was
    // measured 0.7 ms/step slower on 16 x 8K: its early-resident CTAs).
    return e == nullptr ? 3 : std::atoi(e);
  }();
  return (mask & cls) != 0;
}

namespace {

__global__ void embed_kernel(const int32_t* __restrict__ tokens, const bf16* __restrict__ table,
                             bf16* __restrict__ x, int hidden, float* __restrict__ ss) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  const int r = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<int64_t>(tokens[r]) * hidden);
  uint4* dst = reinterpret_cast<uint4*>(x + static_cast<int64_t>(r) * hidden);
  float acc = 0.f;
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) {
    const uint4 v = src[i];
    dst[i] = v;
    if (ss) {
      const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(p[j]);
        acc += f.x * f.x + f.y * f.y;
      }
    }
  }
  if (ss) {  // the row's sum of squares, for the RMSNorm fused into the next GEMM
    __shared__ float red[32];
    for (int w = 16; w >= 1; w >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, w);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) t += red[i];
      ss[r] = t;
    }
  }
}

// W[r][c] *= gamma[c]: a layer RMSNorm's gain folded into the projection
// that consumes its output (x·diag(γ)·Wᵀ = x·(W·diag(γ))ᵀ).
__global__ void scale_cols_kernel(bf16* __restrict__ w, int64_t rows, int64_t cols,
                                  const bf16* __restrict__ gamma) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    w[i] = __float2bfloat16_rn(__bfloat162float(w[i]) * __bfloat162float(gamma[i % cols]));
  }
}

__global__ void rmsnorm_kernel(const bf16* __restrict__ x, const int32_t* __restrict__ src_rows,
                               const bf16* __restrict__ gamma, bf16* __restrict__ y, int hidden,
                               float eps) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  const int r = blockIdx.x;
  const int sr = src_rows ? src_rows[r] : r;
  const bf16* xr = x + static_cast<int64_t>(sr) * hidden;
  float ss = 0.f;
  for (int i = threadIdx.x * 8; i < hidden; i += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + i);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(p[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  __shared__ float red[32];
  for (int w = 16; w >= 1; w >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, w);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int w = 16; w >= 1; w >>= 1) t += __shfl_xor_sync(0xffffffff, t, w);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / static_cast<float>(hidden) + eps);
  bf16* yr = y + static_cast<int64_t>(r) * hidden;
  for (int i = threadIdx.x * 8; i < hidden; i += blockDim.x * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(xr + i);
    // gamma == null: unit gain (a layer norm whose gain is folded into the
    // following projection's weights)
    const uint4 g = gamma ? *reinterpret_cast<const uint4*>(gamma + i)
                          : make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
    const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&g);
    uint4 o;
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(p[j]);
      const float2 gg = __bfloat1622float2(gp[j]);
      op[j] = __floats2bfloat162_rn(f.x * inv * gg.x, f.y * inv * gg.y);
    }
    *reinterpret_cast<uint4*>(yr + i) = o;
  }
}

__global__ void argmax_kernel(const float* __restrict__ logits, int vocab, int32_t* __restrict__ out) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  const int r = blockIdx.x;
  const float* lr = logits + static_cast<int64_t>(r) * vocab;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < vocab; i += blockDim.x) {
    const float v = lr[i];
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  }
  for (int w = 16; w >= 1; w >>= 1) {
    const float b2 = __shfl_xor_sync(0xffffffff, best, w);
    const int i2 = __shfl_xor_sync(0xffffffff, bi, w);
    if (b2 > best || (b2 == best && i2 < bi)) {
      best = b2;
      bi = i2;
    }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) {
    sb[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x >> 5); ++w) {
      if (sb[w] > best || (sb[w] == best && si[w] < bi)) {
        best = sb[w];
        bi = si[w];
      }
    }
    out[r] = bi;
  }
}

__global__ void rope_table_kernel(float2* table, int max_pos, int half, float theta, int hd) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(max_pos) * half) return;
  const int p = static_cast<int>(i / half), j = static_cast<int>(i % half);
  const float inv_freq = powf(theta, -static_cast<float>(2 * j) / static_cast<float>(hd));
  const float ang = static_cast<float>(p) * inv_freq;
  float s, c;
  sincosf(ang, &s, &c);
  table[i] = make_float2(c, s);
}

// layout 0: plain [rows x cols]; 1: fused QKV [3*cols x cols] (q|k|v rows);
// 2: gate_up [rows x cols] in 128-row blocks of 64 gate + 64 up rows.
// A tensor-parallel shard is a window of the logical tensor: destination
// row pr / col c is logical row row_off + pr (layout 1: region pr / part,
// row row_off + pr % part; layout 2: physical row row_off + pr of the
// interleaved layout) and logical col col_off + c of cols_total.
__global__ void init_weight_kernel(bf16* dst, int64_t rows, int64_t cols, uint64_t seed,
                                   int tensor, int layer, int layout, int64_t part,
                                   int64_t row_off, int64_t col_off, int64_t cols_total) {
  const int64_t n = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pr = i / cols, c = i % cols;
    int t = tensor;
    int64_t lr = row_off + pr;
    if (layout == 1) {
      t = tensor + static_cast<int>(pr / part);  // Q, K, V ids are consecutive
      lr = row_off + pr % part;
    } else if (layout == 2) {
      const int64_t g = row_off + pr, blk = g / 128, w = g % 128;
      t = w < 64 ? kTensorGate : kTensorUp;
      lr = blk * 64 + (w % 64);
    }
    dst[i] = __float2bfloat16_rn(synthetic_weight(seed, t, layer, lr, col_off + c, cols_total));
  }
}

__global__ void fill_kernel(bf16* dst, int64_t n, float v) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    dst[i] = __float2bfloat16_rn(v);
  }
}

__global__ void count_slots_kernel(const int32_t* slots, int64_t n, int32_t* counts, int cap) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = slots[i];
    if (s >= 0 && s < cap) atomicAdd(&counts[s], 1);
    else atomicAdd(&counts[cap], 1);  // out-of-range sentinel
  }
}

// result[0] = number of slots assigned (count > 0), result[1] = slots assigned
// more than once + out-of-range entries.
__global__ void check_counts_kernel(const int32_t* counts, int cap, int32_t* result) {
  int used = 0, bad = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
    used += counts[i] > 0;
    bad += counts[i] > 1;
  }
  for (int w = 16; w >= 1; w >>= 1) {
    used += __shfl_xor_sync(0xffffffff, used, w);
    bad += __shfl_xor_sync(0xffffffff, bad, w);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&result[0], used);
    atomicAdd(&result[1], bad);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&result[1], counts[cap]);
}

__global__ void copy_slots_kernel(const bf16* __restrict__ sk, const bf16* __restrict__ sv,
                                  const int32_t* __restrict__ ss, bf16* __restrict__ dk,
                                  bf16* __restrict__ dv, const int32_t* __restrict__ ds,
                                  int layers, int64_t sstride, int64_t dstride, int hidden) {
  const int t = blockIdx.x, layer = blockIdx.y;
  const int64_t so = static_cast<int64_t>(layer) * sstride + static_cast<int64_t>(ss[t]) * hidden;
  const int64_t dof = static_cast<int64_t>(layer) * dstride + static_cast<int64_t>(ds[t]) * hidden;
  const uint4* a = reinterpret_cast<const uint4*>(sk + so);
  const uint4* b = reinterpret_cast<const uint4*>(sv + so);
  uint4* c = reinterpret_cast<uint4*>(dk + dof);
  uint4* d = reinterpret_cast<uint4*>(dv + dof);
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) {
    c[i] = a[i];
    d[i] = b[i];
  }
}

}  // namespace

void embed(const int32_t* tokens, const bf16* table, bf16* x, int rows, int hidden,
           cudaStream_t s, float* ss) {
  if (rows <= 0) return;
  launch_pdl(2, embed_kernel, dim3(rows), dim3(128), 0, s, tokens, table, x, hidden, ss);
  count_launch();
}

void rmsnorm(const bf16* x, const int32_t* src_rows, const bf16* gamma, bf16* y, int rows,
             int hidden, float eps, cudaStream_t s) {
  if (rows <= 0) return;
  const int threads = hidden >= 2048 ? 256 : 64;
  launch_pdl(2, rmsnorm_kernel, dim3(rows), dim3(threads), 0, s, x, src_rows, gamma, y, hidden, eps);
  count_launch();
}

void argmax_rows(const float* logits, int rows, int vocab, int32_t* out, cudaStream_t s) {
  if (rows <= 0) return;
  launch_pdl(2, argmax_kernel, dim3(rows), dim3(1024), 0, s, logits, vocab, out);
  count_launch();
}

void rope_table(float2* table, int max_pos, int head_dim, float theta, cudaStream_t s) {
  const int half = head_dim / 2;
  const int64_t n = static_cast<int64_t>(max_pos) * half;
  rope_table_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(table, max_pos, half,
                                                                           theta, head_dim);
  count_launch();
}

void init_weight(bf16* dst, int64_t rows, int64_t cols, uint64_t seed, int tensor, int layer,
                 int layout, cudaStream_t s) {
  init_weight_kernel<<<4096, 256, 0, s>>>(dst, rows, cols, seed, tensor, layer, layout, cols, 0,
                                          0, cols);
  count_launch();
}

void init_weight_shard(bf16* dst, int64_t rows, int64_t cols, uint64_t seed, int tensor,
                       int layer, int layout, int64_t part, int64_t row_off, int64_t col_off,
                       int64_t cols_total, cudaStream_t s) {
  init_weight_kernel<<<4096, 256, 0, s>>>(dst, rows, cols, seed, tensor, layer, layout, part,
                                          row_off, col_off, cols_total);
  count_launch();
}

// Tensor-parallel all-reduce of a row-parallel projection (O, down), fused
// with the residual and the next layer norm (unit gain: gains are folded into
// the consuming projections): x += the planes' fp32 partials summed in plane
// order (every plane computes the same bits; the other planes' partials are
// read over NVLink) — or, as the second half of a reduce-scatter, one row
// block whose partials the GEMM epilogues already stored here, x and xn then
// stored to every plane that needs them (the all-gather); one CTA per row, the row's new
// residual kept in registers, xn = x_new * rsqrt(mean(x_new^2) + eps) exactly
// as rmsnorm_kernel computes it from the stored bf16 x.
struct TpOuts {
  bf16* p[kMaxTp];
  int n;
};

template <int kPer, int kNP>  // 8-column groups per thread, partials (planes)
__global__ void tp_reduce_norm_kernel(const bf16* x, TpParts parts, TpOuts x_out, TpOuts xn_out,
                                      int hidden, float eps) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * hidden;
  // every load of the row slice issued before the first add (kPer x kNP x 32 B
  // of partials + kPer x 16 B of x in flight per thread)
  float4 pa[kPer][kNP][2];
  uint4 xs[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int c = (threadIdx.x + u * blockDim.x) * 8;
    if (c < hidden) {
#pragma unroll
      for (int q = 0; q < kNP; ++q) {
        const float4* pp = reinterpret_cast<const float4*>(parts.p[q] + base + c);
        pa[u][q][0] = pp[0];
        pa[u][q][1] = pp[1];
      }
      xs[u] = *reinterpret_cast<const uint4*>(x + base + c);
    }
  }
  uint4 keep[kPer];
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int c = (threadIdx.x + u * blockDim.x) * 8;
    if (c >= hidden) break;
    // the planes' partials in plane order, then the residual
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < kNP; ++q) {
      const float4 a = pa[u][q][0], b = pa[u][q][1];
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
    }
    const uint4 xv = xs[u];
    const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(xp[j]);
      acc[2 * j] = f.x + acc[2 * j];
      acc[2 * j + 1] = f.y + acc[2 * j + 1];
    }
    uint4 o;
    o.x = ptx::pack_bf16(acc[0], acc[1]);
    o.y = ptx::pack_bf16(acc[2], acc[3]);
    o.z = ptx::pack_bf16(acc[4], acc[5]);
    o.w = ptx::pack_bf16(acc[6], acc[7]);
#pragma unroll
    for (int q = 0; q < kMaxTp; ++q) {  // unrolled: the pointer table stays in the param bank
      if (q < x_out.n) *reinterpret_cast<uint4*>(x_out.p[q] + base + c) = o;
    }
    keep[u] = o;
    const __nv_bfloat162* op = reinterpret_cast<const __nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(op[j]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  __shared__ float red[32];
  for (int w = 16; w >= 1; w >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, w);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int w = 16; w >= 1; w >>= 1) t += __shfl_xor_sync(0xffffffff, t, w);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(red[0] / static_cast<float>(hidden) + eps);
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int c = (threadIdx.x + u * blockDim.x) * 8;
    if (c >= hidden) break;
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&keep[u]);
    uint4 o;
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(p[j]);
      op[j] = __floats2bfloat162_rn(f.x * inv, f.y * inv);
    }
#pragma unroll
    for (int q = 0; q < kMaxTp; ++q) {
      if (q < xn_out.n) *reinterpret_cast<uint4*>(xn_out.p[q] + base + c) = o;
    }
  }
}

void tp_reduce_residual_norm(const bf16* x, const TpParts& parts, bf16* const* x_out, int n_x,
                             bf16* const* xn_out, int n_xn, int rows, int hidden, float eps,
                             cudaStream_t s) {
  if (rows <= 0) return;
  if (hidden % 8 != 0 || hidden > 256 * 8 * 4) {
    throw std::runtime_error("tp_reduce_residual_norm: hidden % 8 or > 8192");
  }
  if (n_x < 1 || n_x > kMaxTp || n_xn < 1 || n_xn > kMaxTp) {
    throw std::runtime_error("tp_reduce_residual_norm: 1..8 outputs");
  }
  TpOuts xo{}, xno{};
  for (int q = 0; q < n_x; ++q) xo.p[q] = x_out[q];
  for (int q = 0; q < n_xn; ++q) xno.p[q] = xn_out[q];
  xo.n = n_x;
  xno.n = n_xn;
  auto go = [&](auto kern) {
    launch_pdl(2, kern, dim3(rows), dim3(256), 0, s, x, parts, xo, xno, hidden, eps);
  };
  const int per = (hidden + 2047) / 2048;  // 8-column groups per thread at 256 threads
  auto by_np = [&](auto per_c) {
    constexpr int P = decltype(per_c)::value;
    switch (parts.n) {
      case 1: go(tp_reduce_norm_kernel<P, 1>); break;
      case 2: go(tp_reduce_norm_kernel<P, 2>); break;
      case 3: go(tp_reduce_norm_kernel<P, 3>); break;
      case 4: go(tp_reduce_norm_kernel<P, 4>); break;
      case 5: go(tp_reduce_norm_kernel<P, 5>); break;
      case 6: go(tp_reduce_norm_kernel<P, 6>); break;
      case 7: go(tp_reduce_norm_kernel<P, 7>); break;
      case 8: go(tp_reduce_norm_kernel<P, 8>); break;
      default: throw std::runtime_error("tp_reduce_residual_norm: 1..8 partials");
    }
  };
  if (per <= 1) by_np(std::integral_constant<int, 1>{});
  else if (per == 2) by_np(std::integral_constant<int, 2>{});
  else by_np(std::integral_constant<int, 4>{});
  count_launch();
}


void scale_cols(bf16* w, int64_t rows, int64_t cols, const bf16* gamma, cudaStream_t s) {
  scale_cols_kernel<<<2048, 256, 0, s>>>(w, rows, cols, gamma);
  count_launch();
}

void fill_bf16(bf16* dst, int64_t n, float v, cudaStream_t s) {
  fill_kernel<<<1024, 256, 0, s>>>(dst, n, v);
  count_launch();
}

void count_slots(const int32_t* slots, int64_t n, int32_t* counts, int capacity,
                 cudaStream_t s) {
  if (n <= 0) return;
  count_slots_kernel<<<256, 256, 0, s>>>(slots, n, counts, capacity);
  count_launch();
}

void check_counts(const int32_t* counts, int capacity, int32_t* result, cudaStream_t s) {
  check_counts_kernel<<<256, 256, 0, s>>>(counts, capacity, result);
  count_launch();
}

void copy_slots(const bf16* src_k, const bf16* src_v, const int32_t* src_slots, bf16* dst_k,
                bf16* dst_v, const int32_t* dst_slots, int n, int layers,
                int64_t src_layer_stride, int64_t dst_layer_stride, int hidden, cudaStream_t s) {
  if (n <= 0) return;
  copy_slots_kernel<<<dim3(n, layers), 128, 0, s>>>(src_k, src_v, src_slots, dst_k, dst_v,
                                                    dst_slots, layers, src_layer_stride,
                                                    dst_layer_stride, hidden);
  count_launch();
}

}  // namespace esp::k
