// Host-side launchers of the sm_100a kernels of the ESP data path.
#pragma once

#include <cstdlib>

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

namespace esp::k {

using bf16 = __nv_bfloat16;

constexpr int kMaxSlabs = 16;  // instances co-located on one device
constexpr int kMaxPeers = 7;   // other transport domains of one ESP ring
constexpr int kMaxTp = 8;      // tensor-parallel planes of one instance

enum EpiKind : int {
  kEpiStore = 0,     // D = acc (bf16)
  kEpiResidual = 1,  // D += acc (bf16 in place): O-proj / down-proj + residual
  kEpiStoreF32 = 2,  // D = acc (fp32): LM-head logits
  kEpiSiluMul = 3,   // gate/up interleaved in 64-row blocks -> silu(g)*u (bf16)
  kEpiQkvRope = 4,   // q,k,v split + RoPE + ring stripe write + page retention
  kEpiAtomicF32 = 5, // D += acc (fp32 atomics): split-K partial sums (internal)
};

struct GemmEpilogue {
  int kind = kEpiStore;
  void* out = nullptr;  // store / residual / f32 / silu output
  int ldo = 0;          // elements
  // kEpiQkvRope ----------------------------------------------------------
  bf16* q_out = nullptr;  // [M x hidden]
  bf16* k_out = nullptr;  // [M x hidden] ring stripe buffer, nullable
  bf16* v_out = nullptr;
  const int32_t* pos = nullptr;   // [M] token position
  const float2* rope = nullptr;   // [max_pos x head_dim/2] (cos, sin)
  int hidden = 0, head_dim = 0;
  const int32_t* row_inst = nullptr;  // [M] slab index of the resting page, -1 none
  const int32_t* row_slot = nullptr;  // [M] slot within that slab
  const int32_t* kv_rows = nullptr;   // [M] row of k_out/v_out for GEMM row m (null: m)
  bf16* slab_k[kMaxSlabs] = {};       // per co-located instance, this layer's base
  bf16* slab_v[kMaxSlabs] = {};
  // Fused ring transport (ESP prefill across transport domains): every K/V
  // row is also stored, at the same row, into each peer domain's gather
  // buffer (peer / NVLink stores from the epilogue) — the all-gather of the
  // ring's K/V blocks happens inside the QKV GEMM.
  int n_peer = 0;
  bf16* k_peer[kMaxPeers] = {};
  bf16* v_peer[kMaxPeers] = {};
  // Arrival counters of that transport: after a CTA stored a K or V tile to
  // the peers, one system-scope atomic per peer adds rows x columns to
  // arrive[p] (the peer's counter slot of this source domain); the peer's
  // ring-attention producer waits for the layer's running total before it
  // loads this source's blocks (RingWait) — no host or stream round trip.
  int n_arrive = 0;
  unsigned long long* arrive[kMaxPeers] = {};
  // Multi-master decode across domains: q rows go to row q_rows[m] of q_out
  // and of every q_peer (the query broadcast fused into the QKV epilogue).
  const int32_t* q_rows = nullptr;
  int n_qpeer = 0;
  bf16* q_peer[kMaxPeers] = {};
  // RMSNorm fused across decode GEMMs (skinny swap kernel only): a residual
  // epilogue adds each stored row's sum of squares into ss_out[m]; a
  // consumer GEMM (A = the un-normalised x, norm gain folded into its
  // weights) scales row m of its accumulator by rsqrt(ss_in[m]/norm_dim +
  // norm_eps); ss_zero[0..31] is cleared by the kernel (the buffer the next
  // residual GEMM accumulates into — its readers have completed).
  float* ss_out = nullptr;
  const float* ss_in = nullptr;
  float* ss_zero = nullptr;
  int norm_dim = 0;
  float norm_eps = 0.f;
  // Reduce-scatter fused into the fp32 store (tensor-parallel planes): with
  // route_rows > 0, row m of a kEpiStoreF32 tile goes to route[m /
  // route_rows] + (m % route_rows) * ldo — row block q lands, by peer store
  // from the epilogue, in plane q's receive buffer while the GEMM runs.
  int route_rows = 0;
  float* route[kMaxTp] = {};
};

// Schedule selection: kGemmAuto is the production dispatch; the others
// force one path on shapes that would not pick it (kernel tests, via the
// esp_k_gemm hook): the 1-CTA prefill kernel instead of the CTA pair, whole
// skinny tiles only, or skinny stream-K for every shape.
enum GemmPath : int { kGemmAuto = 0, kGemmNoPair = 1, kGemmTilesOnly = 2, kGemmStreamKAll = 3 };

// D[M x N] = A[M x K] . B[N x K]^T with the epilogue above. A and B are
// row-major bf16 (both K-major). N % 128 == 0, K % 64 == 0, any M.
void gemm(const bf16* A, int lda, const bf16* B, int ldb, int M, int N, int K,
          const GemmEpilogue& ep, cudaStream_t s, int path = kGemmAuto);

// ---- attention ------------------------------------------------------------
constexpr int kMaxRounds = 16;  // ESP degree of one ring (the reference tests d <= 16)

// One (ring position, request) segment of striped ring attention: the local
// query stripe rows [q_row0, q_row0+q_len) meet, in round r, the KV stripe
// rows [kv_row0[r], +kv_len[r]) that started at ring position origin[r].
// Key b (stripe index) is visible to query a iff b < a, or b == a and
// origin <= pos_i (striped causal mask; shift[r] = origin > pos_i).
struct RingSegment {
  int32_t q_row0, q_len;
  int32_t n_rounds;
  int32_t kv_row0[kMaxRounds];
  int32_t kv_len[kMaxRounds];
  int32_t shift[kMaxRounds];
  // 0: round r's block is already resident; s + 1: it is stored by source
  // domain s over NVLink and the producer waits on RingWait slot s first.
  int32_t wait_src[kMaxRounds];
};

// Arrival waits of one ring-attention launch (cross-GPU push transport):
// ctr[s] is this domain's counter of the K/V bytes-units source domain s has
// stored into its gather buffer (GemmEpilogue.arrive), target[s] the running
// total that completes the blocks this launch reads.
constexpr int kMaxWaitSrc = 16;
struct RingWait {
  const unsigned long long* ctr = nullptr;
  unsigned long long target[kMaxWaitSrc] = {};
};

// Online-softmax state carried between ring-attention launches (the
// windowed ring: one launch per round over an O(S/d) block window). o is
// [q_rows x heads*head_dim] fp32, the unnormalised output; ml is [q_rows x
// heads] float2 (running max in log2 units, running sum). A launch with a
// carry writes o/ml instead of the bf16 output; carry_in makes it start
// from them; ring_attention_finalize writes out = o / l.
struct RingCarry {
  float* o = nullptr;
  float2* ml = nullptr;
  int carry_in = 0;
};

// K1: striped ring attention over segments; q/out are [q_rows x
// heads*head_dim] and k/v [kv_rows x heads*head_dim] bf16 (segments index
// rows of each). Persistent tcgen05 kernel, two 128-row query tiles per CTA
// (P kept in TMEM); work items are (segment, query-tile PAIR, head) in the
// order build_attention_work lays them out.
void ring_attention(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows,
                    int kv_rows, int heads, int head_dim, const RingSegment* d_segs,
                    const int32_t* d_work, int n_work, float scale, cudaStream_t s,
                    const RingWait* wait = nullptr, const RingCarry* carry = nullptr);
// out[r, :] = o[r, :] / l (bf16) for rows [0, rows) of a carry.
void ring_attention_finalize(const RingCarry& carry, bf16* out, int rows, int heads,
                             int head_dim, cudaStream_t s);

#ifdef ESP_STUDY
// Kernel-study build only (tools/attn_prof.py, `make STUDY=1`): K1 with
// clock64 accounting per role (producer, MMA, 2 softmax warp groups) x 8
// counters into prof[grid x 4 x 8].
void ring_attention_profiled(const bf16* q, const bf16* k, const bf16* v, bf16* out, int q_rows,
                             int kv_rows, int heads, int head_dim, const RingSegment* d_segs,
                             const int32_t* d_work, int n_work, float scale, cudaStream_t s,
                             uint64_t* prof);
#endif

// Work-list builder helper: number of 128-row q tiles of a segment.
inline int q_tiles(int q_len) { return (q_len + 127) / 128; }

// ---- decode ---------------------------------------------------------------
// One chunk of one request's KV on one instance: slots slot_idx[0..n).
struct DecodeChunk {
  const int32_t* slots;
  int32_t n;
  int32_t row;   // request row in the decode batch (row of q)
  int32_t slab;  // index into the slab pointer arrays
  int32_t out;   // index of this chunk's partial in part_o / part_ml
  int32_t dst;   // PartDst entry the partial is stored to (fused gather), else 0
};
// Where split-KV partials go: with o[0] == null the launch's own part_o /
// part_ml; otherwise chunk c's partial is stored to o[c.dst] / ml[c.dst] —
// the master domain's buffers, by peer stores over NVLink (the partial
// gather of multi-master decoding fused into the attention kernel).
constexpr int kMaxPartDst = 8;
struct PartDst {
  float* o[kMaxPartDst] = {};
  float* ml[kMaxPartDst] = {};
};
struct DecodeSlabs {
  const bf16* k[kMaxSlabs];
  const bf16* v[kMaxSlabs];
};
// Split-KV paged attention: partial (o, m, l) per (chunk, head) into
// part_o [n_chunks x heads x head_dim] fp32 and part_ml [n_chunks x heads x 2]
// (or, with dst, into the master domains' buffers by peer stores).
// direct_out: every row has exactly one chunk (short contexts on one
// instance), so each CTA's partial IS the row's attention: it is normalised
// and stored as bf16 [rows x heads*head_dim] and no combine is needed.
// max_chunk: the longest chunk in tokens when the caller knows it (0 =
// unknown: the default kernel); a grid that fits in one wave then takes an
// 8-warp CTA with 64 tokens' K/V loads in flight per iteration.
void decode_attention(const bf16* q, const DecodeChunk* d_chunks, int n_chunks,
                      const DecodeSlabs& slabs, int heads, int head_dim, float scale,
                      float* part_o, float* part_ml, cudaStream_t s,
                      const PartDst* dst = nullptr, bf16* direct_out = nullptr,
                      int max_chunk = 0);
// LSE combine of the partials of each row (chunks row_start[r]..row_start[r+1]).
void decode_combine(const float* part_o, const float* part_ml, const int32_t* row_start,
                    int rows, int heads, int head_dim, bf16* out, cudaStream_t s);
// The same with fp32 output (the fp32 check mode of the decode-attention hook).
void decode_combine_f32(const float* part_o, const float* part_ml, const int32_t* row_start,
                        int rows, int heads, int head_dim, float* out, cudaStream_t s);
// Same, for a subset of rows: out row i combines global row rows[i], whose
// partials are chunk_ids[row_start[g] .. row_start[g+1]).
void decode_combine_rows(const float* part_o, const float* part_ml, const int32_t* row_start,
                         const int32_t* chunk_ids, const int32_t* rows, int n, int heads,
                         int head_dim, bf16* out, cudaStream_t s);

// Proactive retention on pass: copies K/V rows of a ring block that arrived
// from another device into their resting page slots (one layer).
void retain_rows(const bf16* k, const bf16* v, const int32_t* rows, const int32_t* slab,
                 const int32_t* slot, int n, const DecodeSlabs& dst, int hidden, cudaStream_t s);
// out_k/out_v[i] = K/V row of page slot (slab[i], slot[i]) — one layer.
void gather_rows(const DecodeSlabs& src, const int32_t* slab, const int32_t* slot, int n,
                 bf16* out_k, bf16* out_v, int hidden, cudaStream_t s);

// dst[i] = src[rows[i]] (bf16 rows of `hidden`; parity captures).
void copy_rows(const bf16* src, const int32_t* rows, int n, bf16* dst, int hidden, cudaStream_t s);

// ---- small fused ops --------------------------------------------------------
// ss != null: also stores each row's sum of squares (fused-RMSNorm input).
void embed(const int32_t* tokens, const bf16* table, bf16* x, int rows, int hidden,
           cudaStream_t s, float* ss = nullptr);
// y[r] = rmsnorm(x[src_row[r] or r]) * gamma
void rmsnorm(const bf16* x, const int32_t* src_rows, const bf16* gamma, bf16* y, int rows,
             int hidden, float eps, cudaStream_t s);
void argmax_rows(const float* logits, int rows, int vocab, int32_t* out, cudaStream_t s);
void rope_table(float2* table, int max_pos, int head_dim, float theta, cudaStream_t s);
void init_weight(bf16* dst, int64_t rows, int64_t cols, uint64_t seed, int tensor, int layer,
                 int layout, cudaStream_t s);
// A window of a synthetic tensor (tensor-parallel weight shard): logical rows
// row_off.. (layout 1: q|k|v regions of `part` rows each), cols col_off.. of
// cols_total (misc.cu:init_weight_kernel).
void init_weight_shard(bf16* dst, int64_t rows, int64_t cols, uint64_t seed, int tensor,
                       int layer, int layout, int64_t part, int64_t row_off, int64_t col_off,
                       int64_t cols_total, cudaStream_t s);
// Tensor parallelism: the planes' fp32 partials of a row-parallel GEMM
// (device pointers, any GPU of the runtime; row r of part q at p[q] + r*hidden).
struct TpParts {
  const float* p[kMaxTp] = {};
  int n = 0;
};
// x_new = x (rows x hidden) + the partials summed in plane order, xn =
// rmsnorm(x_new) with unit gain — one pass, the row kept in registers. x_new
// is stored to every pointer of x_out (x itself may be one of them), xn to
// every pointer of xn_out (1..8 each; peer pointers: the all-gather of a
// reduce-scatter fused into its reduction).
void tp_reduce_residual_norm(const bf16* x, const TpParts& parts, bf16* const* x_out, int n_x,
                             bf16* const* xn_out, int n_xn, int rows, int hidden, float eps,
                             cudaStream_t s);
void fill_bf16(bf16* dst, int64_t n, float v, cudaStream_t s);
// w[r][c] *= gamma[c] (fold a norm gain into the consuming projection).
void scale_cols(bf16* w, int64_t rows, int64_t cols, const bf16* gamma, cudaStream_t s);
// Page-table conservation: counts how often each slot appears (atomic).
void count_slots(const int32_t* slots, int64_t n, int32_t* counts, int capacity,
                 cudaStream_t s);
void check_counts(const int32_t* counts, int capacity, int32_t* result /*[2]*/, cudaStream_t s);
// KV move: copy slab rows (all layers) between slots / slabs. Layer l of a
// slab starts l * layer_stride elements after its base.
void copy_slots(const bf16* src_k, const bf16* src_v, const int32_t* src_slots, bf16* dst_k,
                bf16* dst_v, const int32_t* dst_slots, int n, int layers,
                int64_t src_layer_stride, int64_t dst_layer_stride, int hidden, cudaStream_t s);

int64_t launch_count();
void count_launch();

// Launch with programmatic stream serialization (PDL) unless ESP_PDL=0: the
// kernel may start while the previous kernel of the stream drains; every
// kernel launched this way executes griddepcontrol.wait before it reads or
// writes anything a predecessor touches (only weights are read earlier).
// cls: 1 skinny GEMM, 2 norm/embed/argmax, 4 decode attention, 8 combine
// (ESP_PDL=<mask>, default 3 = GEMMs + norms; ESP_PDL=0 off).
bool pdl_enabled(int cls);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(int cls, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(cls) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Kernel function attributes (dynamic shared memory, cluster size) belong to
// the device's context: run `set` once per (current device, kernel), so every
// GPU of a multi-device runtime gets them.
template <class F>
inline void once_per_device(const void* kernel, F&& set) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.emplace(dev, kernel).second) set();
}

}  // namespace esp::k
