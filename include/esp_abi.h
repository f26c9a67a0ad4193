/* esp_abi.h — C ABI of the B200-native ESP (elastic sequence parallelism)
 * data path. Plain pointers and sizes only; no C++ or torch types cross it.
 *
 * Two families of entry points:
 *
 *  (1) Pure host planning functions — B200-side restatements of the
 *      reference's hot-path placement mechanics, bit-exact with them:
 *        esp_kv_bytes_per_token      <- cluster.cpp:30-34   (kv_bytes_per_token)
 *        esp_plan_prefill_scale_down <- scheduler.cpp:663-713 (plan_prefill_scale_down)
 *        esp_plan_decode_step        <- scheduler.cpp:726-804 (plan_decode_step_core)
 *        esp_assign_masters          <- esp_mechanics.cpp:220-238
 *        esp_decode_step_comm        <- esp_mechanics.cpp:240-264
 *        esp_build_ring_schedule     <- esp_mechanics.cpp:24-70
 *        esp_proactive_scale_down    <- esp_mechanics.cpp:78-136
 *        esp_reactive_migrate        <- esp_mechanics.cpp:138-218
 *        esp_sib_prefill_time / esp_sib_decode_time <- cost_model.cpp:169-187
 *
 *  (2) The runtime (executor): each elastic instance (reference
 *      ElasticInstance, cluster.hpp:69-78) is a GPU-resident slice of one
 *      token-granular paged KV pool (reference KvPool, cluster.hpp:102-128).
 *      The reference engine commits placements at Engine::apply_decision
 *      (engine.cpp:246-490); a Policy decorator calls
 *        esp_prefill      for every PrefillPlan    (state.hpp:83-96)
 *        esp_decode_step  for every DecodeStepPlan (state.hpp:98-107)
 *        esp_move_kv      for every KvMove         (state.hpp:67-72)
 *        esp_free_request when a request finishes / is evicted (engine.cpp:119-166)
 *      and the device page tables then hold exactly the reference's
 *      Request.placement (cluster.hpp:44, :63) and ElasticInstance.kv_used.
 *
 * Error convention: every int-returning call returns ESP_OK (0) or one of the
 * negative codes below, mapped 1:1 to the reference taxonomy
 * (types.hpp:48-109); nothing throws across the ABI. esp_last_error() gives a
 * thread-local message for the last failure on the calling thread.
 *
 * Threading: one caller thread per runtime (the reference engine is strictly
 * single-threaded, engine.hpp:45). Calls return after their results are
 * host-visible. Caller owns every array it passes (borrowed for the call);
 * the runtime owns device memory, weights, slabs and page tables.
 */
#ifndef ESP_ABI_H_
#define ESP_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define ESP_ABI_VERSION 3

/* ---- error codes (reference types.hpp:48-109) --------------------------- */
enum esp_status {
  ESP_OK = 0,
  ESP_ERR_CONFIG = -1,           /* ConfigError               types.hpp:53-56  */
  ESP_ERR_INFEASIBLE = -2,       /* InfeasiblePlanError       types.hpp:83-86  */
  ESP_ERR_INTERNAL = -3,         /* InternalError             types.hpp:95-98  */
  ESP_ERR_CAPACITY = -4,         /* AllocResult{ok=false}     cluster.hpp:95-98 */
  ESP_ERR_MASTER_FULL = -5,      /* DecodeCommResult{ok=false} esp_mechanics.hpp:104-110 */
  ESP_ERR_UNKNOWN_STRATEGY = -6, /* UnknownStrategyError      types.hpp:58-65  */
  ESP_ERR_CUDA = -7,             /* device failure (no reference counterpart) */
  ESP_ERR_NO_DEVICE = -8         /* compute requested from a placement-only runtime */
};

const char* esp_last_error(void);
int32_t esp_abi_version(void);

/* ---- (1) pure host planning --------------------------------------------- */

/* 2 * layers * hidden_dim * bytes_per_element (cluster.cpp:30-34). Returns -1
 * (and sets ESP_ERR_CONFIG message) on a non-positive field. */
int64_t esp_kv_bytes_per_token(int32_t layers, int32_t hidden_dim, int32_t kv_heads,
                               int32_t bytes_per_element);

/* plan_prefill_scale_down (scheduler.cpp:663-713).
 * in : instances[d] ring order (PrefillPlan.instances), free[d] free slots per
 *      instance (the scheduler's free_override view), input_lens[n_req] in
 *      PrefillPlan.requests order.
 * out: decode_instances[d] (ascending survivors), *n_decode;
 *      per request r: place_n[r] (instance, tokens) pairs in FILL ORDER at
 *      place_inst[r*d + p], place_tok[r*d + p] (a request's tokens are laid
 *      contiguously over them in that order); *ring_volume = (d-1)*sum(len).
 * Returns ESP_ERR_INFEASIBLE when the batch KV exceeds the interval. */
int esp_plan_prefill_scale_down(const int32_t* instances, const int64_t* free, int32_t d,
                                const int64_t* input_lens, int32_t n_req,
                                int32_t* decode_instances, int32_t* n_decode,
                                int32_t* place_inst, int64_t* place_tok, int32_t* place_n,
                                int64_t* ring_volume);

/* One strategy row of the scaling information base (cost_model.hpp:47-52). */
typedef struct esp_sib_record {
  int32_t dop, tp;
  double alpha_p, beta_p, gamma_p;          /* prefill  cost_model.hpp:31-35 */
  double alpha_d, beta_d, gamma_d;          /* decode   cost_model.hpp:40-45 */
  int32_t compute_bound_batch_threshold;
  double tipping_ms;
} esp_sib_record;

/* Sib::prefill_time_sums / decode_time (cost_model.cpp:169-187). Return a
 * negative time and ESP_ERR_UNKNOWN_STRATEGY message if (dop,tp) is absent. */
double esp_sib_prefill_time(const esp_sib_record* sib, int32_t n_rec, int32_t dop, int32_t tp,
                            double sum_len, double sum_len_sq);
double esp_sib_decode_time(const esp_sib_record* sib, int32_t n_rec, int32_t dop, int32_t tp,
                           int32_t batch_size, int64_t resident_kv, int32_t n_masters);

/* plan_decode_step_core (scheduler.cpp:726-804).
 * free_inst/free_tok: free slots keyed by instance (n_free entries, must cover
 * members and idle). idle_pool/n_idle: in-out, consumed from the front.
 * out: *feasible, masters[*n_masters] ascending, add_instances[*n_add]. */
int esp_plan_decode_step(const int32_t* members, int32_t d, int32_t batch_size,
                         const int32_t* free_inst, const int64_t* free_tok, int32_t n_free,
                         int32_t* idle_pool, int32_t* n_idle,
                         const esp_sib_record* sib, int32_t n_rec, int32_t tp,
                         int32_t enable_scale_up,
                         int32_t* feasible, int32_t* masters, int32_t* n_masters,
                         int32_t* add_instances, int32_t* n_add);

/* assign_masters (esp_mechanics.cpp:220-238): master_of[i] is the master of
 * batch[i] (requests dealt in ascending id to the least-loaded master, lowest
 * id on ties). */
int esp_assign_masters(const int64_t* batch, int32_t b, const int32_t* masters, int32_t k,
                       int32_t* master_of);

/* decode_step_comm (esp_mechanics.cpp:240-264). masters[k] with counts[k]
 * requests each, free slots master_free[k]; group width d.
 * Returns ESP_ERR_MASTER_FULL with *full_master set on the first (ascending
 * id) master without room for its appends. */
int esp_decode_step_comm(int32_t d, const int32_t* masters, const int32_t* counts,
                         const int64_t* master_free, int32_t k,
                         int64_t* query_volume, int64_t* overlappable_volume,
                         int32_t* full_master);

/* build_ring_schedule (esp_mechanics.cpp:45-70): round r < d-1, position i
 * sends the block that started at (i-r) mod d to (i+1) mod d.
 * out arrays have (d-1)*d entries, row-major [round][position]. */
int esp_build_ring_schedule(const int32_t* group, const int64_t* segment_tokens, int32_t d,
                            int32_t* from, int32_t* to, int64_t* volume,
                            int64_t* total_comm_volume);

/* proactive_scale_down (esp_mechanics.cpp:78-136) for one aggregate target
 * placement (n_target entries). free_inst/free_tok give pool free slots. */
int esp_proactive_scale_down(const int32_t* ring, const int64_t* segment_tokens, int32_t d,
                             const int32_t* sources, int32_t n_sources,
                             const int32_t* targets, int32_t n_targets,
                             const int32_t* target_inst, const int64_t* target_tok,
                             int32_t n_target,
                             const int32_t* free_inst, const int64_t* free_tok, int32_t n_free,
                             int64_t* extra_migration_volume,
                             int64_t* transient_buffer_tokens);

/* reactive_migrate (esp_mechanics.cpp:138-218), the migration baseline. */
int esp_reactive_migrate(const int32_t* sources, int32_t n_sources, const int32_t* targets,
                         int32_t n_targets, int64_t total_tokens,
                         const int32_t* free_inst, const int64_t* free_tok, int32_t n_free,
                         int32_t* feasible, int32_t* blocked_instance,
                         int64_t* per_source_headroom, int32_t* final_inst,
                         int64_t* final_tok, int32_t* n_final, int64_t* migration_volume);

/* ---- (2) runtime ---------------------------------------------------------- */

typedef struct esp_runtime esp_runtime;

/* Llama-architecture geometry (LWM-7B: 32, 4096, 32, 128, 11008, 32000). */
typedef struct esp_model_config {
  int32_t layers;
  int32_t hidden;     /* = heads * head_dim */
  int32_t heads;      /* query heads == kv heads (MHA, as LWM-7B) */
  int32_t head_dim;   /* 64 or 128 */
  int32_t ffn;        /* multiple of 128 */
  int32_t vocab;
  float rms_eps;      /* 1e-5 */
  float rope_theta;   /* 10000 */
  uint64_t weight_seed;
} esp_model_config;

/* n_instances elastic instances. instance_device[i] is the CUDA device
 * ordinal of instance i (several instances may share a device); NULL creates
 * a PLACEMENT-ONLY runtime (page tables and slot allocators, no device
 * memory, no kernels: compute calls then fail with ESP_ERR_NO_DEVICE).
 * kv_capacity_tokens: token slots per instance (ElasticInstance.kv_capacity);
 * <= 0 sizes it from free HBM. */
int esp_runtime_create(const esp_model_config* cfg, int32_t n_instances,
                       const int32_t* instance_device, int64_t kv_capacity_tokens,
                       esp_runtime** out);
/* Tensor-parallel instances (StrategyKey.tp, types.hpp:36-41;
 * the paper's TP = 2 x ESP = 4): every instance spans tp GPUs,
 * plane r on plane_device[r] holding heads [r heads/tp, (r+1) heads/tp) of
 * its KV and the Megatron shards of the weights (QKV / gate_up column-
 * parallel, O / down row-parallel, all-reduced over peer memory). Slot ids,
 * page tables and counters are those of a tp = 1 runtime, so every other
 * entry point keeps its meaning; ESP rings run co-located inside each plane.
 * tp in 2..8 dividing heads, hidden / tp % 128 == 0, ffn / tp % 64 == 0;
 * kv_capacity_tokens > 0 (KV moves copy every plane's shard; KV readback
 * and attention capture assemble the planes' column shards; chunked-
 * prefill chunks run per plane over their head shard). */
int esp_runtime_create_tp(const esp_model_config* cfg, int32_t n_instances, int32_t tp,
                          const int32_t* plane_device, int64_t kv_capacity_tokens,
                          esp_runtime** out);
void esp_runtime_destroy(esp_runtime* rt);

int esp_instance_info(const esp_runtime* rt, int32_t instance, int64_t* capacity,
                      int64_t* used);

/* ESP prefill of one PrefillPlan (state.hpp:83-96) as a striped ring over
 * ring[dop] with proactive scale-down: every token's K/V lands in a page slot
 * of its resting instance (retain pairs) during the ring pass itself. */
typedef struct esp_prefill_args {
  int32_t n_requests;
  const int64_t* request_ids;      /* PrefillPlan.requests (longest first)   */
  const int64_t* input_lens;
  const int32_t* tokens;           /* concatenated prompts; NULL if placement-only */
  int32_t dop;
  const int32_t* ring;             /* PrefillPlan.instances                  */
  const int32_t* retain_n;         /* per request: #(instance, tokens) pairs */
  const int32_t* retain_instance;  /* concatenated, token order              */
  const int64_t* retain_tokens;
  int32_t* first_token_out;        /* [n_requests] greedy token, nullable    */
  float* logits_out;               /* [n_requests x vocab] fp32, nullable    */
  double* device_ms_out;           /* device time of the pass, nullable      */
} esp_prefill_args;
int esp_prefill(esp_runtime* rt, const esp_prefill_args* args);

/* One multi-master decoding iteration (DecodeStepPlan, state.hpp:98-107):
 * members = group instances after scale-up, masters = plan.masters. The
 * runtime recomputes assign_masters exactly as the engine does
 * (engine.cpp:401), appends each request's new KV token on its master, runs
 * split-KV attention on every instance holding the request's KV and combines
 * the partial (o, lse) at the master. */
typedef struct esp_decode_args {
  int32_t n_members;
  const int32_t* members;
  int32_t n_masters;
  const int32_t* masters;
  int32_t batch_size;
  const int64_t* batch;            /* GroupState.batch                      */
  const int32_t* in_tokens;        /* [b] or NULL: each request's last token */
  int32_t* out_tokens;             /* [b] greedy tokens, nullable            */
  float* logits_out;               /* [b x vocab], nullable                  */
  double* device_ms_out;
  /* Chunked prefill riding on this step (DecodeStepPlan.chunk_request /
   * chunk_tokens / chunk_placement, state.hpp:98-107; the chunked policy,
   * policies.cpp:297-405; committed at engine.cpp:432-462). chunk_tokens == 0:
   * none (a zero-initialised struct has no chunk). The chunk's tokens take slots on chunk_instance[i] (chunk_tokens_on[i]
   * tokens each, ascending instance = KvPlacement order); its queries attend
   * to every earlier token of the request and causally within the chunk.
   * chunk_final = 1 when the chunk completes the prompt (engine.cpp:570-579):
   * the request's first generated token is written to *chunk_first_token_out. */
  int64_t chunk_request;
  int64_t chunk_tokens;
  int32_t chunk_n;
  const int32_t* chunk_instance;
  const int64_t* chunk_tokens_on;
  const int32_t* chunk_token_ids;  /* [chunk_tokens] prompt ids, NULL on a placement-only runtime */
  int32_t chunk_final;
  int32_t* chunk_first_token_out;  /* nullable */
  float* chunk_logits_out;         /* [vocab] when chunk_final, nullable */
} esp_decode_args;
int esp_decode_step(esp_runtime* rt, const esp_decode_args* args);

/* KvMove (state.hpp:67-72): move `tokens` of request's KV from -> to (the
 * request's most recent tokens on `from` go first). */
int esp_move_kv(esp_runtime* rt, int64_t request, int32_t from, int32_t to, int64_t tokens);

/* Releases every slot of the request (finish / evict / recompute). */
int esp_free_request(esp_runtime* rt, int64_t request);

/* Page-table readback for parity: (instance, token count) pairs ascending by
 * instance — exactly the shape of the reference KvPlacement map. */
int esp_query_placement(const esp_runtime* rt, int64_t request, int32_t* inst,
                        int64_t* tokens, int32_t cap, int32_t* n);

/* Recounts, ON THE DEVICE, the slots each instance's slab has assigned and
 * checks them against the host counters and page tables (the device-side
 * analogue of KvPool::check_conservation, cluster.cpp:113-132). */
int esp_check_conservation(esp_runtime* rt);

/* Token history of a request (prompt + generated), for parity tests. */
int esp_request_tokens(const esp_runtime* rt, int64_t request, int32_t* out, int32_t cap,
                       int32_t* n);

/* The ring and scale-down the last esp_prefill executed, as the reference's
 * mechanics account them (through the runtime's restatements of
 * build_ring_schedule, esp_mechanics.cpp:45-70, and proactive_scale_down,
 * :78-136):
 *   ring_volume_tokens       RingSchedule::total_comm_volume = (d-1) * sum
 *   cross_domain_tokens      the part of it whose hops cross co-location
 *                            domains (GPUs): NVLink traffic, per K or V row
 *                            and layer
 *   nvlink_bytes             cross_domain_tokens * 2 (K, V) * hidden * 2 B
 *                            * layers: the ring's NVLink bytes of the pass
 *   transient_buffer_tokens  ceil(sum / d), the circulating stripe
 *   extra_migration_tokens   0 whenever the resting instances are ring
 *                            members (retention rides the ring), else -1
 *   device_ms                device time of the pass (max over GPUs)
 *   kv_ring_rows             (ABI 3) K/V rows of ring buffer one GPU held
 *                            (max over GPUs): every block of the layer on
 *                            one GPU or with the all-gather push (x2 layer
 *                            parities); own block + 2 receive slots, O(S/d),
 *                            with the windowed ring */
typedef struct esp_prefill_stats {
  int64_t ring_volume_tokens;
  int64_t cross_domain_tokens;
  int64_t nvlink_bytes;
  int64_t transient_buffer_tokens;
  int64_t extra_migration_tokens;
  double device_ms;
  int64_t kv_ring_rows;
} esp_prefill_stats;
int esp_last_prefill_stats(const esp_runtime* rt, esp_prefill_stats* out);

/* Parity readback of a request's KV cache, one layer: K (after RoPE) and V
 * rows in TOKEN order (position 0 first), wherever the page tables put them
 * (any instance, any slot), as bf16 [n x hidden] into host buffers k_out /
 * v_out of cap rows (tp > 1: plane p's head shard in columns [p hidden/tp,
 * (p+1) hidden/tp)). *n = the request's KV token count; with cap < *n
 * nothing is copied (size query). Device runtimes only (ESP_ERR_NO_DEVICE). */
int esp_read_kv(esp_runtime* rt, int64_t request, int32_t layer, void* k_out, void* v_out,
                int64_t cap, int64_t* n);

/* Parity capture of the NEXT esp_prefill (single-request plan): the
 * attention outputs (before the O projection) of the prompt positions
 * pos[0..n) in every layer. esp_captured_attention then copies them as bf16
 * [layers x n x hidden] (cap rows of hidden; *n_rows = layers * n; with
 * cap < *n_rows nothing is copied). */
int esp_capture_attention(esp_runtime* rt, const int64_t* pos, int64_t n);
int esp_captured_attention(esp_runtime* rt, void* out, int64_t cap, int64_t* n_rows);

/* 1 in *ok iff every mapped chunk of the instance's K and V slabs is
 * read/write for CUDA device `device` (cuMemGetAccess) — the VMM mappings
 * a cross-GPU ring / KV move dereferences from another device. */
int esp_slab_access(const esp_runtime* rt, int32_t instance, int32_t device, int32_t* ok);

/* Measured ProfileSample records ({"kind":"profile","dop","tp","lengths",
 * "measured_ms"}, cost_model.cpp:243-248) appended to a JSONL file. */
int esp_dump_profiles(const esp_runtime* rt, const char* path);

/* Measured decode steps (one per esp_decode_step that carries no chunk), as
 * the arguments of Sib::decode_time (cost_model.cpp:175-187) the engine
 * charges them with (engine.cpp:420-425): dop = members, batch, masters,
 * resident = KV tokens of the batch after the append; ms = device time.
 * Copies min(cap, available) samples; *n = available. The reference has no
 * decode profile record (it hand-sets alpha_d/beta_d/gamma_d). */
int esp_decode_samples(const esp_runtime* rt, int32_t* dop, int32_t* batch, int32_t* masters,
                       int64_t* resident, double* ms, int64_t cap, int64_t* n);

/* Measured-SIB fit: least squares y ~ c[0] + c[1]*x1 + c[2]*x2
 * with fit_prefill_coefficients' admissibility rule (cost_model.cpp:86-135:
 * unit-norm columns, most negative coefficient dropped until all >= 0).
 * Prefill: x1 = sum of lengths, x2 = sum of squares -> alpha_p, beta_p,
 * gamma_p. Decode: x1 = batch (/ masters above the compute-bound threshold),
 * x2 = resident / dop -> alpha_d, beta_d, gamma_d. ESP_ERR_CONFIG when n < 3
 * or the design is rank deficient (the reference's UnderdeterminedError). */
int esp_fit_cost(const double* x1, const double* x2, const double* y, int64_t n, double* coef);

/* Per-phase device timing (CUDA events around each launch on the runtime's
 * stream) while profiling is on. Phases: 0 embed, 1 rmsnorm, 2 QKV GEMM(+RoPE
 * +ring write+retention), 3 ring attention, 4 O GEMM, 5 gate_up GEMM, 6 down
 * GEMM, 7 LM head, 8 argmax, 9 decode attention, 10 LSE combine; and, always
 * recorded, 11 host enqueue (host wall ms of each single-domain prefill /
 * decode step from the call's entry to its last stream operation).
 * esp_phase_times returns and resets the accumulated ms / launch counts. */
#define ESP_N_PHASES 12
int esp_set_profiling(esp_runtime* rt, int32_t on);
int esp_phase_times(esp_runtime* rt, double* ms, int64_t* launches, int32_t n);

/* Count of kernel launches issued by this runtime so far. */
int64_t esp_launch_count(const esp_runtime* rt);

/* ---- kernel-level hooks (device pointers; for parity/roofline tests) ------- */

/* D[M,N] (bf16, row-major) = A[M,K] (bf16, row-major) x B[N,K]^T (bf16,
 * row-major = K-major). epilogue (low byte): 0 store, 1 D += (residual add,
 * D is read), 2 store fp32 (D is float; the fp32 check mode: bf16 inputs,
 * fp32 accumulation and output), 3 SiLU(gate)*up over 64-row gate/up blocks
 * (D has N/2 columns). Bits 8-15 select the schedule: 0 the production
 * dispatch, 1 the 1-CTA prefill kernel instead of the CTA pair, 2 whole
 * skinny tiles only, 3 skinny stream-K for every shape. */
int esp_k_gemm(const void* A, const void* B, void* D, int32_t M, int32_t N, int32_t K,
               int32_t epilogue, void* stream);

/* Striped ring attention for one instance (ring position i of d) against d
 * KV blocks, bf16 [rows x heads*head_dim] row-major buffers, fp32 softmax.
 * kv_k[r], kv_v[r], kv_len[r], origin[r] describe round r's block. */
int esp_k_ring_attention(const void* q, int32_t q_len, int32_t pos_i, int32_t d,
                         const void* const* kv_k, const void* const* kv_v,
                         const int32_t* kv_len, const int32_t* origin, void* out,
                         int32_t heads, int32_t head_dim, void* stream);
/* The same, for kernel timing: stages once, then launches K1 `repeats`
 * times back to back between CUDA events on `stream`; *ms_per_launch =
 * their average (staging excluded). */
int esp_k_ring_attention_timed(const void* q, int32_t q_len, int32_t pos_i, int32_t d,
                               const void* const* kv_k, const void* const* kv_v,
                               const int32_t* kv_len, const int32_t* origin, void* out,
                               int32_t heads, int32_t head_dim, int32_t repeats,
                               float* ms_per_launch, void* stream);

/* Split-KV paged decode attention + LSE combine over n_chunks chunks of
 * slots: request b's query q[b], chunk c reads slots slot_idx[c][0..n) from
 * slab (k_slab, v_slab rows of heads*head_dim bf16). out: [batch x
 * heads*head_dim] bf16, or fp32 with out_f32 = 1 (the fp32 check mode: the
 * kernels accumulate and combine in fp32; only the output rounding differs). */
int esp_k_decode_attention(const void* q, int32_t batch, const void* const* k_slab,
                           const void* const* v_slab, const int32_t* const* slot_idx,
                           const int32_t* n_slots, const int32_t* chunk_req, int32_t n_chunks,
                           void* out, int32_t heads, int32_t head_dim, int32_t out_f32,
                           void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* ESP_ABI_H_ */
