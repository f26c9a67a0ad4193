// extern "C" surface (include/esp_abi.h). Exceptions stop here: each entry
// point maps esp::Error to its status code and records the message in a
// thread-local buffer for esp_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../kernels/kernels.h"
#include "esp_abi.h"
#include "planner.hpp"
#include "device_ctx.hpp"
#include "runtime.hpp"
#include "sib_fit.hpp"

struct esp_runtime {
  esp::Runtime* impl;
};

namespace {

thread_local std::string g_last_error;

// Device scratch of the kernel hooks: checked allocation, freed on scope
// exit (errors included).
struct DevMem {
  void* p = nullptr;
  explicit DevMem(size_t bytes) { esp::cuda_ok(cudaMalloc(&p, bytes), "cudaMalloc(hook)"); }
  ~DevMem() {
    if (p) cudaFree(p);
  }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ESP_OK;
  } catch (const esp::Error& e) {
    g_last_error = e.what();
    return e.code();
  } catch (const std::exception& e) {
    g_last_error = std::string("internal: ") + e.what();
    return ESP_ERR_INTERNAL;
  }
}

esp::Sib make_sib(const esp_sib_record* sib, int32_t n) {
  std::vector<esp::SibRecord> recs;
  for (int32_t i = 0; i < n; ++i) {
    esp::SibRecord r;
    r.dop = sib[i].dop;
    r.tp = sib[i].tp;
    r.alpha_p = sib[i].alpha_p;
    r.beta_p = sib[i].beta_p;
    r.gamma_p = sib[i].gamma_p;
    r.alpha_d = sib[i].alpha_d;
    r.beta_d = sib[i].beta_d;
    r.gamma_d = sib[i].gamma_d;
    r.threshold = sib[i].compute_bound_batch_threshold;
    r.tipping_ms = sib[i].tipping_ms;
    recs.push_back(r);
  }
  return esp::Sib(std::move(recs));
}

std::map<int32_t, int64_t> free_map(const int32_t* inst, const int64_t* tok, int32_t n) {
  std::map<int32_t, int64_t> m;
  for (int32_t i = 0; i < n; ++i) m[inst[i]] = tok[i];
  return m;
}

}  // namespace

extern "C" {

const char* esp_last_error(void) { return g_last_error.c_str(); }
int32_t esp_abi_version(void) { return ESP_ABI_VERSION; }

int64_t esp_kv_bytes_per_token(int32_t layers, int32_t hidden_dim, int32_t kv_heads,
                               int32_t bytes_per_element) {
  int64_t out = -1;
  guarded([&] { out = esp::kv_bytes_per_token(layers, hidden_dim, kv_heads, bytes_per_element); });
  return out;
}

int esp_plan_prefill_scale_down(const int32_t* instances, const int64_t* free, int32_t d,
                                const int64_t* input_lens, int32_t n_req,
                                int32_t* decode_instances, int32_t* n_decode,
                                int32_t* place_inst, int64_t* place_tok, int32_t* place_n,
                                int64_t* ring_volume) {
  return guarded([&] {
    auto p = esp::plan_prefill_scale_down(std::vector<int32_t>(instances, instances + d),
                                          std::vector<int64_t>(free, free + d),
                                          std::vector<int64_t>(input_lens, input_lens + n_req));
    *n_decode = static_cast<int32_t>(p.decode_instances.size());
    std::copy(p.decode_instances.begin(), p.decode_instances.end(), decode_instances);
    for (int32_t r = 0; r < n_req; ++r) {
      place_n[r] = static_cast<int32_t>(p.fill[r].size());
      for (size_t j = 0; j < p.fill[r].size(); ++j) {
        place_inst[r * d + j] = p.fill[r][j].first;
        place_tok[r * d + j] = p.fill[r][j].second;
      }
    }
    *ring_volume = p.ring_volume;
  });
}

double esp_sib_prefill_time(const esp_sib_record* sib, int32_t n_rec, int32_t dop, int32_t tp,
                            double sum_len, double sum_len_sq) {
  double out = -1;
  if (guarded([&] { out = make_sib(sib, n_rec).prefill_time_sums(sum_len, sum_len_sq, dop, tp); }) !=
      ESP_OK) {
    return -1;
  }
  return out;
}

double esp_sib_decode_time(const esp_sib_record* sib, int32_t n_rec, int32_t dop, int32_t tp,
                           int32_t batch_size, int64_t resident_kv, int32_t n_masters) {
  double out = -1;
  if (guarded([&] {
        out = make_sib(sib, n_rec).decode_time(batch_size, resident_kv, dop, tp, n_masters);
      }) != ESP_OK) {
    return -1;
  }
  return out;
}

int esp_plan_decode_step(const int32_t* members, int32_t d, int32_t batch_size,
                         const int32_t* free_inst, const int64_t* free_tok, int32_t n_free,
                         int32_t* idle_pool, int32_t* n_idle, const esp_sib_record* sib,
                         int32_t n_rec, int32_t tp, int32_t enable_scale_up, int32_t* feasible,
                         int32_t* masters, int32_t* n_masters, int32_t* add_instances,
                         int32_t* n_add) {
  return guarded([&] {
    std::vector<int32_t> idle(idle_pool, idle_pool + *n_idle);
    auto plan = esp::plan_decode_step(std::vector<int32_t>(members, members + d), batch_size,
                                      free_map(free_inst, free_tok, n_free), idle,
                                      make_sib(sib, n_rec), tp, enable_scale_up != 0);
    *feasible = plan.feasible ? 1 : 0;
    *n_masters = static_cast<int32_t>(plan.masters.size());
    std::copy(plan.masters.begin(), plan.masters.end(), masters);
    *n_add = static_cast<int32_t>(plan.add_instances.size());
    std::copy(plan.add_instances.begin(), plan.add_instances.end(), add_instances);
    *n_idle = static_cast<int32_t>(idle.size());
    std::copy(idle.begin(), idle.end(), idle_pool);
  });
}

int esp_assign_masters(const int64_t* batch, int32_t b, const int32_t* masters, int32_t k,
                       int32_t* master_of) {
  return guarded([&] {
    auto a = esp::assign_masters(std::vector<int64_t>(batch, batch + b),
                                 std::vector<int32_t>(masters, masters + k));
    std::map<int64_t, int32_t> of;
    for (const auto& [m, rs] : a) {
      for (int64_t r : rs) of[r] = m;
    }
    for (int32_t i = 0; i < b; ++i) master_of[i] = of[batch[i]];
  });
}

int esp_decode_step_comm(int32_t d, const int32_t* masters, const int32_t* counts,
                         const int64_t* master_free, int32_t k, int64_t* query_volume,
                         int64_t* overlappable_volume, int32_t* full_master) {
  *full_master = -1;
  return guarded([&] {
    std::map<int32_t, std::vector<int64_t>> assign;
    std::map<int32_t, int64_t> free;
    int64_t next = 0;
    for (int32_t i = 0; i < k; ++i) {
      auto& v = assign[masters[i]];
      for (int32_t j = 0; j < counts[i]; ++j) v.push_back(next++);
      free[masters[i]] = master_free[i];
    }
    try {
      auto c = esp::decode_step_comm(d, assign, free);
      *query_volume = c.query_volume;
      *overlappable_volume = c.overlappable_volume;
    } catch (const esp::MasterFullError& e) {
      *full_master = e.instance;
      throw;
    }
  });
}

int esp_build_ring_schedule(const int32_t* group, const int64_t* segment_tokens, int32_t d,
                            int32_t* from, int32_t* to, int64_t* volume,
                            int64_t* total_comm_volume) {
  return guarded([&] {
    if (d < 0) throw esp::InfeasiblePlanError("negative ring width");
    auto ring = esp::build_ring_schedule(std::vector<int32_t>(group, group + d),
                                         std::vector<int64_t>(segment_tokens, segment_tokens + d));
    for (int32_t r = 0; r + 1 < d; ++r) {
      for (int32_t i = 0; i < d; ++i) {
        const auto& t = ring.rounds[r][i];
        from[r * d + i] = t.from;
        to[r * d + i] = t.to;
        volume[r * d + i] = t.volume;
      }
    }
    *total_comm_volume = ring.total_comm_volume();
  });
}

int esp_proactive_scale_down(const int32_t* ring, const int64_t* segment_tokens, int32_t d,
                             const int32_t* sources, int32_t n_sources, const int32_t* targets,
                             int32_t n_targets, const int32_t* target_inst,
                             const int64_t* target_tok, int32_t n_target,
                             const int32_t* free_inst, const int64_t* free_tok, int32_t n_free,
                             int64_t* extra_migration_volume,
                             int64_t* transient_buffer_tokens) {
  return guarded([&] {
    auto sched = esp::build_ring_schedule(std::vector<int32_t>(ring, ring + d),
                                          std::vector<int64_t>(segment_tokens, segment_tokens + d));
    esp::FillOrder tp;
    for (int32_t i = 0; i < n_target; ++i) tp.emplace_back(target_inst[i], target_tok[i]);
    auto r = esp::proactive_scale_down(sched, std::vector<int32_t>(sources, sources + n_sources),
                                       std::vector<int32_t>(targets, targets + n_targets), tp,
                                       free_map(free_inst, free_tok, n_free));
    *extra_migration_volume = r.extra_migration_volume;
    *transient_buffer_tokens = r.transient_buffer_tokens;
  });
}

int esp_reactive_migrate(const int32_t* sources, int32_t n_sources, const int32_t* targets,
                         int32_t n_targets, int64_t total_tokens, const int32_t* free_inst,
                         const int64_t* free_tok, int32_t n_free, int32_t* feasible,
                         int32_t* blocked_instance, int64_t* per_source_headroom,
                         int32_t* final_inst, int64_t* final_tok, int32_t* n_final,
                         int64_t* migration_volume) {
  return guarded([&] {
    auto r = esp::reactive_migrate(free_map(free_inst, free_tok, n_free),
                                   std::vector<int32_t>(sources, sources + n_sources),
                                   std::vector<int32_t>(targets, targets + n_targets),
                                   total_tokens);
    *feasible = r.feasible ? 1 : 0;
    *blocked_instance = r.blocked_instance;
    *per_source_headroom = r.per_source_headroom;
    *migration_volume = r.migration_volume;
    int32_t n = 0;
    for (const auto& [i, t] : r.final_placement) {
      final_inst[n] = i;
      final_tok[n] = t;
      ++n;
    }
    *n_final = n;
  });
}

// ---- runtime -------------------------------------------------------------------
int esp_runtime_create(const esp_model_config* cfg, int32_t n_instances,
                       const int32_t* instance_device, int64_t kv_capacity_tokens,
                       esp_runtime** out) {
  *out = nullptr;
  return guarded([&] {
    auto* rt = new esp_runtime{nullptr};
    try {
      rt->impl = new esp::Runtime(*cfg, n_instances, instance_device, kv_capacity_tokens);
    } catch (...) {
      delete rt;
      throw;
    }
    *out = rt;
  });
}

int esp_runtime_create_tp(const esp_model_config* cfg, int32_t n_instances, int32_t tp,
                          const int32_t* plane_device, int64_t kv_capacity_tokens,
                          esp_runtime** out) {
  *out = nullptr;
  return guarded([&] {
    if (!cfg) throw esp::ConfigError("null model config");
    auto* rt = new esp_runtime{nullptr};
    try {
      rt->impl = new esp::Runtime(*cfg, n_instances, tp, plane_device, kv_capacity_tokens);
    } catch (...) {
      delete rt;
      throw;
    }
    *out = rt;
  });
}

void esp_runtime_destroy(esp_runtime* rt) {
  if (!rt) return;
  delete rt->impl;
  delete rt;
}

int esp_instance_info(const esp_runtime* rt, int32_t instance, int64_t* capacity,
                      int64_t* used) {
  return guarded([&] { rt->impl->instance_info(instance, capacity, used); });
}

int esp_prefill(esp_runtime* rt, const esp_prefill_args* args) {
  return guarded([&] { rt->impl->prefill(*args); });
}

int esp_decode_step(esp_runtime* rt, const esp_decode_args* args) {
  return guarded([&] { rt->impl->decode_step(*args); });
}

int esp_move_kv(esp_runtime* rt, int64_t request, int32_t from, int32_t to, int64_t tokens) {
  return guarded([&] { rt->impl->move_kv(request, from, to, tokens); });
}

int esp_free_request(esp_runtime* rt, int64_t request) {
  return guarded([&] { rt->impl->free_request(request); });
}

int esp_query_placement(const esp_runtime* rt, int64_t request, int32_t* inst, int64_t* tokens,
                        int32_t cap, int32_t* n) {
  return guarded([&] { rt->impl->query_placement(request, inst, tokens, cap, n); });
}

int esp_check_conservation(esp_runtime* rt) {
  return guarded([&] { rt->impl->check_conservation(); });
}

int esp_request_tokens(const esp_runtime* rt, int64_t request, int32_t* out, int32_t cap,
                       int32_t* n) {
  return guarded([&] { rt->impl->request_tokens(request, out, cap, n); });
}

int esp_last_prefill_stats(const esp_runtime* rt, esp_prefill_stats* out) {
  return guarded([&] {
    if (!rt || !out) throw esp::ConfigError("last_prefill_stats: null argument");
    *out = rt->impl->last_prefill_stats();
  });
}

int esp_read_kv(esp_runtime* rt, int64_t request, int32_t layer, void* k_out, void* v_out,
                int64_t cap, int64_t* n) {
  return guarded([&] {
    if (!rt || !n) throw esp::ConfigError("read_kv: null argument");
    if (cap > 0 && (!k_out || !v_out)) throw esp::ConfigError("read_kv: null output");
    rt->impl->read_kv(request, layer, k_out, v_out, cap, n);
  });
}

int esp_capture_attention(esp_runtime* rt, const int64_t* pos, int64_t n) {
  return guarded([&] {
    if (!rt || (n > 0 && !pos) || n < 0) throw esp::ConfigError("capture_attention: bad argument");
    rt->impl->capture_attention(pos, n);
  });
}

int esp_captured_attention(esp_runtime* rt, void* out, int64_t cap, int64_t* n_rows) {
  return guarded([&] {
    if (!rt || !n_rows) throw esp::ConfigError("captured_attention: null argument");
    rt->impl->captured_attention(out, cap, n_rows);
  });
}

int esp_slab_access(const esp_runtime* rt, int32_t instance, int32_t device, int32_t* ok) {
  return guarded([&] {
    if (!rt || !ok) throw esp::ConfigError("slab_access: null argument");
    *ok = rt->impl->slab_accessible(instance, device) ? 1 : 0;
  });
}

int esp_dump_profiles(const esp_runtime* rt, const char* path) {
  return guarded([&] { rt->impl->dump_profiles(path); });
}

int esp_decode_samples(const esp_runtime* rt, int32_t* dop, int32_t* batch, int32_t* masters,
                       int64_t* resident, double* ms, int64_t cap, int64_t* n) {
  return guarded([&] {
    if (!rt || !n) throw esp::ConfigError("decode_samples: null argument");
    const auto& v = rt->impl->decode_profiles();
    *n = static_cast<int64_t>(v.size());
    const int64_t m = std::min<int64_t>(cap, *n);
    if (m > 0 && (!dop || !batch || !masters || !resident || !ms)) {
      throw esp::ConfigError("decode_samples: null output array");
    }
    for (int64_t i = 0; i < m; ++i) {
      const auto& r = v[static_cast<size_t>(i)];
      dop[i] = r.dop;
      batch[i] = r.batch;
      masters[i] = r.masters;
      resident[i] = r.resident;
      ms[i] = r.ms;
    }
  });
}

int esp_fit_cost(const double* x1, const double* x2, const double* y, int64_t n, double* coef) {
  return guarded([&] {
    if (n > 0 && (!x1 || !x2 || !y)) throw esp::ConfigError("fit_cost: null argument");
    if (!coef) throw esp::ConfigError("fit_cost: null output");
    const auto c = esp::fit_cost(x1, x2, y, n > 0 ? static_cast<size_t>(n) : 0);
    for (int i = 0; i < 3; ++i) coef[i] = c[static_cast<size_t>(i)];
  });
}

int esp_set_profiling(esp_runtime* rt, int32_t on) {
  return guarded([&] { rt->impl->set_profiling(on != 0); });
}

int esp_phase_times(esp_runtime* rt, double* ms, int64_t* launches, int32_t n) {
  return guarded([&] { rt->impl->phase_times(ms, launches, n); });
}

int64_t esp_launch_count(const esp_runtime* rt) {
  (void)rt;
  return esp::k::launch_count();
}

// ---- kernel-level hooks ---------------------------------------------------------
int esp_k_gemm(const void* A, const void* B, void* D, int32_t M, int32_t N, int32_t K,
               int32_t epilogue, void* stream) {
  return guarded([&] {
    esp::k::GemmEpilogue ep;
    const int kind = epilogue & 0xFF, path = (epilogue >> 8) & 0xFF;
    if (kind == 0) ep.kind = esp::k::kEpiStore;
    else if (kind == 1) ep.kind = esp::k::kEpiResidual;
    else if (kind == 2) ep.kind = esp::k::kEpiStoreF32;
    else if (kind == 3) ep.kind = esp::k::kEpiSiluMul;
    else throw esp::ConfigError("unknown epilogue");
    if (path > esp::k::kGemmStreamKAll) throw esp::ConfigError("unknown GEMM path");
    if (!A || !B || !D) throw esp::ConfigError("gemm hook: null argument");
    ep.out = D;
    ep.ldo = kind == 3 ? N / 2 : N;
    esp::k::gemm(static_cast<const esp::k::bf16*>(A), K, static_cast<const esp::k::bf16*>(B), K,
                 M, N, K, ep, static_cast<cudaStream_t>(stream), path);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw esp::CudaError(cudaGetErrorString(e));
  });
}

int esp_k_ring_attention(const void* q, int32_t q_len, int32_t pos_i, int32_t d,
                         const void* const* kv_k, const void* const* kv_v, const int32_t* kv_len,
                         const int32_t* origin, void* out, int32_t heads, int32_t head_dim,
                         void* stream) {
  return esp_k_ring_attention_timed(q, q_len, pos_i, d, kv_k, kv_v, kv_len, origin, out, heads,
                                    head_dim, 1, nullptr, stream);
}

int esp_k_ring_attention_timed(const void* q, int32_t q_len, int32_t pos_i, int32_t d,
                               const void* const* kv_k, const void* const* kv_v,
                               const int32_t* kv_len, const int32_t* origin, void* out,
                               int32_t heads, int32_t head_dim, int32_t repeats,
                               float* ms_per_launch, void* stream) {
  // Test hook: stages q and the d KV blocks into one buffer (rows: q, then
  // block 0..d-1) so the production kernel runs on exactly its layout.
  return guarded([&] {
    if (repeats < 1) throw esp::ConfigError("repeats must be >= 1");
    if (d < 1 || d > esp::k::kMaxRounds) throw esp::ConfigError("d out of range");
    if (!q || !kv_k || !kv_v || !kv_len || !origin || !out) {
      throw esp::ConfigError("ring_attention hook: null argument");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t hidden = static_cast<int64_t>(heads) * head_dim;
    int64_t rows = q_len;
    std::vector<int32_t> row0(static_cast<size_t>(d));
    for (int r = 0; r < d; ++r) {
      row0[r] = static_cast<int32_t>(rows);
      rows += kv_len[r];
    }
    if (rows > INT32_MAX) throw esp::ConfigError("ring_attention hook: too many rows");
    using esp::k::bf16;
    const size_t bytes = static_cast<size_t>(rows) * hidden * 2;
    DevMem Q(bytes), K(bytes), V(bytes), O(bytes);
    esp::cuda_ok(cudaMemcpyAsync(Q.p, q, static_cast<size_t>(q_len) * hidden * 2,
                                 cudaMemcpyDeviceToDevice, s), "stage q");
    for (int r = 0; r < d; ++r) {
      const size_t off = static_cast<size_t>(row0[r]) * hidden * 2;
      const size_t n = static_cast<size_t>(kv_len[r]) * hidden * 2;
      esp::cuda_ok(cudaMemcpyAsync(static_cast<char*>(K.p) + off, kv_k[r], n,
                                   cudaMemcpyDeviceToDevice, s), "stage k");
      esp::cuda_ok(cudaMemcpyAsync(static_cast<char*>(V.p) + off, kv_v[r], n,
                                   cudaMemcpyDeviceToDevice, s), "stage v");
    }
    esp::k::RingSegment sg{};
    sg.q_row0 = 0;
    sg.q_len = q_len;
    sg.n_rounds = d;
    for (int r = 0; r < d; ++r) {
      sg.kv_row0[r] = row0[r];
      sg.kv_len[r] = kv_len[r];
      sg.shift[r] = origin[r] > pos_i ? 1 : 0;
    }
    std::vector<int32_t> work;  // the runtime's work order (LPT, head groups)
    esp::build_attention_work({sg}, heads, work);
    DevMem dseg(sizeof(sg)), dwork(work.size() * 4);
    esp::cuda_ok(cudaMemcpyAsync(dseg.p, &sg, sizeof(sg), cudaMemcpyHostToDevice, s), "h2d");
    esp::cuda_ok(cudaMemcpyAsync(dwork.p, work.data(), work.size() * 4, cudaMemcpyHostToDevice, s),
                 "h2d");
    const float scale = 1.0f / std::sqrt(static_cast<float>(head_dim));
    const int nr = static_cast<int>(rows);
    const int n_work = esp::attention_n_work(work);
    const auto* segs = static_cast<const esp::k::RingSegment*>(dseg.p);
    const auto* wk = static_cast<const int32_t*>(dwork.p);
#ifdef ESP_STUDY
    if (std::getenv("ESP_ATTN_PROF") != nullptr) {
      // Kernel study build: cycle accounting of the pipeline roles (stderr).
      const int grid = std::min(n_work, 148);
      DevMem dprof(static_cast<size_t>(grid) * 32 * 8);
      cudaMemsetAsync(dprof.p, 0, static_cast<size_t>(grid) * 32 * 8, s);
      esp::k::ring_attention_profiled(static_cast<bf16*>(Q.p), static_cast<bf16*>(K.p),
                                      static_cast<bf16*>(V.p), static_cast<bf16*>(O.p), nr, nr,
                                      heads, head_dim, segs, wk, n_work, scale, s,
                                      static_cast<uint64_t*>(dprof.p));
      std::vector<uint64_t> h(static_cast<size_t>(grid) * 32);
      cudaMemcpyAsync(h.data(), dprof.p, h.size() * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      const char* roles[4] = {"producer", "mma", "softmax0", "softmax1"};
      for (int r = 0; r < 4; ++r) {
        std::fprintf(stderr, "[attn-prof] %-9s", roles[r]);
        for (int c = 0; c < 8; ++c) {
          double sum = 0;
          for (int b = 0; b < grid; ++b) sum += static_cast<double>(h[(b * 4 + r) * 8 + c]);
          std::fprintf(stderr, " c%d=%.0f", c, sum / grid);
        }
        std::fprintf(stderr, "\n");
      }
    }
#endif
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ms_per_launch) {
      esp::cuda_ok(cudaEventCreate(&e0), "event");
      esp::cuda_ok(cudaEventCreate(&e1), "event");
      esp::cuda_ok(cudaEventRecord(e0, s), "event");
    }
    for (int i = 0; i < repeats; ++i) {
      esp::k::ring_attention(static_cast<bf16*>(Q.p), static_cast<bf16*>(K.p),
                             static_cast<bf16*>(V.p), static_cast<bf16*>(O.p), nr, nr, heads,
                             head_dim, segs, wk, n_work, scale, s);
    }
    esp::cuda_ok(cudaGetLastError(), "ring_attention launch");
    if (ms_per_launch) {
      esp::cuda_ok(cudaEventRecord(e1, s), "event");
      esp::cuda_ok(cudaEventSynchronize(e1), "event");
      float ms = 0.f;
      esp::cuda_ok(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
      *ms_per_launch = ms / static_cast<float>(repeats);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    esp::cuda_ok(cudaMemcpyAsync(out, O.p, static_cast<size_t>(q_len) * hidden * 2,
                                 cudaMemcpyDeviceToDevice, s), "d2d");
    esp::cuda_ok(cudaStreamSynchronize(s), "ring_attention hook");
  });
}

int esp_k_decode_attention(const void* q, int32_t batch, const void* const* k_slab,
                           const void* const* v_slab, const int32_t* const* slot_idx,
                           const int32_t* n_slots, const int32_t* chunk_req, int32_t n_chunks,
                           void* out, int32_t heads, int32_t head_dim, int32_t out_f32,
                           void* stream) {
  return guarded([&] {
    if (n_chunks > esp::k::kMaxSlabs) throw esp::ConfigError("too many chunks for the hook");
    if (!q || !k_slab || !v_slab || !slot_idx || !n_slots || !chunk_req || !out) {
      throw esp::ConfigError("decode_attention hook: null argument");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    esp::k::DecodeSlabs slabs{};
    std::vector<esp::k::DecodeChunk> ch;
    std::vector<std::pair<int32_t, int>> by_row;
    for (int c = 0; c < n_chunks; ++c) {
      if (chunk_req[c] < 0 || chunk_req[c] >= batch) throw esp::ConfigError("chunk row out of range");
      by_row.emplace_back(chunk_req[c], c);
    }
    std::stable_sort(by_row.begin(), by_row.end());
    std::vector<int32_t> row_start(static_cast<size_t>(batch) + 1, 0);
    for (const auto& [row, c] : by_row) {
      slabs.k[c] = static_cast<const esp::k::bf16*>(k_slab[c]);
      slabs.v[c] = static_cast<const esp::k::bf16*>(v_slab[c]);
      // split into the runtime's chunk size, as esp_decode_step does
      for (int32_t c0 = 0; c0 < n_slots[c]; c0 += esp::decode_chunk()) {
        ch.push_back({slot_idx[c] + c0, std::min<int32_t>(esp::decode_chunk(), n_slots[c] - c0), row,
                      c, static_cast<int32_t>(ch.size()), 0});
        row_start[row + 1]++;
      }
    }
    const int32_t n_parts = static_cast<int32_t>(ch.size());
    int max_n = 0;  // the short-chunk kernel when every chunk is <= 64 tokens
    for (const auto& c : ch) max_n = std::max(max_n, static_cast<int>(c.n));
    for (int r = 0; r < batch; ++r) row_start[r + 1] += row_start[r];
    DevMem dch(ch.size() * sizeof(esp::k::DecodeChunk) + 16), drs(row_start.size() * 4);
    DevMem po(static_cast<size_t>(n_parts) * heads * head_dim * 4 + 16);
    DevMem pml(static_cast<size_t>(n_parts) * heads * 2 * 4 + 16);
    esp::cuda_ok(cudaMemcpyAsync(dch.p, ch.data(), ch.size() * sizeof(esp::k::DecodeChunk),
                                 cudaMemcpyHostToDevice, s), "h2d");
    esp::cuda_ok(cudaMemcpyAsync(drs.p, row_start.data(), row_start.size() * 4,
                                 cudaMemcpyHostToDevice, s), "h2d");
    const float scale = 1.0f / std::sqrt(static_cast<float>(head_dim));
    esp::k::decode_attention(static_cast<const esp::k::bf16*>(q),
                             static_cast<const esp::k::DecodeChunk*>(dch.p), n_parts, slabs,
                             heads, head_dim, scale, static_cast<float*>(po.p),
                             static_cast<float*>(pml.p), s, nullptr, nullptr, max_n);
    if (out_f32) {
      esp::k::decode_combine_f32(static_cast<float*>(po.p), static_cast<float*>(pml.p),
                                 static_cast<int32_t*>(drs.p), batch, heads, head_dim,
                                 static_cast<float*>(out), s);
    } else {
      esp::k::decode_combine(static_cast<float*>(po.p), static_cast<float*>(pml.p),
                             static_cast<int32_t*>(drs.p), batch, heads, head_dim,
                             static_cast<esp::k::bf16*>(out), s);
    }
    esp::cuda_ok(cudaGetLastError(), "decode_attention launch");
    esp::cuda_ok(cudaStreamSynchronize(s), "decode_attention hook");
  });
}

}  // extern "C"
