/* CPU numeric oracle — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's
 * cpu_baseline leg). Never linked into or called by the product path.
 *
 * The reference (espsim) has no numeric path: SPEC.md:14 and :283 put
 * attention numerics out of scope, so there is no reference function to
 * restate line by line. This file restates the computation the ESP data path
 * must reproduce, from the paper's own statement that ESP at any degree,
 * placement or master set has "the same accuracy as the original
 * implementations": a DENSE, single-device, causal
 * Llama-2-architecture forward (LWM-1M-Text = Llama-2-7B arch)
 *   embed -> L x [RMSNorm -> QKV -> RoPE -> causal softmax attention -> O
 *   (+res) -> RMSNorm -> SiLU(gate)*up -> down (+res)] -> RMSNorm -> LM head
 *   -> greedy argmax,
 * prefill of the whole prompt followed by KV-cached decode steps, one token
 * appended per step (KV count after step s = input_len + s, engine.cpp:408-419).
 * Parity of this oracle is therefore UNPINNED by the reference (no golden
 * vectors exist for numerics); the placement side is pinned
 * separately against the compiled reference.
 *
 * Weights are the seeded synthetic weights of
 * paper_2404_09526_b200/csrc/kernels/synthetic.h, restated here bit-exactly
 * (splitmix64 -> 4-term Irwin-Hall -> one fp32 multiply -> bf16 RNE).
 *
 * emulate_bf16 = 1 rounds to bf16 at the points where the GPU path stores
 * bf16 (residual stream, norm outputs, q/k/v after RoPE, attention output,
 * SiLU*up); 0 keeps everything fp32 (the "fp32 check mode").
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t layers, hidden, heads, head_dim, ffn, vocab;
  float rms_eps, rope_theta;
  uint64_t weight_seed;
} llama_cfg;

enum { T_EMBED = 1, T_Q = 2, T_K = 3, T_V = 4, T_O = 5, T_GATE = 6, T_UP = 7, T_DOWN = 8, T_LM = 9 };

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static float bf16_round(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return f; /* inf / nan */
  u += 0x7fffu + ((u >> 16) & 1u);                 /* round to nearest even */
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return f;
}

/* synthetic.h: synthetic_weight(), then __float2bfloat16_rn. */
float llama_ref_weight(uint64_t seed, int tensor, int layer, int64_t row, int64_t col,
                       int64_t cols) {
  const uint64_t idx = (uint64_t)row * (uint64_t)cols + (uint64_t)col;
  const uint64_t key = ((uint64_t)tensor << 56) ^ ((uint64_t)layer << 48) ^ idx;
  const uint64_t h = splitmix64(seed ^ splitmix64(key));
  const int32_t s = (int32_t)(h & 0xFFFF) + (int32_t)((h >> 16) & 0xFFFF) +
                    (int32_t)((h >> 32) & 0xFFFF) + (int32_t)(h >> 48);
  const float x = (float)(s - 131070) * 5.2857997e-07f;
  return bf16_round(x);
}

/* A whole synthetic tensor [rows x cols] (tests: loading the same weights
 * into an independent implementation). */
void llama_ref_weights(uint64_t seed, int tensor, int layer, int64_t rows, int64_t cols,
                       float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t k = 0; k < cols; ++k) out[r * cols + k] = llama_ref_weight(seed, tensor, layer, r, k, cols);
  }
}

static float* make_weight(const llama_cfg* c, int tensor, int layer, int64_t rows, int64_t cols) {
  float* w = (float*)malloc(sizeof(float) * rows * cols);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t k = 0; k < cols; ++k) {
      w[r * cols + k] = llama_ref_weight(c->weight_seed, tensor, layer, r, k, cols);
    }
  }
  return w;
}

/* Y[t][o] = sum_k X[t][k] * W[o][k] for many rows: W transposed once into
 * WT[k][o] (o padded to 16), then per 16-output panel (a thread's WT panel
 * stays in its L2 while it walks every row block) a 6 x 16 register tile
 * accumulates X[t][k] * WT[k][o..o+15] over k. */
#define GEMM_MR 6
#define GEMM_NR 16
static void gemm_nt_panels(const float* X, int64_t T, int64_t K, const float* W, int64_t O,
                           float* Y) {
  const int64_t Op = (O + GEMM_NR - 1) / GEMM_NR * GEMM_NR;
  float* WT = (float*)malloc(sizeof(float) * K * Op);
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t kb = 0; kb < K; kb += 32) {
    for (int64_t ob = 0; ob < Op; ob += 32) {
      for (int64_t k = kb; k < kb + 32 && k < K; ++k) {
        for (int64_t o = ob; o < ob + 32 && o < Op; ++o) {
          WT[k * Op + o] = o < O ? W[o * K + k] : 0.f;
        }
      }
    }
  }
  const int64_t np = Op / GEMM_NR;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t p = 0; p < np; ++p) {
    const int64_t o0 = p * GEMM_NR;
    for (int64_t t0 = 0; t0 < T; t0 += GEMM_MR) {
      float acc[GEMM_MR][GEMM_NR];
      const float* xr[GEMM_MR];
      for (int r = 0; r < GEMM_MR; ++r) {
        xr[r] = X + (t0 + r < T ? t0 + r : t0) * K;
        for (int c = 0; c < GEMM_NR; ++c) acc[r][c] = 0.f;
      }
      const float* wk = WT + o0;
      for (int64_t k = 0; k < K; ++k, wk += Op) {
#pragma GCC unroll 6
        for (int r = 0; r < GEMM_MR; ++r) {
          const float xv = xr[r][k];
#pragma omp simd
          for (int c = 0; c < GEMM_NR; ++c) acc[r][c] += xv * wk[c];
        }
      }
      for (int r = 0; r < GEMM_MR && t0 + r < T; ++r) {
        for (int c = 0; c < GEMM_NR && o0 + c < O; ++c) Y[(t0 + r) * O + o0 + c] = acc[r][c];
      }
    }
  }
  free(WT);
}

/* Y[t][o] = sum_k X[t][k] * W[o][k]  (nn.Linear layout). Few rows (decode,
 * LM head of one row): 4x4 blocks of dot products, the weights streamed once. */
static void gemm_nt(const float* X, int64_t T, int64_t K, const float* W, int64_t O, float* Y) {
  if (T >= 64) {
    gemm_nt_panels(X, T, K, W, O, Y);
    return;
  }
  const int64_t tb = (T + 3) / 4, ob = (O + 3) / 4;
#pragma omp parallel for collapse(2) schedule(dynamic, 4)
  for (int64_t oi = 0; oi < ob; ++oi) {
    for (int64_t ti = 0; ti < tb; ++ti) {
      const int64_t t0 = ti * 4, o0 = oi * 4;
      float acc[4][4] = {{0}};
      const float* x[4];
      const float* w[4];
      for (int j = 0; j < 4; ++j) {
        x[j] = X + (t0 + j < T ? t0 + j : t0) * K;
        w[j] = W + (o0 + j < O ? o0 + j : o0) * K;
      }
      for (int a = 0; a < 4; ++a) {
        for (int b = 0; b < 4; ++b) {
          float s = 0.f;
          const float* xa = x[a];
          const float* wb = w[b];
#pragma omp simd reduction(+ : s)
          for (int64_t k = 0; k < K; ++k) s += xa[k] * wb[k];
          acc[a][b] = s;
        }
      }
      for (int a = 0; a < 4; ++a) {
        if (t0 + a >= T) continue;
        for (int b = 0; b < 4; ++b) {
          if (o0 + b < O) Y[(t0 + a) * O + o0 + b] = acc[a][b];
        }
      }
    }
  }
}

static void rmsnorm(const float* x, int64_t T, int64_t H, float eps, int rb, float* y) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    double ss = 0;
    for (int64_t i = 0; i < H; ++i) ss += (double)x[t * H + i] * x[t * H + i];
    const float inv = 1.0f / sqrtf((float)(ss / (double)H) + eps);
    for (int64_t i = 0; i < H; ++i) {
      const float v = x[t * H + i] * inv; /* gamma = 1 */
      y[t * H + i] = rb ? bf16_round(v) : v;
    }
  }
}

static void rope_rows(float* q, int64_t T, int heads, int hd, const int64_t* pos, float theta) {
  const int half = hd / 2;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    for (int h = 0; h < heads; ++h) {
      float* v = q + t * (int64_t)heads * hd + (int64_t)h * hd;
      for (int j = 0; j < half; ++j) {
        const float inv_freq = powf(theta, -(float)(2 * j) / (float)hd);
        const float ang = (float)pos[t] * inv_freq;
        const float c = cosf(ang), s = sinf(ang);
        const float x1 = v[j], x2 = v[j + half];
        v[j] = x1 * c - x2 * s;
        v[j + half] = x2 * c + x1 * s;
      }
    }
  }
}

typedef struct {
  float *wq, *wk, *wv, *wo, *wg, *wu, *wd;
} layer_w;

typedef struct {
  llama_cfg c;
  float *emb, *lm;
  layer_w* L;
  float **kc, **vc; /* per layer KV cache [cap x H] */
  int64_t cap, len;
  int rb;
} model;

static void model_init(model* m, const llama_cfg* c, int64_t cap, int rb) {
  m->c = *c;
  m->rb = rb;
  const int64_t H = c->hidden, F = c->ffn, V = c->vocab;
  m->emb = make_weight(c, T_EMBED, 0, V, H);
  m->lm = make_weight(c, T_LM, 0, V, H);
  m->L = (layer_w*)calloc((size_t)c->layers, sizeof(layer_w));
  m->kc = (float**)calloc((size_t)c->layers, sizeof(float*));
  m->vc = (float**)calloc((size_t)c->layers, sizeof(float*));
  for (int l = 0; l < c->layers; ++l) {
    m->L[l].wq = make_weight(c, T_Q, l, H, H);
    m->L[l].wk = make_weight(c, T_K, l, H, H);
    m->L[l].wv = make_weight(c, T_V, l, H, H);
    m->L[l].wo = make_weight(c, T_O, l, H, H);
    m->L[l].wg = make_weight(c, T_GATE, l, F, H);
    m->L[l].wu = make_weight(c, T_UP, l, F, H);
    m->L[l].wd = make_weight(c, T_DOWN, l, H, F);
    m->kc[l] = (float*)malloc(sizeof(float) * cap * H);
    m->vc[l] = (float*)malloc(sizeof(float) * cap * H);
  }
  m->cap = cap;
  m->len = 0;
}

static void model_free(model* m) {
  free(m->emb);
  free(m->lm);
  for (int l = 0; l < m->c.layers; ++l) {
    free(m->L[l].wq); free(m->L[l].wk); free(m->L[l].wv); free(m->L[l].wo);
    free(m->L[l].wg); free(m->L[l].wu); free(m->L[l].wd);
    free(m->kc[l]); free(m->vc[l]);
  }
  free(m->L);
  free(m->kc);
  free(m->vc);
}

/* Causal softmax attention of nq query rows (absolute positions qpos[],
 * ascending; row i sees keys 0..qpos[i]) against the cache K/V [* x H]:
 * per (head, row) s_j = q.k_j / sqrt(hd), p_j = exp(s_j - max) (two-pass,
 * exact max), o = sum_j p_j v_j / sum_j p_j, rounded to bf16 when rb.
 * Blocked for the CPU (the GPU path's tiling is irrelevant here): the keys of
 * one head are transposed once to [hd][nk] so a block of query rows computes
 * its scores vectorised over keys, and P.V vectorised over the head dim with
 * each V row read once per block. */
#define ATT_RB 16
#define ATT_KC 64
static void attend(const float* q, int64_t nq, const int64_t* qpos, const float* K,
                   const float* V, int64_t H, int heads, int hd, int rb, float* out) {
  if (nq <= 0) return;
  const int64_t nk = qpos[nq - 1] + 1;
  if (nq < ATT_RB) { /* decode-sized: keys read row by row, no transpose */
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t r = 0; r < nq; ++r) {
      for (int h = 0; h < heads; ++h) {
        const int64_t kr = qpos[r] + 1;
        const float* qv = q + r * H + (int64_t)h * hd;
        float* sc = (float*)malloc(sizeof(float) * kr);
        const float scale = 1.0f / sqrtf((float)hd);
        float mx = -3.0e38f;
        for (int64_t j = 0; j < kr; ++j) {
          const float* kv = K + j * H + (int64_t)h * hd;
          float acc = 0.f;
#pragma omp simd reduction(+ : acc)
          for (int d = 0; d < hd; ++d) acc += qv[d] * kv[d];
          sc[j] = acc * scale;
          mx = sc[j] > mx ? sc[j] : mx;
        }
        double sum = 0;
        for (int64_t j = 0; j < kr; ++j) {
          sc[j] = expf(sc[j] - mx);
          sum += sc[j];
        }
        float o[128];
        for (int d = 0; d < hd; ++d) o[d] = 0.f;
        for (int64_t j = 0; j < kr; ++j) {
          const float p = sc[j];
          const float* vv = V + j * H + (int64_t)h * hd;
#pragma omp simd
          for (int d = 0; d < hd; ++d) o[d] += p * vv[d];
        }
        float* dst = out + r * H + (int64_t)h * hd;
        const double inv = 1.0 / sum;
        for (int d = 0; d < hd; ++d) {
          const float v = (float)(o[d] * inv);
          dst[d] = rb ? bf16_round(v) : v;
        }
        free(sc);
      }
    }
    return;
  }
  const int64_t nkp = (nk + ATT_KC - 1) / ATT_KC * ATT_KC;
  float* KT = (float*)malloc(sizeof(float) * (size_t)heads * hd * nkp);
#pragma omp parallel for collapse(2) schedule(static)
  for (int h = 0; h < heads; ++h) {
    for (int d = 0; d < hd; ++d) {
      float* dst = KT + ((int64_t)h * hd + d) * nkp;
      for (int64_t j = 0; j < nk; ++j) dst[j] = K[j * H + (int64_t)h * hd + d];
      for (int64_t j = nk; j < nkp; ++j) dst[j] = 0.f;
    }
  }
  const float scale = 1.0f / sqrtf((float)hd);
  const int64_t nb = (nq + ATT_RB - 1) / ATT_RB;
#pragma omp parallel
  {
    float* sc = (float*)malloc(sizeof(float) * ATT_RB * nkp);
#pragma omp for collapse(2) schedule(dynamic, 1)
    for (int64_t bi = nb - 1; bi >= 0; --bi) { /* dearest (latest) blocks first */
      for (int h = 0; h < heads; ++h) {
        const int64_t r0 = bi * ATT_RB;
        const int64_t r1 = r0 + ATT_RB < nq ? r0 + ATT_RB : nq;
        const int64_t kmax = qpos[r1 - 1] + 1;
        const float* kt = KT + (int64_t)h * hd * nkp;
        double inv[ATT_RB];
        for (int64_t r = r0; r < r1; ++r) {
          const float* qv = q + r * H + (int64_t)h * hd;
          float* srow = sc + (r - r0) * nkp;
          const int64_t kr = qpos[r] + 1;
          for (int64_t j0 = 0; j0 < kr; j0 += ATT_KC) {
            float acc[ATT_KC];
            for (int jj = 0; jj < ATT_KC; ++jj) acc[jj] = 0.f;
            for (int d = 0; d < hd; ++d) {
              const float qd = qv[d];
              const float* kd = kt + (int64_t)d * nkp + j0;
#pragma omp simd
              for (int jj = 0; jj < ATT_KC; ++jj) acc[jj] += qd * kd[jj];
            }
            for (int jj = 0; jj < ATT_KC; ++jj) srow[j0 + jj] = acc[jj] * scale;
          }
          float mx = -3.0e38f;
          for (int64_t j = 0; j < kr; ++j) mx = srow[j] > mx ? srow[j] : mx;
          double sum = 0;
          for (int64_t j = 0; j < kr; ++j) {
            srow[j] = expf(srow[j] - mx);
            sum += srow[j];
          }
          for (int64_t j = kr; j < kmax; ++j) srow[j] = 0.f; /* causal: unseen keys */
          inv[r - r0] = 1.0 / sum;
        }
        float o[ATT_RB][128];
        for (int64_t r = r0; r < r1; ++r) {
          for (int d = 0; d < hd; ++d) o[r - r0][d] = 0.f;
        }
        for (int64_t j = 0; j < kmax; ++j) {
          const float* vv = V + j * H + (int64_t)h * hd;
          for (int64_t r = r0; r < r1; ++r) {
            const float p = sc[(r - r0) * nkp + j];
            float* orow = o[r - r0];
#pragma omp simd
            for (int d = 0; d < hd; ++d) orow[d] += p * vv[d];
          }
        }
        for (int64_t r = r0; r < r1; ++r) {
          float* dst = out + r * H + (int64_t)h * hd;
          for (int d = 0; d < hd; ++d) {
            const float v = (float)(o[r - r0][d] * inv[r - r0]);
            dst[d] = rb ? bf16_round(v) : v;
          }
        }
      }
    }
    free(sc);
  }
  free(KT);
}

/* Optional per-call captures of a prefill (parity at BASELINE sizes):
 *   attn[l][i][:]   attention output (pre O-proj) of the row at position
 *                   attn_pos[i] in layer l            (n_attn rows, nullable)
 *   kcap/vcap[l][i] the cached K (after RoPE) / V of the row at kv_pos[i]
 *                   in layer l                         (n_kv rows, nullable)
 * With `last_only`, the LAST layer computes queries, attention, O and MLP
 * only for the captured rows and the final row (logits need nothing else);
 * every earlier layer is computed in full. */
typedef struct {
  int64_t n_attn;
  const int64_t* attn_pos;
  float* attn;
  int64_t n_kv;
  const int64_t* kv_pos;
  float* kcap;
  float* vcap;
  int last_only;
} probe_t;

/* Runs T new tokens (positions len..len+T-1) through the model, appending
 * their K/V; writes fp32 logits of the LAST new token into `logits`. */
static void forward(model* m, const int32_t* tok, int64_t T, float* logits, const probe_t* pr) {
  const llama_cfg* c = &m->c;
  const int64_t H = c->hidden, F = c->ffn, V = c->vocab;
  const int heads = c->heads, hd = c->head_dim;
  const int rb = m->rb;
  const int64_t p0 = m->len, T0 = T;
  float* x = (float*)malloc(sizeof(float) * T * H);
  float* xn = (float*)malloc(sizeof(float) * T * H);
  float* q = (float*)malloc(sizeof(float) * T * H);
  float* k = (float*)malloc(sizeof(float) * T * H);
  float* v = (float*)malloc(sizeof(float) * T * H);
  float* att = (float*)malloc(sizeof(float) * T * H);
  float* tmp = (float*)malloc(sizeof(float) * T * H);
  float* g = (float*)malloc(sizeof(float) * T * F);
  float* u = (float*)malloc(sizeof(float) * T * F);
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * T);
  int64_t* sel = (int64_t*)malloc(sizeof(int64_t) * (T + 1)); /* last-layer rows (local) */
  int64_t* selpos = (int64_t*)malloc(sizeof(int64_t) * (T + 1));
  for (int64_t t = 0; t < T; ++t) {
    pos[t] = p0 + t;
    memcpy(x + t * H, m->emb + (int64_t)tok[t] * H, sizeof(float) * H);
  }
  for (int l = 0; l < c->layers; ++l) {
    layer_w* w = &m->L[l];
    const int partial = pr && pr->last_only && l == c->layers - 1 && T > 1;
    /* rows whose queries / outputs this layer needs (all, or the probes + last) */
    int64_t ns = 0;
    if (partial) {
      char* want = (char*)calloc((size_t)T, 1);
      for (int64_t i = 0; i < pr->n_attn; ++i) {
        const int64_t t = pr->attn_pos[i] - p0;
        if (t >= 0 && t < T) want[t] = 1;
      }
      want[T - 1] = 1;
      for (int64_t t = 0; t < T; ++t) {
        if (want[t]) sel[ns++] = t;
      }
      free(want);
    } else {
      for (int64_t t = 0; t < T; ++t) sel[ns++] = t;
    }
    for (int64_t i = 0; i < ns; ++i) selpos[i] = pos[sel[i]];
    rmsnorm(x, T, H, c->rms_eps, rb, xn);
    gemm_nt(xn, T, H, w->wk, H, k);
    gemm_nt(xn, T, H, w->wv, H, v);
    rope_rows(k, T, heads, hd, pos, c->rope_theta);
    if (partial) { /* compact the selected rows */
      for (int64_t i = 0; i < ns; ++i) {
        memmove(xn + i * H, xn + sel[i] * H, sizeof(float) * H);
        memmove(x + i * H, x + sel[i] * H, sizeof(float) * H);
      }
    }
    gemm_nt(xn, ns, H, w->wq, H, q);
    rope_rows(q, ns, heads, hd, selpos, c->rope_theta);
    if (rb) {
      for (int64_t i = 0; i < ns * H; ++i) q[i] = bf16_round(q[i]);
      for (int64_t i = 0; i < T * H; ++i) {
        k[i] = bf16_round(k[i]);
        v[i] = bf16_round(v[i]);
      }
    }
    memcpy(m->kc[l] + p0 * H, k, sizeof(float) * T * H);
    memcpy(m->vc[l] + p0 * H, v, sizeof(float) * T * H);
    if (pr && pr->n_kv > 0 && pr->kcap) {
      for (int64_t i = 0; i < pr->n_kv; ++i) {
        const int64_t p = pr->kv_pos[i];
        memcpy(pr->kcap + ((int64_t)l * pr->n_kv + i) * H, m->kc[l] + p * H, sizeof(float) * H);
        memcpy(pr->vcap + ((int64_t)l * pr->n_kv + i) * H, m->vc[l] + p * H, sizeof(float) * H);
      }
    }
    attend(q, ns, selpos, m->kc[l], m->vc[l], H, heads, hd, rb, att);
    if (pr && pr->n_attn > 0 && pr->attn) {
      for (int64_t i = 0; i < pr->n_attn; ++i) {
        for (int64_t j = 0; j < ns; ++j) {
          if (selpos[j] == pr->attn_pos[i]) {
            memcpy(pr->attn + ((int64_t)l * pr->n_attn + i) * H, att + j * H, sizeof(float) * H);
            break;
          }
        }
      }
    }
    int64_t nr = ns;
    const float* a_in = att;
    if (partial) { /* only the final row continues to the logits */
      memmove(x, x + (ns - 1) * H, sizeof(float) * H);
      a_in = att + (ns - 1) * H;
      nr = 1;
    }
    gemm_nt(a_in, nr, H, w->wo, H, tmp);
    for (int64_t i = 0; i < nr * H; ++i) {
      const float r = x[i] + tmp[i];
      x[i] = rb ? bf16_round(r) : r;
    }
    rmsnorm(x, nr, H, c->rms_eps, rb, xn);
    gemm_nt(xn, nr, H, w->wg, F, g);
    gemm_nt(xn, nr, H, w->wu, F, u);
    for (int64_t i = 0; i < nr * F; ++i) {
      const float a = g[i] / (1.0f + expf(-g[i])) * u[i];
      g[i] = rb ? bf16_round(a) : a;
    }
    gemm_nt(g, nr, F, w->wd, H, tmp);
    for (int64_t i = 0; i < nr * H; ++i) {
      const float r = x[i] + tmp[i];
      x[i] = rb ? bf16_round(r) : r;
    }
    if (partial) T = 1; /* x now holds the final row only */
  }
  rmsnorm(x + (T - 1) * H, 1, H, c->rms_eps, rb, xn);
  gemm_nt(xn, 1, H, m->lm, V, logits);
  m->len = p0 + T0;
  free(x); free(xn); free(q); free(k); free(v); free(att); free(tmp); free(g); free(u);
  free(pos); free(sel); free(selpos);
}

static int32_t argmax(const float* l, int64_t V) {
  int64_t b = 0;
  for (int64_t i = 1; i < V; ++i) {
    if (l[i] > l[b]) b = i;
  }
  return (int32_t)b;
}

/* Prefill `prompt` (S tokens), then n_steps decode steps. Step s feeds
 * forced[s-1] when forced != NULL (teacher forcing on the GPU's tokens), else
 * the oracle's own previous greedy token. out_tokens[0..n_steps] and
 * out_logits[(n_steps+1) x vocab] (nullable) hold each step's greedy token
 * and logits. Returns 0. */
int llama_ref_generate(const llama_cfg* c, const int32_t* prompt, int64_t S, int n_steps,
                       const int32_t* forced, int emulate_bf16, int32_t* out_tokens,
                       float* out_logits, int n_threads) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  model m;
  model_init(&m, c, S + n_steps + 1, emulate_bf16);
  float* lg = (float*)malloc(sizeof(float) * c->vocab);
  forward(&m, prompt, S, lg, NULL);
  out_tokens[0] = argmax(lg, c->vocab);
  if (out_logits) memcpy(out_logits, lg, sizeof(float) * c->vocab);
  for (int s = 1; s <= n_steps; ++s) {
    int32_t in = forced ? forced[s - 1] : out_tokens[s - 1];
    forward(&m, &in, 1, lg, NULL);
    out_tokens[s] = argmax(lg, c->vocab);
    if (out_logits) memcpy(out_logits + (int64_t)s * c->vocab, lg, sizeof(float) * c->vocab);
  }
  free(lg);
  model_free(&m);
  return 0;
}

/* Prefill only, with captures (see probe_t): attention outputs of the rows at
 * attn_pos[n_attn] and the cached K/V rows at kv_pos[n_kv], per layer
 * ([layers][n][hidden] fp32, nullable). last_only: the last layer computes
 * only the captured rows and the final one. Writes the final row's logits
 * (nullable) and returns its greedy token. */
int32_t llama_ref_prefill_probe(const llama_cfg* c, const int32_t* prompt, int64_t S,
                                int emulate_bf16, int64_t n_attn, const int64_t* attn_pos,
                                float* attn_out, int64_t n_kv, const int64_t* kv_pos,
                                float* k_out, float* v_out, int last_only, float* logits_out,
                                int n_threads) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  model m;
  model_init(&m, c, S, emulate_bf16);
  float* lg = (float*)malloc(sizeof(float) * c->vocab);
  probe_t pr = {n_attn, attn_pos, attn_out, n_kv, kv_pos, k_out, v_out, last_only};
  forward(&m, prompt, S, lg, &pr);
  const int32_t tok = argmax(lg, c->vocab);
  if (logits_out) memcpy(logits_out, lg, sizeof(float) * c->vocab);
  free(lg);
  model_free(&m);
  return tok;
}

static float bf16_to_f32(uint16_t h) {
  const uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* One decode step at position n_ctx for a request whose KV cache is GIVEN
 * (bf16 [layers][n_ctx][hidden], token order, after RoPE) — the teacher-
 * forced check of multi-master decoding: the cache is read back from the
 * device, so the step's arithmetic (q, split-KV attention + LSE combine
 * across instances, O, MLP, LM head) is checked on its own. Outputs (each
 * nullable): logits [vocab], the step's new K/V rows [layers][hidden] and
 * attention outputs [layers][hidden]. Returns the greedy token. */
int32_t llama_ref_decode_cached(const llama_cfg* c, int64_t n_ctx, const uint16_t* k_cache,
                                const uint16_t* v_cache, int32_t token, int emulate_bf16,
                                float* logits_out, float* k_new, float* v_new, float* attn_out,
                                int n_threads) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  model m;
  model_init(&m, c, n_ctx + 1, emulate_bf16);
  const int64_t H = c->hidden;
  for (int l = 0; l < c->layers; ++l) {
    const uint16_t* ks = k_cache + (int64_t)l * n_ctx * H;
    const uint16_t* vs = v_cache + (int64_t)l * n_ctx * H;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_ctx * H; ++i) {
      m.kc[l][i] = bf16_to_f32(ks[i]);
      m.vc[l][i] = bf16_to_f32(vs[i]);
    }
  }
  m.len = n_ctx;
  float* lg = (float*)malloc(sizeof(float) * c->vocab);
  int64_t at = n_ctx;
  float* kc = k_new ? k_new : (float*)malloc(sizeof(float) * c->layers * H);
  float* vc = v_new ? v_new : (float*)malloc(sizeof(float) * c->layers * H);
  probe_t pr = {attn_out ? 1 : 0, &at, attn_out, 1, &at, kc, vc, 0};
  forward(&m, &token, 1, lg, &pr);
  const int32_t tok = argmax(lg, c->vocab);
  if (logits_out) memcpy(logits_out, lg, sizeof(float) * c->vocab);
  if (!k_new) free(kc);
  if (!v_new) free(vc);
  free(lg);
  model_free(&m);
  return tok;
}

/* CPU decode baseline (bench.py cpu_baseline.decode): one decode step of a
 * batch of `batch` requests, each over its own n_ctx-token cache (random bf16
 * values; every request reads n_ctx x layers x 2 rows, as on the GPU), the
 * model built once outside the timed region. Returns the wall ms of one
 * step (all requests, all layers, LM head) or -1. */
double llama_ref_decode_sample(const llama_cfg* c, int64_t n_ctx, int batch, int n_threads) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  model m;
  model_init(&m, c, n_ctx + 1, 0);
  const int64_t H = c->hidden;
  for (int l = 0; l < c->layers; ++l) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_ctx * H; ++i) {
      const uint64_t h = splitmix64((uint64_t)i ^ ((uint64_t)l << 40));
      m.kc[l][i] = bf16_round((float)(int32_t)(h & 0xFFFF) / 32768.0f - 1.0f);
      m.vc[l][i] = bf16_round((float)(int32_t)((h >> 16) & 0xFFFF) / 32768.0f - 1.0f);
    }
  }
  float* lg = (float*)malloc(sizeof(float) * c->vocab);
  const double t0 = omp_get_wtime();
  for (int b = 0; b < batch; ++b) {
    m.len = n_ctx;
    int32_t tok = (int32_t)(b * 7919 % c->vocab);
    forward(&m, &tok, 1, lg, NULL);
  }
  const double ms = (omp_get_wtime() - t0) * 1e3;
  free(lg);
  model_free(&m);
  return ms;
}

int llama_ref_max_threads(void) { return omp_get_max_threads(); }
