/*
 * pf_oracle.c -- plain-C restatement of the reference's PipeFusion hot path.
 * TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
 * bench.py's CPU baseline as the checker; never linked into the product.
 *
 * Every function cites the reference source it restates
 * (/root/reference/proj/src/...). Arithmetic is the same scalar sequence as
 * the reference so results are bitwise identical (pinned by
 * tests/test_oracle.py against oracle/_ref, the reference itself).
 */
#include "pf_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG */
/* std::mt19937_64 (the standard's parameters), as seeded by the reference. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* next_uniform, toy_model.cpp:28-30 */
static double next_uniform(mt64* r) {
  return (double)(mt64_next(r) >> 11) * 0x1.0p-52 - 1.0;
}

/* fill_matrix, toy_model.cpp:32-40 (row-major traversal) */
static void fill_matrix(mt64* r, double* m, int rows, int cols, double scale) {
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m[(size_t)i * cols + j] = next_uniform(r) * scale;
}

/* ---------------------------------------------------------------- model */
struct pfo_model {
  int layers, hs, heads, mlp;
  double* w;  /* per layer: wq, wk, wv, wo, win, wout back to back */
  double* cb; /* [hs] */
};

static size_t layer_stride(const pfo_model* m) {
  return 4 * (size_t)m->hs * m->hs + 2 * (size_t)m->hs * m->mlp;
}

static void set_err(char* err, int cap, const char* msg) {
  if (err && cap > 0) {
    strncpy(err, msg, (size_t)cap - 1);
    err[cap - 1] = 0;
  }
}

/* build_toy_model, toy_model.cpp:44-82 */
pfo_model* pfo_build(uint64_t seed, int layers, int hs, int heads, double mlp_ratio,
                     char* err, int cap) {
  if (layers < 1) {
    set_err(err, cap, "toy model needs layers >= 1");
    return NULL;
  }
  if (hs < 1 || heads < 1) {
    set_err(err, cap, "toy model needs hidden_size >= 1 and heads >= 1");
    return NULL;
  }
  if (hs % heads != 0) {
    char b[160];
    snprintf(b, sizeof b, "hidden_size (%d) must be divisible by heads (%d)", hs, heads);
    set_err(err, cap, b);
    return NULL;
  }
  const int mlp = (int)lround(mlp_ratio * hs);
  if (mlp < 1) {
    set_err(err, cap, "mlp_ratio * hidden_size must be >= 1");
    return NULL;
  }
  pfo_model* m = (pfo_model*)calloc(1, sizeof(pfo_model));
  m->layers = layers;
  m->hs = hs;
  m->heads = heads;
  m->mlp = mlp;
  m->w = (double*)malloc(layer_stride(m) * (size_t)layers * sizeof(double));
  m->cb = (double*)malloc((size_t)hs * sizeof(double));
  mt64 r;
  mt64_seed(&r, seed);
  const double scale = 1.0 / sqrt((double)hs);
  for (int l = 0; l < layers; ++l) {
    for (int i = 0; i < 6; ++i) {
      const int rows = i == 5 ? mlp : hs;
      const int cols = i == 4 ? mlp : hs;
      fill_matrix(&r, (double*)pfo_weight(m, l, i), rows, cols, scale);
    }
  }
  fill_matrix(&r, m->cb, 1, hs, 1.0);
  return m;
}

void pfo_free(pfo_model* m) {
  if (!m) return;
  free(m->w);
  free(m->cb);
  free(m);
}

int pfo_mlp_hidden(const pfo_model* m) { return m->mlp; }

const double* pfo_weight(const pfo_model* m, int layer, int idx) {
  const size_t hh = (size_t)m->hs * m->hs, hm = (size_t)m->hs * m->mlp;
  const size_t off[6] = {0, hh, 2 * hh, 3 * hh, 4 * hh, 4 * hh + hm};
  return m->w + layer_stride(m) * (size_t)layer + off[idx];
}

const double* pfo_condition_bias(const pfo_model* m) { return m->cb; }

/* n values of next_uniform (toy_model.cpp:28-30) from mt19937_64(seed): the
 * raw stream test specs build their parameters from. */
void pfo_uniform_stream(uint64_t seed, int64_t n, double* out) {
  mt64 r;
  mt64_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = next_uniform(&r);
}

/* make_initial_latent, toy_model.cpp:84-91 */
void pfo_latent(uint64_t seed, int64_t p, int hs, double* out) {
  mt64 r;
  mt64_seed(&r, seed ^ 0x9e3779b97f4a7c15ULL);
  fill_matrix(&r, out, (int)p, hs, 1.0);
}

/* ---------------------------------------------------------------- kernels */
/* matmul_rows, toy_model.cpp:93-102: strict left-to-right k, product rounded
 * then added (out.row(i) += x(i,k) * w.row(k)). */
void pfo_matmul_rows(const double* x, int64_t rows, int64_t k, const double* w,
                     int64_t n, double* out) {
  for (int64_t i = 0; i < rows; ++i) {
    double* o = out + i * n;
    for (int64_t c = 0; c < n; ++c) o[c] = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) {
      const double s = x[i * k + kk];
      const double* wr = w + kk * n;
      for (int64_t c = 0; c < n; ++c) {
        const double t = s * wr[c];
        o[c] = o[c] + t;
      }
    }
  }
}

/* attention_rows, toy_model.cpp:104-143 */
void pfo_attention_rows(const double* q, int64_t rows, const double* kf,
                        const double* vf, int64_t kv_rows, int64_t hs, int heads,
                        double* out) {
  const int64_t dh = hs / heads;
  const double inv_sqrt_dh = 1.0 / sqrt((double)dh);
  double* scores = (double*)malloc((size_t)(kv_rows > 0 ? kv_rows : 1) * sizeof(double));
  double* acc = (double*)malloc((size_t)(dh > 0 ? dh : 1) * sizeof(double));
  for (int64_t i = 0; i < rows; ++i) {
    for (int h = 0; h < heads; ++h) {
      const int64_t c0 = (int64_t)h * dh;
      double score_max = -INFINITY;
      for (int64_t j = 0; j < kv_rows; ++j) {
        double s = 0.0;
        for (int64_t d = 0; d < dh; ++d) s += q[i * hs + c0 + d] * kf[j * hs + c0 + d];
        s *= inv_sqrt_dh;
        scores[j] = s;
        if (s > score_max) score_max = s;
      }
      double z = 0.0;
      for (int64_t d = 0; d < dh; ++d) acc[d] = 0.0;
      for (int64_t j = 0; j < kv_rows; ++j) {
        const double e = exp(scores[j] - score_max);
        z += e;
        for (int64_t d = 0; d < dh; ++d) acc[d] += e * vf[j * hs + c0 + d];
      }
      for (int64_t d = 0; d < dh; ++d) out[i * hs + c0 + d] = acc[d] / z;
    }
  }
  free(scores);
  free(acc);
}

static void add_inplace(double* h, const double* t, size_t n) {
  for (size_t i = 0; i < n; ++i) h[i] = h[i] + t[i];
}

/* toy_layer_forward = toy_layer_project (toy_model.cpp:145-149), the
 * in-place K/V row write (:174-175) and toy_layer_finish (:151-167). */
static void layer_forward_p(const pfo_model* m, int layer, double* h, int64_t rows,
                            double* kbuf, double* vbuf, int64_t p, int64_t row0) {
  const int64_t hs = m->hs, mlp = m->mlp;
  const size_t rh = (size_t)rows * hs;
  double* q = (double*)malloc(rh * sizeof(double));
  double* a = (double*)malloc(rh * sizeof(double));
  double* t = (double*)malloc(rh * sizeof(double));
  double* z = (double*)malloc((size_t)rows * mlp * sizeof(double));
  pfo_matmul_rows(h, rows, hs, pfo_weight(m, layer, 0), hs, q);
  pfo_matmul_rows(h, rows, hs, pfo_weight(m, layer, 1), hs, kbuf + row0 * hs);
  pfo_matmul_rows(h, rows, hs, pfo_weight(m, layer, 2), hs, vbuf + row0 * hs);
  pfo_attention_rows(q, rows, kbuf, vbuf, p, hs, m->heads, a);
  pfo_matmul_rows(a, rows, hs, pfo_weight(m, layer, 3), hs, t);
  add_inplace(h, t, rh);
  pfo_matmul_rows(h, rows, hs, pfo_weight(m, layer, 4), mlp, z);
  for (size_t i = 0; i < (size_t)rows * mlp; ++i) z[i] = tanh(z[i]);
  pfo_matmul_rows(z, rows, mlp, pfo_weight(m, layer, 5), hs, t);
  add_inplace(h, t, rh);
  free(q);
  free(a);
  free(t);
  free(z);
}

void pfo_layer_forward(const pfo_model* m, int layer, double* h, int64_t rows,
                       double* kbuf, double* vbuf, int64_t p, int64_t row0) {
  layer_forward_p(m, layer, h, rows, kbuf, vbuf, p, row0);
}

static int all_finite(const double* h, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(h[i])) return 0;
  return 1;
}

/* toy_forward, toy_model.cpp:182-197 (scratch buffers per call) */
static int toy_forward(const pfo_model* m, const double* x, int64_t p, int timestep,
                       double* h, char* err, int cap) {
  const int64_t hs = m->hs;
  const size_t n = (size_t)p * hs;
  double* kb = (double*)calloc(n, sizeof(double));
  double* vb = (double*)calloc(n, sizeof(double));
  for (int64_t i = 0; i < p; ++i)
    for (int64_t c = 0; c < hs; ++c) h[i * hs + c] = x[i * hs + c] + m->cb[c];
  int rc = 0;
  for (int l = 0; l < m->layers; ++l) {
    layer_forward_p(m, l, h, p, kb, vb, p, 0);
    if (!all_finite(h, n)) {
      char b[160];
      snprintf(b, sizeof b, "non-finite activation at timestep %d, layer %d", timestep, l);
      set_err(err, cap, b);
      rc = 1;
      break;
    }
  }
  free(kb);
  free(vb);
  return rc;
}

/* serial_reference, toy_model.cpp:201-214 */
int pfo_serial(const pfo_model* m, const double* x_in, int64_t p, int steps, double eta,
               double* out, char* err, int cap) {
  if (steps < 1) {
    set_err(err, cap, "serial_reference needs steps >= 1");
    return 2;
  }
  const size_t n = (size_t)p * m->hs;
  double* h = (double*)malloc(n * sizeof(double));
  memcpy(out, x_in, n * sizeof(double));
  int rc = 0;
  for (int t = steps - 1; t >= 0 && rc == 0; --t) {
    rc = toy_forward(m, out, p, t, h, err, cap);
    if (rc) break;
    for (size_t i = 0; i < n; ++i) out[i] = out[i] - eta * h[i];
  }
  free(h);
  return rc;
}

/* ---------------------------------------------------------------- pipefusion */
/* check_pipefusion_args (execute.cpp:97-131) + run_pipefusion_inline
 * (execute.cpp:167-223) with stage_forward_full/_patch (:134-165) and the
 * staleness accounting (:51-73). */
int pfo_pipefusion(const pfo_model* m, const double* x_in, int64_t p, int steps,
                   int workers, int patches, int warmup, double eta, double* out,
                   int64_t* fresh_out, int64_t* stale_out, double* ff, int64_t ff_cap,
                   char* err, int cap) {
  char b[200];
  if (steps < 1) { set_err(err, cap, "steps must be >= 1"); return 2; }
  if (workers < 1 || patches < 1) {
    set_err(err, cap, "workers and patches must be >= 1");
    return 2;
  }
  if (warmup < 0 || warmup > steps) {
    set_err(err, cap, "warmup must lie in [0, steps]");
    return 2;
  }
  if (m->layers % workers != 0) {
    snprintf(b, sizeof b, "layer count %d is not divisible by workers %d", m->layers, workers);
    set_err(err, cap, b);
    return 2;
  }
  if (p % patches != 0) {
    snprintf(b, sizeof b, "seq_len %lld is not divisible by patches %d", (long long)p, patches);
    set_err(err, cap, b);
    return 2;
  }
  const int64_t hs = m->hs;
  const int lps = m->layers / workers;
  const int64_t r = p / patches;
  const size_t n = (size_t)p * hs;
  const int L = m->layers;
  const int steady = steps - warmup;

  double* x = out;
  memcpy(x, x_in, n * sizeof(double));
  double* kb = (double*)calloc(n * (size_t)L, sizeof(double));
  double* vb = (double*)calloc(n * (size_t)L, sizeof(double));
  int* src = (int*)malloc(sizeof(int) * (size_t)L * patches);
  for (int i = 0; i < L * patches; ++i) src[i] = steps; /* sentinel */
  double* h = (double*)malloc(n * sizeof(double));
  double* eps = (double*)calloc(n, sizeof(double));
  double* pending = (double*)calloc(n, sizeof(double));
  const int64_t per_worker = (int64_t)patches * steady;
  int64_t fresh = 0, stale = 0;
  int rc = 0;

  for (int w = 0; w < warmup && rc == 0; ++w) {
    const int t = steps - 1 - w;
    for (int64_t i = 0; i < p; ++i)
      for (int64_t c = 0; c < hs; ++c) h[i * hs + c] = x[i * hs + c] + m->cb[c];
    for (int d = 0; d < workers && rc == 0; ++d) {
      for (int lf = 0; lf < lps; ++lf) {
        const int l = d * lps + lf;
        for (int pi = 0; pi < patches; ++pi) src[l * patches + pi] = t;
        fresh += patches;
        layer_forward_p(m, l, h, p, kb + n * l, vb + n * l, p, 0);
        if (!all_finite(h, n)) {
          snprintf(b, sizeof b, "non-finite activation at timestep %d, layer %d", t, l);
          set_err(err, cap, b);
          rc = 1;
          break;
        }
      }
    }
    if (rc) break;
    for (size_t i = 0; i < n; ++i) x[i] = x[i] - eta * h[i];
  }

  for (int q = 0; q < steady && rc == 0; ++q) {
    const int t = steady - 1 - q;
    for (int j = 0; j < patches && rc == 0; ++j) {
      const size_t off = (size_t)j * r * hs, cnt = (size_t)r * hs;
      if (q > 0)
        for (size_t i = 0; i < cnt; ++i) x[off + i] = x[off + i] - eta * pending[off + i];
      for (int64_t i = 0; i < r; ++i)
        for (int64_t c = 0; c < hs; ++c) h[i * hs + c] = x[off + i * hs + c] + m->cb[c];
      for (int d = 0; d < workers && rc == 0; ++d) {
        for (int lf = 0; lf < lps; ++lf) {
          const int l = d * lps + lf;
          int* sv = src + l * patches;
          sv[j] = t;
          for (int pi = 0; pi < patches; ++pi) {
            if (sv[pi] == t) ++fresh;
            else if (sv[pi] == t + 1) ++stale;
            else {
              snprintf(b, sizeof b,
                       "staleness bound violated: patch %d carries timestep %d while "
                       "computing timestep %d", pi, sv[pi], t);
              set_err(err, cap, b);
              rc = 1;
              break;
            }
          }
          if (rc) break;
          layer_forward_p(m, l, h, r, kb + n * l, vb + n * l, p, (int64_t)j * r);
          if (!all_finite(h, cnt)) {
            snprintf(b, sizeof b, "non-finite activation at timestep %d, layer %d", t, l);
            set_err(err, cap, b);
            rc = 1;
            break;
          }
        }
        if (rc) break;
        /* fresh_fraction(src[first local layer], t), execute.cpp:67-73,164 */
        {
          const int* s0 = src + (d * lps) * patches;
          int f = 0;
          for (int pi = 0; pi < patches; ++pi) f += (s0[pi] == t);
          const int64_t k = (int64_t)d * per_worker + (int64_t)q * patches + j;
          if (ff && k < ff_cap) ff[k] = (double)f / (double)patches;
        }
      }
      if (rc) break;
      memcpy(eps + off, h, cnt * sizeof(double));
    }
    if (rc) break;
    memcpy(pending, eps, n * sizeof(double));
  }
  if (rc == 0 && steady > 0)
    for (size_t i = 0; i < n; ++i) x[i] = x[i] - eta * pending[i];

  if (fresh_out) *fresh_out = fresh;
  if (stale_out) *stale_out = stale;
  free(kb);
  free(vb);
  free(src);
  free(h);
  free(eps);
  free(pending);
  return rc;
}

/* divergence, toy_model.cpp:216-228. Norms summed in column-major order,
 * the traversal of the Eigen-shim build of the reference (oracle/_ref). */
static double colmajor_sqnorm_diff(const double* a, const double* b, int64_t rows,
                                   int64_t cols) {
  double s = 0.0;
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) {
      const double d = b ? a[r * cols + c] - b[r * cols + c] : a[r * cols + c];
      s += d * d;
    }
  return s;
}

double pfo_divergence(const double* a, const double* b, int64_t rows, int64_t cols) {
  const double den = sqrt(colmajor_sqnorm_diff(b, NULL, rows, cols));
  if (den == 0.0) return NAN;
  return sqrt(colmajor_sqnorm_diff(a, b, rows, cols)) / den;
}

/* auto_warmup, toy_model.cpp:230-249 */
int pfo_auto_warmup(const pfo_model* m, const double* x_in, int64_t p, int steps,
                    double eta, double threshold, int* warmup, int* met) {
  const size_t n = (size_t)p * m->hs;
  double* x = (double*)malloc(n * sizeof(double));
  double* h = (double*)malloc(n * sizeof(double));
  double* nx = (double*)malloc(n * sizeof(double));
  memcpy(x, x_in, n * sizeof(double));
  *warmup = steps;
  *met = 0;
  for (int k = 1; k <= steps; ++k) {
    const int t = steps - k;
    if (toy_forward(m, x, p, t, h, NULL, 0)) break;
    for (size_t i = 0; i < n; ++i) nx[i] = x[i] - eta * h[i];
    const double denom = sqrt(colmajor_sqnorm_diff(x, NULL, p, m->hs));
    double change = 0.0;
    {
      double s = 0.0;
      for (int64_t c = 0; c < m->hs; ++c)
        for (int64_t r = 0; r < p; ++r) {
          const double d = nx[r * m->hs + c] - x[r * m->hs + c];
          s += d * d;
        }
      change = sqrt(s);
    }
    const double rel = denom > 0.0 ? change / denom : (change == 0.0 ? 0.0 : INFINITY);
    memcpy(x, nx, n * sizeof(double));
    if (rel < threshold) {
      *warmup = k;
      *met = 1;
      break;
    }
  }
  free(x);
  free(h);
  free(nx);
  return 0;
}

/* ---------------------------------------------------------------- schedule */
/* build_pipefusion_schedule, schedule.cpp:87-142 */
int pfo_schedule(int n, int m, int steps, int warmup, int* patch, int* timestep,
                 int* kind, int cap, int* warmup_slots, int* steady_slots) {
  if (n < 1 || m < 1 || steps < 1 || warmup < 0 || warmup > steps) return -1;
  const int steady = steps - warmup;
  const int stride = m > n ? m : n;
  const int ws = warmup * n * m;
  const int ss = steady > 0 ? (steady - 1) * stride + m + n - 1 : 0;
  const int cells = (ws + ss) * n;
  *warmup_slots = ws;
  *steady_slots = ss;
  if (cells > cap) return -1;
  for (int i = 0; i < cells; ++i) {
    patch[i] = -1;
    timestep[i] = -1;
    kind[i] = 2; /* Bubble */
  }
  for (int w = 0; w < warmup; ++w) {
    const int t = steps - 1 - w;
    for (int d = 0; d < n; ++d)
      for (int j = 0; j < m; ++j) {
        const int idx = (w * n * m + d * m + j) * n + d;
        patch[idx] = j;
        timestep[idx] = t;
        kind[idx] = 0;
      }
  }
  for (int q = 0; q < steady; ++q) {
    const int t = steady - 1 - q;
    for (int d = 0; d < n; ++d)
      for (int j = 0; j < m; ++j) {
        const int idx = (ws + d + q * stride + j) * n + d;
        patch[idx] = j;
        timestep[idx] = t;
        kind[idx] = 1;
      }
  }
  return cells;
}

/* fresh_area_series, freshness.cpp:35-75 (observer = lowest active device) */
int pfo_fresh_series(int n, int m, int steps, int warmup, double* out, int cap) {
  int ws, ss;
  const int total_cells = (warmup * n * m +
                           ((steps - warmup) > 0 ? (steps - warmup - 1) * (m > n ? m : n) + m + n - 1 : 0)) * n;
  int* patch = (int*)malloc(sizeof(int) * (size_t)(total_cells > 0 ? total_cells : 1));
  int* ts = (int*)malloc(sizeof(int) * (size_t)(total_cells > 0 ? total_cells : 1));
  int* kind = (int*)malloc(sizeof(int) * (size_t)(total_cells > 0 ? total_cells : 1));
  const int cells = pfo_schedule(n, m, steps, warmup, patch, ts, kind, total_cells, &ws, &ss);
  const int slots = cells < 0 ? 0 : cells / n;
  for (int s = 0; s < slots && s < cap; ++s) {
    int obs = -1;
    for (int d = 0; d < n; ++d)
      if (patch[s * n + d] >= 0) { obs = s * n + d; break; }
    int fresh = 0;
    for (int j = 0; j < m; ++j) {
      int age = 0;
      if (obs >= 0 && kind[obs] == 1) age = (j <= patch[obs]) ? 0 : 1;
      fresh += (age == 0);
    }
    out[s] = (double)fresh / m;
  }
  free(patch);
  free(ts);
  free(kind);
  return slots;
}
