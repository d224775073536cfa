/*
 * px_oracle.c -- fp64 restatement of the PixArt-alpha block variant
 * run under the reference's PipeFusion schedule.
 * TEST INFRASTRUCTURE ONLY: used by tests/ as the checker for the GPU
 * `block=pixart` path; never linked into the product.
 *
 * The reference (/root/reference/proj) has no PixArt semantics: its toy
 * block is toy_model.cpp:145-177. This file keeps everything of the
 * reference's run loop (run_pipefusion_inline, execute.cpp:167-223: warmup,
 * patch order, in-place K/V row writes, staleness accounting, sampler
 * x -= eta*eps, h = x_j + condition_bias) and swaps the block for the
 * PixArt-alpha DiT block (arXiv 2310.00426 §2.3 / the public PixArtBlock):
 *
 *   shift1, scale1, gate1, shift2, scale2, gate2 = sst[l] + tv(t)   (adaLN-single)
 *   a  = LN(h) * (1 + scale1) + shift1                  (LN: no affine, eps 1e-6)
 *   q, k, v = a Wqkv + bqkv          k, v rows written in place at row0
 *   h += gate1 * (attention(q, K_full, V_full) Wo + bo)
 *   h += attention(h Wqc + bqc, Kc, Vc) Woc + boc       (cross-attention, Kc/Vc
 *                                                        = y Wkc + bkc, y Wvc + bvc)
 *   a2 = LN(h) * (1 + scale2) + shift2
 *   h += gate2 * (gelu_tanh(a2 W1 + b1) W2 + b2)
 *
 * Timestep embedding (DiT/PixArt t_embedder + t_block), at timestep index t
 * of a run of S steps: tau = 1000 t / S; sinusoid(tau) [256]
 * = [cos(tau f_i), sin(tau f_i)], f_i = exp(-ln(10000) i / 128);
 * temb = silu(sinusoid Wt1 + bt1) Wt2 + bt2; tv = silu(temb) Wt0 + bt0 [6 hs].
 *
 * Parameters come from one mt19937_64 stream seeded with seed ^ PX_SEED_XOR,
 * drawn as U[-1,1) = (rng() >> 11) 2^-52 - 1 (the reference's next_uniform,
 * toy_model.cpp:28-30), row-major in the order listed in px_build below;
 * matrices are scaled by 1/sqrt(fan_in), biases by 0.1, sst by 1/sqrt(hs),
 * condition_bias by 1. The text tokens y [T x hs] are U[-1,1) from
 * seed ^ PX_TEXT_XOR.
 */
#include "pf_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define PX_SEED_XOR 0x5049584152542d41ULL /* "PIXART-A" */
#define PX_TEXT_XOR 0x5458542d544f4b53ULL /* "TXT-TOKS" */
#define PX_FREQ 256

/* ---- mt19937_64 (same generator as pf_oracle.c, kept file-local) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} px_mt;

static void px_seed(px_mt* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t px_next(px_mt* r) {
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

static void px_fill(px_mt* r, double* m, size_t n, double scale) {
  for (size_t i = 0; i < n; ++i) m[i] = ((double)(px_next(r) >> 11) * 0x1.0p-52 - 1.0) * scale;
}

/* ---- model ---- */
enum {
  PX_WQKV, PX_BQKV, PX_WO, PX_BO, PX_WQC, PX_BQC, PX_WKC, PX_BKC, PX_WVC, PX_BVC,
  PX_WOC, PX_BOC, PX_W1, PX_B1, PX_W2, PX_B2, PX_SST, PX_NPARAM
};

struct pxo_model {
  int layers, hs, heads, mlp, T;
  size_t off[PX_NPARAM + 1]; /* per-layer parameter offsets */
  double* w;                 /* layers * off[PX_NPARAM] */
  double *wt1, *bt1, *wt2, *bt2, *wt0, *bt0, *cb;
  double* y;  /* [T x hs] text tokens */
  double* kc; /* per layer [T x hs] */
  double* vc;
};

static size_t px_param_size(int id, int hs, int mlp) {
  const size_t h = (size_t)hs, m = (size_t)mlp;
  switch (id) {
    case PX_WQKV: return h * 3 * h;
    case PX_BQKV: return 3 * h;
    case PX_W1: return h * m;
    case PX_B1: return m;
    case PX_W2: return m * h;
    case PX_SST: return 6 * h;
    case PX_WO: case PX_WQC: case PX_WKC: case PX_WVC: case PX_WOC: return h * h;
    default: return h; /* biases of width hs */
  }
}

static double px_param_scale(int id, int hs, int mlp) {
  switch (id) {
    case PX_WQKV: case PX_WO: case PX_WQC: case PX_WKC: case PX_WVC: case PX_WOC: case PX_W1:
      return 1.0 / sqrt((double)hs);
    case PX_W2: return 1.0 / sqrt((double)mlp);
    case PX_SST: return 1.0 / sqrt((double)hs);
    default: return 0.1;
  }
}

const double* pxo_param(const pxo_model* m, int layer, int id) {
  return m->w + m->off[PX_NPARAM] * (size_t)layer + m->off[id];
}

const double* pxo_global(const pxo_model* m, int id) {
  switch (id) {
    case 0: return m->wt1;
    case 1: return m->bt1;
    case 2: return m->wt2;
    case 3: return m->bt2;
    case 4: return m->wt0;
    case 5: return m->bt0;
    case 6: return m->cb;
    default: return m->y;
  }
}

int pxo_mlp_hidden(const pxo_model* m) { return m->mlp; }

static void mm(const double* x, int64_t rows, int64_t k, const double* w, int64_t n,
               const double* bias, double* out) {
  pfo_matmul_rows(x, rows, k, w, n, out);
  if (bias)
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t c = 0; c < n; ++c) out[i * n + c] += bias[c];
}

static void px_cross_kv(pxo_model* m) {
  const size_t th = (size_t)m->T * m->hs;
  for (int l = 0; l < m->layers; ++l) {
    mm(m->y, m->T, m->hs, pxo_param(m, l, PX_WKC), m->hs, pxo_param(m, l, PX_BKC), m->kc + th * l);
    mm(m->y, m->T, m->hs, pxo_param(m, l, PX_WVC), m->hs, pxo_param(m, l, PX_BVC), m->vc + th * l);
  }
}

pxo_model* pxo_build(uint64_t seed, int layers, int hs, int heads, double mlp_ratio, int T) {
  if (layers < 1 || hs < 1 || heads < 1 || hs % heads != 0 || T < 1) return NULL;
  const int mlp = (int)lround(mlp_ratio * hs);
  if (mlp < 1) return NULL;
  pxo_model* m = (pxo_model*)calloc(1, sizeof(pxo_model));
  m->layers = layers;
  m->hs = hs;
  m->heads = heads;
  m->mlp = mlp;
  m->T = T;
  m->off[0] = 0;
  for (int i = 0; i < PX_NPARAM; ++i) m->off[i + 1] = m->off[i] + px_param_size(i, hs, mlp);
  m->w = (double*)malloc(m->off[PX_NPARAM] * (size_t)layers * sizeof(double));
  const size_t h = (size_t)hs;
  m->wt1 = (double*)malloc(PX_FREQ * h * sizeof(double));
  m->bt1 = (double*)malloc(h * sizeof(double));
  m->wt2 = (double*)malloc(h * h * sizeof(double));
  m->bt2 = (double*)malloc(h * sizeof(double));
  m->wt0 = (double*)malloc(h * 6 * h * sizeof(double));
  m->bt0 = (double*)malloc(6 * h * sizeof(double));
  m->cb = (double*)malloc(h * sizeof(double));
  m->y = (double*)malloc((size_t)T * h * sizeof(double));
  m->kc = (double*)malloc((size_t)layers * T * h * sizeof(double));
  m->vc = (double*)malloc((size_t)layers * T * h * sizeof(double));
  px_mt r;
  px_seed(&r, seed ^ PX_SEED_XOR);
  for (int l = 0; l < layers; ++l)
    for (int i = 0; i < PX_NPARAM; ++i)
      px_fill(&r, m->w + m->off[PX_NPARAM] * (size_t)l + m->off[i], px_param_size(i, hs, mlp),
              px_param_scale(i, hs, mlp));
  px_fill(&r, m->wt1, PX_FREQ * h, 1.0 / sqrt((double)PX_FREQ));
  px_fill(&r, m->bt1, h, 0.1);
  px_fill(&r, m->wt2, h * h, 1.0 / sqrt((double)hs));
  px_fill(&r, m->bt2, h, 0.1);
  px_fill(&r, m->wt0, h * 6 * h, 1.0 / sqrt((double)hs));
  px_fill(&r, m->bt0, 6 * h, 0.1);
  px_fill(&r, m->cb, h, 1.0);
  px_mt rt;
  px_seed(&rt, seed ^ PX_TEXT_XOR);
  px_fill(&rt, m->y, (size_t)T * h, 1.0);
  px_cross_kv(m);
  return m;
}

void pxo_set_text(pxo_model* m, const double* y) {
  memcpy(m->y, y, (size_t)m->T * m->hs * sizeof(double));
  px_cross_kv(m);
}

void pxo_free(pxo_model* m) {
  if (!m) return;
  free(m->w);
  free(m->wt1); free(m->bt1); free(m->wt2); free(m->bt2); free(m->wt0); free(m->bt0);
  free(m->cb); free(m->y); free(m->kc); free(m->vc);
  free(m);
}

static double silu(double x) { return x / (1.0 + exp(-x)); }

/* tv(t) [6 hs] for timestep index t of a run of `steps` steps. */
void pxo_tvec(const pxo_model* m, int t, int steps, double* tv) {
  const int hs = m->hs;
  double sin_[PX_FREQ];
  const double tau = 1000.0 * (double)t / (double)steps;
  for (int i = 0; i < PX_FREQ / 2; ++i) {
    const double f = exp(-log(10000.0) * (double)i / (double)(PX_FREQ / 2));
    sin_[i] = cos(tau * f);
    sin_[PX_FREQ / 2 + i] = sin(tau * f);
  }
  double* e1 = (double*)malloc((size_t)hs * sizeof(double));
  double* e2 = (double*)malloc((size_t)hs * sizeof(double));
  mm(sin_, 1, PX_FREQ, m->wt1, hs, m->bt1, e1);
  for (int i = 0; i < hs; ++i) e1[i] = silu(e1[i]);
  mm(e1, 1, hs, m->wt2, hs, m->bt2, e2);
  for (int i = 0; i < hs; ++i) e2[i] = silu(e2[i]);
  mm(e2, 1, hs, m->wt0, 6 * hs, m->bt0, tv);
  free(e1);
  free(e2);
}

/* a = LN(h) * (1 + scale) + shift, per row (biased variance, eps 1e-6). */
static void ln_modulate(const double* h, int64_t rows, int hs, const double* shift,
                        const double* scale, double* a) {
  for (int64_t i = 0; i < rows; ++i) {
    const double* hr = h + i * hs;
    double mu = 0.0, var = 0.0;
    for (int c = 0; c < hs; ++c) mu += hr[c];
    mu /= hs;
    for (int c = 0; c < hs; ++c) var += (hr[c] - mu) * (hr[c] - mu);
    var /= hs;
    const double rstd = 1.0 / sqrt(var + 1e-6);
    for (int c = 0; c < hs; ++c) a[i * hs + c] = (hr[c] - mu) * rstd * (1.0 + scale[c]) + shift[c];
  }
}

static double gelu_tanh(double x) {
  const double k = 0.7978845608028654; /* sqrt(2/pi) */
  return 0.5 * x * (1.0 + tanh(k * (x + 0.044715 * x * x * x)));
}

/* One PixArt block over rows [row0, row0+rows) (see the header). mod = sst[l] + tv. */
void pxo_layer_forward_mod(const pxo_model* m, int l, const double* mod, double* h,
                           int64_t rows, double* kbuf, double* vbuf, int64_t p, int64_t row0) {
  const int hs = m->hs, mlp = m->mlp;
  const size_t rh = (size_t)rows * hs;
  const double *shift1 = mod, *scale1 = mod + hs, *gate1 = mod + 2 * hs;
  const double *shift2 = mod + 3 * hs, *scale2 = mod + 4 * hs, *gate2 = mod + 5 * hs;
  double* a = (double*)malloc(rh * sizeof(double));
  double* qkv = (double*)malloc(rh * 3 * sizeof(double));
  double* q = (double*)malloc(rh * sizeof(double));
  double* o = (double*)malloc(rh * sizeof(double));
  double* t = (double*)malloc(rh * sizeof(double));
  double* z = (double*)malloc((size_t)rows * mlp * sizeof(double));

  ln_modulate(h, rows, hs, shift1, scale1, a);
  mm(a, rows, hs, pxo_param(m, l, PX_WQKV), 3 * hs, pxo_param(m, l, PX_BQKV), qkv);
  for (int64_t i = 0; i < rows; ++i)
    for (int c = 0; c < hs; ++c) {
      q[i * hs + c] = qkv[i * 3 * hs + c];
      kbuf[(row0 + i) * hs + c] = qkv[i * 3 * hs + hs + c];
      vbuf[(row0 + i) * hs + c] = qkv[i * 3 * hs + 2 * hs + c];
    }
  pfo_attention_rows(q, rows, kbuf, vbuf, p, hs, m->heads, o);
  mm(o, rows, hs, pxo_param(m, l, PX_WO), hs, pxo_param(m, l, PX_BO), t);
  for (size_t i = 0; i < rh; ++i) h[i] += gate1[i % hs] * t[i];

  const size_t th = (size_t)m->T * hs;
  mm(h, rows, hs, pxo_param(m, l, PX_WQC), hs, pxo_param(m, l, PX_BQC), q);
  pfo_attention_rows(q, rows, m->kc + th * l, m->vc + th * l, m->T, hs, m->heads, o);
  mm(o, rows, hs, pxo_param(m, l, PX_WOC), hs, pxo_param(m, l, PX_BOC), t);
  for (size_t i = 0; i < rh; ++i) h[i] += t[i];

  ln_modulate(h, rows, hs, shift2, scale2, a);
  mm(a, rows, hs, pxo_param(m, l, PX_W1), mlp, pxo_param(m, l, PX_B1), z);
  for (size_t i = 0; i < (size_t)rows * mlp; ++i) z[i] = gelu_tanh(z[i]);
  mm(z, rows, mlp, pxo_param(m, l, PX_W2), hs, pxo_param(m, l, PX_B2), t);
  for (size_t i = 0; i < rh; ++i) h[i] += gate2[i % hs] * t[i];

  free(a); free(qkv); free(q); free(o); free(t); free(z);
}

static void layer_mod(const pxo_model* m, int l, const double* tv, double* mod) {
  const double* sst = pxo_param(m, l, PX_SST);
  for (int i = 0; i < 6 * m->hs; ++i) mod[i] = sst[i] + tv[i];
}

void pxo_layer_forward(const pxo_model* m, int l, int t, int steps, double* h, int64_t rows,
                       double* kbuf, double* vbuf, int64_t p, int64_t row0) {
  double* tv = (double*)malloc(6 * (size_t)m->hs * sizeof(double));
  double* mod = (double*)malloc(6 * (size_t)m->hs * sizeof(double));
  pxo_tvec(m, t, steps, tv);
  layer_mod(m, l, tv, mod);
  pxo_layer_forward_mod(m, l, mod, h, rows, kbuf, vbuf, p, row0);
  free(tv);
  free(mod);
}

static int px_finite(const double* h, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(h[i])) return 0;
  return 1;
}

static void set_err(char* err, int cap, const char* msg) {
  if (err && cap > 0) {
    strncpy(err, msg, (size_t)cap - 1);
    err[cap - 1] = 0;
  }
}

/* serial_reference (toy_model.cpp:201-214) with the PixArt block. */
int pxo_serial(const pxo_model* m, const double* x_in, int64_t p, int steps, double eta,
               double* out, char* err, int cap) {
  if (steps < 1) {
    set_err(err, cap, "serial_reference needs steps >= 1");
    return 2;
  }
  const int hs = m->hs;
  const size_t n = (size_t)p * hs;
  double* h = (double*)malloc(n * sizeof(double));
  double* kb = (double*)malloc(n * sizeof(double));
  double* vb = (double*)malloc(n * sizeof(double));
  double* tv = (double*)malloc(6 * (size_t)hs * sizeof(double));
  double* mod = (double*)malloc(6 * (size_t)hs * sizeof(double));
  memcpy(out, x_in, n * sizeof(double));
  int rc = 0;
  for (int t = steps - 1; t >= 0 && rc == 0; --t) {
    pxo_tvec(m, t, steps, tv);
    for (int64_t i = 0; i < p; ++i)
      for (int c = 0; c < hs; ++c) h[i * hs + c] = out[i * hs + c] + m->cb[c];
    memset(kb, 0, n * sizeof(double));
    memset(vb, 0, n * sizeof(double));
    for (int l = 0; l < m->layers; ++l) {
      layer_mod(m, l, tv, mod);
      pxo_layer_forward_mod(m, l, mod, h, p, kb, vb, p, 0);
      if (!px_finite(h, n)) {
        char b[160];
        snprintf(b, sizeof b, "non-finite activation at timestep %d, layer %d", t, l);
        set_err(err, cap, b);
        rc = 1;
        break;
      }
    }
    if (rc) break;
    for (size_t i = 0; i < n; ++i) out[i] = out[i] - eta * h[i];
  }
  free(h); free(kb); free(vb); free(tv); free(mod);
  return rc;
}

/* run_pipefusion_inline (execute.cpp:97-223) with the PixArt block; same
 * schedule, staleness accounting and sampler as pfo_pipefusion. */
int pxo_pipefusion(const pxo_model* m, const double* x_in, int64_t p, int steps, int workers,
                   int patches, int warmup, double eta, double* out, int64_t* fresh_out,
                   int64_t* stale_out, char* err, int cap) {
  char b[200];
  if (steps < 1) { set_err(err, cap, "steps must be >= 1"); return 2; }
  if (workers < 1 || patches < 1) { set_err(err, cap, "workers and patches must be >= 1"); return 2; }
  if (warmup < 0 || warmup > steps) { set_err(err, cap, "warmup must lie in [0, steps]"); return 2; }
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
  const int hs = m->hs, L = m->layers;
  const int64_t r = p / patches;
  const size_t n = (size_t)p * hs;
  const int steady = steps - warmup;
  double* x = out;
  memcpy(x, x_in, n * sizeof(double));
  double* kb = (double*)calloc(n * (size_t)L, sizeof(double));
  double* vb = (double*)calloc(n * (size_t)L, sizeof(double));
  int* src = (int*)malloc(sizeof(int) * (size_t)L * patches);
  for (int i = 0; i < L * patches; ++i) src[i] = steps;
  double* h = (double*)malloc(n * sizeof(double));
  double* eps = (double*)calloc(n, sizeof(double));
  double* pending = (double*)calloc(n, sizeof(double));
  double* tv = (double*)malloc(6 * (size_t)hs * sizeof(double));
  double* mod = (double*)malloc(6 * (size_t)hs * sizeof(double));
  int64_t fresh = 0, stale = 0;
  int rc = 0;
  (void)workers;

  for (int w = 0; w < warmup && rc == 0; ++w) {
    const int t = steps - 1 - w;
    pxo_tvec(m, t, steps, tv);
    for (int64_t i = 0; i < p; ++i)
      for (int c = 0; c < hs; ++c) h[i * hs + c] = x[i * hs + c] + m->cb[c];
    for (int l = 0; l < L && rc == 0; ++l) {
      for (int pi = 0; pi < patches; ++pi) src[l * patches + pi] = t;
      fresh += patches;
      layer_mod(m, l, tv, mod);
      pxo_layer_forward_mod(m, l, mod, h, p, kb + n * l, vb + n * l, p, 0);
      if (!px_finite(h, n)) {
        snprintf(b, sizeof b, "non-finite activation at timestep %d, layer %d", t, l);
        set_err(err, cap, b);
        rc = 1;
      }
    }
    if (rc) break;
    for (size_t i = 0; i < n; ++i) x[i] = x[i] - eta * h[i];
  }
  for (int q = 0; q < steady && rc == 0; ++q) {
    const int t = steady - 1 - q;
    pxo_tvec(m, t, steps, tv);
    for (int j = 0; j < patches && rc == 0; ++j) {
      const size_t off = (size_t)j * r * hs, cnt = (size_t)r * hs;
      if (q > 0)
        for (size_t i = 0; i < cnt; ++i) x[off + i] = x[off + i] - eta * pending[off + i];
      for (int64_t i = 0; i < r; ++i)
        for (int c = 0; c < hs; ++c) h[i * hs + c] = x[off + i * hs + c] + m->cb[c];
      for (int l = 0; l < L && rc == 0; ++l) {
        int* sv = src + l * patches;
        sv[j] = t;
        for (int pi = 0; pi < patches; ++pi) {
          if (sv[pi] == t) ++fresh;
          else if (sv[pi] == t + 1) ++stale;
          else {
            snprintf(b, sizeof b,
                     "staleness bound violated: patch %d carries timestep %d while computing "
                     "timestep %d", pi, sv[pi], t);
            set_err(err, cap, b);
            rc = 1;
            break;
          }
        }
        if (rc) break;
        layer_mod(m, l, tv, mod);
        pxo_layer_forward_mod(m, l, mod, h, r, kb + n * l, vb + n * l, p, (int64_t)j * r);
        if (!px_finite(h, cnt)) {
          snprintf(b, sizeof b, "non-finite activation at timestep %d, layer %d", t, l);
          set_err(err, cap, b);
          rc = 1;
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
  free(kb); free(vb); free(src); free(h); free(eps); free(pending); free(tv); free(mod);
  return rc;
}
