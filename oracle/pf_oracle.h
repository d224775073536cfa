/*
 * pf_oracle.h -- plain-C restatement of the reference's PipeFusion path.
 * TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's CPU
 * baseline). Never linked into the product library.
 *
 * Pinned bit-for-bit against the reference itself (oracle/_ref, built from
 * /root/reference by oracle/Makefile) and against the reference's golden
 * values (tests/golden/).
 *
 * All matrices are row-major double.
 */
#ifndef PF_ORACLE_H_
#define PF_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pfo_model pfo_model;

/* build_toy_model, toy_model.cpp:44-82. Returns NULL on invalid shape (the
 * message is copied into err). */
pfo_model* pfo_build(uint64_t seed, int layers, int hs, int heads, double mlp_ratio,
                     char* err, int cap);
void pfo_free(pfo_model* m);
int pfo_mlp_hidden(const pfo_model* m);
/* idx: 0 w_q, 1 w_k, 2 w_v, 3 w_o [hs x hs], 4 w_mlp_in [hs x mlp],
 * 5 w_mlp_out [mlp x hs]; pointer into the model. */
const double* pfo_weight(const pfo_model* m, int layer, int idx);
const double* pfo_condition_bias(const pfo_model* m);

/* n next_uniform values of mt19937_64(seed) */
void pfo_uniform_stream(uint64_t seed, int64_t n, double* out);

/* make_initial_latent, toy_model.cpp:84-91 */
void pfo_latent(uint64_t seed, int64_t p, int hs, double* out);

/* matmul_rows, toy_model.cpp:93-102: out[rows x n] = x[rows x k] . w[k x n] */
void pfo_matmul_rows(const double* x, int64_t rows, int64_t k, const double* w,
                     int64_t n, double* out);
/* attention_rows, toy_model.cpp:104-143 */
void pfo_attention_rows(const double* q, int64_t rows, const double* kf,
                        const double* vf, int64_t kv_rows, int64_t hs, int heads,
                        double* out);
/* toy_layer_forward, toy_model.cpp:169-177 (h [rows x hs] in place; K/V
 * buffers [p x hs] receive rows [row0, row0+rows)). */
void pfo_layer_forward(const pfo_model* m, int layer, double* h, int64_t rows,
                       double* kbuf, double* vbuf, int64_t p, int64_t row0);

/* serial_reference, toy_model.cpp:201-214. Returns 0, 1 (numeric), 2 (validation). */
int pfo_serial(const pfo_model* m, const double* x, int64_t p, int steps, double eta,
               double* out, char* err, int cap);

/* run_pipefusion_inline, execute.cpp:97-223 (+ StalenessStats). ff receives
 * workers x patches*(steps-warmup) fresh fractions (worker-major). */
int pfo_pipefusion(const pfo_model* m, const double* x, int64_t p, int steps,
                   int workers, int patches, int warmup, double eta, double* out,
                   int64_t* fresh, int64_t* stale, double* ff, int64_t ff_cap,
                   char* err, int cap);

/* divergence, toy_model.cpp:216-228 (sequential-sum Frobenius norms). */
double pfo_divergence(const double* a, const double* b, int64_t rows, int64_t cols);

/* auto_warmup, toy_model.cpp:230-249 */
int pfo_auto_warmup(const pfo_model* m, const double* x, int64_t p, int steps,
                    double eta, double threshold, int* warmup, int* met);

/* build_pipefusion_schedule, schedule.cpp:87-142: fills slot-major grids of
 * total_slots x devices cells; returns the cell count (or -1 if cap too small). */
int pfo_schedule(int n, int m, int steps, int warmup, int* patch, int* timestep,
                 int* kind, int cap, int* warmup_slots, int* steady_slots);
/* fresh_area_series, freshness.cpp:64-75 */
int pfo_fresh_series(int n, int m, int steps, int warmup, double* out, int cap);


/* ---- PixArt-alpha block variant (px_oracle.c) ---- */
typedef struct pxo_model pxo_model;
/* Parameter ids per layer (x.W orientation, [in x out] row-major). */
enum {
  PXO_WQKV = 0, PXO_BQKV, PXO_WO, PXO_BO, PXO_WQC, PXO_BQC, PXO_WKC, PXO_BKC, PXO_WVC,
  PXO_BVC, PXO_WOC, PXO_BOC, PXO_W1, PXO_B1, PXO_W2, PXO_B2, PXO_SST
};
pxo_model* pxo_build(uint64_t seed, int layers, int hs, int heads, double mlp_ratio, int T);
void pxo_free(pxo_model* m);
int pxo_mlp_hidden(const pxo_model* m);
const double* pxo_param(const pxo_model* m, int layer, int id);
/* 0 wt1 [256 x hs], 1 bt1, 2 wt2 [hs x hs], 3 bt2, 4 wt0 [hs x 6hs], 5 bt0,
 * 6 condition_bias [hs], 7 text tokens y [T x hs] */
const double* pxo_global(const pxo_model* m, int id);
void pxo_set_text(pxo_model* m, const double* y);
void pxo_tvec(const pxo_model* m, int t, int steps, double* tv);
void pxo_layer_forward(const pxo_model* m, int layer, int t, int steps, double* h,
                       int64_t rows, double* kbuf, double* vbuf, int64_t p, int64_t row0);
int pxo_serial(const pxo_model* m, const double* x, int64_t p, int steps, double eta,
               double* out, char* err, int cap);
int pxo_pipefusion(const pxo_model* m, const double* x, int64_t p, int steps, int workers,
                   int patches, int warmup, double eta, double* out, int64_t* fresh,
                   int64_t* stale, char* err, int cap);

#ifdef __cplusplus
}
#endif

#endif
