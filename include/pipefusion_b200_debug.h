/*
 * pipefusion_b200_debug.h -- kernel-level test entry points (device pointers).
 *
 * Not part of the drop-in boundary: these exist so the unit tests can check a
 * single sm_100a kernel against a plain fp32 computation of the same op.
 *   pf_debug_gemm       <- ditsim::matmul_rows      (toy_model.cpp:93-102)
 *   pf_debug_attention  <- ditsim::attention_rows   (toy_model.cpp:104-143)
 */
#ifndef PIPEFUSION_B200_DEBUG_H_
#define PIPEFUSION_B200_DEBUG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C[r, n] = sum_k A[row0 + r, k] * B[n, k] for r < rows, n < N.
 * A: bf16 [total_rows x K] row-major, B: bf16 [N x K] row-major,
 * C: fp32 [rows x N] (row r of the block at C + r*N).
 * Returns 0 on success, else a cudaError_t value. */
int pf_debug_gemm(const void* A, const void* B, float* C, int rows, int row0,
                  int total_rows, int N, int K, void* stream);

/* Attention of query rows [row0, row0+rows) of q against all P rows of k/v.
 * q, k, v: bf16 [P x hs] row-major (head h = columns [h*dh, (h+1)*dh)).
 * out: bf16 [P x hs] (rows [row0, row0+rows) written).
 * Returns 0 on success, else a cudaError_t value. */
int pf_debug_attention(const void* q, const void* k, const void* v, void* out,
                       int P, int rows, int row0, int heads, int hs,
                       void* stream);
/* Same with the production V layout for padded head dims (dh < dhp): the
 * row-sum column (V column dh = 1, AttnLaunch::v_sum_col) when v_sum_col. */
int pf_debug_attention_ex(const void* q, const void* k, const void* v, void* out,
                          int P, int rows, int row0, int heads, int hs, void* stream,
                          int v_sum_col);

/* Debug timeline: enable=1 allocates a device trace buffer that subsequent
 * pf_debug_attention launches fill with clock64 stamps of CTA (0,0,0);
 * host (8192 uint64, may be NULL) receives the current contents; enable=0
 * frees it. */
int pf_debug_attention_trace(int enable, unsigned long long* host);
// Per-CTA timeline (8 slots x 256 CTAs, globaltimer ns) of the 1-SM GEMM
// kernel launches that follow; debug instrumentation, not part of the product.
int pf_debug_gemm_trace(int enable, unsigned long long* host);
// Host only (no GPU): the attention schedule the library picks for a launch of
// `rows` query rows over `P` KV rows (the 128-row-block kernel). out[7] =
// {query-tile groups per head, KV blocks per item, units, persistent CTAs,
// items cut (0/1), merged in-kernel (0/1), whole items round-robin (0/1)}.
int pf_debug_attn_schedule(int P, int rows, int heads, int dhp, int sm_count, long long* out);

/* Failure injection for the channel-close tests (rank mode): ctx's next runs
 * throw when its plan loop reaches op `op` (-1 disables), after which the
 * rank closes the pipeline (pf_rank_reset reopens it). ctx is a pf_ctx*.
 * Returns a pf_status value. */
struct pf_ctx;
int pf_debug_fail_at(struct pf_ctx* ctx, int op);
/* Makes global layer `layer`'s out-projection weight NaN (non-finite
 * activations from that layer on). Returns a pf_status value. */
int pf_debug_poison_layer(struct pf_ctx* ctx, int layer);

#ifdef __cplusplus
}
#endif

#endif
