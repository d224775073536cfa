// Internal launch API of the sm_100a kernels (host side). Not part of the
// C ABI: the runtime (runtime.cpp) and the debug entry points use it.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <utility>

namespace pf {

using bf16 = __nv_bfloat16;

// Tensor maps (cuTensorMapEncodeTiled via the runtime's driver entry point).
// 2-D bf16 tensor: `inner` contiguous elements per row, `outer` rows,
// `row_bytes` between rows. Box = box_inner x box_outer elements.
bool encode_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t inner,
                         uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                         uint32_t box_outer, int swizzle_bytes);

bool encode_tmap_f32_2d(CUtensorMap* map, const void* base, uint64_t inner,
                        uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                        uint32_t box_outer, int swizzle_bytes);

int device_sm_count(int device);

// Launch with programmatic dependent launch enabled (the kernel calls
// ptx::pdl_wait() before its first dependent memory access). PF_NO_PDL=1 in
// the environment turns the attribute off (plain stream serialisation).
bool pdl_enabled();
// Per-thread switch: launches enqueued by this thread skip PDL while set
// (patch lanes: early-launched CTAs waiting on their predecessor would hold
// SMs the other lanes could use).
bool& pdl_thread_off();
// Kernel launches issued by the calling thread. Every launch site in the
// library bumps it; the runtime reports per-run deltas (pf_last_launch_count).
int64_t& launch_counter();
cudaError_t set_gemm_trace(unsigned long long* buf);  // debug timeline (gemm_sm100.cuh)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++launch_counter();
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

enum class Epi : int { StoreF32 = 0, QKV = 1, Residual = 2, Tanh = 3, Gelu = 4, Fold = 5 };

struct EpiParams {
  // StoreF32: out_f32[row*ld + n] = acc
  // Residual: h = out_f32[row*ld + n] + acc; out_f32 = h; out_bf16 = bf16(h);
  //           non-finite h -> atomicMin(flag, code)
  // Tanh:     out_bf16[row*ld + n] = bf16(tanh(acc))
  // Fold:     out_f32[row*ld + n] = acc + (row odd ? bias[n] : 0)
  // QKV:      n in [0,hs): q, [hs,2hs): k, [2hs,3hs): v, each [heads][P][dhp]
  float* out_f32 = nullptr;
  bf16* out_bf16 = nullptr;
  int ld = 0;
  bf16* q = nullptr;
  bf16* k = nullptr;
  bf16* v = nullptr;
  int hs = 0, dh = 0, dhp = 0, P = 0;
  int* flag = nullptr;
  int code = 0;
  // Residual only: tensor maps over out_f32 (fp32, box 32 x 128, SW128) and
  // out_bf16 (bf16, box 64 x 128, SW128) enable the TMA epilogue.
  // 64-row box over the A operand (bf16, SW128): enables the 4-CTA-cluster
  // 2-SM kernel that multicasts A across N-adjacent tile pairs
  const CUtensorMap* a_half = nullptr;
  const CUtensorMap* tm_h32 = nullptr;
  const CUtensorMap* tm_hb = nullptr;
  // tm_h32 / tm_hb (and the _dst maps) end at row row0 + rows: a partial last
  // row tile may use the TMA epilogue (its stores are clipped by the maps)
  bool tma_clip = false;
  // Residual: write the updated rows (fp32 and bf16 copy) to these buffers /
  // maps instead of out_f32 / out_bf16 (which are still read): a stage's last
  // layer storing its output directly into the next stage's landing buffers.
  float* out_f32_dst = nullptr;
  bf16* out_bf16_dst = nullptr;
  const CUtensorMap* tm_h32_dst = nullptr;
  const CUtensorMap* tm_hb_dst = nullptr;
  // ---- PixArt block extensions (all optional) ----
  // Residual: h += gate[n] * (acc + bias[n]); out_bf16 = bf16(h * (1 + colscale[n]));
  //           stats_out[(n/32) * stats_ld + row] = (sum, sum of squares) of h
  //           over the chunk's 32 columns (LayerNorm statistics for the consumer).
  // QKV/Gelu: affine epilogue  y = a_row * acc + b_row * c1[n] + c2[n]  where,
  //           with stats_in, (a_row, b_row) = (rstd, -rstd * mean) of the A row
  //           (LayerNorm folded through the GEMM: the A operand holds
  //           h * (1 + scale) and c1 = (1 + scale) . W, c2 = shift . W + bias),
  //           else (1, 0); Gelu then applies gelu_tanh and stores bf16.
  const float* bias = nullptr;
  const float* gate = nullptr;
  const float* colscale = nullptr;
  float2* stats_out = nullptr;
  const float2* stats_in = nullptr;
  int stats_ld = 0;    // rows of the stats buffer (= P)
  int ln_cols = 0;     // LayerNorm width (hs): stats_in holds ln_cols / 32 chunks
  float ln_eps = 1e-6f;
  const float* c1 = nullptr;
  const float* c2 = nullptr;
  // Split-K workspace (fp32) and per-tile counters (zeroed, left zeroed by
  // the kernel) for skinny GEMMs; null disables split-K.
  float* splitk_ws = nullptr;
  size_t splitk_ws_floats = 0;
  int* splitk_counters = nullptr;
  int splitk_counter_cap = 0;
  bool mod() const { return bias || gate || colscale || stats_out; }
};

// Tensor maps over a weight B [N x K] (K-major bf16) for both GEMM paths:
// one_sm: box 64 x gemm_bn_1sm(N); two_sm: box 64 x gemm_bn_2sm(N)/2.
struct WeightMaps {
  CUtensorMap one_sm;
  CUtensorMap two_sm;
  CUtensorMap two_sm_res[3];  // box 64 x {64, 96, 128}: CTA-pair residual tiles BN 128/192/256
};
int gemm_bn_1sm(int N);
int gemm_bn_2sm(int N);
bool make_weight_maps(WeightMaps* maps, const bf16* w, int N, int K);

// D[rows x N] = A[row0 .. row0+rows, 0..K) . B[N x K]^T, epilogue `kind`.
// `a` is a tensor map over the whole A buffer (box 64 x 128, SW128). Row
// blocks of >= 256 rows use the 2-SM (CTA pair) kernel, smaller ones the
// 1-SM kernel.
cudaError_t gemm(const CUtensorMap& a, const WeightMaps& b, int rows, int row0,
                 int N, int K, Epi kind, const EpiParams& ep, int sm_count,
                 cudaStream_t stream);

// Attention of query rows [row0, row0+rows) against all P kv rows.
// stream-K attention: one merge flag per softmax warp of each CTA
constexpr int kAttnFlagsPerCta = 16;
constexpr int kAttnPrefetchRegions = 4;

struct AttnLaunch {
  // P: kv rows per head (buffer height); Q rows per head = q_stride (0 -> P)
  int dhp, P, rows, row0, heads, dh, hs;
  float scale;           // 1/sqrt(dh)
  bf16* out;             // [P][hs]
  float* work;           // split-KV partials (may be null if splits == 1)
  size_t work_floats;    // capacity of `work`
  unsigned long long* trace = nullptr;  // debug timeline (see AttnParams)
  int q_stride = 0;      // cross-attention: Q buffer [heads][q_stride][dhp]
  // DistriFusion: kv rows [fresh_lo, fresh_hi) (multiples of 128) come from
  // k2/v2 (this worker's fresh K/V), the rest from k/v (previous step)
  int fresh_lo = 0, fresh_hi = 0;
  const CUtensorMap* k2 = nullptr;
  const CUtensorMap* v2 = nullptr;
  // [sm_count * kAttnFlagsPerCta] zero-initialised flags for the in-kernel merge of cut items
  // (left zero after every launch); null -> merge in a separate kernel
  int* flags = nullptr;
  // weights of the following kernels to pull into L2 during the attention
  // (16-byte aligned regions; bytes 0 = unused)
  const void* prefetch[kAttnPrefetchRegions] = {};
  size_t prefetch_bytes[kAttnPrefetchRegions] = {};
  // K / V tensor maps with attn3_kv_rows(dhp)-row boxes: the triple-buffered
  // kernel (attn3_sm100.cuh) runs when present and no k2 / v2 is given
  const CUtensorMap* k3 = nullptr;
  const CUtensorMap* v3 = nullptr;
  // every V row (k/v, k2/v2) holds 1.0 in padding column dh (dh < dhp,
  // v_ones_col): the PV MMA then produces the softmax row sum in O column dh
  // and the softmax warps skip their per-element sum
  bool v_sum_col = false;
};
// KV rows per block of the kernel a launch uses (128, or 112 for the
// triple-buffered kernel) and the schedule for a given block size
int attn_block_rows(const AttnLaunch& a);
// KV rows per block (and K / V tensor-map box rows) of the triple-buffered kernel
int attn3_kv_rows(int dhp);
int attn_grid(const AttnLaunch& a, int sm_count, int bn = 128);
// The attention launch's schedule (host only): query-tile groups per head,
// KV blocks per item, units, persistent CTAs, whether items are cut and
// whether the cut items are merged in-kernel.
struct AttnSchedule {
  int nq = 0, blocks = 0, grid = 0;
  long long units = 0;
  bool cut = false, fused = false;
  // whole items dealt round-robin (CTA c: items c, c + grid, ...): the CTAs
  // running at one time then share a few heads' K/V, for launches whose K/V
  // exceed the L2 (stream-K's contiguous ranges would span every head at once)
  bool strided = false;
};
AttnSchedule attn_schedule(const AttnLaunch& a, int sm_count, int bn = 128);
// partial-result workspace the attention needs on a device with sm_count SMs
size_t attn_work_floats(int dhp, int sm_count);
cudaError_t attention(const CUtensorMap& q, const CUtensorMap& k,
                      const CUtensorMap& v, const AttnLaunch& a, int sm_count,
                      cudaStream_t stream);

// Sampler / patch split-merge (HBM-bound, vectorised).
// rows [row0, row0+rows) of [* x hs] fp32 matrices:
//   if (update) x -= eta * eps;  h32 = x + cb;  hb = bf16(h32)
cudaError_t patch_prepare(float* x, const float* eps, const float* cb,
                          float* h32, bf16* hb, int row0, int rows, int hs,
                          float eta, bool update, cudaStream_t stream);
// x[i] -= eta * src[i], i < n
cudaError_t latent_update(float* x, const float* src, float eta, size_t n,
                          cudaStream_t stream);
// fp64 host-layout latent (row- or column-major) <-> fp32 row-major device latent
cudaError_t latent_from_f64(const double* src, float* dst, int64_t rows, int cols, bool col_major,
                            cudaStream_t stream);
cudaError_t latent_to_f64(const float* src, double* dst, int64_t rows, int cols, bool col_major,
                          cudaStream_t stream);
// V buffers [rows][dhp] with dh < dhp: column dh = 1 (the attention's
// row-sum column, AttnLaunch::v_sum_col); the other padding columns stay 0
cudaError_t v_ones_col(bf16* v, size_t rows, int dhp, int dh, cudaStream_t stream);
// hb[i] = bf16(h32[i]), i < n
cudaError_t to_bf16(const float* h32, bf16* hb, size_t n, cudaStream_t stream);
// ---- PixArt block conditioning (pixart.cu) ----
// sinusoid(1000 t / S) rows for t < S: [S x 256] (cos | sin)
cudaError_t px_sinusoid(float* out, int S, cudaStream_t stream);
// out[s][n] = act(sum_k act(in[s][k]) W[n][k] + b[n]); W fp32 [N x K]
cudaError_t px_gemv(const float* in, int S, int K, const float* W, const float* b, int N,
                    float* out, bool silu_in, bool silu_out, cudaStream_t stream);
// mod[l][s][:] = sst[l][:] + tv[s][:]   (w6 = 6 hs)
cudaError_t px_mod(const float* sst, int nl, const float* tv, int S, int w6, float* mod,
                   cudaStream_t stream);
// GEMM operands of the LayerNorm fold (see pixart.cu): per local layer a
// [rpad x hs] bf16 block with rows 2s = 1 + scale_s, 2s+1 = shift_s, for the
// attention (aq: mod columns [0, 2hs)) and MLP (am: [3hs, 5hs)) branches.
// gemm(..., Epi::Fold) then gives c1 (row 2s) and c2 = shift . W + b (row 2s+1).
cudaError_t px_fold_rows(const float* mod, int nl, int S, int hs, bf16* aq, bf16* am,
                         int rpad, cudaStream_t stream);
// rows [row0, row0+rows): if (update) x -= eta eps; h32 = x + cb;
// hb = bf16(h32 (1 + scale)); stats[(c/32) stats_ld + row] = (sum, sum^2)
cudaError_t px_patch_prepare(float* x, const float* eps, const float* cb, const float* scale,
                             float* h32, bf16* hb, float2* stats, int stats_ld, int row0,
                             int rows, int hs, float eta, bool update, cudaStream_t stream);

// ---- MMDiT blocks (mmdit.cu; spec oracle/mmdit_oracle.py) ----
// key of tensor `tid` of a model seeded with `seed` (splitmix64 stream)
uint64_t mm_tensor_key(uint64_t seed, uint64_t tid);
// parameter tensor [K x N] (x.W orientation) -> kind 0: bf16 [N x K] (K-major),
// 1: fp32 [K x N] * scale, 2: fp32 1 + 0.1 u (gains), 3: fp32 [N x K] * scale
cudaError_t mm_fill(void* dst, uint64_t key, int64_t K, int64_t N, float scale, int kind,
                    cudaStream_t stream);
// out[s][n] (row pitch ld_out) = in[s] . W[n] + b[n], W bf16 [N x K], s < S
cudaError_t mm_gemv_bf16(const float* in, int S, int K, const bf16* W, const float* b, int N,
                         float* out, int ld_out, cudaStream_t stream);
// QK-norm (+ Flux RoPE) in place on joint rows [row0, row0+rows) of the
// head-major q [heads][q_rows][dhp] and k [heads][k_rows][dhp]
cudaError_t mm_qk_norm_rope(bf16* q, bf16* k, int heads, int q_rows, int k_rows, int dhp, int dh,
                            int row0, int rows, int J, const float* gq_img, const float* gk_img,
                            const float* gq_txt, const float* gk_txt, bool rope, int side,
                            cudaStream_t stream);

// Deterministic fp64 reductions (fixed grid and order), for auto_warmup and
// divergence (toy_model.cpp:216-249). `work`: sumsq_work_bytes() of scratch.
// out[0] = sum x^2, out[1] = sum (eta eps)^2  over n fp32 elements
size_t sumsq_work_bytes();
cudaError_t sumsq_latent(const float* x, const float* eps, double eta, size_t n, void* work,
                         double* out, cudaStream_t stream);
// out[0] = sum (a - b)^2, out[1] = sum b^2  over n fp64 elements
cudaError_t sumsq_diff(const double* a, const double* b, size_t n, void* work, double* out,
                       cudaStream_t stream);

// ---- fp32 parity mode (parity_f32.cu; CUDA cores, test infrastructure) ----
// C[M x N] (ldc) <- A[M x K] (lda) . B[K x N] (ldb), all fp32 row-major:
//   kF32Store: C = acc;  kF32Residual: C += acc (non-finite -> atomicMin(flag, code));
//   kF32Tanh: C = tanh(acc)
enum F32Epi : int { kF32Store = 0, kF32Residual = 1, kF32Tanh = 2 };
cudaError_t gemm_f32(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M,
                     int N, int K, int epi, int* flag, int code, cudaStream_t stream);
// rows query rows of q [rows x hs] against k, v [P x hs] (row-major, head h =
// columns [h dh, (h+1) dh)) -> out [rows x hs]
cudaError_t attention_f32(const float* q, const float* k, const float* v, float* out, int rows,
                          int P, int heads, int dh, int hs, float scale, cudaStream_t stream);

// Device-side finite-check flag reset: *flag = INT_MAX
cudaError_t reset_flag(int* flag, cudaStream_t stream);

}  // namespace pf
