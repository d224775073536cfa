// Internal launch API of the sm_100a kernels (host side). Not part of the
// C ABI: the runtime (runtime.cpp) and the debug entry points use it.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

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

enum class Epi : int { StoreF32 = 0, QKV = 1, Residual = 2, Tanh = 3 };

struct EpiParams {
  // StoreF32: out_f32[row*ld + n] = acc
  // Residual: h = out_f32[row*ld + n] + acc; out_f32 = h; out_bf16 = bf16(h);
  //           non-finite h -> atomicMin(flag, code)
  // Tanh:     out_bf16[row*ld + n] = bf16(tanh(acc))
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
  const CUtensorMap* tm_h32 = nullptr;
  const CUtensorMap* tm_hb = nullptr;
};

// Tensor maps over a weight B [N x K] (K-major bf16) for both GEMM paths:
// one_sm: box 64 x gemm_bn_1sm(N); two_sm: box 64 x gemm_bn_2sm(N)/2.
struct WeightMaps {
  CUtensorMap one_sm;
  CUtensorMap two_sm;
  CUtensorMap two_sm_128;  // box 64 x 64: CTA-pair tiles of N = 128 (residual GEMMs)
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
struct AttnLaunch {
  int dhp, P, rows, row0, heads, dh, hs;
  float scale;           // 1/sqrt(dh)
  bf16* out;             // [P][hs]
  float* work;           // split-KV partials (may be null if splits == 1)
  size_t work_floats;    // capacity of `work`
  unsigned long long* trace = nullptr;  // debug timeline (see AttnParams)
};
int attn_splits(const AttnLaunch& a, int sm_count);
size_t attn_work_floats(int dhp, int heads, int rows, int splits);
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
// hb[i] = bf16(h32[i]), i < n
cudaError_t to_bf16(const float* h32, bf16* hb, size_t n, cudaStream_t stream);
// Device-side finite-check flag reset: *flag = INT_MAX
cudaError_t reset_flag(int* flag, cudaStream_t stream);

}  // namespace pf
