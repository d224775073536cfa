// fp32 parity mode of the toy block (pf_create_toy_ex(..., PF_PRECISION_FP32)).
//
// The product path computes the toy layer (toy_model.cpp:145-177) with bf16
// tcgen05 GEMMs and attention (fp32 accumulation). At the benchmarked depth
// (28 layers) the reference's stale-K/V dynamics amplify bf16 operand
// rounding past the 1e-2 gate after one step (1.9e-2 at S=1),
// so the executor -- schedule, patch split/merge, in-place K/V row writes,
// sampler, stage hand-off -- is anchored at the C2 shape with the same
// executor running these fp32 CUDA-core kernels instead (A.6: fp32 stays
// at ~1e-5 over S <= 4). They are parity infrastructure, not a fast path:
// a 64 x 64 register-tiled SIMT GEMM and one CTA per (query row, head)
// attention with the scores staged in shared memory.
#include <cfloat>
#include <climits>
#include <cmath>

#include "kernels.h"

namespace pf {
namespace {

constexpr int kT = 64;   // C tile
constexpr int kBK = 16;  // k-slab

// C[m, n] (ldc) <- epi(sum_k A[m, k] (lda) * B[k, n] (ldb)), 256 threads, 4 x 4 per thread.
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, int lda,
                                                       const float* __restrict__ B, int ldb,
                                                       float* __restrict__ C, int ldc, int M,
                                                       int N, int K, int epi, int* flag,
                                                       int code) {
  __shared__ float As[kBK][kT + 4];
  __shared__ float Bs[kBK][kT];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kBK) {
    for (int i = threadIdx.x; i < kT * kBK; i += 256) {
      const int mm = i / kBK, kk = i % kBK;  // A tile, transposed into As[k][m]
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[size_t(gm) * lda + gk] : 0.f;
      const int kb = i / kT, nb = i % kT;
      const int gkb = k0 + kb, gn = n0 + nb;
      Bs[kb][nb] = (gkb < K && gn < N) ? B[size_t(gkb) * ldb + gn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      float* c = C + size_t(gm) * ldc + gn;
      if (epi == kF32Residual) {
        const float h = *c + acc[i][j];
        *c = h;
        bad |= !isfinite(h);
      } else if (epi == kF32Tanh) {
        *c = tanhf(acc[i][j]);
      } else {
        *c = acc[i][j];
      }
    }
  }
  if (bad && flag) atomicMin(flag, code);
}

// One CTA per (query row, head): out[i, h*dh + d] = sum_j softmax_j(q.k_j scale) v_j[d]
// over all P kv rows (toy_model.cpp:104-143; zero rows are not masked).
__global__ void __launch_bounds__(128) attn_f32_kernel(const float* __restrict__ q,
                                                       const float* __restrict__ k,
                                                       const float* __restrict__ v,
                                                       float* __restrict__ out, int P, int hs,
                                                       int dh, float scale) {
  extern __shared__ float sm[];
  float* qs = sm;        // [dh]
  float* s = sm + dh;    // [P]
  __shared__ float red[32];
  const int i = blockIdx.x, h = blockIdx.y;
  const float* qi = q + size_t(i) * hs + size_t(h) * dh;
  for (int d = threadIdx.x; d < dh; d += blockDim.x) qs[d] = qi[d];
  __syncthreads();
  float mx = -FLT_MAX;
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    const float* kj = k + size_t(j) * hs + size_t(h) * dh;
    float acc = 0.f;
    for (int d = 0; d < dh; ++d) acc = fmaf(qs[d], kj[d], acc);
    acc *= scale;
    s[j] = acc;
    mx = fmaxf(mx, acc);
  }
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
  for (int o = 16; o; o /= 2) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < nw; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float z = 0.f;
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    const float e = expf(s[j] - mx);
    s[j] = e;
    z += e;
  }
  for (int o = 16; o; o /= 2) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  z = 0.f;
  for (int w = 0; w < nw; ++w) z += red[w];
  const float inv = 1.f / z;
  float* oi = out + size_t(i) * hs + size_t(h) * dh;
  for (int d = threadIdx.x; d < dh; d += blockDim.x) {
    const float* vd = v + size_t(h) * dh + d;
    float acc = 0.f;
    for (int j = 0; j < P; ++j) acc = fmaf(s[j], vd[size_t(j) * hs], acc);
    oi[d] = acc * inv;
  }
}

}  // namespace

cudaError_t gemm_f32(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M,
                     int N, int K, int epi, int* flag, int code, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 grid((N + kT - 1) / kT, (M + kT - 1) / kT);
  ++launch_counter();
  gemm_f32_kernel<<<grid, 256, 0, stream>>>(A, lda, B, ldb, C, ldc, M, N, K, epi, flag, code);
  return cudaGetLastError();
}

cudaError_t attention_f32(const float* q, const float* k, const float* v, float* out, int rows,
                          int P, int heads, int dh, int hs, float scale, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const size_t smem = size_t(dh + P) * sizeof(float);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(
        attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
  }
  ++launch_counter();
  attn_f32_kernel<<<dim3(unsigned(rows), unsigned(heads)), 128, smem, stream>>>(
      q, k, v, out, P, hs, dh, scale);
  return cudaGetLastError();
}

}  // namespace pf
