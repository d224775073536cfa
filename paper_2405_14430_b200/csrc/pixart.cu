// Conditioning and LayerNorm-fold kernels of the PixArt-alpha block variant
// (`block = pixart`; the fp64 specification is
// oracle/px_oracle.c). All of these are small and bandwidth- or
// latency-bound; the block's dense work stays in the tcgen05 GEMMs, whose
// epilogues (kernels.cu: EpiQKVAffine, EpiGeluAffine, resid_chunk<true>)
// apply LayerNorm, adaLN modulate/gate, biases and GELU.
//
// Per run, for every timestep index t of the S-step schedule:
//   sinusoid(tau_t)            px_sinusoid_kernel      [S x 256]
//   e1 = silu(sin Wt1 + bt1)   px_gemv_kernel          [S x hs]
//   silu(temb), temb = e1 Wt2 + bt2   px_gemv_kernel   [S x hs]
//   tv = silu(temb) Wt0 + bt0  px_gemv_kernel         [S x 6hs]
//   mod[l][t] = sst[l] + tv[t] px_mod_kernel           [layers x S x 6hs]
//   c1[l][t] = (1 + scale) . W, c2[l][t] = shift . W + b   px_fold_rows_kernel
//                              (bf16 rows) + one tcgen05 GEMM per layer and branch
// where W is the bf16 QKV (scale/shift of the attention branch) or MLP-in
// weight (MLP branch): the LayerNorm-modulated GEMM operand
//   LN(h)(1+s) + sh  =  rstd * h(1+s) - rstd*mean*(1+s) + sh
// becomes  a = bf16(h * (1 + s))  (written by the producing epilogue) and
//   y = rstd * (a . W) - rstd*mean * c1 + c2.
#include <cmath>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace pf {
namespace {

constexpr int kFreq = 256;

__global__ void px_sinusoid_kernel(float* __restrict__ out, int S) {
  const int s = blockIdx.x;
  const int i = threadIdx.x;  // 0 .. 127
  const double tau = 1000.0 * double(s) / double(S);
  const double f = exp(-log(10000.0) * double(i) / double(kFreq / 2));
  out[size_t(s) * kFreq + i] = float(cos(tau * f));
  out[size_t(s) * kFreq + kFreq / 2 + i] = float(sin(tau * f));
}

__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

// out[s][n] = act_out( sum_k act_in(in[s][k]) * W[n][k] + b[n] ), s < S.
// One warp per output column n and 16 timesteps per pass; W rows are read
// coalesced once per pass, the inputs come from L1.
constexpr int kGemvS = 16;
__global__ void px_gemv_kernel(const float* __restrict__ in, int S, int K,
                               const float* __restrict__ W, const float* __restrict__ b, int N,
                               float* __restrict__ out, int silu_in, int silu_out) {
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const int n = blockIdx.x * (blockDim.x >> 5) + warp;
  const int s0 = blockIdx.y * kGemvS;
  if (n >= N) return;
  float acc[kGemvS];
#pragma unroll
  for (int j = 0; j < kGemvS; ++j) acc[j] = 0.f;
  const float* wr = W + size_t(n) * K;
  for (int k = lane; k < K; k += 32) {
    const float w = __ldg(wr + k);
#pragma unroll
    for (int j = 0; j < kGemvS; ++j) {
      if (s0 + j < S) {
        float x = __ldg(in + size_t(s0 + j) * K + k);
        if (silu_in) x = silu(x);
        acc[j] = fmaf(x, w, acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kGemvS; ++j) {
    float v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[j] = v;
  }
  if (lane == 0) {
    const float bn = b ? b[n] : 0.f;
#pragma unroll
    for (int j = 0; j < kGemvS; ++j) {
      if (s0 + j < S) {
        float v = acc[j] + bn;
        if (silu_out) v = silu(v);
        out[size_t(s0 + j) * N + n] = v;
      }
    }
  }
}

// mod[l][s][i] = sst[l][i] + tv[s][i]
__global__ void px_mod_kernel(const float* __restrict__ sst, int nl, const float* __restrict__ tv,
                              int S, int w6, float* __restrict__ mod) {
  const size_t total = size_t(nl) * S * w6;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const int c = int(i % w6);
    const size_t ls = i / w6;
    const int s = int(ls % S);
    const int l = int(ls / S);
    mod[i] = sst[size_t(l) * w6 + c] + tv[size_t(s) * w6 + c];
  }
}

// GEMM operands of the LayerNorm fold: for every local layer l and timestep s
//   aq[l][2s] = 1 + scale_msa, aq[l][2s+1] = shift_msa   (attention branch)
//   am[l][2s] = 1 + scale_mlp, am[l][2s+1] = shift_mlp   (MLP branch)
// as bf16 rows of hs; rows >= 2S of each [rpad x hs] block stay zero.
__global__ void px_fold_rows_kernel(const float* __restrict__ mod, int nl, int S, int hs,
                                    bf16* __restrict__ aq, bf16* __restrict__ am, int rpad) {
  const size_t total = size_t(nl) * S * hs;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
       i += size_t(gridDim.x) * blockDim.x) {
    const int k = int(i % hs);
    const size_t ls = i / hs;
    const int sidx = int(ls % S);
    const int l = int(ls / S);
    const float* m = mod + ls * 6 * hs;
    const size_t r0 = (size_t(l) * rpad + 2 * sidx) * hs + k;
    aq[r0] = __float2bfloat16_rn(1.f + m[hs + k]);
    aq[r0 + hs] = __float2bfloat16_rn(m[k]);
    am[r0] = __float2bfloat16_rn(1.f + m[4 * hs + k]);
    am[r0 + hs] = __float2bfloat16_rn(m[3 * hs + k]);
  }
}

// Patch split + deferred sampler update for the PixArt block (the toy
// block's patch_prepare_kernel plus the first layer's LayerNorm inputs):
//   x_j -= eta eps_j (update);  h = x_j + cb;  hb = bf16(h (1 + scale));
//   stats[(c/32) * stats_ld + row] = (sum, sum^2) of h over 32-column chunks.
// 4 columns per thread; the 8 lanes of one 32-column chunk reduce by shuffle.
__global__ void px_patch_prepare_kernel(float* __restrict__ x, const float* __restrict__ eps,
                                        const float* __restrict__ cb,
                                        const float* __restrict__ scale,
                                        float* __restrict__ h32, bf16* __restrict__ hb,
                                        float2* __restrict__ stats, int stats_ld, int row0,
                                        size_t n4, int hs4, float eta, int update) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i0 = size_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); i0 < n4; i0 += stride) {
    const size_t i = i0 + (threadIdx.x & 31);
    const bool ok = i < n4;  // n4 % 8 == 0: whole 8-lane groups are in or out
    float4 hv = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t row = ok ? i / size_t(hs4) : 0;
    const int c4 = ok ? int(i % size_t(hs4)) : 0;
    if (ok) {
      const size_t off = (size_t(row0) + row) * size_t(hs4) * 4 + 4 * size_t(c4);
      float4 xv = *reinterpret_cast<const float4*>(x + off);
      if (update) {
        const float4 ev = *reinterpret_cast<const float4*>(eps + off);
        xv.x -= eta * ev.x;
        xv.y -= eta * ev.y;
        xv.z -= eta * ev.z;
        xv.w -= eta * ev.w;
        *reinterpret_cast<float4*>(x + off) = xv;
      }
      const float4 bv = *reinterpret_cast<const float4*>(cb + 4 * c4);
      hv = make_float4(xv.x + bv.x, xv.y + bv.y, xv.z + bv.z, xv.w + bv.w);
      *reinterpret_cast<float4*>(h32 + off) = hv;
      const float4 sc = *reinterpret_cast<const float4*>(scale + 4 * c4);
      uint2 pk;
      pk.x = ptx::pack_bf16x2(hv.x * (1.f + sc.x), hv.y * (1.f + sc.y));
      pk.y = ptx::pack_bf16x2(hv.z * (1.f + sc.z), hv.w * (1.f + sc.w));
      *reinterpret_cast<uint2*>(hb + off) = pk;
    }
    float s = (hv.x + hv.y) + (hv.z + hv.w);
    float ss = (hv.x * hv.x + hv.y * hv.y) + (hv.z * hv.z + hv.w * hv.w);
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if (ok && (c4 & 7) == 0)
      stats[size_t(c4 >> 3) * stats_ld + size_t(row0) + row] = make_float2(s, ss);
  }
}

int grid_for(size_t n, int per_block) {
  size_t g = (n + per_block - 1) / per_block;
  if (g > 148 * 8) g = 148 * 8;
  return int(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t px_sinusoid(float* out, int S, cudaStream_t stream) {
  ++launch_counter();
  px_sinusoid_kernel<<<S, kFreq / 2, 0, stream>>>(out, S);
  return cudaGetLastError();
}

cudaError_t px_gemv(const float* in, int S, int K, const float* W, const float* b, int N,
                    float* out, bool silu_in, bool silu_out, cudaStream_t stream) {
  dim3 grid((N + 7) / 8, (S + kGemvS - 1) / kGemvS);
  ++launch_counter();
  px_gemv_kernel<<<grid, 256, 0, stream>>>(in, S, K, W, b, N, out, silu_in ? 1 : 0,
                                           silu_out ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t px_mod(const float* sst, int nl, const float* tv, int S, int w6, float* mod,
                   cudaStream_t stream) {
  const size_t n = size_t(nl) * S * w6;
  ++launch_counter();
  px_mod_kernel<<<grid_for(n, 256), 256, 0, stream>>>(sst, nl, tv, S, w6, mod);
  return cudaGetLastError();
}

cudaError_t px_fold_rows(const float* mod, int nl, int S, int hs, bf16* aq, bf16* am,
                         int rpad, cudaStream_t stream) {
  if (2 * S > rpad) return cudaErrorInvalidValue;
  const size_t n = size_t(nl) * S * hs;
  ++launch_counter();
  px_fold_rows_kernel<<<grid_for(n, 256), 256, 0, stream>>>(mod, nl, S, hs, aq, am, rpad);
  return cudaGetLastError();
}

cudaError_t px_patch_prepare(float* x, const float* eps, const float* cb, const float* scale,
                             float* h32, bf16* hb, float2* stats, int stats_ld, int row0,
                             int rows, int hs, float eta, bool update, cudaStream_t stream) {
  if (hs % 32 != 0) return cudaErrorInvalidValue;
  const size_t n4 = size_t(rows) * hs / 4;
  return launch_pdl(px_patch_prepare_kernel, dim3(grid_for(n4, 256)), dim3(256), 0, stream, x,
                    eps, cb, scale, h32, hb, stats, stats_ld, row0, n4, hs / 4, eta,
                    update ? 1 : 0);
}

}  // namespace pf
