// Kernels of the MMDiT block variants (`block = mmdit`: SD3-medium-style
// double-stream joint blocks and Flux.1-style single-stream blocks; BASELINE
// configs 4 and 5). The fp64 specification is oracle/mmdit_oracle.py; the
// dense work runs in the tcgen05 GEMMs and the attention kernel, whose
// epilogues apply LayerNorm (folded), adaLN-Zero modulate/gate, biases and
// GELU exactly as for the PixArt block (pixart.cu). What is specific here:
//
//   mm_fill_kernel       counter-based parameter generation on the device
//                        (splitmix64 per element, see mmdit_oracle.py) so a
//                        12B-parameter Flux model is built in HBM in seconds
//   mm_gemv_bf16_kernel  adaLN-Zero modulation vectors silu(c_t) Wmod + bmod
//                        for every timestep (bf16 weights, fp32 accumulate)
//   mm_qk_norm_rope_kernel  per-head RMSNorm of q and k (QK-norm) and the
//                        Flux axial RoPE, in place on the head-major q / K
//                        buffers after the QKV GEMM (one warp per row and head)
#include <cmath>
#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

namespace pf {
namespace {

constexpr uint64_t kGold = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMixI = 0xD1B54A32D192ED03ull;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + kGold;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double mm_uniform(uint64_t key, uint64_t i) {
  const uint64_t z = splitmix64(key ^ (i * kMixI));
  return double(z >> 11) * 0x1.0p-52 - 1.0;
}

// Tensor [K x N] (x.W orientation, element i = k N + n) of `key`:
//   kind 0: bf16 dst[n K + k] (K-major GEMM operand / GEMV rows)
//   kind 1: fp32 dst[i] = scale u
//   kind 2: fp32 dst[i] = 1 + 0.1 u   (RMSNorm gains)
//   kind 3: fp32 dst[n K + k] = scale u  (transposed fp32, px_gemv rows)
__global__ void mm_fill_kernel(void* dst, uint64_t key, int64_t K, int64_t N, float scale,
                               int kind) {
  const int64_t total = K * N;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < total;
       j += int64_t(gridDim.x) * blockDim.x) {
    if (kind == 0 || kind == 3) {
      const int64_t n = j / K, k = j - n * K;  // output index j = n K + k
      const double u = mm_uniform(key, uint64_t(k * N + n));
      if (kind == 0)
        static_cast<bf16*>(dst)[j] = __float2bfloat16_rn(float(u * double(scale)));
      else
        static_cast<float*>(dst)[j] = float(u * double(scale));
    } else {
      const double u = mm_uniform(key, uint64_t(j));
      static_cast<float*>(dst)[j] = kind == 1 ? float(u * double(scale)) : float(1.0 + 0.1 * u);
    }
  }
}

// out[s][n] = sum_k in[s][k] W[n][k] + b[n] (+ b2[n]); W bf16 [N x K].
// One warp per output column, 16 timesteps per pass (as px_gemv_kernel).
constexpr int kGemvS = 16;
__global__ void mm_gemv_bf16_kernel(const float* __restrict__ in, int S, int K,
                                    const bf16* __restrict__ W, const float* __restrict__ b,
                                    int N, float* __restrict__ out, int ld_out) {
  const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
  const int n = blockIdx.x * (blockDim.x >> 5) + warp;
  const int s0 = blockIdx.y * kGemvS;
  if (n >= N) return;
  float acc[kGemvS];
#pragma unroll
  for (int j = 0; j < kGemvS; ++j) acc[j] = 0.f;
  const bf16* wr = W + size_t(n) * K;
  for (int k = 2 * lane; k < K; k += 64) {
    const float2 w = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(wr + k));
#pragma unroll
    for (int j = 0; j < kGemvS; ++j)
      if (s0 + j < S) {
        const float2 x = *reinterpret_cast<const float2*>(in + size_t(s0 + j) * K + k);
        acc[j] = fmaf(x.x, w.x, fmaf(x.y, w.y, acc[j]));
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
    for (int j = 0; j < kGemvS; ++j)
      if (s0 + j < S) out[size_t(s0 + j) * ld_out + n] = acc[j] + bn;
  }
}

// In place on q [heads][q_rows][dhp] and k [heads][k_rows][dhp], joint rows
// [row0, row0 + rows): per head x <- x / sqrt(mean(x^2) + 1e-6) * g (g of the
// row's stream: rows < J text, else image), then (rope) the axial rotation of
// mmdit_oracle.rope with position ids (0, 0, 0) for text rows and
// (0, i / side, i % side) for image row i. One warp per (row, head, q|k);
// lane l owns the element pairs l, l + 32, ... of the head.
__global__ void mm_qk_norm_rope_kernel(bf16* __restrict__ q, bf16* __restrict__ k, int heads,
                                       int q_rows, int k_rows, int dhp, int dh, int row0,
                                       int rows, int J, const float* __restrict__ gq_img,
                                       const float* __restrict__ gk_img,
                                       const float* __restrict__ gq_txt,
                                       const float* __restrict__ gk_txt, int rope, int side) {
  ptx::pdl_wait();  // the QKV GEMM's q / k rows
  ptx::pdl_launch();
  const int lane = int(threadIdx.x & 31);
  const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t total = int64_t(rows) * heads * 2;
  if (wid >= total) return;
  const int which = int(wid & 1);  // 0: q, 1: k
  const int64_t rh = wid >> 1;
  const int head = int(rh % heads);
  const int row = row0 + int(rh / heads);
  const bool txt = row < J;
  const float* g = which == 0 ? (txt ? gq_txt : gq_img) : (txt ? gk_txt : gk_img);
  bf16* base = (which == 0 ? q + (size_t(head) * q_rows + row) * dhp
                           : k + (size_t(head) * k_rows + row) * dhp);
  constexpr int kMaxPairs = 2;  // dh <= 128
  const int npairs = dh / 2;
  float2 v[kMaxPairs];
  float ss = 0.f;
#pragma unroll
  for (int t = 0; t < kMaxPairs; ++t) {
    const int p = lane + 32 * t;
    v[t] = make_float2(0.f, 0.f);
    if (p < npairs) {
      v[t] = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(base + 2 * p));
      ss += v[t].x * v[t].x + v[t].y * v[t].y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / float(dh) + 1e-6f);
  const int img = row - J;
  const float pos1 = txt ? 0.f : float(img / side), pos2 = txt ? 0.f : float(img % side);
  const int d0 = dh / 8, d1 = 7 * dh / 16;
#pragma unroll
  for (int t = 0; t < kMaxPairs; ++t) {
    const int p = lane + 32 * t;
    if (p >= npairs) continue;
    float x0 = v[t].x * inv * g[2 * p], x1 = v[t].y * inv * g[2 * p + 1];
    if (rope) {
      const int e = 2 * p;
      int off, d;
      float pos;
      if (e < d0) { off = 0; d = d0; pos = 0.f; }
      else if (e < d0 + d1) { off = d0; d = d1; pos = pos1; }
      else { off = d0 + d1; d = d1; pos = pos2; }
      const int j = (e - off) / 2;
      // theta^(-2j/d) with theta = 10000
      const float w = expf(-9.210340371976184f * float(2 * j) / float(d));
      float sn, cs;
      sincosf(pos * w, &sn, &cs);
      const float y0 = cs * x0 - sn * x1, y1 = sn * x0 + cs * x1;
      x0 = y0;
      x1 = y1;
    }
    *reinterpret_cast<__nv_bfloat162*>(base + 2 * p) = __floats2bfloat162_rn(x0, x1);
  }
}

// Vectorised variant for dhp / 8 in {2, 4, 8, 16}: G = dhp / 8 lanes per
// (row, head, q|k) item, 8 elements (one 16-byte vector) per lane, the RMS
// reduction over the item's G lanes; 32 / G items per warp.
template <int G>
__global__ void mm_qk_norm_rope_vec_kernel(bf16* __restrict__ q, bf16* __restrict__ k, int heads,
                                           int q_rows, int k_rows, int dhp, int dh, int row0,
                                           int rows, int J, const float* __restrict__ gq_img,
                                           const float* __restrict__ gk_img,
                                           const float* __restrict__ gq_txt,
                                           const float* __restrict__ gk_txt, int rope, int side) {
  ptx::pdl_wait();
  ptx::pdl_launch();
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t item = tid / G;
  const int sub = int(tid % G);
  const int64_t total = int64_t(rows) * heads * 2;
  const bool live = item < total;
  const int64_t it = live ? item : 0;
  const int which = int(it & 1);
  const int64_t rh = it >> 1;
  const int head = int(rh % heads);
  const int row = row0 + int(rh / heads);
  const bool txt = row < J;
  const float* g = which == 0 ? (txt ? gq_txt : gq_img) : (txt ? gk_txt : gk_img);
  bf16* base = (which == 0 ? q + (size_t(head) * q_rows + row) * dhp
                           : k + (size_t(head) * k_rows + row) * dhp) + 8 * sub;
  float x[8];
  uint4 raw = live ? *reinterpret_cast<const uint4*>(base) : make_uint4(0, 0, 0, 0);
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(h2[j]);
    x[2 * j] = f.x;
    x[2 * j + 1] = f.y;
  }
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) ss += x[j] * x[j];  // padding columns are zero
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (!live) return;
  const float inv = rsqrtf(ss / float(dh) + 1e-6f);
  const int img = row - J;
  const float pos1 = txt ? 0.f : float(img / side), pos2 = txt ? 0.f : float(img % side);
  const int d0 = dh / 8, d1 = 7 * dh / 16;
  uint4 outv;
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&outv);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int e = 8 * sub + 2 * j;
    float y0 = 0.f, y1 = 0.f;
    if (e < dh) {
      y0 = x[2 * j] * inv * g[e];
      y1 = x[2 * j + 1] * inv * g[e + 1];
      if (rope) {
        int off, d;
        float pos;
        if (e < d0) { off = 0; d = d0; pos = 0.f; }
        else if (e < d0 + d1) { off = d0; d = d1; pos = pos1; }
        else { off = d0 + d1; d = d1; pos = pos2; }
        const int jj = (e - off) / 2;
        const float w = expf(-9.210340371976184f * float(2 * jj) / float(d));
        float sn, cs;
        sincosf(pos * w, &sn, &cs);
        const float z0 = cs * y0 - sn * y1, z1 = sn * y0 + cs * y1;
        y0 = z0;
        y1 = z1;
      }
    }
    o2[j] = __floats2bfloat162_rn(y0, y1);
  }
  *reinterpret_cast<uint4*>(base) = outv;
}

int fill_grid(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return int(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

}  // namespace

uint64_t mm_tensor_key(uint64_t seed, uint64_t tid) { return splitmix64(seed + tid * kGold); }

cudaError_t mm_fill(void* dst, uint64_t key, int64_t K, int64_t N, float scale, int kind,
                    cudaStream_t stream) {
  ++launch_counter();
  mm_fill_kernel<<<fill_grid(K * N), 256, 0, stream>>>(dst, key, K, N, scale, kind);
  return cudaGetLastError();
}

cudaError_t mm_gemv_bf16(const float* in, int S, int K, const bf16* W, const float* b, int N,
                         float* out, int ld_out, cudaStream_t stream) {
  if (K % 64 != 0) return cudaErrorInvalidValue;
  dim3 grid(unsigned((N + 7) / 8), unsigned((S + kGemvS - 1) / kGemvS));
  ++launch_counter();
  mm_gemv_bf16_kernel<<<grid, 256, 0, stream>>>(in, S, K, W, b, N, out, ld_out);
  return cudaGetLastError();
}

cudaError_t mm_qk_norm_rope(bf16* q, bf16* k, int heads, int q_rows, int k_rows, int dhp, int dh,
                            int row0, int rows, int J, const float* gq_img, const float* gk_img,
                            const float* gq_txt, const float* gk_txt, bool rope, int side,
                            cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  if (dh > 128 || dh % 2 != 0) return cudaErrorInvalidValue;
  const int G = dhp / 8;
  if (G == 2 || G == 4 || G == 8 || G == 16) {
    const int64_t threads = int64_t(rows) * heads * 2 * G;
    const unsigned blocks = unsigned((threads + 255) / 256);
    const int sd = side < 1 ? 1 : side;
    const int rp = rope ? 1 : 0;
    switch (G) {
      case 2:
        return launch_pdl(mm_qk_norm_rope_vec_kernel<2>, dim3(blocks), dim3(256), 0, stream, q,
                          k, heads, q_rows, k_rows, dhp, dh, row0, rows, J, gq_img, gk_img,
                          gq_txt, gk_txt, rp, sd);
      case 4:
        return launch_pdl(mm_qk_norm_rope_vec_kernel<4>, dim3(blocks), dim3(256), 0, stream, q,
                          k, heads, q_rows, k_rows, dhp, dh, row0, rows, J, gq_img, gk_img,
                          gq_txt, gk_txt, rp, sd);
      case 8:
        return launch_pdl(mm_qk_norm_rope_vec_kernel<8>, dim3(blocks), dim3(256), 0, stream, q,
                          k, heads, q_rows, k_rows, dhp, dh, row0, rows, J, gq_img, gk_img,
                          gq_txt, gk_txt, rp, sd);
      default:
        return launch_pdl(mm_qk_norm_rope_vec_kernel<16>, dim3(blocks), dim3(256), 0, stream, q,
                          k, heads, q_rows, k_rows, dhp, dh, row0, rows, J, gq_img, gk_img,
                          gq_txt, gk_txt, rp, sd);
    }
  }
  const int64_t warps = int64_t(rows) * heads * 2;
  const unsigned blocks = unsigned((warps * 32 + 255) / 256);
  return launch_pdl(mm_qk_norm_rope_kernel, dim3(blocks), dim3(256), 0, stream, q, k, heads,
                    q_rows, k_rows, dhp, dh, row0, rows, J, gq_img, gk_img, gq_txt, gk_txt,
                    rope ? 1 : 0, side < 1 ? 1 : side);
}

}  // namespace pf
