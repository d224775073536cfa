// Kernel-level test entry points (include/pipefusion_b200_debug.h).
#include <cmath>
#include <vector>

#include "kernels.h"
#include "pipefusion_b200_debug.h"

namespace {

// Repack [P x hs] row-major bf16 into the attention layouts
// (Q/K/V: [heads][P][dhp]), zero padded.
__global__ void pack_heads_kernel(const pf::bf16* __restrict__ src, pf::bf16* __restrict__ qk,
                                  pf::bf16* __restrict__ vt, int P, int hs, int heads, int dh,
                                  int dhp) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P * hs) return;
  const int r = idx / hs, c = idx % hs;
  const int h = c / dh, d = c % dh;
  if (qk) qk[(size_t(h) * P + r) * dhp + d] = src[idx];
  if (vt) vt[(size_t(h) * dhp + d) * P + r] = src[idx];
}

}  // namespace

extern "C" int pf_debug_gemm(const void* A, const void* B, float* C, int rows,
                             int row0, int total_rows, int N, int K, void* stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  CUtensorMap ta;
  pf::WeightMaps tb;
  if (!pf::encode_tmap_bf16_2d(&ta, A, uint64_t(K), uint64_t(total_rows), uint64_t(K) * 2,
                               64, 128, 128))
    return int(cudaErrorInvalidValue);
  if (!pf::make_weight_maps(&tb, static_cast<const pf::bf16*>(B), N, K))
    return int(cudaErrorInvalidValue);
  CUtensorMap ta_half;
  if (!pf::encode_tmap_bf16_2d(&ta_half, A, uint64_t(K), uint64_t(total_rows), uint64_t(K) * 2,
                               64, 64, 128))
    return int(cudaErrorInvalidValue);
  pf::EpiParams ep;
  ep.a_half = &ta_half;
  ep.out_f32 = C - size_t(row0) * N;  // epilogue indexes by global row
  ep.ld = N;
  // split-K workspace as the runtime attaches it (skinny problems split K)
  static float* ws = nullptr;
  static int* counters = nullptr;
  constexpr size_t kWsFloats = size_t(4) << 20;
  constexpr int kCounters = 4096;
  if (!ws) {
    cudaMalloc(reinterpret_cast<void**>(&ws), kWsFloats * 4);
    cudaMalloc(reinterpret_cast<void**>(&counters), kCounters * sizeof(int));
    cudaMemset(counters, 0, kCounters * sizeof(int));
  }
  ep.splitk_ws = ws;
  ep.splitk_ws_floats = kWsFloats;
  ep.splitk_counters = counters;
  ep.splitk_counter_cap = kCounters;
  return int(pf::gemm(ta, tb, rows, row0, N, K, pf::Epi::StoreF32, ep,
                      pf::device_sm_count(dev), static_cast<cudaStream_t>(stream)));
}

// Debug-only: record the per-CTA timeline of the next 1-SM GEMM launches into
// a device buffer; `host` (2048 slots) receives it.
extern "C" int pf_debug_gemm_trace(int enable, unsigned long long* host) {
  static unsigned long long* buf = nullptr;
  if (enable && !buf) {
    cudaMalloc(reinterpret_cast<void**>(&buf), 2048 * 8);
    cudaMemset(buf, 0, 2048 * 8);
    pf::set_gemm_trace(buf);
  }
  if (host && buf) cudaMemcpy(host, buf, 2048 * 8, cudaMemcpyDeviceToHost);
  if (!enable && buf) {
    pf::set_gemm_trace(nullptr);
    cudaFree(buf);
    buf = nullptr;
  }
  return int(cudaGetLastError());
}

// Host-only: the stream-K attention schedule the library picks for a launch
// (no GPU needed). out = {nq, blocks, units, grid, cut, fused, strided}.
extern "C" int pf_debug_attn_schedule(int P, int rows, int heads, int dhp, int sm_count,
                                      long long* out) {
  if (!out || P <= 0 || rows <= 0 || heads <= 0 || dhp <= 0 || sm_count <= 0) return 1;
  static int dummy_flags = 0;
  pf::AttnLaunch a{dhp, P, rows, 0, heads, dhp, heads * dhp, 1.f, nullptr, nullptr, 0};
  a.flags = &dummy_flags;  // the runtime always provides merge flags
  const pf::AttnSchedule sc = pf::attn_schedule(a, sm_count, pf::attn_block_rows(a));
  out[0] = sc.nq;
  out[1] = sc.blocks;
  out[2] = sc.units;
  out[3] = sc.grid;
  out[4] = sc.cut ? 1 : 0;
  out[5] = sc.fused ? 1 : 0;
  out[6] = sc.strided ? 1 : 0;
  return 0;
}

namespace {
// device buffer: 8192 clock64 slots of CTA 0, then 4 per CTA (globaltimer at
// entry / after griddepcontrol.wait / exit, SM id) for up to 1024 CTAs
constexpr int kTraceSlots = 8192 + 4 * 1024 + 1024;  // + epilogue probes of CTA 0
unsigned long long* g_attn_trace = nullptr;
}

// Debug-only: record the clock64 timeline of CTA (0,0,0) of the next
// pf_debug_attention launches into `host` (8192 slots) when enabled.
extern "C" int pf_debug_attention_trace(int enable, unsigned long long* host) {
  if (enable && !g_attn_trace) {
    cudaMalloc(reinterpret_cast<void**>(&g_attn_trace), kTraceSlots * 8);
    cudaMemset(g_attn_trace, 0, kTraceSlots * 8);
  }
  if (host && g_attn_trace)
    cudaMemcpy(host, g_attn_trace, kTraceSlots * 8, cudaMemcpyDeviceToHost);
  if (!enable && g_attn_trace) {
    cudaFree(g_attn_trace);
    g_attn_trace = nullptr;
  }
  return int(cudaGetLastError());
}

extern "C" int pf_debug_attention(const void* q, const void* k, const void* v, void* out,
                                  int P, int rows, int row0, int heads, int hs,
                                  void* stream) {
  return pf_debug_attention_ex(q, k, v, out, P, rows, row0, heads, hs, stream, 0);
}

extern "C" int pf_debug_attention_ex(const void* q, const void* k, const void* v, void* out,
                                     int P, int rows, int row0, int heads, int hs,
                                     void* stream, int v_sum_col) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaGetDevice(&dev);
  const int dh = hs / heads;
  const int dhp = (dh + 15) / 16 * 16;
  pf::bf16 *qp = nullptr, *kp = nullptr, *vp = nullptr;
  float* work = nullptr;
  int* flags = nullptr;
  const size_t n = size_t(heads) * P * dhp;
  cudaMallocAsync(reinterpret_cast<void**>(&qp), n * 2, s);
  cudaMallocAsync(reinterpret_cast<void**>(&kp), n * 2, s);
  cudaMallocAsync(reinterpret_cast<void**>(&vp), n * 2, s);
  cudaMemsetAsync(qp, 0, n * 2, s);
  cudaMemsetAsync(kp, 0, n * 2, s);
  cudaMemsetAsync(vp, 0, n * 2, s);
  const int total = P * hs;
  ++pf::launch_counter();
  pack_heads_kernel<<<(total + 255) / 256, 256, 0, s>>>(static_cast<const pf::bf16*>(q), qp,
                                                         nullptr, P, hs, heads, dh, dhp);
  ++pf::launch_counter();
  pack_heads_kernel<<<(total + 255) / 256, 256, 0, s>>>(static_cast<const pf::bf16*>(k), kp,
                                                         nullptr, P, hs, heads, dh, dhp);
  ++pf::launch_counter();
  pack_heads_kernel<<<(total + 255) / 256, 256, 0, s>>>(static_cast<const pf::bf16*>(v), vp,
                                                         nullptr, P, hs, heads, dh, dhp);
  const bool sumcol = v_sum_col && dh < dhp;
  if (sumcol) pf::v_ones_col(vp, size_t(heads) * P, dhp, dh, s);
  CUtensorMap tq, tk, tv;
  bool ok = pf::encode_tmap_bf16_2d(&tq, qp, dhp, uint64_t(heads) * P, uint64_t(dhp) * 2, 16,
                                    128, 32) &&
            pf::encode_tmap_bf16_2d(&tk, kp, dhp, uint64_t(heads) * P, uint64_t(dhp) * 2, 16,
                                    128, 32) &&
            pf::encode_tmap_bf16_2d(&tv, vp, dhp, uint64_t(heads) * P, uint64_t(dhp) * 2, 16,
                                    128, 32);
  CUtensorMap tk3, tv3;
  const uint32_t b3 = uint32_t(pf::attn3_kv_rows(dhp));
  const bool kv3 = pf::encode_tmap_bf16_2d(&tk3, kp, dhp, uint64_t(heads) * P,
                                           uint64_t(dhp) * 2, 16, b3, 32) &&
                   pf::encode_tmap_bf16_2d(&tv3, vp, dhp, uint64_t(heads) * P,
                                           uint64_t(dhp) * 2, 16, b3, 32);
  int err = ok ? 0 : int(cudaErrorInvalidValue);
  if (ok) {
    pf::AttnLaunch a{dhp, P, rows, row0, heads, dh, hs, float(1.0 / std::sqrt(double(dh))),
                     static_cast<pf::bf16*>(out), nullptr, 0, g_attn_trace};
    if (kv3) {
      a.k3 = &tk3;
      a.v3 = &tv3;
    }
    const int sms = pf::device_sm_count(dev);
    a.work_floats = pf::attn_work_floats(dhp, sms);
    cudaMallocAsync(reinterpret_cast<void**>(&work), a.work_floats * 4, s);
    a.work = work;
    cudaMallocAsync(reinterpret_cast<void**>(&flags), size_t(sms) * pf::kAttnFlagsPerCta * sizeof(int), s);
    cudaMemsetAsync(flags, 0, size_t(sms) * pf::kAttnFlagsPerCta * sizeof(int), s);
    a.flags = flags;
    a.v_sum_col = sumcol;
    err = int(pf::attention(tq, tk, tv, a, sms, s));
  }
  cudaStreamSynchronize(s);
  cudaFreeAsync(qp, s);
  cudaFreeAsync(kp, s);
  cudaFreeAsync(vp, s);
  if (work) cudaFreeAsync(work, s);
  if (flags) cudaFreeAsync(flags, s);
  cudaStreamSynchronize(s);
  if (!err) err = int(cudaGetLastError());
  return err;
}
