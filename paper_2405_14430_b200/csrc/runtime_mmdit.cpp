// MMDiT blocks on the PipeFusion executor (block = kBlockMMDiT): the
// SD3-medium / Flux.1 configurations of BASELINE.json (configs 4 and 5).
// Specification: oracle/mmdit_oracle.py (fp64). The reference has no such
// blocks (its only block is toy_model.cpp:145-177); the executor around
// them -- schedule, patch order, in-place K/V row writes, stale/fresh
// accounting, sampler -- is the reference's run_pipefusion loop
// (execute.cpp:167-223) as for every other block, with the joint-row
// convention of the joint block (T text rows first; they re-enter with
// patch 0 of every step).
//
// Per double-stream layer and stream (text rows: stream 1, image rows: 0):
//   QKV GEMM     LayerNorm folded into the epilogue (stats_in + c1/c2 of the
//                layer, stream and timestep), bias in c2
//   QK-norm      mm_qk_norm_rope (per-head RMSNorm, Flux RoPE) in place
//   attention    all rows of the patch over the P + T joint K/V rows
//   out-proj     residual epilogue: + gate1 (acc + bo); operand h (1 + scale2),
//                LayerNorm stats of h
//   MLP-in       GELU epilogue with the folded LayerNorm (c1/c2 of scale2/shift2)
//   MLP-out      residual: + gate2 (acc + b2); operand h (1 + scale1 of the
//                next layer's stream), stats
// Single-stream layers run QKV and MLP-in from the same modulated input,
// then out-proj (+ gate (acc + b2)) and MLP-out (+ gate acc) residuals.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "runtime.h"
#include "runtime_internal.h"

namespace pf {
namespace {

enum { P_WQKV, P_BQKV, P_WO, P_BO, P_W1, P_B1, P_W2, P_B2, P_WMOD, P_BMOD, P_GQ, P_GK };
enum { G_WT1, G_BT1, G_WT2, G_BT2, G_YP, G_CB, G_Y };
constexpr uint64_t kGlobalTid = uint64_t(1) << 20;
constexpr int kFreq = 256;

uint64_t tid_of(int layer, int stream, int k) {
  return uint64_t(layer) * 64 + uint64_t(stream) * 32 + uint64_t(k);
}

template <class T>
T* mm_dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) throw CudaError("cudaMalloc failed (MMDiT)");
  if (cudaMemset(p, 0, n * sizeof(T)) != cudaSuccess) throw CudaError("cudaMemset failed");
  return static_cast<T*>(p);
}

void mm_free(void* p) {
  if (p) cudaFree(p);
}


}  // namespace

void Engine::mm_alloc_stage(Stage& s) {
  const ModelShape& m = shape_;
  const size_t hs = size_t(m.hs), mlp = size_t(m.mlp), dh = size_t(m.dh);
  const size_t P = size_t(m.rows_total());
  for (int lf = 0; lf < s.layer_count; ++lf) {
    StageLayer& L = s.layers[size_t(lf)];
    const bool dbl = mm_double(s.first_layer + lf);
    const size_t w6 = dbl ? 6 * hs : 3 * hs;
    L.bqkv = mm_dalloc<float>(3 * hs);
    L.bo = mm_dalloc<float>(hs);
    L.b1 = mm_dalloc<float>(mlp);
    L.b2 = mm_dalloc<float>(hs);
    L.wmod = mm_dalloc<bf16>(w6 * hs);
    L.bmod = mm_dalloc<float>(w6);
    L.gq = mm_dalloc<float>(dh);
    L.gk = mm_dalloc<float>(dh);
    if (!dbl) continue;
    L.t_wqkv = mm_dalloc<bf16>(3 * hs * hs);
    L.t_wo = mm_dalloc<bf16>(hs * hs);
    L.t_win = mm_dalloc<bf16>(mlp * hs);
    L.t_wout = mm_dalloc<bf16>(hs * mlp);
    if (!make_weight_maps(&L.tm_t_wqkv, L.t_wqkv, int(3 * hs), int(hs)) ||
        !make_weight_maps(&L.tm_t_wo, L.t_wo, int(hs), int(hs)) ||
        !make_weight_maps(&L.tm_t_win, L.t_win, int(mlp), int(hs)) ||
        !make_weight_maps(&L.tm_t_wout, L.t_wout, int(hs), int(mlp)))
      throw CudaError("cuTensorMapEncodeTiled failed for a text-stream weight");
    L.t_bqkv = mm_dalloc<float>(3 * hs);
    L.t_bo = mm_dalloc<float>(hs);
    L.t_b1 = mm_dalloc<float>(mlp);
    L.t_b2 = mm_dalloc<float>(hs);
    L.t_wmod = mm_dalloc<bf16>(w6 * hs);
    L.t_bmod = mm_dalloc<float>(w6);
    L.t_gq = mm_dalloc<float>(dh);
    L.t_gk = mm_dalloc<float>(dh);
  }
  const int next = s.first_layer + s.layer_count;
  if (next < m.layers) {
    const bool dbl = mm_double(next);
    const size_t w6 = dbl ? 6 * hs : 3 * hs;
    for (int st = 0; st < (dbl ? 2 : 1); ++st) {
      s.mm_next_wmod[st] = mm_dalloc<bf16>(w6 * hs);
      s.mm_next_bmod[st] = mm_dalloc<float>(w6);
    }
  }
  PxStage& px = s.px;
  px.wt1 = mm_dalloc<float>(hs * kFreq);
  px.bt1 = mm_dalloc<float>(hs);
  px.wt2 = mm_dalloc<float>(hs * hs);
  px.bt2 = mm_dalloc<float>(hs);
  s.mm_bcond = mm_dalloc<float>(hs);
  px.stats = mm_dalloc<float2>((hs / 32) * P);
  px.zeros = mm_dalloc<float>(hs);
}

void Engine::mm_free_stage(Stage& s) {
  for (StageLayer& L : s.layers) {
    for (float* p : {L.t_bqkv, L.t_bo, L.t_b1, L.t_b2, L.bmod, L.t_bmod, L.gq, L.gk, L.t_gq,
                     L.t_gk})
      mm_free(p);
    mm_free(L.wmod);
    mm_free(L.t_wmod);
  }
  for (int st = 0; st < 2; ++st) {
    mm_free(s.mm_next_wmod[st]);
    mm_free(s.mm_next_bmod[st]);
    s.mm_next_wmod[st] = nullptr;
    s.mm_next_bmod[st] = nullptr;
  }
  mm_free(s.mm_bcond);
  s.mm_bcond = nullptr;
}

void Engine::mm_generate(uint64_t seed) {
  const ModelShape& m = shape_;
  if (m.block != kBlockMMDiT) throw ValidationError("model is not an MMDiT block model");
  const int64_t hs = m.hs, mlp = m.mlp, dh = m.dh;
  const float rh = float(1.0 / std::sqrt(double(hs))), rm = float(1.0 / std::sqrt(double(mlp)));
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    auto fill = [&](void* dst, uint64_t tid, int64_t K, int64_t N, float scale, int kind) {
      check(mm_fill(dst, mm_tensor_key(seed, tid), K, N, scale, kind, s.stream),
               "MMDiT parameter generation");
    };
    auto stream_params = [&](int l, int st, bf16* wqkv, float* bqkv, bf16* wo, float* bo,
                             bf16* w1, float* b1, bf16* w2, float* b2, bf16* wmod, float* bmod,
                             float* gq, float* gk) {
      const int64_t w6 = mm_double(l) ? 6 * hs : 3 * hs;
      if (wqkv) {
        fill(wqkv, tid_of(l, st, P_WQKV), hs, 3 * hs, rh, 0);
        fill(bqkv, tid_of(l, st, P_BQKV), 1, 3 * hs, 0.1f, 1);
        fill(wo, tid_of(l, st, P_WO), hs, hs, rh, 0);
        fill(bo, tid_of(l, st, P_BO), 1, hs, 0.1f, 1);
        fill(w1, tid_of(l, st, P_W1), hs, mlp, rh, 0);
        fill(b1, tid_of(l, st, P_B1), 1, mlp, 0.1f, 1);
        fill(w2, tid_of(l, st, P_W2), mlp, hs, rm, 0);
        fill(b2, tid_of(l, st, P_B2), 1, hs, 0.1f, 1);
        fill(gq, tid_of(l, st, P_GQ), 1, dh, 0.f, 2);
        fill(gk, tid_of(l, st, P_GK), 1, dh, 0.f, 2);
      }
      fill(wmod, tid_of(l, st, P_WMOD), hs, w6, rh, 0);
      fill(bmod, tid_of(l, st, P_BMOD), 1, w6, 0.1f, 1);
    };
    for (int lf = 0; lf < s.layer_count; ++lf) {
      StageLayer& L = s.layers[size_t(lf)];
      const int l = s.first_layer + lf;
      stream_params(l, 0, L.wqkv, L.bqkv, L.wo, L.bo, L.win, L.b1, L.wout, L.b2, L.wmod, L.bmod,
                    L.gq, L.gk);
      if (mm_double(l))
        stream_params(l, 1, L.t_wqkv, L.t_bqkv, L.t_wo, L.t_bo, L.t_win, L.t_b1, L.t_wout,
                      L.t_b2, L.t_wmod, L.t_bmod, L.t_gq, L.t_gk);
    }
    const int next = s.first_layer + s.layer_count;
    for (int st = 0; st < 2; ++st)
      if (s.mm_next_wmod[st])
        stream_params(next, st, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, s.mm_next_wmod[st], s.mm_next_bmod[st], nullptr, nullptr);
    PxStage& px = s.px;
    fill(px.wt1, kGlobalTid + G_WT1, kFreq, hs, float(1.0 / std::sqrt(double(kFreq))), 3);
    fill(px.bt1, kGlobalTid + G_BT1, 1, hs, 0.1f, 1);
    fill(px.wt2, kGlobalTid + G_WT2, hs, hs, rh, 3);
    fill(px.bt2, kGlobalTid + G_BT2, 1, hs, 0.1f, 1);
    fill(s.mm_bcond, kGlobalTid + G_YP, 1, hs, 1.0f, 1);
    if (s.cb) fill(s.cb, kGlobalTid + G_CB, 1, hs, 1.0f, 1);
    if (s.text) fill(s.text, kGlobalTid + G_Y, m.T, hs, 1.0f, 1);
    PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
    // conditioning bias bt2 + y_pooled
    std::vector<float> a(static_cast<size_t>(hs)), b(static_cast<size_t>(hs));
    PF_CUDA_CHECK(cudaMemcpy(a.data(), px.bt2, a.size() * 4, cudaMemcpyDeviceToHost));
    PF_CUDA_CHECK(cudaMemcpy(b.data(), s.mm_bcond, b.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < a.size(); ++i) b[i] += a[i];
    PF_CUDA_CHECK(cudaMemcpy(s.mm_bcond, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
  }
}

void Engine::mm_alloc_run(Stage& s, int steps) {
  const ModelShape& m = shape_;
  PxStage& px = s.px;
  if (steps <= px.steps_cap) return;
  DeviceGuard g(s.device);
  sync_own();  // a replayed graph may still read the old buffers
  drop_graphs();
  for (float* p : {px.sinus, px.e1, px.temb, px.tv, px.mod, px.foldq, px.foldm}) mm_free(p);
  mm_free(px.fold_aq);
  mm_free(px.fold_am);
  const size_t S = size_t(steps), hs = size_t(m.hs), nb = size_t(s.layer_count) * 2;
  px.sinus = mm_dalloc<float>(S * kFreq);
  px.e1 = mm_dalloc<float>(S * hs);
  px.temb = mm_dalloc<float>(S * hs);
  px.tv = nullptr;
  px.mod = mm_dalloc<float>((nb + 2) * S * 6 * hs);
  px.fold_rpad = int((2 * S + 127) / 128 * 128);
  const size_t rp = size_t(px.fold_rpad);
  px.fold_aq = mm_dalloc<bf16>(nb * rp * hs);
  px.fold_am = mm_dalloc<bf16>(nb * rp * hs);
  px.tm_aq.resize(nb);
  px.tm_am.resize(nb);
  for (size_t b = 0; b < nb; ++b) {
    if (!encode_tmap_bf16_2d(&px.tm_aq[b], px.fold_aq + b * rp * hs, hs, rp, hs * 2, 64, 128,
                             128) ||
        !encode_tmap_bf16_2d(&px.tm_am[b], px.fold_am + b * rp * hs, hs, rp, hs * 2, 64, 128,
                             128))
      throw CudaError("cuTensorMapEncodeTiled failed for a LayerNorm fold operand");
  }
  px.foldq = mm_dalloc<float>(nb * 2 * S * 3 * hs);
  px.foldm = mm_dalloc<float>(nb * 2 * S * size_t(m.mlp));
  px.steps_cap = steps;
}

// Per-run conditioning of one stage: silu(c_t) for every timestep index,
// the adaLN-Zero modulation vectors of each local layer (and of the next
// stage's first layer) per stream, and the LayerNorm fold vectors.
// px.mod layout: [(local layer) x 2 streams][S][6 hs]; single-stream layers
// hold (shift, scale, gate) twice per row and the same vectors for both
// streams, so every consumer reads (shift1, scale1, gate1, shift2, scale2,
// gate2) of its row's stream.
void Engine::mm_conditioning(Stage& s, int steps) {
  const ModelShape& m = shape_;
  PxStage& px = s.px;
  const int hs = m.hs, w6 = 6 * hs, nl = s.layer_count, S = steps;
  prof_begin(s, kPxCond, 0, 0);
  check(px_sinusoid(px.sinus, S, s.stream), "sinusoid");
  check(px_gemv(px.sinus, S, kFreq, px.wt1, px.bt1, hs, px.e1, false, true, s.stream),
        "t_embedder.0");
  check(px_gemv(px.e1, S, hs, px.wt2, s.mm_bcond, hs, px.temb, false, true, s.stream),
        "conditioning");
  const int next = s.first_layer + nl;
  for (int lf = 0; lf <= nl; ++lf) {
    const int l = s.first_layer + lf;
    if (lf == nl && next >= m.layers) break;
    const bool dbl = mm_double(l);
    for (int st = 0; st < 2; ++st) {
      float* dst = px.mod + (size_t(lf) * 2 + st) * S * w6;
      const bf16* W;
      const float* b;
      if (lf < nl) {
        const StageLayer& L = s.layers[size_t(lf)];
        W = (st && dbl) ? L.t_wmod : L.wmod;
        b = (st && dbl) ? L.t_bmod : L.bmod;
      } else {
        W = s.mm_next_wmod[st && dbl ? 1 : 0];
        b = s.mm_next_bmod[st && dbl ? 1 : 0];
      }
      if (dbl) {
        check(mm_gemv_bf16(px.temb, S, hs, W, b, w6, dst, w6, s.stream), "adaLN-Zero");
      } else if (st == 0) {
        check(mm_gemv_bf16(px.temb, S, hs, W, b, 3 * hs, dst, w6, s.stream), "adaLN-Zero");
        PF_CUDA_CHECK(cudaMemcpy2DAsync(dst + 3 * hs, size_t(w6) * 4, dst, size_t(w6) * 4,
                                        size_t(3 * hs) * 4, size_t(S), cudaMemcpyDeviceToDevice,
                                        s.stream));
      } else {
        PF_CUDA_CHECK(cudaMemcpyAsync(dst, dst - size_t(S) * w6, size_t(S) * w6 * 4,
                                      cudaMemcpyDeviceToDevice, s.stream));
      }
    }
  }
  check(px_fold_rows(px.mod, 2 * nl, S, hs, px.fold_aq, px.fold_am, px.fold_rpad, s.stream),
        "LayerNorm fold operands");
  for (int lf = 0; lf < nl; ++lf) {
    StageLayer& L = s.layers[size_t(lf)];
    const bool dbl = mm_double(s.first_layer + lf);
    for (int st = 0; st < 2; ++st) {
      const size_t b = size_t(lf) * 2 + st;
      const bool t = st && dbl;
      EpiParams fq;
      fq.out_f32 = px.foldq + b * 2 * S * 3 * hs;
      fq.ld = 3 * hs;
      fq.bias = t ? L.t_bqkv : L.bqkv;
      check(gemm(px.tm_aq[b], t ? L.tm_t_wqkv : L.tm_wqkv, 2 * S, 0, 3 * hs, hs, Epi::Fold, fq,
                 s.sm_count, s.stream), "LayerNorm fold (attention)");
      EpiParams fm;
      fm.out_f32 = px.foldm + b * 2 * S * m.mlp;
      fm.ld = m.mlp;
      fm.bias = t ? L.t_b1 : L.b1;
      check(gemm(px.tm_am[b], t ? L.tm_t_win : L.tm_win, 2 * S, 0, m.mlp, hs, Epi::Fold, fm,
                 s.sm_count, s.stream), "LayerNorm fold (MLP)");
    }
  }
  prof_end(s);
  px_steps_ = S;
}

// Image rows [row0, row0 + rows) of patch prepare (execute.cpp:198-203) with
// the operand of the first layer's image-stream LayerNorm.
void Engine::mm_patch_prepare(Stage& s0, float* x_dev, bool update, int row0, int rows, int t,
                              float eta) {
  const ModelShape& m = shape_;
  const size_t hs = size_t(m.hs), J = size_t(m.J());
  const float* scale1 = s0.px.mod + size_t(t) * 6 * hs + hs;  // layer 0, stream 0
  check(pf::px_patch_prepare(x_dev, s0.eps, s0.cb, scale1, s0.h32 + J * hs, s0.hb + J * hs,
                             s0.px.stats + J, int(m.rows_total()), row0, rows, m.hs, eta, update,
                             s0.stream),
        "patch_prepare (MMDiT)");
}

// The text rows re-enter from the text tokens (stream 1 of layer 0).
void Engine::mm_text_prepare(Stage& s0, int t) {
  const ModelShape& m = shape_;
  const size_t hs = size_t(m.hs), S = size_t(px_steps_);
  const float* scale1 = s0.px.mod + (S + size_t(t)) * 6 * hs + hs;  // layer 0, stream 1
  check(pf::px_patch_prepare(s0.text, nullptr, s0.px.zeros, scale1, s0.h32, s0.hb, s0.px.stats,
                             int(m.rows_total()), 0, int(m.J()), m.hs, 0.f, false, s0.stream),
        "text rows (MMDiT)");
}

void Engine::layer_forward_mm(Stage& s, int lf, int rows, int row0, int t, int code) {
  const ModelShape& m = shape_;
  StageLayer& L = s.layers[size_t(lf)];
  PxStage& px = s.px;
  const int hs = m.hs, w6 = 6 * hs, S = px_steps_, J = int(m.J()), Pt = int(m.rows_total());
  const int gl = s.first_layer + lf;
  const bool dbl = mm_double(gl);
  const double dhs = hs, mlp = m.mlp;
  auto modv = [&](int layer_local, int st) {
    return px.mod + ((size_t(layer_local) * 2 + st) * S + t) * w6;
  };
  const bool last_model_layer = gl + 1 == m.layers;
  auto next_scale1 = [&](int st) -> const float* {
    return last_model_layer ? nullptr : modv(lf + 1, st) + hs;
  };
  auto foldq = [&](int st) { return px.foldq + ((size_t(lf) * 2 + st) * 2 * S + 2 * t) * 3 * hs; };
  auto foldm = [&](int st) {
    return px.foldm + ((size_t(lf) * 2 + st) * 2 * S + 2 * t) * size_t(m.mlp);
  };
  // joint rows of the two streams: text [row0, J), image [max(row0, J), row0 + rows)
  const int t_rows = row0 < J ? std::min(row0 + rows, J) - row0 : 0;
  const int i_row0 = std::max(row0, J), i_rows = row0 + rows - i_row0;
  auto parts = [&](auto&& fn) {
    if (!dbl) {
      fn(0, row0, rows);
      return;
    }
    if (t_rows > 0) fn(1, row0, t_rows);
    if (i_rows > 0) fn(0, i_row0, i_rows);
  };
  auto wmap = [&](int st, const WeightMaps& a, const WeightMaps& b) -> const WeightMaps& {
    return st ? b : a;
  };
  // text rows (a partial last row tile): residual epilogue through maps that
  // end at the last text row, so the TMA stores clip there (not into the
  // image rows that follow); a redirected store keeps the register path
  auto text_maps = [&](int st, EpiParams& e) {
    if (st != 1 || e.out_f32_dst) return;
    e.tm_h32 = &s.tm_h32_txt;
    e.tm_hb = &s.tm_hb_txt;
    e.tma_clip = true;
  };

  EpiParams res;
  res.out_f32 = s.h32;
  res.out_bf16 = s.hb;
  res.ld = hs;
  res.flag = s.flag;
  res.code = code;
  res.tm_h32 = &s.tm_h32;
  res.tm_hb = &s.tm_hb;
  res.stats_ld = Pt;

  if (lane_wait_) PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, lane_wait_, 0));
  // 1. q, k, v = (LN(h)(1 + scale1) + shift1) Wqkv + bqkv per stream
  parts([&](int st, int r0, int n) {
    EpiParams qkv;
    qkv.q = s.q;
    qkv.k = L.k;
    qkv.v = L.v;
    qkv.hs = hs;
    qkv.dh = m.dh;
    qkv.dhp = m.dhp;
    qkv.P = Pt;
    qkv.stats_in = px.stats;
    qkv.stats_ld = Pt;
    qkv.ln_cols = hs;
    qkv.c1 = foldq(st);
    qkv.c2 = qkv.c1 + 3 * hs;
    prof_begin(s, kGemmQKV, 2.0 * n * dhs * 3 * dhs, 0);
    check(gemm(s.tm_hb, wmap(st, L.tm_wqkv, L.tm_t_wqkv), n, r0, 3 * hs, hs, Epi::QKV,
               sk(s, qkv), s.sm_count, s.stream), "gemm qkv (MMDiT)");
    prof_end(s);
  });
  if (!dbl) {  // single-stream: the MLP branch reads the same modulated input
    EpiParams ge;
    ge.out_bf16 = s.z;
    ge.ld = m.mlp;
    ge.stats_in = px.stats;
    ge.stats_ld = Pt;
    ge.ln_cols = hs;
    ge.c1 = foldm(0);
    ge.c2 = ge.c1 + m.mlp;
    prof_begin(s, kGemmMlpIn, 2.0 * rows * dhs * mlp, 0);
    check(gemm(s.tm_hb, L.tm_win, rows, row0, m.mlp, hs, Epi::Gelu, sk(s, ge), s.sm_count,
               s.stream), "gemm mlp-in (MMDiT single)");
    prof_end(s);
  }
  // 2. QK RMSNorm (+ RoPE) on this block's q / k rows
  const float* gq_t = dbl ? L.t_gq : L.gq;
  const float* gk_t = dbl ? L.t_gk : L.gk;
  check(mm_qk_norm_rope(s.q, L.k, m.heads, Pt, Pt, m.dhp, m.dh, row0, rows, J, L.gq, L.gk, gq_t,
                        gk_t, m.rope != 0, int(std::lround(std::floor(std::sqrt(double(m.P))))),
                        s.stream),
        "qk norm / rope");
  // 3. attention over the joint K/V rows
  AttnLaunch a{m.dhp, Pt, rows, row0, m.heads, m.dh, hs, float(1.0 / std::sqrt(double(m.dh))),
               s.attn, s.attn_work, s.attn_work_floats};
  a.flags = s.attn_flags;
  a.v_sum_col = m.dh < m.dhp;
  if (L.has_kv3) {
    a.k3 = &L.tm_k3;
    a.v3 = &L.tm_v3;
  }
  prof_begin(s, kAttention, 4.0 * rows * double(Pt) * dhs, 0);
  check(attention(s.tm_q, L.tm_k, L.tm_v, a, s.sm_count, s.stream), "attention (MMDiT)");
  prof_end(s);
  if (lane_rec_) PF_CUDA_CHECK(cudaEventRecord(lane_rec_, s.stream));

  auto redirect = [&](EpiParams& e) {
    if (!redirect_) return;  // last layer of a rank: store straight into the next stage
    e.out_f32_dst = redirect_->h32;
    e.out_bf16_dst = redirect_->hb;
    e.tm_h32_dst = redirect_->tm_h32;
    e.tm_hb_dst = redirect_->tm_hb;
    if (redirect_->stats) e.stats_out = redirect_->stats;
  };
  if (dbl) {
    // 4. h += gate1 (attn Wo + bo); operand h (1 + scale2) + LayerNorm stats
    parts([&](int st, int r0, int n) {
      EpiParams r1 = res;
      r1.bias = st ? L.t_bo : L.bo;
      r1.gate = modv(lf, st) + 2 * hs;
      r1.colscale = modv(lf, st) + 4 * hs;
      r1.stats_out = px.stats;
      text_maps(st, r1);
      prof_begin(s, kGemmOut, 2.0 * n * dhs * dhs, 0);
      check(gemm(s.tm_attn, wmap(st, L.tm_wo, L.tm_t_wo), n, r0, hs, hs, Epi::Residual,
                 sk(s, r1), s.sm_count, s.stream), "gemm out-proj (MMDiT)");
      prof_end(s);
    });
    // 5. z = gelu_tanh((LN(h)(1 + scale2) + shift2) W1 + b1)
    parts([&](int st, int r0, int n) {
      EpiParams ge;
      ge.out_bf16 = s.z;
      ge.ld = m.mlp;
      ge.stats_in = px.stats;
      ge.stats_ld = Pt;
      ge.ln_cols = hs;
      ge.c1 = foldm(st);
      ge.c2 = ge.c1 + m.mlp;
      prof_begin(s, kGemmMlpIn, 2.0 * n * dhs * mlp, 0);
      check(gemm(s.tm_hb, wmap(st, L.tm_win, L.tm_t_win), n, r0, m.mlp, hs, Epi::Gelu,
                 sk(s, ge), s.sm_count, s.stream), "gemm mlp-in (MMDiT)");
      prof_end(s);
    });
    // 6. h += gate2 (z W2 + b2); operand of the next layer's LayerNorm
    parts([&](int st, int r0, int n) {
      EpiParams r3 = res;
      r3.bias = st ? L.t_b2 : L.b2;
      r3.gate = modv(lf, st) + 5 * hs;
      r3.colscale = next_scale1(st);
      r3.stats_out = px.stats;
      redirect(r3);
      text_maps(st, r3);
      prof_begin(s, kGemmMlpOut, 2.0 * n * dhs * mlp, 0);
      check(gemm(s.tm_z, wmap(st, L.tm_wout, L.tm_t_wout), n, r0, hs, m.mlp, Epi::Residual,
                 sk(s, r3), s.sm_count, s.stream), "gemm mlp-out (MMDiT)");
      prof_end(s);
    });
    return;
  }
  // single-stream: h += gate (attn Wo + b2) ; h += gate (z W2)
  const float* gate = modv(lf, 0) + 2 * hs;
  EpiParams r1 = res;
  r1.bias = L.b2;
  r1.gate = gate;
  prof_begin(s, kGemmOut, 2.0 * rows * dhs * dhs, 0);
  check(gemm(s.tm_attn, L.tm_wo, rows, row0, hs, hs, Epi::Residual, sk(s, r1), s.sm_count,
             s.stream), "gemm out-proj (MMDiT single)");
  prof_end(s);
  EpiParams r3 = res;
  r3.gate = gate;
  r3.colscale = next_scale1(0);
  r3.stats_out = px.stats;
  redirect(r3);
  prof_begin(s, kGemmMlpOut, 2.0 * rows * dhs * mlp, 0);
  check(gemm(s.tm_z, L.tm_wout, rows, row0, hs, m.mlp, Epi::Residual, sk(s, r3), s.sm_count,
             s.stream), "gemm mlp-out (MMDiT single)");
  prof_end(s);
}

// Parameter bytes per stage (bf16 matrices, fp32 vectors) by block kind.
size_t Engine::param_bytes() const {
  const ModelShape& m = shape_;
  const size_t hs = size_t(m.hs), mlp = size_t(m.mlp), dh = size_t(m.dh);
  const size_t mats = (4 * hs * hs + 2 * hs * mlp) * 2;  // Wqkv, Wo, W1, W2 (bf16)
  const size_t vecs = (5 * hs + mlp) * 4;                  // bqkv, bo, b1, b2 (fp32)
  size_t total = 0;
  for (const Stage& s : stages_) {
    for (int lf = 0; lf < s.layer_count; ++lf) {
      const int l = s.first_layer + lf;
      switch (m.block) {
        case kBlockMMDiT: {
          const int streams = mm_double(l) ? 2 : 1;
          const size_t w6 = mm_double(l) ? 6 * hs : 3 * hs;
          total += size_t(streams) * (mats + vecs + w6 * hs * 2 + w6 * 4 + 2 * dh * 4);
          break;
        }
        case kBlockJoint:
          total += size_t(l < m.double_layers ? 2 : 1) * mats;
          break;
        case kBlockPixArt:
          total += mats + vecs + 4 * hs * hs * 2 + 4 * hs * 4 + 6 * hs * 4;
          break;
        default:
          total += mats;
      }
    }
  }
  return total;
}

size_t Engine::kv_bytes() const {
  const ModelShape& m = shape_;
  size_t layers = 0;
  for (const Stage& s : stages_) layers += size_t(s.layer_count);
  return layers * 2 * size_t(m.heads) * size_t(m.rows_total()) * size_t(m.dhp) * 2;
}

}  // namespace pf
