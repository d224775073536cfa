// PipeFusion runtime (see runtime.h for the mapping onto the reference).
#include "runtime.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <sstream>

namespace pf {

#define PF_CUDA_CHECK(expr)                                                  \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      std::ostringstream _os;                                                \
      _os << "CUDA error " << cudaGetErrorString(_e) << " at " << __FILE__   \
          << ":" << __LINE__ << " (" #expr ")";                              \
      throw CudaError(_os.str());                                            \
    }                                                                        \
  } while (0)

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  PF_CUDA_CHECK(cudaMalloc(&p, n * sizeof(T)));
  PF_CUDA_CHECK(cudaMemset(p, 0, n * sizeof(T)));
  return static_cast<T*>(p);
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

CUtensorMap tmap(const void* base, uint64_t inner, uint64_t outer,
                 uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
                 int swizzle) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  if (!encode_tmap_bf16_2d(&m, base, inner, outer, row_bytes, box_inner,
                           box_outer, swizzle)) {
    std::ostringstream os;
    os << "cuTensorMapEncodeTiled failed (inner=" << inner << " outer=" << outer
       << " box=" << box_inner << "x" << box_outer << ")";
    throw CudaError(os.str());
  }
  return m;
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::ostringstream os;
    os << "CUDA error " << cudaGetErrorString(e) << " launching " << what;
    throw CudaError(os.str());
  }
}

}  // namespace

void validate_shape(const ModelShape& s) {
  if (s.layers < 1) throw ValidationError("toy model needs layers >= 1");
  if (s.hs < 1 || s.heads < 1)
    throw ValidationError("toy model needs hidden_size >= 1 and heads >= 1");
  if (s.hs % s.heads != 0) {
    std::ostringstream os;
    os << "hidden_size (" << s.hs << ") must be divisible by heads (" << s.heads
       << ")";
    throw ValidationError(os.str());
  }
  if (s.mlp < 1) throw ValidationError("mlp_ratio * hidden_size must be >= 1");
  if (s.P < 1) throw ValidationError("latent needs seq_len >= 1 and hidden_size >= 1");
  // Device-layout constraints of the CUDA backend (16-byte TMA row pitch).
  if (s.hs % 8 != 0 || s.mlp % 8 != 0)
    throw ValidationError("CUDA backend needs hidden_size and mlp hidden size divisible by 8");
  if (s.P % 8 != 0) throw ValidationError("CUDA backend needs seq_len divisible by 8");
  if (s.hs / s.heads > 128) throw ValidationError("CUDA backend supports head dim <= 128");
}

Engine::Engine(const ModelShape& shape_in, const std::vector<int>& devices)
    : shape_(shape_in) {
  shape_.dh = shape_.hs / std::max(shape_.heads, 1);
  shape_.dhp = (shape_.dh + 15) / 16 * 16;
  validate_shape(shape_);
  const int n = int(devices.size());
  if (n < 1) throw ValidationError("workers and patches must be >= 1");
  if (n > shape_.layers) {
    std::ostringstream os;
    os << "layer count " << shape_.layers << " is not divisible by workers " << n
       << " (fewer layers than stages)";
    throw ValidationError(os.str());
  }
  int dev_count = 0;
  PF_CUDA_CHECK(cudaGetDeviceCount(&dev_count));
  for (int d : devices) {
    if (d < 0 || d >= dev_count) {
      std::ostringstream os;
      os << "CUDA device " << d << " not present (" << dev_count << " visible)";
      throw ValidationError(os.str());
    }
  }
  stages_.resize(size_t(n));
  try {
    for (int d = 0; d < n; ++d) {
      Stage& s = stages_[size_t(d)];
      s.device = devices[size_t(d)];
      // Balanced contiguous split; equals the reference's d*L/N .. (d+1)*L/N
      // when N divides L (execute.cpp:107-112, 138-139), and relaxes it
      // otherwise (e.g. 28 layers on 8 stages).
      const int first = int(int64_t(d) * shape_.layers / n);
      const int last = int(int64_t(d + 1) * shape_.layers / n);
      alloc_stage(s, first, last - first, d == 0);
    }
    // Peer access between neighbouring stages on distinct devices.
    for (int d = 0; d < n; ++d) {
      const int a = stages_[size_t(d)].device;
      const int b = stages_[size_t((d + 1) % n)].device;
      if (a == b) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, a, b);
      if (ok) {
        DeviceGuard g(a);
        cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      }
    }
  } catch (...) {
    for (Stage& s : stages_) free_stage(s);
    throw;
  }
}

Engine::~Engine() {
  if (ev_start_) {
    DeviceGuard g(stages_[0].device);
    cudaEventDestroy(ev_start_);
  }
  for (auto& kv : graphs_)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (size_t d = 0; d < prof_pool_.size() && d < stages_.size(); ++d) {
    DeviceGuard g(stages_[d].device);
    for (cudaEvent_t e : prof_pool_[d]) cudaEventDestroy(e);
  }
  for (Stage& s : stages_) free_stage(s);
}

void Engine::alloc_stage(Stage& s, int first, int count, bool is_first) {
  DeviceGuard g(s.device);
  const ModelShape& m = shape_;
  const size_t P = size_t(m.P), hs = size_t(m.hs), mlp = size_t(m.mlp);
  const size_t heads = size_t(m.heads), dhp = size_t(m.dhp);
  s.first_layer = first;
  s.layer_count = count;
  s.sm_count = device_sm_count(s.device);
  PF_CUDA_CHECK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  PF_CUDA_CHECK(cudaEventCreateWithFlags(&s.ev_fwd, cudaEventDisableTiming));
  s.h32 = dalloc<float>(P * hs);
  s.hb = dalloc<bf16>(P * hs);
  s.q = dalloc<bf16>(heads * P * dhp);
  s.attn = dalloc<bf16>(P * hs);
  s.z = dalloc<bf16>(P * mlp);
  s.flag = dalloc<int>(1);
  // Split-KV workspace sized for the worst case (a single 128-row q tile).
  {
    AttnLaunch probe{int(dhp), int(P), 128, 0, int(heads), m.dh, int(hs), 1.f,
                     nullptr, nullptr, 0};
    const int splits = attn_splits(probe, s.sm_count);
    size_t need = 0;
    // any rows >= 128 use fewer splits per tile; bound by splits * tiles
    for (int rows = 128; rows <= int(P) + 127; rows += 128) {
      probe.rows = rows;
      need = std::max(need, attn_work_floats(int(dhp), int(heads), rows,
                                             attn_splits(probe, s.sm_count)));
    }
    (void)splits;
    s.attn_work_floats = need;
    s.attn_work = need ? dalloc<float>(need) : nullptr;
  }
  s.tm_hb = tmap(s.hb, hs, P, hs * 2, 64, 128, 128);
  if (!encode_tmap_f32_2d(&s.tm_h32, s.h32, hs, P, hs * 4, 32, 128, 128))
    throw CudaError("cuTensorMapEncodeTiled failed for the residual stream");
  s.tm_attn = tmap(s.attn, hs, P, hs * 2, 64, 128, 128);
  s.tm_z = tmap(s.z, mlp, P, mlp * 2, 64, 128, 128);
  s.tm_q = tmap(s.q, dhp, heads * P, dhp * 2, 16, 128, 32);
  s.layers.resize(size_t(count));
  for (StageLayer& L : s.layers) {
    L.wqkv = dalloc<bf16>(3 * hs * hs);
    L.wo = dalloc<bf16>(hs * hs);
    L.win = dalloc<bf16>(mlp * hs);
    L.wout = dalloc<bf16>(hs * mlp);
    L.k = dalloc<bf16>(heads * P * dhp);
    L.v = dalloc<bf16>(heads * P * dhp);
    if (!make_weight_maps(&L.tm_wqkv, L.wqkv, int(3 * hs), int(hs)) ||
        !make_weight_maps(&L.tm_wo, L.wo, int(hs), int(hs)) ||
        !make_weight_maps(&L.tm_win, L.win, int(mlp), int(hs)) ||
        !make_weight_maps(&L.tm_wout, L.wout, int(hs), int(mlp)))
      throw CudaError("cuTensorMapEncodeTiled failed for a weight matrix");
    L.tm_k = tmap(L.k, dhp, heads * P, dhp * 2, 16, 128, 32);
    L.tm_v = tmap(L.v, dhp, heads * P, dhp * 2, 16, 128, 32);
  }
  if (is_first) {
    s.x = dalloc<float>(P * hs);
    s.cb = dalloc<float>(hs);
  }
}

void Engine::free_stage(Stage& s) {
  if (!s.stream && !s.h32) return;
  DeviceGuard g(s.device);
  if (s.stream) cudaStreamSynchronize(s.stream);
  for (StageLayer& L : s.layers) {
    dfree(L.wqkv); dfree(L.wo); dfree(L.win); dfree(L.wout);
    dfree(L.k); dfree(L.v);
  }
  s.layers.clear();
  dfree(s.h32); dfree(s.hb); dfree(s.q); dfree(s.attn); dfree(s.z);
  dfree(s.attn_work); dfree(s.flag); dfree(s.x); dfree(s.cb);
  if (s.eps && s.eps != s.h32) dfree(s.eps);
  for (cudaEvent_t e : s.ev_eps) cudaEventDestroy(e);
  s.ev_eps.clear();
  if (s.ev_fwd) cudaEventDestroy(s.ev_fwd);
  if (s.stream) cudaStreamDestroy(s.stream);
  s = Stage{};
}

int Engine::stage_of_layer(int layer) const {
  for (int d = 0; d < stage_count(); ++d) {
    const Stage& s = stages_[size_t(d)];
    if (layer >= s.first_layer && layer < s.first_layer + s.layer_count) return d;
  }
  return -1;
}

void Engine::load_layer(int layer, const HostMatrix (&w)[6]) {
  const int d = stage_of_layer(layer);
  if (d < 0) throw ValidationError("layer index out of range");
  Stage& s = stages_[size_t(d)];
  StageLayer& L = s.layers[size_t(layer - s.first_layer)];
  const int hs = shape_.hs, mlp = shape_.mlp;
  // Transpose to N x K (K-major) bf16: dst[n*K + k] = W[k][n].
  auto pack = [](const HostMatrix& W, std::vector<bf16>& dst, size_t n_off, int K) {
    for (int n = 0; n < W.cols; ++n)
      for (int k = 0; k < K; ++k)
        dst[(n_off + size_t(n)) * size_t(K) + size_t(k)] = __float2bfloat16_rn(float(W.at(k, n)));
  };
  std::vector<bf16> qkv(size_t(3) * hs * hs), wo(size_t(hs) * hs),
      win(size_t(mlp) * hs), wout(size_t(hs) * mlp);
  pack(w[0], qkv, 0, hs);
  pack(w[1], qkv, size_t(hs), hs);
  pack(w[2], qkv, size_t(2) * hs, hs);
  pack(w[3], wo, 0, hs);
  pack(w[4], win, 0, hs);
  pack(w[5], wout, 0, mlp);
  DeviceGuard g(s.device);
  PF_CUDA_CHECK(cudaMemcpy(L.wqkv, qkv.data(), qkv.size() * 2, cudaMemcpyHostToDevice));
  PF_CUDA_CHECK(cudaMemcpy(L.wo, wo.data(), wo.size() * 2, cudaMemcpyHostToDevice));
  PF_CUDA_CHECK(cudaMemcpy(L.win, win.data(), win.size() * 2, cudaMemcpyHostToDevice));
  PF_CUDA_CHECK(cudaMemcpy(L.wout, wout.data(), wout.size() * 2, cudaMemcpyHostToDevice));
}

void Engine::load_condition_bias(const double* cb) {
  std::vector<float> v(size_t(shape_.hs));
  for (int i = 0; i < shape_.hs; ++i) v[size_t(i)] = float(cb[i]);
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  PF_CUDA_CHECK(cudaMemcpy(s.cb, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
}

// One toy DiT layer over rows [row0, row0+rows) (toy_model.cpp:169-177):
// fused QKV projection writing this block's K/V rows into the full buffers,
// attention over all P rows, out-proj residual, tanh MLP, MLP residual.
void Engine::layer_forward(Stage& s, int lf, int rows, int row0, int code) {
  const ModelShape& m = shape_;
  StageLayer& L = s.layers[size_t(lf)];
  const double r = rows, hs = m.hs, mlp = m.mlp, P = double(m.P);
  EpiParams qkv;
  qkv.q = s.q;
  qkv.k = L.k;
  qkv.v = L.v;
  qkv.hs = m.hs;
  qkv.dh = m.dh;
  qkv.dhp = m.dhp;
  qkv.P = int(m.P);
  prof_begin(s, kGemmQKV, 2 * r * hs * 3 * hs, 0);
  check(gemm(s.tm_hb, L.tm_wqkv, rows, row0, 3 * m.hs, m.hs, Epi::QKV, qkv,
             s.sm_count, s.stream), "gemm qkv");
  prof_end(s);
  AttnLaunch a{m.dhp, int(m.P), rows, row0, m.heads, m.dh, m.hs,
               float(1.0 / std::sqrt(double(m.dh))), s.attn, s.attn_work,
               s.attn_work_floats};
  prof_begin(s, kAttention, 4 * r * P * hs, 0);
  check(attention(s.tm_q, L.tm_k, L.tm_v, a, s.sm_count, s.stream), "attention");
  prof_end(s);
  EpiParams res;
  res.out_f32 = s.h32;
  res.out_bf16 = s.hb;
  res.ld = m.hs;
  res.flag = s.flag;
  res.code = code;
  if (m.hs % 32 == 0) {
    res.tm_h32 = &s.tm_h32;
    res.tm_hb = &s.tm_hb;
  }
  prof_begin(s, kGemmOut, 2 * r * hs * hs, 0);
  check(gemm(s.tm_attn, L.tm_wo, rows, row0, m.hs, m.hs, Epi::Residual, res,
             s.sm_count, s.stream), "gemm out-proj");
  prof_end(s);
  EpiParams th;
  th.out_bf16 = s.z;
  th.ld = m.mlp;
  prof_begin(s, kGemmMlpIn, 2 * r * hs * mlp, 0);
  check(gemm(s.tm_hb, L.tm_win, rows, row0, m.mlp, m.hs, Epi::Tanh, th,
             s.sm_count, s.stream), "gemm mlp-in");
  prof_end(s);
  prof_begin(s, kGemmMlpOut, 2 * r * hs * mlp, 0);
  check(gemm(s.tm_z, L.tm_wout, rows, row0, m.hs, m.mlp, Epi::Residual, res,
             s.sm_count, s.stream), "gemm mlp-out");
  prof_end(s);
  const int splits = attn_splits(a, s.sm_count);
  launches_ += 5 + (splits > 1 ? 1 : 0);
}

cudaEvent_t Engine::prof_event(int stage) {
  if (prof_pool_.size() < stages_.size()) prof_pool_.resize(stages_.size());
  if (prof_used_.size() < stages_.size()) prof_used_.resize(stages_.size(), 0);
  auto& pool = prof_pool_[size_t(stage)];
  size_t& used = prof_used_[size_t(stage)];
  if (used == pool.size()) {
    cudaEvent_t e;
    PF_CUDA_CHECK(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

void Engine::prof_begin(Stage& s, int kind, double flops, double bytes) {
  if (!profiling_) return;
  const int d = int(&s - stages_.data());
  ProfRec r{kind, d, prof_event(d), prof_event(d), flops, bytes};
  PF_CUDA_CHECK(cudaEventRecord(r.a, s.stream));
  prof_.push_back(r);
}

void Engine::prof_end(Stage& s) {
  if (!profiling_) return;
  PF_CUDA_CHECK(cudaEventRecord(prof_.back().b, s.stream));
}

KernelProfile Engine::collect_profile() {
  KernelProfile out;
  for (const ProfRec& r : prof_) {
    DeviceGuard g(stages_[size_t(r.stage)].device);
    PF_CUDA_CHECK(cudaEventSynchronize(r.b));
    float ms = 0.f;
    PF_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
    out.ms[r.kind] += ms;
    out.launches[r.kind] += 1;
    out.flops[r.kind] += r.flops;
    out.bytes[r.kind] += r.bytes;
  }
  return out;
}

// Stage-boundary transfer of rows [row0, row0+rows) of the residual stream:
// stage d -> stage d+1 (activation, fp32 + its bf16 operand copy), or last
// stage -> stage 0 (noise estimate eps, fp32). Stream-ordered on the sender;
// the receiver's stream waits on an event (the reference's Channel::push/pop,
// channel.hpp:33-57).
void Engine::send_rows(int from, int row0, int rows) {
  const int n = stage_count();
  Stage& src = stages_[size_t(from)];
  const size_t off = size_t(row0) * shape_.hs;
  const size_t cnt = size_t(rows) * shape_.hs;
  DeviceGuard g(src.device);
  if (from + 1 < n) {
    Stage& dst = stages_[size_t(from + 1)];
    PF_CUDA_CHECK(cudaMemcpyAsync(dst.h32 + off, src.h32 + off, cnt * 4,
                                  cudaMemcpyDefault, src.stream));
    PF_CUDA_CHECK(cudaMemcpyAsync(dst.hb + off, src.hb + off, cnt * 2,
                                  cudaMemcpyDefault, src.stream));
    PF_CUDA_CHECK(cudaEventRecord(src.ev_fwd, src.stream));
    DeviceGuard g2(dst.device);
    PF_CUDA_CHECK(cudaStreamWaitEvent(dst.stream, src.ev_fwd, 0));
  } else if (n > 1) {
    Stage& s0 = stages_[0];
    PF_CUDA_CHECK(cudaMemcpyAsync(s0.eps + off, src.h32 + off, cnt * 4,
                                  cudaMemcpyDefault, src.stream));
  }
}

void Engine::enqueue_run(float* x_dev, int steps, int patches, int warmup,
                         float eta, cudaStream_t caller, RunStats* stats) {
  const ModelShape& m = shape_;
  const int n = stage_count();
  // check_pipefusion_args (execute.cpp:97-131), with the layer divisibility
  // relaxed (stages may hold L/N rounded up or down).
  if (steps < 1) throw ValidationError("steps must be >= 1");
  if (patches < 1) throw ValidationError("workers and patches must be >= 1");
  if (warmup < 0 || warmup > steps) throw ValidationError("warmup must lie in [0, steps]");
  if (m.P % patches != 0) {
    std::ostringstream os;
    os << "seq_len " << m.P << " is not divisible by patches " << patches;
    throw ValidationError(os.str());
  }
  const int r = int(m.P / patches);
  if (patches > 1 && r % 8 != 0) {
    std::ostringstream os;
    os << "CUDA backend needs seq_len / patches divisible by 8 (got " << r << ")";
    throw ValidationError(os.str());
  }
  Stage& s0 = stages_[0];
  prepare_run(patches);

  // Host bookkeeping: StageBuffers::src (execute.cpp:38-49), sentinel = steps.
  std::vector<std::vector<std::vector<int>>> src(static_cast<size_t>(n));
  RunStats local;
  RunStats& st = stats ? *stats : local;
  st.fresh = 0;
  st.stale = 0;
  st.fresh_fraction.assign(size_t(n), {});
  for (int d = 0; d < n; ++d)
    src[size_t(d)].assign(size_t(stages_[size_t(d)].layer_count),
                          std::vector<int>(size_t(patches), steps));
  codes_.clear();
  launches_ = 0;
  prof_.clear();
  prof_used_.assign(stages_.size(), 0);

  // Fork: every stage stream waits for the caller's prior work.
  cudaEvent_t ev_start = ev_start_;
  {
    DeviceGuard g(s0.device);
    PF_CUDA_CHECK(cudaEventRecord(ev_start, caller));
  }
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, ev_start, 0));
    check(reset_flag(s.flag, s.stream), "reset_flag");
    ++launches_;
    // StageBuffers are zero-initialised per run (execute.cpp:42-48). Without
    // warmup the zero rows are read as stale context, so clear them; with
    // warmup every row is rewritten before it is read.
    if (warmup == 0) {
      const size_t kv = size_t(m.heads) * size_t(m.P) * size_t(m.dhp) * sizeof(bf16);
      for (StageLayer& L : s.layers) {
        PF_CUDA_CHECK(cudaMemsetAsync(L.k, 0, kv, s.stream));
        PF_CUDA_CHECK(cudaMemsetAsync(L.v, 0, kv, s.stream));
      }
    }
  }
  auto next_code = [&](int t, int layer) {
    codes_.emplace_back(t, layer);
    return int(codes_.size()) - 1;
  };

  // ---- warmup: synchronous full-sequence steps (execute.cpp:181-190)
  for (int w = 0; w < warmup; ++w) {
    const int t = steps - 1 - w;
    {
      DeviceGuard g(s0.device);
      prof_begin(s0, kSampler, 0, double(m.P) * m.hs * (4 + 4 + 2));
      check(patch_prepare(x_dev, nullptr, s0.cb, s0.h32, s0.hb, 0, int(m.P), m.hs,
                          0.f, false, s0.stream), "patch_prepare");
      prof_end(s0);
      ++launches_;
    }
    for (int d = 0; d < n; ++d) {
      Stage& s = stages_[size_t(d)];
      DeviceGuard g(s.device);
      for (int lf = 0; lf < s.layer_count; ++lf) {
        auto& sv = src[size_t(d)][size_t(lf)];
        std::fill(sv.begin(), sv.end(), t);
        st.fresh += patches;
        layer_forward(s, lf, int(m.P), 0, next_code(t, s.first_layer + lf));
      }
      send_rows(d, 0, int(m.P));
    }
    if (n > 1) {
      Stage& last = stages_[size_t(n - 1)];
      DeviceGuard g(last.device);
      PF_CUDA_CHECK(cudaEventRecord(s0.ev_eps[0], last.stream));
      DeviceGuard g0(s0.device);
      PF_CUDA_CHECK(cudaStreamWaitEvent(s0.stream, s0.ev_eps[0], 0));
    }
    DeviceGuard g(s0.device);
    prof_begin(s0, kSampler, 0, double(m.P) * m.hs * 12);
    check(latent_update(x_dev, s0.eps, eta, size_t(m.P) * m.hs, s0.stream), "latent_update");
    prof_end(s0);
    ++launches_;
  }

  // ---- steady: patch pipeline (execute.cpp:192-212)
  const int steady = steps - warmup;
  for (int q = 0; q < steady; ++q) {
    const int t = steady - 1 - q;
    for (int j = 0; j < patches; ++j) {
      const int row0 = j * r;
      {
        DeviceGuard g(s0.device);
        if (q > 0 && n > 1)
          PF_CUDA_CHECK(cudaStreamWaitEvent(s0.stream, s0.ev_eps[size_t(j)], 0));
        prof_begin(s0, kSampler, 0, double(r) * m.hs * (q > 0 ? 4 + 4 + 4 + 4 + 2 : 4 + 4 + 2));
        check(patch_prepare(x_dev, s0.eps, s0.cb, s0.h32, s0.hb, row0, r, m.hs, eta,
                            q > 0, s0.stream), "patch_prepare");
        prof_end(s0);
        ++launches_;
      }
      for (int d = 0; d < n; ++d) {
        Stage& s = stages_[size_t(d)];
        DeviceGuard g(s.device);
        for (int lf = 0; lf < s.layer_count; ++lf) {
          auto& sv = src[size_t(d)][size_t(lf)];
          sv[size_t(j)] = t;
          // check_staleness_and_count (execute.cpp:51-65)
          for (size_t pi = 0; pi < sv.size(); ++pi) {
            if (sv[pi] == t) {
              ++st.fresh;
            } else if (sv[pi] == t + 1) {
              ++st.stale;
            } else {
              std::ostringstream os;
              os << "staleness bound violated: patch " << pi << " carries timestep "
                 << sv[pi] << " while computing timestep " << t;
              throw NumericError(os.str());
            }
          }
          layer_forward(s, lf, r, row0, next_code(t, s.first_layer + lf));
        }
        // fresh_fraction(src[0], t) after the stage (execute.cpp:67-73,164)
        {
          const auto& s0v = src[size_t(d)][0];
          int fresh = 0;
          for (int v : s0v) fresh += (v == t);
          st.fresh_fraction[size_t(d)].push_back(double(fresh) / double(s0v.size()));
        }
        send_rows(d, row0, r);
        if (d == n - 1 && n > 1)
          PF_CUDA_CHECK(cudaEventRecord(s0.ev_eps[size_t(j)], s.stream));
      }
    }
  }
  if (steady > 0) {
    DeviceGuard g(s0.device);
    if (n > 1)
      for (int j = 0; j < patches; ++j)
        PF_CUDA_CHECK(cudaStreamWaitEvent(s0.stream, s0.ev_eps[size_t(j)], 0));
    prof_begin(s0, kSampler, 0, double(m.P) * m.hs * 12);
    check(latent_update(x_dev, s0.eps, eta, size_t(m.P) * m.hs, s0.stream), "latent_update");
    prof_end(s0);
    ++launches_;
  }

  // Join: the caller's stream waits for every stage.
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    PF_CUDA_CHECK(cudaEventRecord(s.ev_fwd, s.stream));
    DeviceGuard g0(s0.device);
    PF_CUDA_CHECK(cudaStreamWaitEvent(caller, s.ev_fwd, 0));
  }
}

// Allocations and events a run needs, created outside any stream capture.
void Engine::prepare_run(int patches) {
  const int n = stage_count();
  Stage& s0 = stages_[0];
  if (!ev_start_) {
    DeviceGuard g(s0.device);
    PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_start_, cudaEventDisableTiming));
  }
  if (n > 1 && !s0.eps) {
    DeviceGuard g(s0.device);
    s0.eps = dalloc<float>(size_t(shape_.P) * shape_.hs);
  }
  if (n == 1) s0.eps = s0.h32;
  if (int(s0.ev_eps.size()) < patches) {
    DeviceGuard g(stages_[size_t(n - 1)].device);
    while (int(s0.ev_eps.size()) < patches) {
      cudaEvent_t e;
      PF_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      s0.ev_eps.push_back(e);
    }
  }
}

void Engine::run(float* x_dev, int steps, int patches, int warmup, float eta,
                 cudaStream_t caller, RunStats* stats) {
  if (patches >= 1) prepare_run(patches);
  bool single_device = true;
  for (const Stage& s : stages_) single_device &= s.device == stages_[0].device;
  if (!graphs_enabled_ || profiling_ || caller == nullptr || !single_device) {
    enqueue_run(x_dev, steps, patches, warmup, eta, caller, stats);
    return;
  }
  uint32_t eta_bits;
  std::memcpy(&eta_bits, &eta, sizeof(eta_bits));
  const GraphKey key{x_dev, steps, patches, warmup, eta_bits, caller};
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    GraphEntry e;
    DeviceGuard g(stages_[0].device);
    PF_CUDA_CHECK(cudaStreamBeginCapture(caller, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t graph = nullptr;
    try {
      enqueue_run(x_dev, steps, patches, warmup, eta, caller, &e.stats);
    } catch (...) {
      cudaStreamEndCapture(caller, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    PF_CUDA_CHECK(cudaStreamEndCapture(caller, &graph));
    cudaError_t err = cudaGraphInstantiate(&e.exec, graph, 0);
    cudaGraphDestroy(graph);
    PF_CUDA_CHECK(err);
    e.launches = launches_;
    e.codes = codes_;
    it = graphs_.emplace(key, std::move(e)).first;
  }
  DeviceGuard g(stages_[0].device);
  PF_CUDA_CHECK(cudaGraphLaunch(it->second.exec, caller));
  launches_ = it->second.launches;
  codes_ = it->second.codes;
  if (stats) *stats = it->second.stats;
}

void Engine::finish(cudaStream_t caller) {
  {
    DeviceGuard g(stages_[0].device);
    PF_CUDA_CHECK(cudaStreamSynchronize(caller));
  }
  int first = INT_MAX;
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
    int f = INT_MAX;
    PF_CUDA_CHECK(cudaMemcpy(&f, s.flag, sizeof(int), cudaMemcpyDeviceToHost));
    first = std::min(first, f);
  }
  if (first != INT_MAX && first >= 0 && size_t(first) < codes_.size()) {
    std::ostringstream os;
    os << "non-finite activation at timestep " << codes_[size_t(first)].first
       << ", layer " << codes_[size_t(first)].second;
    throw NumericError(os.str());
  }
}

void Engine::layer_forward_host(int layer, double* h, int64_t rows, int64_t row0,
                                double* k_buf, double* v_buf, bool col_major) {
  const ModelShape& m = shape_;
  const int d = stage_of_layer(layer);
  if (d < 0) throw ValidationError("layer index out of range");
  if (rows < 1 || row0 < 0 || row0 + rows > m.P)
    throw ValidationError("row block outside the K/V buffer");
  Stage& s = stages_[size_t(d)];
  StageLayer& L = s.layers[size_t(layer - s.first_layer)];
  const int64_t P = m.P;
  const int hs = m.hs;
  auto idx = [&](int64_t r, int64_t c, int64_t nrows) {
    return col_major ? size_t(c * nrows + r) : size_t(r * hs + c);
  };
  // Host -> device: h rows into h32/hb at row0; K, V into the padded layouts.
  std::vector<float> h32(size_t(rows) * hs);
  std::vector<bf16> hb(size_t(rows) * hs);
  for (int64_t r = 0; r < rows; ++r)
    for (int c = 0; c < hs; ++c) {
      const float v = float(h[idx(r, c, rows)]);
      h32[size_t(r) * hs + c] = v;
      hb[size_t(r) * hs + c] = __float2bfloat16_rn(v);
    }
  std::vector<bf16> kd(size_t(m.heads) * P * m.dhp, __float2bfloat16_rn(0.f));
  std::vector<bf16> vd(size_t(m.heads) * P * m.dhp, __float2bfloat16_rn(0.f));
  for (int64_t r = 0; r < P; ++r)
    for (int c = 0; c < hs; ++c) {
      const int head = c / m.dh, dd = c % m.dh;
      kd[(size_t(head) * P + r) * m.dhp + dd] = __float2bfloat16_rn(float(k_buf[idx(r, c, P)]));
      vd[(size_t(head) * P + r) * m.dhp + dd] = __float2bfloat16_rn(float(v_buf[idx(r, c, P)]));
    }
  DeviceGuard g(s.device);
  PF_CUDA_CHECK(cudaMemcpyAsync(s.h32 + row0 * hs, h32.data(), h32.size() * 4,
                                cudaMemcpyHostToDevice, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(s.hb + row0 * hs, hb.data(), hb.size() * 2,
                                cudaMemcpyHostToDevice, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(L.k, kd.data(), kd.size() * 2, cudaMemcpyHostToDevice, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(L.v, vd.data(), vd.size() * 2, cudaMemcpyHostToDevice, s.stream));
  check(reset_flag(s.flag, s.stream), "reset_flag");
  codes_.assign(1, {0, layer});
  launches_ = 1;
  layer_forward(s, layer - s.first_layer, int(rows), int(row0), 0);
  PF_CUDA_CHECK(cudaMemcpyAsync(h32.data(), s.h32 + row0 * hs, h32.size() * 4,
                                cudaMemcpyDeviceToHost, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(kd.data(), L.k, kd.size() * 2, cudaMemcpyDeviceToHost, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(vd.data(), L.v, vd.size() * 2, cudaMemcpyDeviceToHost, s.stream));
  PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
  for (int64_t r = 0; r < rows; ++r)
    for (int c = 0; c < hs; ++c) h[idx(r, c, rows)] = double(h32[size_t(r) * hs + c]);
  for (int64_t r = 0; r < P; ++r)
    for (int c = 0; c < hs; ++c) {
      const int head = c / m.dh, dd = c % m.dh;
      k_buf[idx(r, c, P)] = double(__bfloat162float(kd[(size_t(head) * P + r) * m.dhp + dd]));
      v_buf[idx(r, c, P)] = double(__bfloat162float(vd[(size_t(head) * P + r) * m.dhp + dd]));
    }
  int f = INT_MAX;
  PF_CUDA_CHECK(cudaMemcpy(&f, s.flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (f != INT_MAX) {
    std::ostringstream os;
    os << "non-finite activation at timestep 0, layer " << layer;
    throw NumericError(os.str());
  }
}

}  // namespace pf
