// PipeFusion runtime (see runtime.h for the mapping onto the reference).
#include "runtime.h"
#include "runtime_internal.h"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <chrono>
#include <mutex>
#include <random>
#include <sstream>
#include <thread>
#include <type_traits>

#include <unistd.h>

namespace pf {

namespace {

// Patch lanes run without programmatic dependent launch: an early-launched
// grid waiting on its predecessor holds SMs the other lanes could use
// (C2 M = 8: 0.201 vs 0.207 s; PF_LANES_PDL=1 keeps PDL). Scoped, per thread.
struct PdlOff {
  bool prev;
  explicit PdlOff(bool lanes) : prev(pdl_thread_off()) { set(lanes); }
  void set(bool lanes) {
    static const bool keep = [] {
      const char* e = std::getenv("PF_LANES_PDL");
      return e && e[0] == '1';
    }();
    pdl_thread_off() = lanes && !keep;
  }
  ~PdlOff() { pdl_thread_off() = prev; }
};

// Counts the kernels a run enqueues (launch_counter() delta over its scope).
struct LaunchTally {
  int64_t& out;
  int64_t base;
  explicit LaunchTally(int64_t& o) : out(o), base(launch_counter()) {}
  ~LaunchTally() { out = launch_counter() - base; }
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



// Graph nodes of captured stream memory operations (batch mem-op nodes):
// enumerated once after capture, their values patched before a replay.
struct GraphMemOps {
  CUresult (*node_type)(CUgraphNode, CUgraphNodeType*) = nullptr;
  CUresult (*get)(CUgraphNode, CUDA_BATCH_MEM_OP_NODE_PARAMS*) = nullptr;
  CUresult (*exec_set)(CUgraphExec, CUgraphNode, const CUDA_BATCH_MEM_OP_NODE_PARAMS*) = nullptr;
};

const GraphMemOps& graph_memops() {
  static GraphMemOps g;
  static std::once_flag once;
  std::call_once(once, [&] {
    auto get = [](const char* name, auto& fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
    };
    get("cuGraphNodeGetType", g.node_type);
    get("cuGraphBatchMemOpNodeGetParams", g.get);
    get("cuGraphExecBatchMemOpNodeSetParams", g.exec_set);
  });
  if (!g.node_type || !g.get || !g.exec_set)
    throw CudaError("graph batch memory-operation entry points are unavailable");
  return g;
}

// Per-process identity for PeerBlob: hostname + boot id, and a random nonce.
uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ULL) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ULL;
  return h;
}
uint64_t host_identity() {
  static const uint64_t id = [] {
    char host[256] = {0};
    gethostname(host, sizeof(host) - 1);
    std::string boot;
    if (FILE* f = std::fopen("/proc/sys/kernel/random/boot_id", "r")) {
      char buf[64] = {0};
      if (std::fgets(buf, sizeof(buf), f)) boot = buf;
      std::fclose(f);
    }
    return fnv1a(boot, fnv1a(host));
  }();
  return id;
}
uint64_t process_nonce() {
  static const uint64_t n = [] {
    std::random_device rd;
    return (uint64_t(rd()) << 32) ^ uint64_t(rd()) ^ uint64_t(getpid());
  }();
  return n;
}

constexpr uint32_t kAbortSpan = 1u << 30;  // abort value = run base + kAbortSpan

// stream memory operations (rank mode), defined with the rank-mode code
void stream_wait_geq(cudaStream_t st, const uint32_t* addr, uint32_t value, int device);
void stream_write(cudaStream_t st, uint32_t* addr, uint32_t value, int device);

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
  if (s.block != kBlockToy && s.block != kBlockPixArt && s.block != kBlockJoint &&
      s.block != kBlockMMDiT)
    throw ValidationError("unknown block kind");
  if (s.joint_rows() && s.T < 1)
    throw ValidationError("joint block needs at least one text token");
  if (s.joint_rows() && (s.double_layers < 0 || s.double_layers > s.layers))
    throw ValidationError("double-stream layer count must lie in [0, layers]");
  if (s.precision != kPrecBf16 && s.precision != kPrecFp32)
    throw ValidationError("unknown precision");
  if (s.precision == kPrecFp32 && s.block != kBlockToy)
    throw ValidationError("the fp32 parity mode supports the toy block only");
  if (s.block == kBlockMMDiT) {
    if (s.hs % 64 != 0) throw ValidationError("MMDiT block needs hidden_size divisible by 64");
    if (s.rope && s.dh % 32 != 0)
      throw ValidationError("RoPE needs a head dim divisible by 32 (axes dh/8, 7dh/16, 7dh/16)");
  }
  if (s.block == kBlockPixArt) {
    if (s.hs % 32 != 0)
      throw ValidationError("PixArt block needs hidden_size divisible by 32");
    if (s.T < 1) throw ValidationError("PixArt block needs at least one text token");
  }
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
  if (!stages_.empty()) {
    DeviceGuard g(stages_[0].device);
    if (send_stream_) cudaStreamSynchronize(send_stream_);
    for (void* p : ipc_opened_) cudaIpcCloseMemHandle(p);
    for (bf16* p : df_sk_) dfree(p);
    for (bf16* p : df_sv_) dfree(p);
    if (ev_replayed_) cudaEventDestroy(ev_replayed_);
    for (cudaEvent_t e : ev_sent_) cudaEventDestroy(e);
    if (ev_compute_) cudaEventDestroy(ev_compute_);
    for (cudaEvent_t e : ev_write_)
      if (e) cudaEventDestroy(e);
    if (send_stream_) cudaStreamDestroy(send_stream_);
    if (abort_stream_) cudaStreamDestroy(abort_stream_);
    dfree(sig_);
  }
  drop_graphs();
  for (size_t d = 0; d < prof_pool_.size() && d < stages_.size(); ++d) {
    DeviceGuard g(stages_[d].device);
    for (cudaEvent_t e : prof_pool_[d]) cudaEventDestroy(e);
  }
  if (tl_origin_) {
    DeviceGuard g(stages_[0].device);
    cudaEventDestroy(tl_origin_);
  }
  for (Stage& s : stages_) free_stage(s);
}

void Engine::alloc_stage(Stage& s, int first, int count, bool is_first) {
  DeviceGuard g(s.device);
  const ModelShape& m = shape_;
  // activation / K/V buffers hold the joint rows (text rows first, joint block)
  const size_t P = size_t(m.rows_total()), hs = size_t(m.hs), mlp = size_t(m.mlp);
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
  // split-K workspace: enough for ~2 waves of 128 x 128 partial tiles
  s.splitk_ws_floats = size_t(4) << 20;
  s.splitk_ws = dalloc<float>(s.splitk_ws_floats);
  s.splitk_counter_cap = 4096;
  s.splitk_counters = dalloc<int>(size_t(s.splitk_counter_cap));
  // stream-K attention partials (at most two cut segments per CTA)
  s.attn_work_floats = attn_work_floats(int(dhp), s.sm_count);
  s.attn_work = dalloc<float>(s.attn_work_floats);
  s.attn_flags = dalloc<int>(size_t(s.sm_count) * kAttnFlagsPerCta);
  PF_CUDA_CHECK(cudaMemset(s.attn_flags, 0, size_t(s.sm_count) * kAttnFlagsPerCta * sizeof(int)));
  s.tm_hb = tmap(s.hb, hs, P, hs * 2, 64, 128, 128);
  s.tm_hb_half = tmap(s.hb, hs, P, hs * 2, 64, 64, 128);
  if (!encode_tmap_f32_2d(&s.tm_h32, s.h32, hs, P, hs * 4, 32, 128, 128))
    throw CudaError("cuTensorMapEncodeTiled failed for the residual stream");
  if (m.joint_rows() && hs % 32 == 0) {
    if (!encode_tmap_f32_2d(&s.tm_h32_txt, s.h32, hs, size_t(m.T), hs * 4, 32, 128, 128))
      throw CudaError("cuTensorMapEncodeTiled failed for the text rows");
    s.tm_hb_txt = tmap(s.hb, hs, size_t(m.T), hs * 2, 64, 128, 128);
  }
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
    {
      const uint32_t b3 = uint32_t(attn3_kv_rows(int(dhp)));
      L.tm_k3 = tmap(L.k, dhp, heads * P, dhp * 2, 16, b3, 32);
      L.tm_v3 = tmap(L.v, dhp, heads * P, dhp * 2, 16, b3, 32);
      L.has_kv3 = true;
    }
    check(v_ones_col(L.v, heads * P, int(dhp), m.dh, nullptr), "v_ones_col");
    if (m.precision == kPrecFp32) {
      L.w32 = dalloc<float>(4 * hs * hs + 2 * hs * mlp);
      L.k32 = dalloc<float>(P * hs);
      L.v32 = dalloc<float>(P * hs);
    }
  }
  if (m.precision == kPrecFp32) {
    s.q32 = dalloc<float>(P * hs);
    s.attn32 = dalloc<float>(P * hs);
    s.z32 = dalloc<float>(P * mlp);
  }
  s.zeros = dalloc<float>(hs);
  if (is_first) {
    s.x = dalloc<float>(size_t(m.P) * hs);
    s.cb = dalloc<float>(hs);
    if (m.joint_rows()) s.text = dalloc<float>(size_t(m.T) * hs);
  }
  if (m.block == kBlockJoint) {
    for (int lf = 0; lf < count; ++lf) {
      if (first + lf >= m.double_layers) continue;  // single-stream: shared weights
      StageLayer& L = s.layers[size_t(lf)];
      L.t_wqkv = dalloc<bf16>(3 * hs * hs);
      L.t_wo = dalloc<bf16>(hs * hs);
      L.t_win = dalloc<bf16>(mlp * hs);
      L.t_wout = dalloc<bf16>(hs * mlp);
      if (!make_weight_maps(&L.tm_t_wqkv, L.t_wqkv, int(3 * hs), int(hs)) ||
          !make_weight_maps(&L.tm_t_wo, L.t_wo, int(hs), int(hs)) ||
          !make_weight_maps(&L.tm_t_win, L.t_win, int(mlp), int(hs)) ||
          !make_weight_maps(&L.tm_t_wout, L.t_wout, int(hs), int(mlp)))
        throw CudaError("cuTensorMapEncodeTiled failed for a text-stream weight");
    }
  }
  if (m.block == kBlockMMDiT) mm_alloc_stage(s);
  if (m.block == kBlockPixArt) {
    const size_t T = size_t(m.T), Tpad = (T + 127) / 128 * 128;
    const size_t kvc_rows = heads * T + 128;  // + one TMA box of zero rows
    for (StageLayer& L : s.layers) {
      L.bqkv = dalloc<float>(3 * hs);
      L.bo = dalloc<float>(hs);
      L.bqc = dalloc<float>(hs);
      L.bkvc = dalloc<float>(2 * hs);
      L.boc = dalloc<float>(hs);
      L.b1 = dalloc<float>(mlp);
      L.b2 = dalloc<float>(hs);
      L.wqc = dalloc<bf16>(hs * hs);
      L.wkvc = dalloc<bf16>(2 * hs * hs);
      L.woc = dalloc<bf16>(hs * hs);
      L.kc = dalloc<bf16>(kvc_rows * dhp);
      L.vc = dalloc<bf16>(kvc_rows * dhp);
      check(v_ones_col(L.vc, kvc_rows, int(dhp), m.dh, nullptr), "v_ones_col");
      if (!make_weight_maps(&L.tm_wqc, L.wqc, int(hs), int(hs)) ||
          !make_weight_maps(&L.tm_wkvc, L.wkvc, int(2 * hs), int(hs)) ||
          !make_weight_maps(&L.tm_woc, L.woc, int(hs), int(hs)))
        throw CudaError("cuTensorMapEncodeTiled failed for a cross-attention weight");
      L.tm_kc = tmap(L.kc, dhp, kvc_rows, dhp * 2, 16, 128, 32);
      L.tm_vc = tmap(L.vc, dhp, kvc_rows, dhp * 2, 16, 128, 32);
    }
    PxStage& px = s.px;
    px.wt1 = dalloc<float>(hs * kPxFreq);
    px.bt1 = dalloc<float>(hs);
    px.wt2 = dalloc<float>(hs * hs);
    px.bt2 = dalloc<float>(hs);
    px.wt0 = dalloc<float>(6 * hs * hs);
    px.bt0 = dalloc<float>(6 * hs);
    px.sst = dalloc<float>(size_t(count + 1) * 6 * hs);
    px.text = dalloc<bf16>(Tpad * hs);
    px.tm_text = tmap(px.text, hs, Tpad, hs * 2, 64, 128, 128);
    px.stats = dalloc<float2>((hs / 32) * P);
    px.zeros = dalloc<float>(hs);
  }
}

// Per-run PixArt buffers, sized for `steps` timesteps (outside any capture).
// Growing them frees the old buffers, which captured graphs of earlier runs
// still reference: those graphs are dropped first.
void Engine::px_alloc_run(Stage& s, int steps) {
  const ModelShape& m = shape_;
  PxStage& px = s.px;
  if (steps <= px.steps_cap) return;
  DeviceGuard g(s.device);
  sync_own();  // a replayed graph may still read the old buffers
  drop_graphs();
  for (float* p : {px.sinus, px.e1, px.temb, px.tv, px.mod, px.foldq, px.foldm}) dfree(p);
  dfree(px.fold_aq);
  dfree(px.fold_am);
  const size_t S = size_t(steps), hs = size_t(m.hs), nl = size_t(s.layer_count);
  px.sinus = dalloc<float>(S * kPxFreq);
  px.e1 = dalloc<float>(S * hs);
  px.temb = dalloc<float>(S * hs);
  px.tv = dalloc<float>(S * 6 * hs);
  px.mod = dalloc<float>((nl + 1) * S * 6 * hs);
  px.fold_rpad = int((2 * S + 127) / 128 * 128);
  const size_t rp = size_t(px.fold_rpad);
  px.fold_aq = dalloc<bf16>(nl * rp * hs);
  px.fold_am = dalloc<bf16>(nl * rp * hs);
  px.tm_aq.resize(nl);
  px.tm_am.resize(nl);
  for (size_t l = 0; l < nl; ++l) {
    px.tm_aq[l] = tmap(px.fold_aq + l * rp * hs, hs, rp, hs * 2, 64, 128, 128);
    px.tm_am[l] = tmap(px.fold_am + l * rp * hs, hs, rp, hs * 2, 64, 128, 128);
  }
  px.foldq = dalloc<float>(nl * 2 * S * 3 * hs);
  px.foldm = dalloc<float>(nl * 2 * S * size_t(m.mlp));
  px.steps_cap = steps;
}

void Engine::drop_graphs() {
  for (auto& kv : graphs_) {
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (kv.second.graph) cudaGraphDestroy(kv.second.graph);
  }
  graphs_.clear();
}

void Engine::free_stage(Stage& s) {
  if (!s.stream && !s.h32) return;
  DeviceGuard g(s.device);
  if (s.stream) cudaStreamSynchronize(s.stream);
  for (StageLayer& L : s.layers) {
    dfree(L.wqkv); dfree(L.wo); dfree(L.win); dfree(L.wout);
    dfree(L.k); dfree(L.v);
    dfree(L.w32); dfree(L.k32); dfree(L.v32);
  }
  if (shape_.block == kBlockMMDiT) mm_free_stage(s);
  for (StageLayer& L : s.layers) {
    for (float* p : {L.bqkv, L.bo, L.bqc, L.bkvc, L.boc, L.b1, L.b2}) dfree(p);
    dfree(L.k2); dfree(L.v2);
    dfree(L.t_wqkv); dfree(L.t_wo); dfree(L.t_win); dfree(L.t_wout);
    dfree(L.wqc); dfree(L.wkvc); dfree(L.woc); dfree(L.kc); dfree(L.vc);
  }
  {
    PxStage& px = s.px;
    for (float* p : {px.wt1, px.bt1, px.wt2, px.bt2, px.wt0, px.bt0, px.sst, px.zeros, px.sinus,
                     px.e1, px.temb, px.tv, px.mod, px.foldq, px.foldm})
      dfree(p);
    dfree(px.fold_aq);
    dfree(px.fold_am);
    dfree(px.text);
    dfree(px.stats);
  }
  s.layers.clear();
  dfree(s.h32); dfree(s.hb); dfree(s.q); dfree(s.attn); dfree(s.z);
  dfree(s.q32); dfree(s.attn32); dfree(s.z32);
  if (s.lane != 0) use_lane(s, 0);
  for (Stage::Lane& ln : s.extra) {
    dfree(ln.attn_work); dfree(ln.attn_flags); dfree(ln.splitk_ws); dfree(ln.splitk_counters);
    if (ln.stream) cudaStreamDestroy(ln.stream);
  }
  for (auto& v : s.ev_attn)
    for (cudaEvent_t e : v) cudaEventDestroy(e);
  for (cudaEvent_t e : s.ev_lane)
    if (e) cudaEventDestroy(e);
  dfree(s.attn_work); dfree(s.attn_flags); dfree(s.flag); dfree(s.splitk_ws); dfree(s.splitk_counters);
  dfree(s.zeros); dfree(s.text); dfree(s.x); dfree(s.cb);
  if (s.eps_owned) dfree(s.eps);
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

namespace {
// One stream's six toy matrices (x.W orientation) -> bf16 N x K (K-major).
void upload_toy_weights(int device, int hs, int mlp, const HostMatrix* w, bf16* wqkv, bf16* wo,
                        bf16* win, bf16* wout) {
  auto pack = [](const HostMatrix& W, std::vector<bf16>& dst, size_t n_off, int K) {
    for (int n = 0; n < W.cols; ++n)
      for (int k = 0; k < K; ++k)
        dst[(n_off + size_t(n)) * size_t(K) + size_t(k)] = __float2bfloat16_rn(float(W.at(k, n)));
  };
  std::vector<bf16> qkv(size_t(3) * hs * hs), o(size_t(hs) * hs), in(size_t(mlp) * hs),
      out(size_t(hs) * mlp);
  pack(w[0], qkv, 0, hs);
  pack(w[1], qkv, size_t(hs), hs);
  pack(w[2], qkv, size_t(2) * hs, hs);
  pack(w[3], o, 0, hs);
  pack(w[4], in, 0, hs);
  pack(w[5], out, 0, mlp);
  DeviceGuard g(device);
  PF_CUDA_CHECK(cudaMemcpy(wqkv, qkv.data(), qkv.size() * 2, cudaMemcpyHostToDevice));
  PF_CUDA_CHECK(cudaMemcpy(wo, o.data(), o.size() * 2, cudaMemcpyHostToDevice));
  PF_CUDA_CHECK(cudaMemcpy(win, in.data(), in.size() * 2, cudaMemcpyHostToDevice));
  PF_CUDA_CHECK(cudaMemcpy(wout, out.data(), out.size() * 2, cudaMemcpyHostToDevice));
}
}  // namespace

void Engine::load_layer(int layer, const HostMatrix (&w)[6]) {
  const int d = stage_of_layer(layer);
  if (d < 0 && rank_mode() && layer >= 0 && layer < shape_.layers) return;  // another rank's
  if (d < 0) throw ValidationError("layer index out of range");
  Stage& s = stages_[size_t(d)];
  StageLayer& L = s.layers[size_t(layer - s.first_layer)];
  upload_toy_weights(s.device, shape_.hs, shape_.mlp, w, L.wqkv, L.wo, L.win, L.wout);
  if (L.w32) {  // fp32 parity mode: x.W orientation, row-major
    const size_t hs = size_t(shape_.hs), mlp = size_t(shape_.mlp);
    std::vector<float> f(4 * hs * hs + 2 * hs * mlp);
    size_t off = 0;
    for (int i = 0; i < 6; ++i) {
      for (int r = 0; r < w[i].rows; ++r)
        for (int c = 0; c < w[i].cols; ++c) f[off + size_t(r) * w[i].cols + c] = float(w[i].at(r, c));
      off += size_t(w[i].rows) * size_t(w[i].cols);
    }
    DeviceGuard g(s.device);
    PF_CUDA_CHECK(cudaMemcpy(L.w32, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
  }
}

void Engine::load_layer_joint(int layer, const HostMatrix (&w)[12]) {
  if (shape_.block != kBlockJoint) throw ValidationError("model is not a joint-block model");
  const int d = stage_of_layer(layer);
  if (d < 0 && rank_mode() && layer >= 0 && layer < shape_.layers) return;
  if (d < 0) throw ValidationError("layer index out of range");
  Stage& s = stages_[size_t(d)];
  StageLayer& L = s.layers[size_t(layer - s.first_layer)];
  upload_toy_weights(s.device, shape_.hs, shape_.mlp, w, L.wqkv, L.wo, L.win, L.wout);
  if (layer < shape_.double_layers)
    upload_toy_weights(s.device, shape_.hs, shape_.mlp, w + 6, L.t_wqkv, L.t_wo, L.t_win,
                       L.t_wout);
}

void Engine::load_condition_bias(const double* cb) {
  std::vector<float> v(size_t(shape_.hs));
  for (int i = 0; i < shape_.hs; ++i) v[size_t(i)] = float(cb[i]);
  Stage& s = stages_[0];
  if (!s.cb) return;  // rank mode, rank > 0: the sampler lives on rank 0
  DeviceGuard g(s.device);
  PF_CUDA_CHECK(cudaMemcpy(s.cb, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
}

// fp32 parity mode of the toy layer (same order as toy_model.cpp:169-177):
// Q, K, V projections with K/V written into rows [row0, row0+rows) of the
// full buffers before attending, attention over all P rows, out-proj
// residual, tanh MLP, MLP residual -- on the fp32 residual stream h32.
void Engine::layer_forward_f32(Stage& s, int lf, int rows, int row0, int code) {
  const ModelShape& m = shape_;
  StageLayer& L = s.layers[size_t(lf)];
  const int hs = m.hs, mlp = m.mlp;
  const size_t o = size_t(row0) * size_t(hs), hh = size_t(hs) * size_t(hs);
  const float* h = s.h32 + o;
  const float *wq = L.w32, *wk = wq + hh, *wv = wk + hh, *wo = wv + hh, *win = wo + hh,
              *wout = win + size_t(hs) * size_t(mlp);
  const double r = rows, dhs = hs, dmlp = mlp, P = double(m.P);
  if (lane_wait_) PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, lane_wait_, 0));
  prof_begin(s, kGemmQKV, 2 * r * dhs * 3 * dhs, 0);
  check(gemm_f32(h, hs, wq, hs, s.q32 + o, hs, rows, hs, hs, kF32Store, nullptr, 0, s.stream),
        "gemm q (fp32)");
  check(gemm_f32(h, hs, wk, hs, L.k32 + o, hs, rows, hs, hs, kF32Store, nullptr, 0, s.stream),
        "gemm k (fp32)");
  check(gemm_f32(h, hs, wv, hs, L.v32 + o, hs, rows, hs, hs, kF32Store, nullptr, 0, s.stream),
        "gemm v (fp32)");
  prof_end(s);
  prof_begin(s, kAttention, 4 * r * P * dhs, 0);
  check(attention_f32(s.q32 + o, L.k32, L.v32, s.attn32 + o, rows, int(m.P), m.heads, m.dh, hs,
                      float(1.0 / std::sqrt(double(m.dh))), s.stream),
        "attention (fp32)");
  prof_end(s);
  if (lane_rec_) PF_CUDA_CHECK(cudaEventRecord(lane_rec_, s.stream));
  prof_begin(s, kGemmOut, 2 * r * dhs * dhs, 0);
  check(gemm_f32(s.attn32 + o, hs, wo, hs, s.h32 + o, hs, rows, hs, hs, kF32Residual, s.flag,
                 code, s.stream),
        "gemm out-proj (fp32)");
  prof_end(s);
  prof_begin(s, kGemmMlpIn, 2 * r * dhs * dmlp, 0);
  check(gemm_f32(s.h32 + o, hs, win, mlp, s.z32 + size_t(row0) * mlp, mlp, rows, mlp, hs,
                 kF32Tanh, nullptr, 0, s.stream),
        "gemm mlp-in (fp32)");
  prof_end(s);
  float* dst = redirect_ ? redirect_->h32 : s.h32;
  if (dst != s.h32)  // rank mode, last layer: residual base then the successor's rows
    PF_CUDA_CHECK(cudaMemcpyAsync(dst + o, s.h32 + o, size_t(rows) * hs * 4,
                                  cudaMemcpyDefault, s.stream));
  prof_begin(s, kGemmMlpOut, 2 * r * dhs * dmlp, 0);
  check(gemm_f32(s.z32 + size_t(row0) * mlp, mlp, wout, hs, dst + o, hs, rows, hs, mlp,
                 kF32Residual, s.flag, code, s.stream),
        "gemm mlp-out (fp32)");
  prof_end(s);
}

// One toy DiT layer over rows [row0, row0+rows) (toy_model.cpp:169-177):
// fused QKV projection writing this block's K/V rows into the full buffers,
// attention over all P rows, out-proj residual, tanh MLP, MLP residual.
void Engine::layer_forward(Stage& s, int lf, int rows, int row0, int code, const KvView* kv) {
  const ModelShape& m = shape_;
  if (m.precision == kPrecFp32) {
    if (kv) throw ValidationError("the fp32 parity mode does not run DistriFusion");
    layer_forward_f32(s, lf, rows, row0, code);
    return;
  }
  StageLayer& L = s.layers[size_t(lf)];
  const double r = rows, hs = m.hs, mlp = m.mlp, P = double(m.P);
  EpiParams qkv;
  qkv.q = s.q;
  qkv.k = kv ? kv->k : L.k;
  qkv.v = kv ? kv->v : L.v;
  qkv.hs = m.hs;
  qkv.dh = m.dh;
  qkv.dhp = m.dhp;
  qkv.P = int(m.P);
  qkv.a_half = &s.tm_hb_half;
  if (lane_wait_) PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, lane_wait_, 0));
  prof_begin(s, kGemmQKV, 2 * r * hs * 3 * hs, 0);
  check(gemm(s.tm_hb, L.tm_wqkv, rows, row0, 3 * m.hs, m.hs, Epi::QKV, sk(s, qkv),
             s.sm_count, s.stream), "gemm qkv");
  prof_end(s);
  AttnLaunch a{m.dhp, int(m.P), rows, row0, m.heads, m.dh, m.hs,
               float(1.0 / std::sqrt(double(m.dh))), s.attn, s.attn_work,
               s.attn_work_floats};
  a.flags = s.attn_flags;
  a.v_sum_col = m.dh < m.dhp;  // V buffers carry the row-sum column
  if (L.has_kv3) {
    a.k3 = &L.tm_k3;
    a.v3 = &L.tm_v3;
  }
  // pull this layer's out-proj / MLP weights and the next layer's (or, after
  // the stage's last layer, the next patch's first layer's) QKV weights into
  // L2 while the attention runs: small patches otherwise stream them from HBM
  // at latency-bound rates
  if (prefetch_weights_) {
    const StageLayer& nx = s.layers[size_t(lf + 1 < s.layer_count ? lf + 1 : 0)];
    a.prefetch[0] = L.wo;
    a.prefetch_bytes[0] = size_t(m.hs) * m.hs * 2;
    a.prefetch[1] = L.win;
    a.prefetch_bytes[1] = size_t(m.mlp) * m.hs * 2;
    a.prefetch[2] = L.wout;
    a.prefetch_bytes[2] = size_t(m.hs) * m.mlp * 2;
    a.prefetch[3] = nx.wqkv;
    a.prefetch_bytes[3] = size_t(3) * m.hs * m.hs * 2;
  }
  if (kv && kv->sk) {
    // merged K/V: the previous step's rows with this worker's fresh rows
    const size_t pitch = size_t(m.P) * m.dhp * sizeof(bf16);
    const size_t bytes = size_t(m.heads) * pitch;
    const size_t off = size_t(row0) * m.dhp, width = size_t(rows) * m.dhp * sizeof(bf16);
    PF_CUDA_CHECK(cudaMemcpyAsync(kv->sk, kv->prev_k, bytes, cudaMemcpyDeviceToDevice, s.stream));
    PF_CUDA_CHECK(cudaMemcpyAsync(kv->sv, kv->prev_v, bytes, cudaMemcpyDeviceToDevice, s.stream));
    PF_CUDA_CHECK(cudaMemcpy2DAsync(kv->sk + off, pitch, kv->k + off, pitch, width,
                                    size_t(m.heads), cudaMemcpyDeviceToDevice, s.stream));
    PF_CUDA_CHECK(cudaMemcpy2DAsync(kv->sv + off, pitch, kv->v + off, pitch, width,
                                    size_t(m.heads), cudaMemcpyDeviceToDevice, s.stream));
  } else if (kv && kv->fresh_lo < kv->fresh_hi) {
    a.k2 = kv->tm_k2;
    a.v2 = kv->tm_v2;
    a.fresh_lo = kv->fresh_lo;
    a.fresh_hi = kv->fresh_hi;
  }
  prof_begin(s, kAttention, 4 * r * P * hs, 0);
  if (kv) {  // DistriFusion: the whole-buffer views run the serial path's kernel
    a.k3 = kv->k3;
    a.v3 = kv->v3;
  }
  const CUtensorMap& akm = kv ? (kv->sk ? *kv->tm_sk : *kv->tm_k) : L.tm_k;
  const CUtensorMap& avm = kv ? (kv->sk ? *kv->tm_sv : *kv->tm_v) : L.tm_v;
  check(attention(s.tm_q, akm, avm, a, s.sm_count, s.stream), "attention");
  prof_end(s);
  if (lane_rec_) PF_CUDA_CHECK(cudaEventRecord(lane_rec_, s.stream));
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
  check(gemm(s.tm_attn, L.tm_wo, rows, row0, m.hs, m.hs, Epi::Residual, sk(s, res),
             s.sm_count, s.stream), "gemm out-proj");
  prof_end(s);
  EpiParams th;
  th.out_bf16 = s.z;
  th.ld = m.mlp;
  th.a_half = &s.tm_hb_half;
  prof_begin(s, kGemmMlpIn, 2 * r * hs * mlp, 0);
  check(gemm(s.tm_hb, L.tm_win, rows, row0, m.mlp, m.hs, Epi::Tanh, sk(s, th),
             s.sm_count, s.stream), "gemm mlp-in");
  prof_end(s);
  EpiParams res_out = res;
  if (redirect_) {  // last layer of a rank: store straight into the next stage
    res_out.out_f32_dst = redirect_->h32;
    res_out.out_bf16_dst = redirect_->hb;
    res_out.tm_h32_dst = redirect_->tm_h32;
    res_out.tm_hb_dst = redirect_->tm_hb;
  }
  prof_begin(s, kGemmMlpOut, 2 * r * hs * mlp, 0);
  check(gemm(s.tm_z, L.tm_wout, rows, row0, m.hs, m.mlp, Epi::Residual, sk(s, res_out),
             s.sm_count, s.stream), "gemm mlp-out");
  prof_end(s);
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
void Engine::send_rows(int from, int row0, int rows, int patch, int t) {
  const int n = stage_count();
  Stage& src = stages_[size_t(from)];
  const size_t off = size_t(row0) * shape_.hs;
  const size_t cnt = size_t(rows) * shape_.hs;
  DeviceGuard g(src.device);
  if (n > 1) tl_begin(from, 1, patch, t, src.stream);
  if (from + 1 < n) {
    Stage& dst = stages_[size_t(from + 1)];
    PF_CUDA_CHECK(cudaMemcpyAsync(dst.h32 + off, src.h32 + off, cnt * 4,
                                  cudaMemcpyDefault, src.stream));
    PF_CUDA_CHECK(cudaMemcpyAsync(dst.hb + off, src.hb + off, cnt * 2,
                                  cudaMemcpyDefault, src.stream));
    if (shape_.ln_stats()) {
      // LayerNorm partial sums of the rows ([hs/32][P + T] float2)
      const size_t pitch = size_t(shape_.rows_total()) * sizeof(float2);
      PF_CUDA_CHECK(cudaMemcpy2DAsync(dst.px.stats + row0, pitch, src.px.stats + row0, pitch,
                                      size_t(rows) * sizeof(float2), size_t(shape_.hs / 32),
                                      cudaMemcpyDefault, src.stream));
    }
    tl_end(src.stream);  // before the handoff event: its stamp bounds the receiver's start
    PF_CUDA_CHECK(cudaEventRecord(src.ev_fwd, src.stream));
    DeviceGuard g2(dst.device);
    PF_CUDA_CHECK(cudaStreamWaitEvent(dst.stream, src.ev_fwd, 0));
  } else if (n > 1) {
    // eps: image rows only, image-indexed on stage 0 (joint rows start at J)
    Stage& s0 = stages_[0];
    const int64_t J = shape_.J();
    const int64_t i0 = std::max<int64_t>(row0, J), i1 = int64_t(row0) + rows;
    if (i1 > i0)
      PF_CUDA_CHECK(cudaMemcpyAsync(s0.eps + size_t(i0 - J) * shape_.hs,
                                    src.h32 + size_t(i0) * shape_.hs,
                                    size_t(i1 - i0) * shape_.hs * 4, cudaMemcpyDefault,
                                    src.stream));
    tl_end(src.stream);
  }
}

// Extra lanes of a stage (allocated on first use, outside stream capture).
void Engine::alloc_lanes(Stage& s, int lanes) {
  if (s.lanes_alloc >= lanes) return;
  DeviceGuard g(s.device);
  for (int k = s.lanes_alloc; k < lanes; ++k) {
    Stage::Lane& ln = s.extra[k];
    PF_CUDA_CHECK(cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking));
    ln.attn_work = dalloc<float>(s.attn_work_floats);
    ln.attn_flags = dalloc<int>(size_t(s.sm_count) * kAttnFlagsPerCta);
    PF_CUDA_CHECK(cudaMemset(ln.attn_flags, 0,
                             size_t(s.sm_count) * kAttnFlagsPerCta * sizeof(int)));
    ln.splitk_ws = dalloc<float>(s.splitk_ws_floats);
    ln.splitk_counters = dalloc<int>(size_t(s.splitk_counter_cap));
    PF_CUDA_CHECK(cudaMemset(ln.splitk_counters, 0, size_t(s.splitk_counter_cap) * sizeof(int)));
  }
  for (int k = 0; k < lanes; ++k) {
    auto& v = s.ev_attn[k];
    while (v.size() < size_t(s.layer_count)) {
      cudaEvent_t e;
      PF_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      v.push_back(e);
    }
    if (!s.ev_lane[k]) PF_CUDA_CHECK(cudaEventCreateWithFlags(&s.ev_lane[k], cudaEventDisableTiming));
  }
  s.lanes_alloc = lanes;
}

void Engine::use_lane(Stage& s, int lane) {
  if (s.lane == lane) return;
  auto swap_in = [&](Stage::Lane& ln) {
    std::swap(s.stream, ln.stream);
    std::swap(s.attn_work, ln.attn_work);
    std::swap(s.attn_flags, ln.attn_flags);
    std::swap(s.splitk_ws, ln.splitk_ws);
    std::swap(s.splitk_counters, ln.splitk_counters);
  };
  if (s.lane != 0) swap_in(s.extra[s.lane]);  // lane 0's resources back in place
  if (lane != 0) swap_in(s.extra[lane]);
  s.lane = lane;
}

// check_pipefusion_args (execute.cpp:97-131), with the layer divisibility
// relaxed (stages may hold L/N rounded up or down).
void Engine::validate_run(int steps, int patches, int warmup) const {
  const ModelShape& m = shape_;
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
}

void Engine::enqueue_run(float* x_dev, int steps, int patches, int warmup,
                         float eta, cudaStream_t caller, RunStats* stats) {
  const ModelShape& m = shape_;
  const int n = stage_count();
  validate_run(steps, patches, warmup);
  const int r = int(m.P / patches);
  Stage& s0 = stages_[0];
  prepare_run(patches, steps);
  const bool px = m.block == kBlockPixArt;
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
  LaunchTally tally(launches_);
  prof_.clear();
  prof_used_.assign(stages_.size(), 0);

  // Fork: every stage stream waits for the caller's prior work.
  cudaEvent_t ev_start = ev_start_;
  tl_.clear();
  {
    DeviceGuard g(s0.device);
    if (timeline_on_) {
      if (!tl_origin_) PF_CUDA_CHECK(cudaEventCreate(&tl_origin_));
      PF_CUDA_CHECK(cudaEventRecord(tl_origin_, caller));
    }
    PF_CUDA_CHECK(cudaEventRecord(ev_start, caller));
  }
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, ev_start, 0));
    check(reset_flag(s.flag, s.stream), "reset_flag");
    // StageBuffers are zero-initialised per run (execute.cpp:42-48). Without
    // warmup the zero rows are read as stale context, so clear them; with
    // warmup every row is rewritten before it is read.
    if (warmup == 0) {
      const size_t kv = size_t(m.heads) * size_t(m.rows_total()) * size_t(m.dhp) * sizeof(bf16);
      for (StageLayer& L : s.layers) {
        PF_CUDA_CHECK(cudaMemsetAsync(L.k, 0, kv, s.stream));
        PF_CUDA_CHECK(cudaMemsetAsync(L.v, 0, kv, s.stream));
        check(v_ones_col(L.v, kv / (size_t(m.dhp) * sizeof(bf16)), m.dhp, m.dh, s.stream),
              "v_ones_col");
        if (L.k32) {
          const size_t n32 = size_t(m.rows_total()) * size_t(m.hs) * sizeof(float);
          PF_CUDA_CHECK(cudaMemsetAsync(L.k32, 0, n32, s.stream));
          PF_CUDA_CHECK(cudaMemsetAsync(L.v32, 0, n32, s.stream));
        }
      }
    }
  }
  auto next_code = [&](int t, int layer) {
    codes_.emplace_back(t, layer);
    return int(codes_.size()) - 1;
  };
  const bool mm = m.block == kBlockMMDiT;
  if (px || mm)
    for (Stage& s : stages_) {
      DeviceGuard g(s.device);
      if (px) px_conditioning(s, steps);
      else mm_conditioning(s, steps);
    }
  const bool joint = m.joint_rows();
  const int J = int(m.J());  // joint block: text rows [0, J) precede the image rows
  auto forward = [&](Stage& s, int lf, int rows, int row0, int t, int code) {
    if (px) layer_forward_px(s, lf, rows, row0, t, code);
    else if (mm) layer_forward_mm(s, lf, rows, row0, t, code);
    else if (joint && s.first_layer + lf < m.double_layers)
      layer_forward_joint(s, lf, rows, row0, code);
    else if (joint)
      layer_forward_single(s, lf, rows, row0, code);
    else layer_forward(s, lf, rows, row0, code);
  };
  // joint block: the text stream re-enters from the text tokens every step
  auto text_prepare = [&](int t) {
    if (mm) {
      mm_text_prepare(s0, t);
      return;
    }
    check(patch_prepare(s0.text, nullptr, s0.zeros, s0.h32, s0.hb, 0, J, m.hs, 0.f, false,
                        s0.stream), "text rows");
  };
  float* h32_img = s0.h32 + size_t(J) * m.hs;  // image row 0 of the activations
  bf16* hb_img = s0.hb + size_t(J) * m.hs;

  const size_t n_lat = size_t(m.P) * m.hs;
  if (tap_ && tap_->traj) {
    DeviceGuard g(s0.device);
    PF_CUDA_CHECK(cudaMemcpyAsync(tap_->traj, x_dev, n_lat * 4, cudaMemcpyDeviceToDevice,
                                  s0.stream));
  }
  // ---- warmup: synchronous full-sequence steps (execute.cpp:181-190)
  for (int w = 0; w < warmup; ++w) {
    const int t = steps - 1 - w;
    {
      DeviceGuard g(s0.device);
      tl_begin(0, 0, -1, t, s0.stream);
      prof_begin(s0, kSampler, 0, double(m.P) * m.hs * (4 + 4 + 2));
      if (joint) text_prepare(t);
      if (px)
        px_patch_prepare(x_dev, false, 0, int(m.P), t, 0.f);
      else if (mm)
        mm_patch_prepare(s0, x_dev, false, 0, int(m.P), t, 0.f);
      else
        check(patch_prepare(x_dev, nullptr, s0.cb, h32_img, hb_img, 0, int(m.P), m.hs,
                            0.f, false, s0.stream), "patch_prepare");
      prof_end(s0);
    }
    for (int d = 0; d < n; ++d) {
      Stage& s = stages_[size_t(d)];
      DeviceGuard g(s.device);
      if (d > 0) tl_begin(d, 0, -1, t, s.stream);
      for (int lf = 0; lf < s.layer_count; ++lf) {
        auto& sv = src[size_t(d)][size_t(lf)];
        std::fill(sv.begin(), sv.end(), t);
        st.fresh += patches;
        forward(s, lf, int(m.rows_total()), 0, t, next_code(t, s.first_layer + lf));
      }
      tl_end(s.stream);
      send_rows(d, 0, int(m.rows_total()), -1, t);
    }
    if (n > 1) {
      Stage& last = stages_[size_t(n - 1)];
      DeviceGuard g(last.device);
      PF_CUDA_CHECK(cudaEventRecord(s0.ev_eps[0], last.stream));
      DeviceGuard g0(s0.device);
      PF_CUDA_CHECK(cudaStreamWaitEvent(s0.stream, s0.ev_eps[0], 0));
    }
    DeviceGuard g(s0.device);
    if (tap_ && tap_->sums)  // auto_warmup's ||x|| and ||x_next - x|| (toy_model.cpp:238-241)
      check(sumsq_latent(x_dev, s0.eps, double(eta), n_lat, tap_->work, tap_->sums + 2 * w,
                         s0.stream), "sumsq_latent");
    prof_begin(s0, kSampler, 0, double(m.P) * m.hs * 12);
    check(latent_update(x_dev, s0.eps, eta, size_t(m.P) * m.hs, s0.stream), "latent_update");
    prof_end(s0);
    if (tap_ && tap_->traj)
      PF_CUDA_CHECK(cudaMemcpyAsync(tap_->traj + size_t(w + 1) * n_lat, x_dev, n_lat * 4,
                                    cudaMemcpyDeviceToDevice, s0.stream));
  }

  // ---- steady: patch pipeline (execute.cpp:192-212)
  const int steady = steps - warmup;
  // Lanes (one stage, M >= 2): patch j runs on lane j % lanes, so
  // the kernels of consecutive patches overlap; small patches leave most of
  // the GPU idle in per-kernel latency otherwise. The only cross-patch
  // dependency inside a stage is the K/V buffer: patch j's QKV GEMM of layer
  // l overwrites its rows, which the previous patch's layer-l attention
  // reads (stale), and patch j's attention reads the previous patch's fresh
  // rows -- so QKV(j, l) waits for ATTN(j-1, l) (ev_attn). Everything else a
  // patch touches is its own rows or its lane's scratch.
  const int nl = steady > 0 ? lanes_for(patches) : 1;
  const bool lanes = nl > 1;
  if (lanes) {
    DeviceGuard g(s0.device);
    PF_CUDA_CHECK(cudaEventRecord(s0.ev_lane[0], s0.stream));
    for (int k = 1; k < nl; ++k)
      PF_CUDA_CHECK(cudaStreamWaitEvent(s0.extra[k].stream, s0.ev_lane[0], 0));
  }
  int prev_lane = -1;  // lane of the previously enqueued steady patch
  PdlOff pdl_off(lanes);
  // On a throw mid-loop: clear the lane hand-off events and leave the stage
  // on lane 0 with every lane joined (errors ignored: the run is abandoned).
  struct LaneUnwind {
    Engine* e;
    Stage& s;
    int nl;
    bool armed = true;
    ~LaneUnwind() {
      if (!armed) return;
      e->lane_wait_ = e->lane_rec_ = nullptr;
      e->use_lane(s, 0);
      for (int k = 1; k < nl; ++k) {
        cudaEventRecord(s.ev_lane[k], s.extra[k].stream);
        cudaStreamWaitEvent(s.stream, s.ev_lane[k], 0);
      }
      cudaGetLastError();
    }
  } lane_unwind{this, s0, nl};
  for (int q = 0; q < steady; ++q) {
    const int t = steady - 1 - q;
    for (int j = 0; j < patches; ++j) {
      if (lanes) use_lane(s0, j % nl);
      const int row0 = j * r;  // image rows of patch j
      // the block's joint rows: the text rows travel with patch 0
      const int brow0 = joint && j > 0 ? J + row0 : 0;
      const int brows = joint && j == 0 ? J + r : r;
      {
        DeviceGuard g(s0.device);
        if (q > 0 && n > 1)
          PF_CUDA_CHECK(cudaStreamWaitEvent(s0.stream, s0.ev_eps[size_t(j)], 0));
        tl_begin(0, 0, j, t, s0.stream);
        prof_begin(s0, kSampler, 0, double(r) * m.hs * (q > 0 ? 4 + 4 + 4 + 4 + 2 : 4 + 4 + 2));
        if (joint && j == 0) text_prepare(t);
        if (px)
          px_patch_prepare(x_dev, q > 0, row0, r, t, eta);
        else if (mm)
          mm_patch_prepare(s0, x_dev, q > 0, row0, r, t, eta);
        else
          check(patch_prepare(x_dev, s0.eps, s0.cb, h32_img, hb_img, row0, r, m.hs, eta,
                              q > 0, s0.stream), "patch_prepare");
        prof_end(s0);
      }
      for (int d = 0; d < n; ++d) {
        Stage& s = stages_[size_t(d)];
        DeviceGuard g(s.device);
        if (d > 0) tl_begin(d, 0, j, t, s.stream);
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
          if (lanes) {
            lane_wait_ = prev_lane >= 0 ? s.ev_attn[prev_lane][size_t(lf)] : nullptr;
            lane_rec_ = s.ev_attn[j % nl][size_t(lf)];
          }
          forward(s, lf, joint ? brows : r, joint ? brow0 : row0, t,
                  next_code(t, s.first_layer + lf));
          lane_wait_ = lane_rec_ = nullptr;
        }
        // fresh_fraction(src[0], t) after the stage (execute.cpp:67-73,164)
        {
          const auto& s0v = src[size_t(d)][0];
          int fresh = 0;
          for (int v : s0v) fresh += (v == t);
          st.fresh_fraction[size_t(d)].push_back(double(fresh) / double(s0v.size()));
        }
        tl_end(s.stream);
        send_rows(d, joint ? brow0 : row0, joint ? brows : r, j, t);
        if (d == n - 1 && n > 1)
          PF_CUDA_CHECK(cudaEventRecord(s0.ev_eps[size_t(j)], s.stream));
      }
      prev_lane = j % nl;
    }
  }
  pdl_off.set(false);
  lane_unwind.armed = false;
  if (lanes) {  // join the other lanes back into lane 0
    DeviceGuard g(s0.device);
    use_lane(s0, 0);
    for (int k = 1; k < nl; ++k) {
      PF_CUDA_CHECK(cudaEventRecord(s0.ev_lane[k], s0.extra[k].stream));
      PF_CUDA_CHECK(cudaStreamWaitEvent(s0.stream, s0.ev_lane[k], 0));
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
void Engine::prepare_run(int patches, int steps) {
  const int n = stage_count();
  Stage& s0 = stages_[0];
  if (shape_.block == kBlockPixArt && steps >= 1)
    for (Stage& s : stages_) px_alloc_run(s, steps);
  if (shape_.block == kBlockMMDiT && steps >= 1)
    for (Stage& s : stages_) mm_alloc_run(s, steps);
  if (!ev_start_) {
    DeviceGuard g(s0.device);
    PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_start_, cudaEventDisableTiming));
  }
  if (n > 1 && !s0.eps_owned) {
    DeviceGuard g(s0.device);
    s0.eps = dalloc<float>(size_t(shape_.P) * shape_.hs);
    s0.eps_owned = true;
  }
  if (n == 1) s0.eps = s0.h32 + size_t(shape_.J()) * shape_.hs;  // image rows of h
  if (lanes_for(patches) > 1) alloc_lanes(s0, lanes_for(patches));
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
  if (rank_mode()) {
    run_rank(x_dev, steps, patches, warmup, eta, caller, stats);
    return;
  }
  if (patches >= 1) prepare_run(patches, steps);
  bool single_device = true;
  for (const Stage& s : stages_) single_device &= s.device == stages_[0].device;
  if (!graphs_enabled_ || profiling_ || timeline_on_ || caller == nullptr || !single_device ||
      tap_) {
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
  if (!ev_replayed_) PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_replayed_, cudaEventDisableTiming));
  PF_CUDA_CHECK(cudaEventRecord(ev_replayed_, caller));
  launches_ = it->second.launches;
  codes_ = it->second.codes;
  if (stats) *stats = it->second.stats;
}

void Engine::finish(cudaStream_t caller) {
  {
    DeviceGuard g(stages_[0].device);
    wait_stream(caller);
    if (send_stream_) wait_stream(send_stream_);
  }
  int first = INT_MAX;
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    wait_stream(s.stream);
    int f = INT_MAX;
    PF_CUDA_CHECK(cudaMemcpy(&f, s.flag, sizeof(int), cudaMemcpyDeviceToHost));
    first = std::min(first, f);
  }
  // the root cause (this rank's own non-finite activation) is preferred over
  // the cascade (a neighbour closed the channel), as execute.cpp:357-374
  if (first != INT_MAX && first >= 0 && size_t(first) < codes_.size()) {
    std::ostringstream os;
    os << "non-finite activation at timestep " << codes_[size_t(first)].first
       << ", layer " << codes_[size_t(first)].second;
    throw NumericError(os.str());
  }
  if (rank_mode() && run_epoch_ > 0) {
    if (broken_) throw NumericError("channel closed mid-run (no progress from a peer rank)");
    uint32_t aborted = 0;
    DeviceGuard g(stages_[0].device);
    PF_CUDA_CHECK(cudaMemcpy(&aborted, sig_ + 2, sizeof(aborted), cudaMemcpyDeviceToHost));
    if (aborted == run_epoch_) throw NumericError("channel closed mid-run");
  }
}

void Engine::wait_stream(cudaStream_t st) {
  if (!rank_mode()) {
    PF_CUDA_CHECK(cudaStreamSynchronize(st));
    return;
  }
  // Watchdog: a peer that died or stopped enqueueing leaves this rank's
  // signal waits blocked forever. After rank_timeout_s_ without completion,
  // release them (own pages) and the neighbours' (the pipeline is closed).
  using clock = std::chrono::steady_clock;
  auto t0 = clock::now();
  bool aborted = false;
  int spins = 0;
  for (;;) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) PF_CUDA_CHECK(e);
    const double waited = std::chrono::duration<double>(clock::now() - t0).count();
    if (waited > rank_timeout_s_) {
      if (aborted) throw NumericError("channel closed mid-run (stream did not drain after abort)");
      watchdog_abort();
      aborted = true;
      t0 = clock::now();
    }
    if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

void Engine::prepare_rank_run(int patches, int steps) {
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  if (shape_.block == kBlockPixArt) px_alloc_run(s, steps);
  if (shape_.block == kBlockMMDiT) mm_alloc_run(s, steps);
  while (int(ev_sent_.size()) < patches) {
    cudaEvent_t e;
    PF_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev_sent_.push_back(e);
  }
  if (!ev_start_) PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_start_, cudaEventDisableTiming));
  for (cudaEvent_t& e : ev_write_)
    if (!e) PF_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const int nl = std::min(lanes_, patches);
  if (nl > 1) alloc_lanes(s, nl);
}

void Engine::run_rank(float* x_dev, int steps, int patches, int warmup, float eta,
                      cudaStream_t caller, RunStats* stats, bool launch) {
  if (!connected_) throw ValidationError("rank-mode engine is not connected to its peers");
  if (broken_)
    throw NumericError("channel closed mid-run (an earlier run of this pipeline was aborted; "
                       "call pf_rank_reset on every rank)");
  // identical on every rank: fails everywhere before anything is enqueued
  validate_run(steps, patches, warmup);
  if (launch) ++run_epoch_;
  DeviceGuard g(stages_[0].device);
  bool graph = graphs_enabled_ && !profiling_ && !timeline_on_ && caller != nullptr &&
               fail_at_op_ < 0;
  if (shared_device_peer_) graph = false;  // see connect_peers
  if (!launch && !graph) return;
  static const bool dbg = [] {
    const char* e = std::getenv("PF_RANK_DEBUG");
    return e && e[0] == '1';
  }();
  auto trace = [&](const char* what) {
    if (dbg) std::fprintf(stderr, "[rank %d] %s\n", rank_, what);
  };
  try {
    if (!graph) {
      enqueue_rank_run(x_dev, steps, patches, warmup, eta, caller, stats);
      return;
    }
    if (rank_ == 0 && !x_dev) throw ValidationError("NULL latent pointer");
    trace("prepare");
    prepare_rank_run(patches, steps);
    trace("prepared");
    const GraphMemOps& gm = graph_memops();
    uint32_t eta_bits;
    std::memcpy(&eta_bits, &eta, sizeof(eta_bits));
    const GraphKey key{x_dev, steps, patches, warmup, eta_bits, caller};
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
      // Capture this rank's plan once. The signal waits / writes become
      // batch mem-op nodes whose values hold the capture-time base; later
      // replays patch them to their own base (message counters never reset).
      GraphEntry e;
      const uint32_t in0 = msgs_in_base_, out0 = msgs_out_base_;
      PF_CUDA_CHECK(cudaStreamBeginCapture(caller, cudaStreamCaptureModeThreadLocal));
      cudaGraph_t graph_h = nullptr;
      try {
        enqueue_rank_run(x_dev, steps, patches, warmup, eta, caller, &e.stats);
      } catch (...) {
        // nothing of the plan was executed: close the run and play the
        // message protocol without compute, then report the root cause
        const std::exception_ptr failure = std::current_exception();
        cudaStreamEndCapture(caller, &graph_h);
        if (graph_h) cudaGraphDestroy(graph_h);
        cudaGetLastError();
        msgs_in_base_ = in0;
        msgs_out_base_ = out0;
        close_channels();
        enqueue_rank_run(x_dev, steps, patches, warmup, eta, caller, nullptr, true);
        std::rethrow_exception(failure);
      }
      PF_CUDA_CHECK(cudaStreamEndCapture(caller, &graph_h));
      trace("captured");
      msgs_in_base_ = in0;  // the capture executed nothing
      msgs_out_base_ = out0;
      e.graph = graph_h;
      e.base = in0;
      e.launches = launches_;
      e.codes = codes_;
      size_t n = 0;
      PF_CUDA_CHECK(cudaGraphGetNodes(graph_h, nullptr, &n));
      std::vector<cudaGraphNode_t> nodes(n);
      PF_CUDA_CHECK(cudaGraphGetNodes(graph_h, nodes.data(), &n));
      for (cudaGraphNode_t nd : nodes) {
        CUgraphNodeType t;
        if (gm.node_type(reinterpret_cast<CUgraphNode>(nd), &t) != CUDA_SUCCESS)
          throw CudaError("cuGraphNodeGetType failed");
        if (t != CU_GRAPH_NODE_TYPE_BATCH_MEM_OP) continue;
        CUDA_BATCH_MEM_OP_NODE_PARAMS prm;
        if (gm.get(reinterpret_cast<CUgraphNode>(nd), &prm) != CUDA_SUCCESS)
          throw CudaError("cuGraphBatchMemOpNodeGetParams failed");
        GraphEntry::MemOpNode mn;
        mn.node = nd;
        for (unsigned k = 0; k < prm.count; ++k) {
          const CUstreamBatchMemOpParams& op = prm.paramArray[k];
          uint32_t v = 0;
          if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_32) v = op.waitValue.value;
          else if (op.operation == CU_STREAM_MEM_OP_WRITE_VALUE_32) v = op.writeValue.value;
          else throw CudaError("unexpected memory operation in a captured rank plan");
          mn.delta.push_back(v - in0);
        }
        e.memops.push_back(std::move(mn));
      }
      PF_CUDA_CHECK(cudaGraphInstantiate(&e.exec, graph_h, 0));
      trace("instantiated");
      it = graphs_.emplace(key, std::move(e)).first;
    }
    GraphEntry& e = it->second;
    if (!launch) return;  // prepare_graph: built, not replayed
    if (e.base != msgs_in_base_) {
      for (GraphEntry::MemOpNode& mn : e.memops) {
        CUDA_BATCH_MEM_OP_NODE_PARAMS prm;
        if (gm.get(reinterpret_cast<CUgraphNode>(mn.node), &prm) != CUDA_SUCCESS)
          throw CudaError("cuGraphBatchMemOpNodeGetParams failed");
        std::vector<CUstreamBatchMemOpParams> ops(prm.paramArray, prm.paramArray + prm.count);
        for (size_t k = 0; k < ops.size(); ++k) {
          const uint32_t v = msgs_in_base_ + mn.delta[k];
          if (ops[k].operation == CU_STREAM_MEM_OP_WAIT_VALUE_32) ops[k].waitValue.value = v;
          else ops[k].writeValue.value = v;
        }
        prm.paramArray = ops.data();
        if (gm.exec_set(reinterpret_cast<CUgraphExec>(e.exec),
                        reinterpret_cast<CUgraphNode>(mn.node), &prm) != CUDA_SUCCESS)
          throw CudaError("cuGraphExecBatchMemOpNodeSetParams failed");
      }
      e.base = msgs_in_base_;
    }
    run_base_ = msgs_in_base_;
    trace("launch");
    PF_CUDA_CHECK(cudaGraphLaunch(e.exec, caller));
    if (!ev_replayed_)
      PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_replayed_, cudaEventDisableTiming));
    PF_CUDA_CHECK(cudaEventRecord(ev_replayed_, caller));
    trace("launched");
    const uint32_t per_run = uint32_t(plan_messages_per_run(steps, patches, warmup));
    msgs_in_base_ += per_run;
    msgs_out_base_ += per_run;
    launches_ = e.launches;
    codes_ = e.codes;
    if (stats) *stats = e.stats;
  } catch (const ValidationError&) {
    if (rank_ == 0 && !x_dev) {  // rank 0 alone: the peers are waiting for it
      close_channels();
      enqueue_rank_run(nullptr, steps, patches, warmup, eta, caller, nullptr, true);
    }
    throw;
  }
}

void Engine::close_channels() {
  if (!rank_mode() || !connected_) return;
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  std::vector<uint32_t*> pages = world_sig_;
  if (pages.empty()) pages = {pred_sig_, succ_sig_};
  pages.push_back(sig_);
  for (uint32_t* page : pages)
    if (page) stream_write(abort_stream_, page + 2, run_epoch_, s.device);
  PF_CUDA_CHECK(cudaStreamSynchronize(abort_stream_));
}

void Engine::watchdog_abort() {
  if (!rank_mode() || !connected_) return;
  broken_ = true;
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  const int dev = s.device;
  close_channels();
  // every wait of this run (own and neighbours') passes: >= base + kAbortSpan
  const uint32_t release = run_base_ + kAbortSpan;
  stream_write(abort_stream_, sig_, release, dev);
  stream_write(abort_stream_, sig_ + 1, release, dev);
  if (succ_sig_) stream_write(abort_stream_, succ_sig_, release, dev);
  if (pred_sig_) stream_write(abort_stream_, pred_sig_ + 1, release, dev);
  cudaStreamSynchronize(abort_stream_);
  cudaGetLastError();
}

void Engine::sync_own() {
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (int k = 1; k < s.lanes_alloc; ++k)
      if (s.extra[k].stream) cudaStreamSynchronize(s.extra[k].stream);
  }
  if (send_stream_) cudaStreamSynchronize(send_stream_);
  if (ev_replayed_) cudaEventSynchronize(ev_replayed_);
  cudaGetLastError();
}

void Engine::rank_reset() {
  if (!rank_mode()) return;
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  PF_CUDA_CHECK(cudaDeviceSynchronize());
  PF_CUDA_CHECK(cudaMemset(sig_, 0, 64 * sizeof(uint32_t)));
  PF_CUDA_CHECK(cudaDeviceSynchronize());
  msgs_in_base_ = msgs_out_base_ = 0;
  run_epoch_ = 0;
  run_base_ = 0;
  broken_ = false;
}

void Engine::debug_poison_layer(int layer) {
  const int d = stage_of_layer(layer);
  if (d < 0) throw ValidationError("layer index out of range");
  Stage& s = stages_[size_t(d)];
  DeviceGuard g(s.device);
  const bf16 nan = __float2bfloat16_rn(NAN);
  bf16* w = s.layers[size_t(layer - s.first_layer)].wo;
  PF_CUDA_CHECK(cudaMemcpy(w, &nan, sizeof(nan), cudaMemcpyHostToDevice));
  drop_graphs();
}

void Engine::layer_forward_host(int layer, double* h, int64_t rows, int64_t row0,
                                double* k_buf, double* v_buf, bool col_major, int t,
                                int steps) {
  const ModelShape& m = shape_;
  if (m.joint_rows())
    throw ValidationError("single-layer entry point not available for the joint block");
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
  if (m.dh < m.dhp)  // the attention's row-sum column (AttnLaunch::v_sum_col)
    for (int64_t r = 0; r < int64_t(m.heads) * P; ++r)
      vd[size_t(r) * m.dhp + m.dh] = __float2bfloat16_rn(1.0f);
  DeviceGuard g(s.device);
  if (m.precision == kPrecFp32) {  // parity mode: fp32 row-major K/V
    std::vector<float> k32(size_t(P) * hs), v32(size_t(P) * hs);
    for (int64_t r = 0; r < P; ++r)
      for (int c = 0; c < hs; ++c) {
        k32[size_t(r) * hs + c] = float(k_buf[idx(r, c, P)]);
        v32[size_t(r) * hs + c] = float(v_buf[idx(r, c, P)]);
      }
    PF_CUDA_CHECK(cudaMemcpy(s.h32 + row0 * hs, h32.data(), h32.size() * 4,
                             cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(L.k32, k32.data(), k32.size() * 4, cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(L.v32, v32.data(), v32.size() * 4, cudaMemcpyHostToDevice));
    LaunchTally tally(launches_);
    check(reset_flag(s.flag, s.stream), "reset_flag");
    codes_.assign(1, {0, layer});
    layer_forward(s, layer - s.first_layer, int(rows), int(row0), 0);
    PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
    PF_CUDA_CHECK(cudaMemcpy(h32.data(), s.h32 + row0 * hs, h32.size() * 4,
                             cudaMemcpyDeviceToHost));
    PF_CUDA_CHECK(cudaMemcpy(k32.data(), L.k32, k32.size() * 4, cudaMemcpyDeviceToHost));
    PF_CUDA_CHECK(cudaMemcpy(v32.data(), L.v32, v32.size() * 4, cudaMemcpyDeviceToHost));
    for (int64_t r = 0; r < rows; ++r)
      for (int c = 0; c < hs; ++c) h[idx(r, c, rows)] = double(h32[size_t(r) * hs + c]);
    for (int64_t r = 0; r < P; ++r)
      for (int c = 0; c < hs; ++c) {
        k_buf[idx(r, c, P)] = double(k32[size_t(r) * hs + c]);
        v_buf[idx(r, c, P)] = double(v32[size_t(r) * hs + c]);
      }
    int f = INT_MAX;
    PF_CUDA_CHECK(cudaMemcpy(&f, s.flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (f != INT_MAX) {
      std::ostringstream os;
      os << "non-finite activation at timestep 0, layer " << layer;
      throw NumericError(os.str());
    }
    return;
  }
  PF_CUDA_CHECK(cudaMemcpyAsync(s.h32 + row0 * hs, h32.data(), h32.size() * 4,
                                cudaMemcpyHostToDevice, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(s.hb + row0 * hs, hb.data(), hb.size() * 2,
                                cudaMemcpyHostToDevice, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(L.k, kd.data(), kd.size() * 2, cudaMemcpyHostToDevice, s.stream));
  PF_CUDA_CHECK(cudaMemcpyAsync(L.v, vd.data(), vd.size() * 2, cudaMemcpyHostToDevice, s.stream));
  LaunchTally tally(launches_);
  check(reset_flag(s.flag, s.stream), "reset_flag");
  codes_.assign(1, {0, layer});
  if (m.block == kBlockPixArt) {
    if (steps < 1 || t < 0 || t >= steps)
      throw ValidationError("timestep index outside [0, steps)");
    px_alloc_run(s, steps);
    px_conditioning(s, steps);
    const int lf = layer - s.first_layer;
    const float* scale1 = s.px.mod + (size_t(lf) * steps + t) * 6 * hs + hs;
    // LayerNorm inputs of the uploaded rows (h32 += 0 in place)
    check(pf::px_patch_prepare(s.h32, nullptr, s.px.zeros, scale1, s.h32, s.hb, s.px.stats,
                               int(P), int(row0), int(rows), hs, 0.f, false, s.stream),
          "px_patch_prepare");
    layer_forward_px(s, lf, int(rows), int(row0), t, 0);
  } else {
    layer_forward(s, layer - s.first_layer, int(rows), int(row0), 0);
  }
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

// ============================================================== joint block
// SD3-style MMDiT double-stream block with the toy block's arithmetic per
// stream: rows [0, T) are the text stream (own weights), rows [T, T + P)
// the image stream; both streams' queries attend over all joint K/V rows.
// A row block [row0, row0 + rows) is the text rows plus image patch 0, or an
// image patch alone.
void Engine::layer_forward_joint(Stage& s, int lf, int rows, int row0, int code) {
  const ModelShape& m = shape_;
  StageLayer& L = s.layers[size_t(lf)];
  const int J = int(m.J()), Pt = int(m.rows_total()), hs = m.hs;
  const int t_rows = row0 < J ? std::min(row0 + rows, J) - row0 : 0;
  const int i_row0 = std::max(row0, J), i_rows = row0 + rows - i_row0;
  auto both = [&](auto&& fn) {
    if (t_rows > 0) fn(true, row0, t_rows);
    if (i_rows > 0) fn(false, i_row0, i_rows);
  };
  const double dhs = hs, mlp = m.mlp;
  EpiParams qkv;
  qkv.q = s.q;
  qkv.k = L.k;
  qkv.v = L.v;
  qkv.hs = hs;
  qkv.dh = m.dh;
  qkv.dhp = m.dhp;
  qkv.P = Pt;
  if (lane_wait_) PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, lane_wait_, 0));
  both([&](bool txt, int r0, int n) {
    prof_begin(s, kGemmQKV, 2.0 * n * dhs * 3 * dhs, 0);
    check(gemm(s.tm_hb, txt ? L.tm_t_wqkv : L.tm_wqkv, n, r0, 3 * hs, hs, Epi::QKV,
               sk(s, qkv), s.sm_count, s.stream), "gemm qkv (joint)");
    prof_end(s);
  });
  AttnLaunch a{m.dhp, Pt, rows, row0, m.heads, m.dh, hs,
               float(1.0 / std::sqrt(double(m.dh))), s.attn, s.attn_work,
               s.attn_work_floats};
  a.flags = s.attn_flags;
  a.v_sum_col = m.dh < m.dhp;  // V buffers carry the row-sum column
  if (L.has_kv3) {
    a.k3 = &L.tm_k3;
    a.v3 = &L.tm_v3;
  }
  prof_begin(s, kAttention, 4.0 * rows * double(Pt) * dhs, 0);
  check(attention(s.tm_q, L.tm_k, L.tm_v, a, s.sm_count, s.stream), "attention (joint)");
  prof_end(s);
  if (lane_rec_) PF_CUDA_CHECK(cudaEventRecord(lane_rec_, s.stream));
  EpiParams res;
  res.out_f32 = s.h32;
  res.out_bf16 = s.hb;
  res.ld = hs;
  res.flag = s.flag;
  res.code = code;
  if (hs % 32 == 0) {
    res.tm_h32 = &s.tm_h32;
    res.tm_hb = &s.tm_hb;
  }
  // text rows: TMA residual through maps that end at the last text row (clipped stores)
  auto clip = [&](bool txt, EpiParams e) {
    if (txt && !e.out_f32_dst && hs % 32 == 0) {
      e.tm_h32 = &s.tm_h32_txt;
      e.tm_hb = &s.tm_hb_txt;
      e.tma_clip = true;
    }
    return e;
  };
  both([&](bool txt, int r0, int n) {
    prof_begin(s, kGemmOut, 2.0 * n * dhs * dhs, 0);
    check(gemm(s.tm_attn, txt ? L.tm_t_wo : L.tm_wo, n, r0, hs, hs, Epi::Residual,
               sk(s, clip(txt, res)), s.sm_count, s.stream), "gemm out-proj (joint)");
    prof_end(s);
  });
  EpiParams th;
  th.out_bf16 = s.z;
  th.ld = m.mlp;
  both([&](bool txt, int r0, int n) {
    prof_begin(s, kGemmMlpIn, 2.0 * n * dhs * mlp, 0);
    check(gemm(s.tm_hb, txt ? L.tm_t_win : L.tm_win, n, r0, m.mlp, hs, Epi::Tanh, sk(s, th),
               s.sm_count, s.stream), "gemm mlp-in (joint)");
    prof_end(s);
  });
  EpiParams res_out = res;
  if (redirect_) {  // last layer of a rank: store straight into the next stage
    res_out.out_f32_dst = redirect_->h32;
    res_out.out_bf16_dst = redirect_->hb;
    res_out.tm_h32_dst = redirect_->tm_h32;
    res_out.tm_hb_dst = redirect_->tm_hb;
  }
  both([&](bool txt, int r0, int n) {
    prof_begin(s, kGemmMlpOut, 2.0 * n * dhs * mlp, 0);
    check(gemm(s.tm_z, txt ? L.tm_t_wout : L.tm_wout, n, r0, hs, m.mlp, Epi::Residual,
               sk(s, clip(txt, res_out)), s.sm_count, s.stream), "gemm mlp-out (joint)");
    prof_end(s);
  });
}

// Flux-style single-stream block with the toy arithmetic: one weight set
// for all joint rows; attention and MLP both read the block input h:
//   h += attention(h Wq, K, V) Wo + tanh(h Win) Wout
void Engine::layer_forward_single(Stage& s, int lf, int rows, int row0, int code) {
  const ModelShape& m = shape_;
  StageLayer& L = s.layers[size_t(lf)];
  const int Pt = int(m.rows_total()), hs = m.hs;
  const double r = rows, dhs = hs, mlp = m.mlp;
  EpiParams qkv;
  qkv.q = s.q;
  qkv.k = L.k;
  qkv.v = L.v;
  qkv.hs = hs;
  qkv.dh = m.dh;
  qkv.dhp = m.dhp;
  qkv.P = Pt;
  if (lane_wait_) PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, lane_wait_, 0));
  prof_begin(s, kGemmQKV, 2 * r * dhs * 3 * dhs, 0);
  check(gemm(s.tm_hb, L.tm_wqkv, rows, row0, 3 * hs, hs, Epi::QKV, sk(s, qkv), s.sm_count,
             s.stream), "gemm qkv (single)");
  prof_end(s);
  EpiParams th;
  th.out_bf16 = s.z;
  th.ld = m.mlp;
  prof_begin(s, kGemmMlpIn, 2 * r * dhs * mlp, 0);
  check(gemm(s.tm_hb, L.tm_win, rows, row0, m.mlp, hs, Epi::Tanh, sk(s, th), s.sm_count,
             s.stream), "gemm mlp-in (single)");
  prof_end(s);
  AttnLaunch a{m.dhp, Pt, rows, row0, m.heads, m.dh, hs,
               float(1.0 / std::sqrt(double(m.dh))), s.attn, s.attn_work,
               s.attn_work_floats};
  a.flags = s.attn_flags;
  a.v_sum_col = m.dh < m.dhp;  // V buffers carry the row-sum column
  if (L.has_kv3) {
    a.k3 = &L.tm_k3;
    a.v3 = &L.tm_v3;
  }
  prof_begin(s, kAttention, 4 * r * double(Pt) * dhs, 0);
  check(attention(s.tm_q, L.tm_k, L.tm_v, a, s.sm_count, s.stream), "attention (single)");
  prof_end(s);
  if (lane_rec_) PF_CUDA_CHECK(cudaEventRecord(lane_rec_, s.stream));
  EpiParams res;
  res.out_f32 = s.h32;
  res.out_bf16 = s.hb;
  res.ld = hs;
  res.flag = s.flag;
  res.code = code;
  if (hs % 32 == 0) {
    res.tm_h32 = &s.tm_h32;
    res.tm_hb = &s.tm_hb;
  }
  prof_begin(s, kGemmOut, 2 * r * dhs * dhs, 0);
  check(gemm(s.tm_attn, L.tm_wo, rows, row0, hs, hs, Epi::Residual, sk(s, res), s.sm_count,
             s.stream), "gemm out-proj (single)");
  prof_end(s);
  EpiParams res_out = res;
  if (redirect_) {
    res_out.out_f32_dst = redirect_->h32;
    res_out.out_bf16_dst = redirect_->hb;
    res_out.tm_h32_dst = redirect_->tm_h32;
    res_out.tm_hb_dst = redirect_->tm_hb;
  }
  prof_begin(s, kGemmMlpOut, 2 * r * dhs * mlp, 0);
  check(gemm(s.tm_z, L.tm_wout, rows, row0, hs, m.mlp, Epi::Residual, sk(s, res_out),
             s.sm_count, s.stream), "gemm mlp-out (single)");
  prof_end(s);
}

// ============================================================== DistriFusion
// run_distrifusion_inline (execute.cpp:431-531): per step, warmup steps run
// layer-lockstep over the full sequence (all shards fresh); steady steps run
// each worker's shard through all layers attending over [its fresh rows |
// every other shard's rows of the previous step], then install all shards.
// Two K/V buffers per layer alternate as "previous step" and "this step":
// every shard's rows of "this step" are rewritten by its worker during the
// step, so swapping the roles afterwards is the reference's install().
void Engine::enqueue_distrifusion(float* x_dev, int steps, int workers, int warmup, float eta,
                                  cudaStream_t caller, RunStats* stats) {
  const ModelShape& m = shape_;
  if (stage_count() != 1 || rank_mode())
    throw ValidationError("DistriFusion runs on a single-stage engine (one device per worker "
                          "in the reference; here the workers share the stage's GPU)");
  if (m.block != kBlockToy) throw ValidationError("DistriFusion is defined for the toy block");
  if (steps < 1) throw ValidationError("steps must be >= 1");
  if (workers < 1) throw ValidationError("workers must be >= 1");
  if (warmup < 0 || warmup > steps) throw ValidationError("warmup must lie in [0, steps]");
  if (m.P % workers != 0) {
    std::ostringstream os;
    os << "seq_len " << m.P << " is not divisible by workers " << workers;
    throw ValidationError(os.str());
  }
  const int r = int(m.P / workers);
  // shards off the attention's 128-row KV blocks: merged K/V copies per worker
  const bool merge = workers > 1 && r % 128 != 0;
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  const size_t kvn = size_t(m.heads) * size_t(m.P) * size_t(m.dhp);
  if (merge)
    while (int(df_sk_.size()) < workers) {
      PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
      df_sk_.push_back(dalloc<bf16>(kvn));
      df_sv_.push_back(dalloc<bf16>(kvn));
      df_tm_sk_.push_back(tmap(df_sk_.back(), m.dhp, size_t(m.heads) * m.P,
                               size_t(m.dhp) * 2, 16, 128, 32));
      df_tm_sv_.push_back(tmap(df_sv_.back(), m.dhp, size_t(m.heads) * m.P,
                               size_t(m.dhp) * 2, 16, 128, 32));
    }
  for (StageLayer& L : s.layers)
    if (!L.k2) {
      PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
      L.k2 = dalloc<bf16>(kvn);
      L.v2 = dalloc<bf16>(kvn);
      check(v_ones_col(L.v2, kvn / size_t(m.dhp), m.dhp, m.dh, nullptr), "v_ones_col");
      L.tm_k2 = tmap(L.k2, m.dhp, size_t(m.heads) * m.P, size_t(m.dhp) * 2, 16, 128, 32);
      L.tm_v2 = tmap(L.v2, m.dhp, size_t(m.heads) * m.P, size_t(m.dhp) * 2, 16, 128, 32);
      if (L.has_kv3) {
        const uint32_t b3 = uint32_t(attn3_kv_rows(m.dhp));
        L.tm_k23 = tmap(L.k2, m.dhp, size_t(m.heads) * m.P, size_t(m.dhp) * 2, 16, b3, 32);
        L.tm_v23 = tmap(L.v2, m.dhp, size_t(m.heads) * m.P, size_t(m.dhp) * 2, 16, b3, 32);
      }
    }
  if (!ev_start_) PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_start_, cudaEventDisableTiming));
  RunStats local;
  RunStats& st = stats ? *stats : local;
  st.fresh = 0;
  st.stale = 0;
  st.fresh_fraction.assign(size_t(workers), {});
  codes_.clear();
  LaunchTally tally(launches_);
  prof_.clear();
  prof_used_.assign(stages_.size(), 0);
  tl_.clear();

  PF_CUDA_CHECK(cudaEventRecord(ev_start_, caller));
  PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, ev_start_, 0));
  check(reset_flag(s.flag, s.stream), "reset_flag");
  // slot 0 = (k, v), slot 1 = (k2, v2); `prev` holds the previous step
  int prev = 0;
  if (warmup == 0)  // StageBuffers are zero-initialised (execute.cpp:42-48)
    for (StageLayer& L : s.layers) {
      PF_CUDA_CHECK(cudaMemsetAsync(L.k, 0, kvn * sizeof(bf16), s.stream));
      PF_CUDA_CHECK(cudaMemsetAsync(L.v, 0, kvn * sizeof(bf16), s.stream));
      check(v_ones_col(L.v, kvn / size_t(m.dhp), m.dhp, m.dh, s.stream), "v_ones_col");
    }
  auto view = [&](StageLayer& L, int fresh_lo, int fresh_hi) {
    const int nxt = 1 - prev;
    KvView kv;
    kv.k = nxt ? L.k2 : L.k;
    kv.v = nxt ? L.v2 : L.v;
    kv.tm_k = prev ? &L.tm_k2 : &L.tm_k;
    kv.tm_v = prev ? &L.tm_v2 : &L.tm_v;
    kv.tm_k2 = nxt ? &L.tm_k2 : &L.tm_k;
    kv.tm_v2 = nxt ? &L.tm_v2 : &L.tm_v;
    kv.fresh_lo = fresh_lo;
    kv.fresh_hi = fresh_hi;
    if (fresh_lo == 0 && fresh_hi == int(m.P)) {  // every row from this step's buffer
      kv.tm_k = kv.tm_k2;
      kv.tm_v = kv.tm_v2;
      kv.fresh_lo = kv.fresh_hi = 0;
      if (L.has_kv3) {
        kv.k3 = nxt ? &L.tm_k23 : &L.tm_k3;
        kv.v3 = nxt ? &L.tm_v23 : &L.tm_v3;
      }
    }
    return kv;
  };
  const size_t hs = size_t(m.hs);
  // Workers of one steady step are independent (each writes only its own
  // shard's rows of this step's K/V buffer and reads the others' rows of the
  // previous step's), so they run on the stage's patch lanes, forked at the
  // start of the step and joined at its end (the next step reads every
  // shard of this step's buffer and overwrites the one this step read).
  const int nl = lanes_for(workers);
  if (nl > 1) alloc_lanes(s, nl);
  for (int step = 0; step < steps; ++step) {
    const int t = steps - 1 - step;
    if (step < warmup) {
      // every worker sees every shard fresh: one full-sequence pass
      check(patch_prepare(x_dev, nullptr, s.cb, s.h32, s.hb, 0, int(m.P), m.hs, 0.f, false,
                          s.stream), "patch_prepare");
      for (int l = 0; l < s.layer_count; ++l) {
        st.fresh += int64_t(workers) * workers;
        codes_.emplace_back(t, l);
        KvView kv = view(s.layers[size_t(l)], 0, int(m.P));
        kv.tm_k = kv.tm_k2;  // attend over this step's buffer only
        kv.tm_v = kv.tm_v2;
        layer_forward(s, l, int(m.P), 0, int(codes_.size()) - 1, &kv);
      }
      check(latent_update(x_dev, s.h32, eta, size_t(m.P) * hs, s.stream), "latent_update");
    } else {
      if (nl > 1) {
        PF_CUDA_CHECK(cudaEventRecord(s.ev_lane[0], s.stream));
        for (int k = 1; k < nl; ++k)
          PF_CUDA_CHECK(cudaStreamWaitEvent(s.extra[k].stream, s.ev_lane[0], 0));
      }
      for (int i = 0; i < workers; ++i) {
        const int row0 = i * r;
        if (nl > 1) use_lane(s, i % nl);
        check(patch_prepare(x_dev, nullptr, s.cb, s.h32, s.hb, row0, r, m.hs, 0.f, false,
                            s.stream), "patch_prepare");
        for (int l = 0; l < s.layer_count; ++l) {
          // own shard fresh (t), the others installed last step (t + 1)
          st.fresh += 1;
          st.stale += workers - 1;
          codes_.emplace_back(t, l);
          KvView kv = view(s.layers[size_t(l)], row0, row0 + r);
          if (merge) {
            StageLayer& L = s.layers[size_t(l)];
            kv.prev_k = prev ? L.k2 : L.k;
            kv.prev_v = prev ? L.v2 : L.v;
            kv.sk = df_sk_[size_t(i)];
            kv.sv = df_sv_[size_t(i)];
            kv.tm_sk = &df_tm_sk_[size_t(i)];
            kv.tm_sv = &df_tm_sv_[size_t(i)];
          }
          layer_forward(s, l, r, row0, int(codes_.size()) - 1, &kv);
        }
        st.fresh_fraction[size_t(i)].push_back(1.0 / double(workers));
        check(latent_update(x_dev + size_t(row0) * hs, s.h32 + size_t(row0) * hs, eta,
                            size_t(r) * hs, s.stream), "latent_update");
      }
      if (nl > 1) {
        use_lane(s, 0);
        for (int k = 1; k < nl; ++k) {
          PF_CUDA_CHECK(cudaEventRecord(s.ev_lane[k], s.extra[k].stream));
          PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, s.ev_lane[k], 0));
        }
      }
    }
    prev = 1 - prev;  // install: this step's buffer becomes the previous step's
  }
  PF_CUDA_CHECK(cudaEventRecord(s.ev_fwd, s.stream));
  PF_CUDA_CHECK(cudaStreamWaitEvent(caller, s.ev_fwd, 0));
}

// ============================================================== timeline
void Engine::tl_begin(int stage, int stream, int patch, int t, cudaStream_t st) {
  if (!timeline_on_) return;
  const int d = stage < int(stages_.size()) ? stage : 0;
  TlRec r{stage, stream, patch, t, prof_event(d), prof_event(d)};
  PF_CUDA_CHECK(cudaEventRecord(r.a, st));
  tl_.push_back(r);
}

void Engine::tl_end(cudaStream_t st) {
  if (!timeline_on_) return;
  PF_CUDA_CHECK(cudaEventRecord(tl_.back().b, st));
}

std::vector<TimelineSpan> Engine::collect_timeline() {
  std::vector<TimelineSpan> out;
  if (!tl_origin_) return out;
  DeviceGuard g(stages_[0].device);
  PF_CUDA_CHECK(cudaEventSynchronize(tl_origin_));
  for (const TlRec& r : tl_) {
    PF_CUDA_CHECK(cudaEventSynchronize(r.b));
    float a = 0.f, b = 0.f;
    PF_CUDA_CHECK(cudaEventElapsedTime(&a, tl_origin_, r.a));
    PF_CUDA_CHECK(cudaEventElapsedTime(&b, tl_origin_, r.b));
    out.push_back({r.stage, r.stream, r.patch, r.t, 1e3 * double(a), 1e3 * double(b - a)});
  }
  return out;
}

// ============================================================== rank mode
namespace {

using MemOpFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct MemOps {
  MemOpFn wait = nullptr, write = nullptr;
  bool flush = false;
};

const MemOps& memops(int device) {
  static MemOps ops;
  static std::once_flag once;
  std::call_once(once, [&] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      ops.wait = reinterpret_cast<MemOpFn>(p);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      ops.write = reinterpret_cast<MemOpFn>(p);
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrCanFlushRemoteWrites, device);
    ops.flush = v != 0;
  });
  if (!ops.wait || !ops.write) throw CudaError("stream memory operations are unavailable");
  return ops;
}

// Stream-ordered "wait until *addr >= value" / "*addr = value" (the
// latter after all prior work of the stream, with a memory barrier).
void stream_wait_geq(cudaStream_t st, const uint32_t* addr, uint32_t value, int device) {
  const MemOps& m = memops(device);
  const unsigned flags = 0x0 /*CU_STREAM_WAIT_VALUE_GEQ*/ | (m.flush ? 0x40000000u : 0u);
  if (m.wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value, flags) !=
      CUDA_SUCCESS)
    throw CudaError("cuStreamWaitValue32 failed");
}

void stream_write(cudaStream_t st, uint32_t* addr, uint32_t value, int device) {
  const MemOps& m = memops(device);
  if (m.write(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), value, 0) !=
      CUDA_SUCCESS)
    throw CudaError("cuStreamWriteValue32 failed");
}


}  // namespace

Engine::Engine(const ModelShape& shape_in, int device, int rank, int world)
    : shape_(shape_in), rank_(rank), world_(world) {
  shape_.dh = shape_.hs / std::max(shape_.heads, 1);
  shape_.dhp = (shape_.dh + 15) / 16 * 16;
  validate_shape(shape_);
  if (world < 1 || rank < 0 || rank >= world)
    throw ValidationError("rank must lie in [0, world)");
  if (world > shape_.layers) {
    std::ostringstream os;
    os << "layer count " << shape_.layers << " is not divisible by workers " << world
       << " (fewer layers than stages)";
    throw ValidationError(os.str());
  }
  int dev_count = 0;
  PF_CUDA_CHECK(cudaGetDeviceCount(&dev_count));
  if (device < 0 || device >= dev_count) {
    std::ostringstream os;
    os << "CUDA device " << device << " not present (" << dev_count << " visible)";
    throw ValidationError(os.str());
  }
  stages_.resize(1);
  Stage& s = stages_[0];
  s.device = device;
  try {
    const int first = int(int64_t(rank) * shape_.layers / world);
    const int last = int(int64_t(rank + 1) * shape_.layers / world);
    alloc_stage(s, first, last - first, rank == 0);
    DeviceGuard g(device);
    PF_CUDA_CHECK(cudaStreamCreateWithFlags(&send_stream_, cudaStreamNonBlocking));
    PF_CUDA_CHECK(cudaStreamCreateWithFlags(&abort_stream_, cudaStreamNonBlocking));
    PF_CUDA_CHECK(cudaEventCreateWithFlags(&ev_compute_, cudaEventDisableTiming));
    // signal page: [0] messages delivered here, [1] acknowledgements from the
    // successor, [2] epoch of a run a neighbour aborted (0: none)
    sig_ = dalloc<uint32_t>(64);
    if (rank == 0 && world > 1) {
      s.eps = dalloc<float>(size_t(shape_.P) * shape_.hs);
      s.eps_owned = true;
    }
  } catch (...) {
    free_stage(s);
    throw;
  }
}

PeerBlob Engine::export_peer() {
  if (!rank_mode()) throw ValidationError("export_peer needs a rank-mode engine");
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  PeerBlob b;
  b.rank = rank_;
  b.world = world_;
  b.device = s.device;
  b.block = shape_.block;
  b.pid = int64_t(getpid());
  b.host_id = host_identity();
  b.nonce = process_nonce();
  std::memset(&b.h_h32, 0, sizeof(b.h_h32));
  std::memset(&b.h_hb, 0, sizeof(b.h_hb));
  std::memset(&b.h_stats, 0, sizeof(b.h_stats));
  std::memset(&b.h_eps, 0, sizeof(b.h_eps));
  std::memset(&b.h_sig, 0, sizeof(b.h_sig));
  PF_CUDA_CHECK(cudaIpcGetMemHandle(&b.h_h32, s.h32));
  PF_CUDA_CHECK(cudaIpcGetMemHandle(&b.h_hb, s.hb));
  PF_CUDA_CHECK(cudaIpcGetMemHandle(&b.h_sig, sig_));
  if (s.px.stats) PF_CUDA_CHECK(cudaIpcGetMemHandle(&b.h_stats, s.px.stats));
  if (s.eps) PF_CUDA_CHECK(cudaIpcGetMemHandle(&b.h_eps, s.eps));
  b.p_h32 = reinterpret_cast<uint64_t>(s.h32);
  b.p_hb = reinterpret_cast<uint64_t>(s.hb);
  b.p_stats = reinterpret_cast<uint64_t>(s.px.stats);
  b.p_eps = reinterpret_cast<uint64_t>(s.eps);
  b.p_sig = reinterpret_cast<uint64_t>(sig_);
  return b;
}

void Engine::connect_peers(const PeerBlob& pred, const PeerBlob& succ) {
  if (!rank_mode()) throw ValidationError("connect_peers needs a rank-mode engine");
  for (const PeerBlob* b : {&pred, &succ}) {
    if (b->magic != 0x50465042) throw ValidationError("peer blob is not a pipefusion endpoint");
    if (b->world != world_ || b->block != shape_.block)
      throw ValidationError("peer was created for a different world or block");
  }
  if (succ.rank != (rank_ + 1) % world_ || pred.rank != (rank_ - 1 + world_) % world_)
    throw ValidationError("peer blobs do not belong to this rank's neighbours");
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  // A neighbour in this process on this device (tests on one GPU): such
  // ranks enqueue their plans op by op instead of replaying CUDA graphs.
  // Measured on B200: instantiating a graph while a peer's replay waits on
  // this rank's signals blocks the host, and several in-process replays
  // with patch lanes can map their waiting branches onto shared hardware
  // queues and stall each other. One rank per GPU (or per process) is the
  // deployment shape and replays graphs.
  shared_device_peer_ = false;
  for (const PeerBlob* b : {&pred, &succ})
    if (b->nonce == process_nonce() && b->pid == int64_t(getpid()) && b->device == s.device)
      shared_device_peer_ = true;
  for (const PeerBlob* b : {&pred, &succ})
    if (b->host_id != host_identity()) {
      std::ostringstream os;
      os << "peer rank " << b->rank << " lives on another host: stage boundaries need peer "
         << "memory (CUDA IPC over NVLink) within one node";
      throw ValidationError(os.str());
    }
  auto open = [&](const PeerBlob& b, const cudaIpcMemHandle_t& h, uint64_t raw) -> void* {
    if (b.nonce == process_nonce() && b.pid == int64_t(getpid())) {
      // same process: UVA pointer; enable peer access when on another device
      if (b.device != s.device) {
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, s.device, b.device);
        if (ok) {
          cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
      }
      return reinterpret_cast<void*>(raw);
    }
    void* p = nullptr;
    PF_CUDA_CHECK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ipc_opened_.push_back(p);
    return p;
  };
  succ_sig_ = static_cast<uint32_t*>(open(succ, succ.h_sig, succ.p_sig));
  pred_sig_ = static_cast<uint32_t*>(open(pred, pred.h_sig, pred.p_sig));
  if (succ.rank == 0) {
    succ_eps_ = static_cast<float*>(open(succ, succ.h_eps, succ.p_eps));
  } else {
    succ_h32_ = static_cast<float*>(open(succ, succ.h_h32, succ.p_h32));
    succ_hb_ = static_cast<bf16*>(open(succ, succ.h_hb, succ.p_hb));
    if (shape_.ln_stats())
      succ_stats_ = static_cast<float2*>(open(succ, succ.h_stats, succ.p_stats));
  }
  // tensor maps over the successor's buffers for the fused send (the last
  // MLP-out GEMM's TMA stores): rank 0's eps (fp32) from the last rank, the
  // next stage's residual stream and bf16 operand otherwise
  const size_t hs = size_t(shape_.hs);
  // the eps buffer holds image rows; activations hold joint rows (text first)
  const size_t P = succ_eps_ ? size_t(shape_.P) : size_t(shape_.rows_total());
  float* dst32 = succ_eps_ ? succ_eps_ : succ_h32_;
  if (!encode_tmap_f32_2d(&tm_peer_h32_, dst32, hs, P, hs * 4, 32, 128, 128))
    throw CudaError("cuTensorMapEncodeTiled failed for a peer buffer");
  peer_out_ = OutRedirect{};
  peer_out_.h32 = dst32;
  peer_out_.tm_h32 = &tm_peer_h32_;
  if (succ_hb_) {
    tm_peer_hb_ = tmap(succ_hb_, hs, P, hs * 2, 64, 128, 128);
    peer_out_.hb = succ_hb_;
    peer_out_.tm_hb = &tm_peer_hb_;
  } else {  // eps only: the bf16 copy stays local (unused)
    peer_out_.hb = s.hb;
    peer_out_.tm_hb = &s.tm_hb;
  }
  peer_out_.stats = succ_stats_;
  connected_ = true;
}

void Engine::connect_world(const std::vector<PeerBlob>& blobs) {
  if (!rank_mode()) throw ValidationError("connect_world needs a rank-mode engine");
  if (int(blobs.size()) != world_) throw ValidationError("connect_world needs one blob per rank");
  for (int r = 0; r < world_; ++r)
    if (blobs[size_t(r)].rank != r) throw ValidationError("peer blobs are not in rank order");
  connect_peers(blobs[size_t((rank_ - 1 + world_) % world_)], blobs[size_t((rank_ + 1) % world_)]);
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  world_sig_.clear();
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) continue;
    const PeerBlob& b = blobs[size_t(r)];
    if (r == (rank_ + 1) % world_) { world_sig_.push_back(succ_sig_); continue; }
    if (r == (rank_ - 1 + world_) % world_) { world_sig_.push_back(pred_sig_); continue; }
    if (b.nonce == process_nonce() && b.pid == int64_t(getpid())) {
      world_sig_.push_back(reinterpret_cast<uint32_t*>(b.p_sig));
    } else {
      void* p = nullptr;
      PF_CUDA_CHECK(cudaIpcOpenMemHandle(&p, b.h_sig, cudaIpcMemLazyEnablePeerAccess));
      ipc_opened_.push_back(p);
      world_sig_.push_back(static_cast<uint32_t*>(p));
    }
  }
}

// One rank's share of run_pipefusion (rank_plan.h): its stage's layers on the
// compute stream, boundary transfers on the send stream, and the message
// protocol as stream-ordered waits/writes on the peers' signal pages.
void Engine::enqueue_rank_run(float* x_dev, int steps, int patches, int warmup, float eta,
                              cudaStream_t caller, RunStats* stats, bool skip_all) {
  const ModelShape& m = shape_;
  if (!connected_) throw ValidationError("rank-mode engine is not connected to its peers");
  validate_run(steps, patches, warmup);
  if (rank_ == 0 && !x_dev) throw ValidationError("NULL latent pointer");
  Stage& s = stages_[0];
  DeviceGuard g(s.device);
  const int dev = s.device;
  const bool px = m.block == kBlockPixArt;
  const int r = int(m.P / patches);
  const size_t hs = size_t(m.hs);
  prepare_rank_run(patches, steps);
  std::vector<bool> sent_before(size_t(patches), false);
  run_base_ = msgs_in_base_;

  RunStats local;
  RunStats& st = stats ? *stats : local;
  st.fresh = 0;
  st.stale = 0;
  st.fresh_fraction.assign(1, {});
  std::vector<std::vector<int>> src(size_t(s.layer_count), std::vector<int>(size_t(patches), steps));
  codes_.clear();
  LaunchTally tally(launches_);
  prof_.clear();
  prof_used_.assign(stages_.size(), 0);

  tl_.clear();
  if (timeline_on_) {
    if (!tl_origin_) PF_CUDA_CHECK(cudaEventCreate(&tl_origin_));
    PF_CUDA_CHECK(cudaEventRecord(tl_origin_, caller));
  }
  PF_CUDA_CHECK(cudaEventRecord(ev_start_, caller));
  PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, ev_start_, 0));
  PF_CUDA_CHECK(cudaStreamWaitEvent(send_stream_, ev_start_, 0));
  check(reset_flag(s.flag, s.stream), "reset_flag");
  if (warmup == 0) {
    const size_t kv = size_t(m.heads) * size_t(m.rows_total()) * size_t(m.dhp) * sizeof(bf16);
    for (StageLayer& L : s.layers) {
      PF_CUDA_CHECK(cudaMemsetAsync(L.k, 0, kv, s.stream));
      PF_CUDA_CHECK(cudaMemsetAsync(L.v, 0, kv, s.stream));
      check(v_ones_col(L.v, kv / (size_t(m.dhp) * sizeof(bf16)), m.dhp, m.dh, s.stream),
            "v_ones_col");
      if (L.k32) {
        const size_t n32 = size_t(m.rows_total()) * size_t(m.hs) * sizeof(float);
        PF_CUDA_CHECK(cudaMemsetAsync(L.k32, 0, n32, s.stream));
        PF_CUDA_CHECK(cudaMemsetAsync(L.v32, 0, n32, s.stream));
      }
    }
  }
  const bool mm = m.block == kBlockMMDiT;
  if (px) px_conditioning(s, steps);
  if (mm) mm_conditioning(s, steps);

  const uint32_t base_in = msgs_in_base_, base_out = msgs_out_base_;
  const auto plan = build_rank_plan(rank_, world_, steps, patches, warmup, m.P);
  // Fused send (default): the stage's last MLP-out GEMM stores the message
  // rows straight into the successor's buffers; the flow-control wait and the
  // signal are stream-ordered around it on the compute stream. PF_RANK_COPY=1
  // keeps the separate copy on the send stream.
  static const bool copy_send = [] {
    const char* e = std::getenv("PF_RANK_COPY");
    return e && e[0] == '1';
  }();
  const bool joint = m.joint_rows();
  const int J = int(m.J());
  // joint block: the eps rows of the last rank are image rows (offset by the
  // text rows), which the GEMM's joint-row stores cannot address: copy them
  const bool fused = !copy_send && !(joint && succ_eps_);
  // Lanes (fused sends, M >= 2): the ops of patch j run on lane
  // j % nl, full-sequence ops on lane 0 (lanes fork after / join before
  // them). Besides the K/V ordering of layer_forward (QKV(j, l) after the
  // previous patch's ATTN(l)), the signal writes must keep plan order: their
  // values are absolute message counts that the peers wait on with >=.
  // A lane blocked in a signal wait (a stream memory operation, invisible to
  // the driver's dependency tracking) stalls every stream sharing its
  // hardware queue: lanes here need CUDA_DEVICE_MAX_CONNECTIONS >= 16 (set
  // before the context is created, as bench.py and the tests do).
  static const bool enough_queues = [] {
    const char* e = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    return e && std::atoi(e) >= 16;
  }();
  const int nl = (fused && enough_queues && !profiling_ && !timeline_on_)
                     ? std::min(lanes_, patches) : 1;
  if (nl > 1) alloc_lanes(s, nl);
  bool forked = false, wrote[2] = {false, false};
  int prev_lane = -1;
  PdlOff pdl_off(false);
  // Signal writes of one counter keep plan order across lanes (chain 0:
  // acknowledgements to the predecessor, chain 1: message counts to the
  // successor); the two counters are independent, so acks of a lane never
  // wait for another lane's compute.
  auto ordered_write = [&](int chain, cudaStream_t st, uint32_t* addr, uint32_t value) {
    if (nl > 1 && wrote[chain]) PF_CUDA_CHECK(cudaStreamWaitEvent(st, ev_write_[chain], 0));
    stream_write(st, addr, value, dev);
    if (nl > 1) {
      PF_CUDA_CHECK(cudaEventRecord(ev_write_[chain], st));
      wrote[chain] = true;
    }
  };
  auto join_lanes = [&]() {
    if (!forked) return;
    use_lane(s, 0);
    for (int k = 1; k < nl; ++k) {
      PF_CUDA_CHECK(cudaEventRecord(s.ev_lane[k], s.extra[k].stream));
      PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, s.ev_lane[k], 0));
    }
    forked = false;
  };
  // Channel close (execute.cpp:345-348): when an op throws, this rank closes
  // the run -- the abort word of every rank's signal page is set -- and
  // finishes its plan in skip mode: the message protocol only (receive
  // waits, acknowledgements, message counts), no compute. Every peer's wait
  // of the run is then satisfied exactly as in a good run, so the counters
  // stay consistent for the next run, and the peers report "channel closed
  // mid-run" from finish(). The op that threw is redone in skip mode (its
  // signal values are absolute, so a repeated write or wait is harmless).
  bool skip = skip_all;
  std::exception_ptr failure;
  auto do_op = [&](size_t oi, const PlanOp& op) {
    if (!skip && int(oi) == fail_at_op_) {
      std::ostringstream os;
      os << "injected failure at plan op " << oi << " of rank " << rank_;
      throw NumericError(os.str());
    }
    if (nl > 1 && !skip) {
      if (op.patch < 0 || op.kind == PlanOp::kLatentUpdate) {
        join_lanes();
      } else {
        if (!forked) {  // lanes start after lane 0's work so far
          use_lane(s, 0);
          PF_CUDA_CHECK(cudaEventRecord(s.ev_lane[0], s.stream));
          for (int k = 1; k < nl; ++k)
            PF_CUDA_CHECK(cudaStreamWaitEvent(s.extra[k].stream, s.ev_lane[0], 0));
          forked = true;
        }
        use_lane(s, op.patch % nl);
      }
      pdl_off.set(forked);
    }
    // plan rows are image rows; joint blocks carry the text rows with the
    // full sequence and with patch 0
    const int row0 = op.row0, rows = op.rows;
    const int brow0 = joint && op.patch > 0 ? J + row0 : row0;
    const int brows = joint && op.patch <= 0 ? J + rows : rows;
    switch (op.kind) {
      case PlanOp::kRecv:
        stream_wait_geq(s.stream, sig_, base_in + uint32_t(op.msg), dev);
        break;
      case PlanOp::kAck:
        ordered_write(0, op.flag && !fused ? send_stream_ : s.stream, pred_sig_ + 1,
                      base_in + uint32_t(op.msg));
        break;
      case PlanOp::kPrepare: {
        if (skip) break;
        // this rank's previous send of the same rows must have finished reading h32
        for (int j = 0; j < patches; ++j)
          if ((op.patch < 0 || op.patch == j) && sent_before[size_t(j)])
            PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, ev_sent_[size_t(j)], 0));
        tl_begin(rank_, 0, op.patch, op.t, s.stream);
        prof_begin(s, kSampler, 0, double(rows) * hs * (op.flag ? 18 : 10));
        if (joint && op.patch <= 0) {  // the text stream re-enters each step
          if (mm)
            mm_text_prepare(s, op.t);
          else
            check(patch_prepare(s.text, nullptr, s.zeros, s.h32, s.hb, 0, J, m.hs, 0.f, false,
                                s.stream), "text rows");
        }
        if (px)
          px_patch_prepare(x_dev, op.flag != 0, row0, rows, op.t, eta);
        else if (mm)
          mm_patch_prepare(s, x_dev, op.flag != 0, row0, rows, op.t, eta);
        else
          check(patch_prepare(x_dev, s.eps, s.cb, s.h32 + size_t(J) * hs, s.hb + size_t(J) * hs,
                              row0, rows, m.hs, eta, op.flag != 0, s.stream), "patch_prepare");
        prof_end(s);
        break;
      }
      case PlanOp::kLatentUpdate:
        if (skip) break;
        prof_begin(s, kSampler, 0, double(m.P) * hs * 12);
        check(latent_update(x_dev, s.eps, eta, size_t(m.P) * hs, s.stream), "latent_update");
        prof_end(s);
        break;
      case PlanOp::kCompute: {
        if (skip) {  // the fused send's protocol part only
          if (fused && oi + 1 < plan.size() && plan[oi + 1].kind == PlanOp::kSend) {
            const PlanOp& sn = plan[oi + 1];
            if (sn.overlap > 0)
              stream_wait_geq(s.stream, sig_ + 1, base_out + uint32_t(sn.overlap), dev);
            ordered_write(1, s.stream, succ_sig_, base_out + uint32_t(sn.msg));
          }
          break;
        }
        const int t = op.t;
        if (rank_ != 0) tl_begin(rank_, 0, op.patch, t, s.stream);
        for (int lf = 0; lf < s.layer_count; ++lf) {
          auto& sv = src[size_t(lf)];
          if (op.patch < 0) {
            std::fill(sv.begin(), sv.end(), t);
            st.fresh += patches;
          } else {
            sv[size_t(op.patch)] = t;
            for (size_t pi = 0; pi < sv.size(); ++pi) {
              if (sv[pi] == t) {
                ++st.fresh;
              } else if (sv[pi] == t + 1) {
                ++st.stale;
              } else {
                std::ostringstream os;
                os << "staleness bound violated: patch " << pi << " carries timestep " << sv[pi]
                   << " while computing timestep " << t;
                throw NumericError(os.str());
              }
            }
          }
          codes_.emplace_back(t, s.first_layer + lf);
          const int code = int(codes_.size()) - 1;
          const bool last = lf == s.layer_count - 1;
          const PlanOp* send = fused && last && oi + 1 < plan.size() &&
                                       plan[oi + 1].kind == PlanOp::kSend
                                   ? &plan[oi + 1]
                                   : nullptr;
          if (send && send->overlap > 0)  // landing rows free at the successor
            stream_wait_geq(s.stream, sig_ + 1, base_out + uint32_t(send->overlap), dev);
          redirect_ = send ? &peer_out_ : nullptr;
          if (nl > 1 && op.patch >= 0) {
            lane_wait_ = prev_lane >= 0 ? s.ev_attn[prev_lane][size_t(lf)] : nullptr;
            lane_rec_ = s.ev_attn[op.patch % nl][size_t(lf)];
          }
          if (px) layer_forward_px(s, lf, rows, row0, t, code);
          else if (mm) layer_forward_mm(s, lf, brows, brow0, t, code);
          else if (joint && s.first_layer + lf < m.double_layers)
            layer_forward_joint(s, lf, brows, brow0, code);
          else if (joint)
            layer_forward_single(s, lf, brows, brow0, code);
          else layer_forward(s, lf, rows, row0, code);
          redirect_ = nullptr;
          lane_wait_ = lane_rec_ = nullptr;
          if (send) {
            ordered_write(1, s.stream, succ_sig_, base_out + uint32_t(send->msg));
            for (int j = 0; j < patches; ++j)
              if (send->patch < 0 || send->patch == j) {
                PF_CUDA_CHECK(cudaEventRecord(ev_sent_[size_t(j)], s.stream));
                sent_before[size_t(j)] = true;
              }
          }
        }
        tl_end(s.stream);
        if (op.patch >= 0) {
          int fresh = 0;
          for (int v : src[0]) fresh += (v == t);
          st.fresh_fraction[0].push_back(double(fresh) / double(patches));
          prev_lane = op.patch % nl;
        }
        break;
      }
      case PlanOp::kSend: {
        if (fused) break;  // stored by the last MLP-out GEMM, signalled after it
        if (skip) {
          if (op.overlap > 0)
            stream_wait_geq(s.stream, sig_ + 1, base_out + uint32_t(op.overlap), dev);
          ordered_write(1, s.stream, succ_sig_, base_out + uint32_t(op.msg));
          break;
        }
        PF_CUDA_CHECK(cudaEventRecord(ev_compute_, s.stream));
        PF_CUDA_CHECK(cudaStreamWaitEvent(send_stream_, ev_compute_, 0));
        if (op.overlap > 0)
          stream_wait_geq(send_stream_, sig_ + 1, base_out + uint32_t(op.overlap), dev);
        tl_begin(rank_, 1, op.patch, op.t, send_stream_);
        const size_t off = size_t(brow0) * hs, cnt = size_t(brows) * hs;
        if (succ_eps_) {  // image rows only, image-indexed at rank 0
          PF_CUDA_CHECK(cudaMemcpyAsync(succ_eps_ + size_t(row0) * hs,
                                        s.h32 + size_t(J + row0) * hs, size_t(rows) * hs * 4,
                                        cudaMemcpyDefault, send_stream_));
        } else {
          PF_CUDA_CHECK(cudaMemcpyAsync(succ_h32_ + off, s.h32 + off, cnt * 4,
                                        cudaMemcpyDefault, send_stream_));
          PF_CUDA_CHECK(cudaMemcpyAsync(succ_hb_ + off, s.hb + off, cnt * 2, cudaMemcpyDefault,
                                        send_stream_));
          if (m.ln_stats()) {
            const size_t pitch = size_t(m.rows_total()) * sizeof(float2);
            PF_CUDA_CHECK(cudaMemcpy2DAsync(succ_stats_ + brow0, pitch, s.px.stats + brow0,
                                            pitch, size_t(brows) * sizeof(float2),
                                            size_t(m.hs / 32), cudaMemcpyDefault,
                                            send_stream_));
          }
        }
        tl_end(send_stream_);
        ordered_write(1, send_stream_, succ_sig_, base_out + uint32_t(op.msg));
        for (int j = 0; j < patches; ++j)
          if (op.patch < 0 || op.patch == j) {
            PF_CUDA_CHECK(cudaEventRecord(ev_sent_[size_t(j)], send_stream_));
            sent_before[size_t(j)] = true;
          }
        break;
      }
    }
  };
  for (size_t oi = 0; oi < plan.size(); ++oi) {
    try {
      do_op(oi, plan[oi]);
    } catch (...) {
      if (skip) throw;  // the protocol itself failed (CUDA error): nothing left to do
      failure = std::current_exception();
      skip = true;
      redirect_ = nullptr;
      lane_wait_ = lane_rec_ = nullptr;
      join_lanes();
      pdl_off.set(false);
      close_channels();
      do_op(oi, plan[oi]);
    }
  }
  const uint32_t per_run = uint32_t(plan_messages_per_run(steps, patches, warmup));
  msgs_in_base_ += per_run;
  msgs_out_base_ += per_run;
  if (nl > 1) join_lanes();
  use_lane(s, 0);
  // join: the caller waits for both streams
  PF_CUDA_CHECK(cudaEventRecord(s.ev_fwd, s.stream));
  PF_CUDA_CHECK(cudaStreamWaitEvent(caller, s.ev_fwd, 0));
  PF_CUDA_CHECK(cudaEventRecord(ev_compute_, send_stream_));
  PF_CUDA_CHECK(cudaStreamWaitEvent(caller, ev_compute_, 0));
  if (failure) std::rethrow_exception(failure);
}

// ============================================================== PixArt block
namespace {
// Transpose an fp64 [K x N] (x.W orientation) matrix to [N x K] (K-major).
template <class T, class Cvt>
std::vector<T> transpose_kn(const double* w, int K, int N, Cvt cvt) {
  std::vector<T> out(size_t(N) * K);
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) out[size_t(n) * K + k] = cvt(w[size_t(k) * N + n]);
  return out;
}
inline bf16 to_bf(double v) { return __float2bfloat16_rn(float(v)); }
inline float to_f(double v) { return float(v); }
std::vector<float> to_f32(const double* v, size_t n) {
  std::vector<float> out(n);
  for (size_t i = 0; i < n; ++i) out[i] = float(v[i]);
  return out;
}
}  // namespace

void Engine::load_layer_px(int layer, const double* const* prm) {
  if (shape_.block != kBlockPixArt) throw ValidationError("model is not a PixArt block model");
  const int d = stage_of_layer(layer);
  if (d < 0 && rank_mode() && layer >= 0 && layer < shape_.layers) {
    // another rank's layer; keep its adaLN row if it is the one after ours
    Stage& s = stages_[0];
    if (layer == s.first_layer + s.layer_count) {
      std::vector<float> sst(size_t(6) * shape_.hs);
      for (size_t i = 0; i < sst.size(); ++i) sst[i] = float(prm[16][i]);
      DeviceGuard g(s.device);
      PF_CUDA_CHECK(cudaMemcpy(s.px.sst + size_t(s.layer_count) * sst.size(), sst.data(),
                               sst.size() * 4, cudaMemcpyHostToDevice));
    }
    return;
  }
  if (d < 0) throw ValidationError("layer index out of range");
  Stage& s = stages_[size_t(d)];
  StageLayer& L = s.layers[size_t(layer - s.first_layer)];
  const int hs = shape_.hs, mlp = shape_.mlp;
  // PXO_* order: WQKV BQKV WO BO WQC BQC WKC BKC WVC BVC WOC BOC W1 B1 W2 B2 SST
  auto up = [&](void* dst, const void* src, size_t bytes) {
    PF_CUDA_CHECK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  };
  DeviceGuard g(s.device);
  auto wqkv = transpose_kn<bf16>(prm[0], hs, 3 * hs, to_bf);
  auto wo = transpose_kn<bf16>(prm[2], hs, hs, to_bf);
  auto wqc = transpose_kn<bf16>(prm[4], hs, hs, to_bf);
  auto wkc = transpose_kn<bf16>(prm[6], hs, hs, to_bf);
  auto wvc = transpose_kn<bf16>(prm[8], hs, hs, to_bf);
  auto woc = transpose_kn<bf16>(prm[10], hs, hs, to_bf);
  auto w1 = transpose_kn<bf16>(prm[12], hs, mlp, to_bf);
  auto w2 = transpose_kn<bf16>(prm[14], mlp, hs, to_bf);
  up(L.wqkv, wqkv.data(), wqkv.size() * 2);
  up(L.wo, wo.data(), wo.size() * 2);
  up(L.wqc, wqc.data(), wqc.size() * 2);
  up(L.wkvc, wkc.data(), wkc.size() * 2);
  up(L.wkvc + size_t(hs) * hs, wvc.data(), wvc.size() * 2);
  up(L.woc, woc.data(), woc.size() * 2);
  up(L.win, w1.data(), w1.size() * 2);
  up(L.wout, w2.data(), w2.size() * 2);
  auto bqkv = to_f32(prm[1], size_t(3) * hs);
  up(L.bqkv, bqkv.data(), bqkv.size() * 4);
  auto bo = to_f32(prm[3], hs);
  up(L.bo, bo.data(), bo.size() * 4);
  auto bqc = to_f32(prm[5], hs);
  up(L.bqc, bqc.data(), bqc.size() * 4);
  auto bkc = to_f32(prm[7], hs);
  auto bvc = to_f32(prm[9], hs);
  up(L.bkvc, bkc.data(), bkc.size() * 4);
  up(L.bkvc + hs, bvc.data(), bvc.size() * 4);
  auto boc = to_f32(prm[11], hs);
  up(L.boc, boc.data(), boc.size() * 4);
  auto b1 = to_f32(prm[13], size_t(mlp));
  up(L.b1, b1.data(), b1.size() * 4);
  auto b2 = to_f32(prm[15], hs);
  up(L.b2, b2.data(), b2.size() * 4);
  auto sst = to_f32(prm[16], size_t(6) * hs);
  const size_t row = size_t(6) * hs;
  up(s.px.sst + size_t(layer - s.first_layer) * row, sst.data(), row * 4);
  // The previous stage's last epilogue folds this layer's adaLN scale into
  // the bf16 operand it sends: keep a copy as that stage's "next" row.
  if (layer == s.first_layer && d > 0) {
    Stage& prev = stages_[size_t(d - 1)];
    DeviceGuard gp(prev.device);
    up(prev.px.sst + size_t(prev.layer_count) * row, sst.data(), row * 4);
  }
}

void Engine::load_px_globals(const double* const* gw) {
  if (shape_.block != kBlockPixArt) throw ValidationError("model is not a PixArt block model");
  const int hs = shape_.hs;
  auto wt1 = transpose_kn<float>(gw[0], kPxFreq, hs, to_f);
  auto bt1 = to_f32(gw[1], hs);
  auto wt2 = transpose_kn<float>(gw[2], hs, hs, to_f);
  auto bt2 = to_f32(gw[3], hs);
  auto wt0 = transpose_kn<float>(gw[4], hs, 6 * hs, to_f);
  auto bt0 = to_f32(gw[5], size_t(6) * hs);
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    PF_CUDA_CHECK(cudaMemcpy(s.px.wt1, wt1.data(), wt1.size() * 4, cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(s.px.bt1, bt1.data(), bt1.size() * 4, cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(s.px.wt2, wt2.data(), wt2.size() * 4, cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(s.px.bt2, bt2.data(), bt2.size() * 4, cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(s.px.wt0, wt0.data(), wt0.size() * 4, cudaMemcpyHostToDevice));
    PF_CUDA_CHECK(cudaMemcpy(s.px.bt0, bt0.data(), bt0.size() * 4, cudaMemcpyHostToDevice));
  }
}

void Engine::set_text(const double* y) {
  if (shape_.joint_rows()) {
    Stage& s0 = stages_[0];
    if (!s0.text) return;  // rank mode, rank > 0: text enters the pipeline on rank 0
    std::vector<float> t(size_t(shape_.T) * shape_.hs);
    for (size_t i = 0; i < t.size(); ++i) t[i] = float(y[i]);
    DeviceGuard g(s0.device);
    PF_CUDA_CHECK(cudaStreamSynchronize(s0.stream));
    PF_CUDA_CHECK(cudaMemcpy(s0.text, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    return;
  }
  if (shape_.block != kBlockPixArt) throw ValidationError("model is not a PixArt block model");
  std::vector<bf16> t(size_t(shape_.T) * shape_.hs);
  for (size_t i = 0; i < t.size(); ++i) t[i] = to_bf(y[i]);
  for (Stage& s : stages_) {
    DeviceGuard g(s.device);
    if (s.stream) PF_CUDA_CHECK(cudaStreamSynchronize(s.stream));
    PF_CUDA_CHECK(cudaMemcpy(s.px.text, t.data(), t.size() * 2, cudaMemcpyHostToDevice));
  }
}

// Per-run conditioning of one stage (adaLN-single, px_oracle.c pxo_tvec):
// timestep embeddings for every t < steps, per-layer modulation vectors,
// LayerNorm fold vectors, and the cross-attention K/V of the text tokens.
void Engine::px_conditioning(Stage& s, int steps) {
  const ModelShape& m = shape_;
  PxStage& px = s.px;
  const int hs = m.hs, w6 = 6 * m.hs, nl = s.layer_count, S = steps;
  prof_begin(s, kPxCond, 0, 0);
  check(px_sinusoid(px.sinus, S, s.stream), "px_sinusoid");
  check(px_gemv(px.sinus, S, kPxFreq, px.wt1, px.bt1, hs, px.e1, false, true, s.stream), "t_embedder.0");
  // temb is only consumed through t_block = Linear(SiLU(temb)): store silu(temb)
  check(px_gemv(px.e1, S, hs, px.wt2, px.bt2, hs, px.temb, false, true, s.stream), "t_embedder.2");
  check(px_gemv(px.temb, S, hs, px.wt0, px.bt0, w6, px.tv, false, false, s.stream), "t_block");
  check(px_mod(px.sst, nl + 1, px.tv, S, w6, px.mod, s.stream), "adaLN modulation");
  check(px_fold_rows(px.mod, nl, S, hs, px.fold_aq, px.fold_am, px.fold_rpad, s.stream),
        "LayerNorm fold operands");
  for (int lf = 0; lf < nl; ++lf) {
    StageLayer& L = s.layers[size_t(lf)];
    EpiParams fq;
    fq.out_f32 = px.foldq + size_t(lf) * 2 * S * 3 * hs;
    fq.ld = 3 * hs;
    fq.bias = L.bqkv;
    check(gemm(px.tm_aq[size_t(lf)], L.tm_wqkv, 2 * S, 0, 3 * hs, hs, Epi::Fold, fq, s.sm_count,
               s.stream), "LayerNorm fold (attention)");
    EpiParams fm;
    fm.out_f32 = px.foldm + size_t(lf) * 2 * S * m.mlp;
    fm.ld = m.mlp;
    fm.bias = L.b1;
    check(gemm(px.tm_am[size_t(lf)], L.tm_win, 2 * S, 0, m.mlp, hs, Epi::Fold, fm, s.sm_count,
               s.stream), "LayerNorm fold (MLP)");
    EpiParams kv;
    kv.q = L.kc;
    kv.k = L.vc;
    kv.hs = hs;
    kv.dh = m.dh;
    kv.dhp = m.dhp;
    kv.P = m.T;
    kv.c2 = L.bkvc;
    check(gemm(px.tm_text, L.tm_wkvc, m.T, 0, 2 * hs, hs, Epi::QKV, kv, s.sm_count, s.stream),
          "cross K/V projection");
  }
  prof_end(s);
  px_steps_ = S;
}

// Stage-0 patch split for the PixArt block: sampler update, h = x + cb, the
// first layer's adaLN-scaled bf16 operand and its LayerNorm statistics.
void Engine::px_patch_prepare(float* x_dev, bool update, int row0, int rows, int t, float eta) {
  Stage& s0 = stages_[0];
  const int hs = shape_.hs;
  const float* scale1 = s0.px.mod + size_t(t) * 6 * hs + hs;  // layer 0 = stage 0, lf 0
  check(pf::px_patch_prepare(x_dev, s0.eps, s0.cb, scale1, s0.h32, s0.hb, s0.px.stats,
                             int(shape_.P), row0, rows, hs, eta, update, s0.stream),
        "px_patch_prepare");
}

// One PixArt block over rows [row0, row0+rows) at timestep index t
// (px_oracle.c pxo_layer_forward_mod).
void Engine::layer_forward_px(Stage& s, int lf, int rows, int row0, int t, int code) {
  const ModelShape& m = shape_;
  StageLayer& L = s.layers[size_t(lf)];
  PxStage& px = s.px;
  const int hs = m.hs, w6 = 6 * hs, S = px_steps_;
  const double r = rows, dhs = hs, mlp = m.mlp, P = double(m.P), T = double(m.T);
  const float* modl = px.mod + (size_t(lf) * S + t) * w6;
  const float* gate1 = modl + 2 * hs;
  const float* scale2 = modl + 4 * hs;
  const float* gate2 = modl + 5 * hs;
  const bool last_model_layer = s.first_layer + lf + 1 == m.layers;
  const float* next_scale1 =
      last_model_layer ? nullptr : px.mod + (size_t(lf + 1) * S + t) * w6 + hs;

  // 1. q, k, v = (LN(h)(1 + scale1) + shift1) Wqkv + bqkv; k, v rows in place
  EpiParams qkv;
  qkv.q = s.q;
  qkv.k = L.k;
  qkv.v = L.v;
  qkv.hs = hs;
  qkv.dh = m.dh;
  qkv.dhp = m.dhp;
  qkv.P = int(m.P);
  qkv.stats_in = px.stats;
  qkv.stats_ld = int(m.P);
  qkv.ln_cols = hs;
  qkv.c1 = px.foldq + (size_t(lf) * 2 * S + 2 * t) * 3 * hs;
  qkv.c2 = qkv.c1 + 3 * hs;
  if (lane_wait_) PF_CUDA_CHECK(cudaStreamWaitEvent(s.stream, lane_wait_, 0));
  prof_begin(s, kGemmQKV, 2 * r * dhs * 3 * dhs, 0);
  check(gemm(s.tm_hb, L.tm_wqkv, rows, row0, 3 * hs, hs, Epi::QKV, sk(s, qkv), s.sm_count, s.stream),
        "gemm qkv");
  prof_end(s);
  // 2. self-attention over the full (fresh + stale) K/V buffer
  AttnLaunch a{m.dhp, int(m.P), rows, row0, m.heads, m.dh, hs,
               float(1.0 / std::sqrt(double(m.dh))), s.attn, s.attn_work,
               s.attn_work_floats};
  a.flags = s.attn_flags;
  a.v_sum_col = m.dh < m.dhp;  // V buffers carry the row-sum column
  if (L.has_kv3) {
    a.k3 = &L.tm_k3;
    a.v3 = &L.tm_v3;
  }
  prof_begin(s, kAttention, 4 * r * P * dhs, 0);
  check(attention(s.tm_q, L.tm_k, L.tm_v, a, s.sm_count, s.stream), "attention");
  prof_end(s);
  if (lane_rec_) PF_CUDA_CHECK(cudaEventRecord(lane_rec_, s.stream));
  // 3. h += gate1 (attn Wo + bo); raw bf16 copy for the cross-attention query
  EpiParams res;
  res.out_f32 = s.h32;
  res.out_bf16 = s.hb;
  res.ld = hs;
  res.flag = s.flag;
  res.code = code;
  res.tm_h32 = &s.tm_h32;
  res.tm_hb = &s.tm_hb;
  res.stats_ld = int(m.P);
  EpiParams r1 = res;
  r1.bias = L.bo;
  r1.gate = gate1;
  prof_begin(s, kGemmOut, 2 * r * dhs * dhs, 0);
  check(gemm(s.tm_attn, L.tm_wo, rows, row0, hs, hs, Epi::Residual, sk(s, r1), s.sm_count, s.stream),
        "gemm out-proj");
  prof_end(s);
  // 4. cross-attention query h Wqc + bqc
  EpiParams cq;
  cq.q = s.q;
  cq.hs = hs;
  cq.dh = m.dh;
  cq.dhp = m.dhp;
  cq.P = int(m.P);
  cq.c2 = L.bqc;
  prof_begin(s, kGemmCrossQ, 2 * r * dhs * dhs, 0);
  check(gemm(s.tm_hb, L.tm_wqc, rows, row0, hs, hs, Epi::QKV, sk(s, cq), s.sm_count, s.stream),
        "gemm cross q");
  prof_end(s);
  // 5. cross-attention over the T text tokens
  AttnLaunch ca{m.dhp, m.T, rows, row0, m.heads, m.dh, hs,
                float(1.0 / std::sqrt(double(m.dh))), s.attn, s.attn_work,
                s.attn_work_floats};
  ca.flags = s.attn_flags;
  ca.v_sum_col = m.dh < m.dhp;
  ca.q_stride = int(m.P);
  prof_begin(s, kCrossAttention, 4 * r * T * dhs, 0);
  check(attention(s.tm_q, L.tm_kc, L.tm_vc, ca, s.sm_count, s.stream), "cross attention");
  prof_end(s);
  // 6. h += cross Woc + boc; operand bf16(h (1 + scale2)) + LayerNorm stats
  EpiParams r2 = res;
  r2.bias = L.boc;
  r2.colscale = scale2;
  r2.stats_out = px.stats;
  prof_begin(s, kGemmCrossOut, 2 * r * dhs * dhs, 0);
  check(gemm(s.tm_attn, L.tm_woc, rows, row0, hs, hs, Epi::Residual, sk(s, r2), s.sm_count, s.stream),
        "gemm cross out-proj");
  prof_end(s);
  // 7. z = gelu_tanh((LN(h)(1 + scale2) + shift2) W1 + b1)
  EpiParams ge;
  ge.out_bf16 = s.z;
  ge.ld = m.mlp;
  ge.stats_in = px.stats;
  ge.stats_ld = int(m.P);
  ge.ln_cols = hs;
  ge.c1 = px.foldm + (size_t(lf) * 2 * S + 2 * t) * m.mlp;
  ge.c2 = ge.c1 + m.mlp;
  prof_begin(s, kGemmMlpIn, 2 * r * dhs * mlp, 0);
  check(gemm(s.tm_hb, L.tm_win, rows, row0, m.mlp, hs, Epi::Gelu, sk(s, ge), s.sm_count, s.stream),
        "gemm mlp-in");
  prof_end(s);
  // 8. h += gate2 (z W2 + b2); operand for the next layer's LayerNorm
  EpiParams r3 = res;
  r3.bias = L.b2;
  r3.gate = gate2;
  r3.colscale = next_scale1;
  r3.stats_out = px.stats;
  if (redirect_) {  // last layer of a rank: store straight into the next stage
    r3.out_f32_dst = redirect_->h32;
    r3.out_bf16_dst = redirect_->hb;
    r3.tm_h32_dst = redirect_->tm_h32;
    r3.tm_hb_dst = redirect_->tm_hb;
    if (redirect_->stats) r3.stats_out = redirect_->stats;
  }
  prof_begin(s, kGemmMlpOut, 2 * r * dhs * mlp, 0);
  check(gemm(s.tm_z, L.tm_wout, rows, row0, hs, m.mlp, Epi::Residual, sk(s, r3), s.sm_count, s.stream),
        "gemm mlp-out");
  prof_end(s);
}

}  // namespace pf
