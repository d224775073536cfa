// PipeFusion runtime on B200: per-stage device state, the patch-pipeline
// scheduler and the staleness bookkeeping. Host C++; the hot arithmetic is in
// kernels.cu.
//
// Mirrors the reference executor (/root/reference/proj/src/execute.cpp):
//   StageBuffers            execute.cpp:38-49    -> Stage (+ StageLayer K/V)
//   check_staleness_and_count :51-65             -> Engine::enqueue_run (host)
//   stage_forward_full      :134-147             -> enqueue_run warmup loop
//   stage_forward_patch     :150-165             -> enqueue_run steady loop
//   toy_layer_forward       toy_model.cpp:169-177 -> Engine::layer_forward
//   run_pipefusion_inline   :167-223             -> Engine::enqueue_run
//   Channel<PatchMsg> sends :239-244, 275-281    -> Engine::send_rows (stream
//                                                   ordered copy + event)
// The worker threads of the reference's Threads backend become CUDA streams:
// the host enqueues the inline order once and stage streams overlap on the
// device exactly where the reference's threads would run concurrently.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <tuple>
#include <string>
#include <vector>

#include "kernels.h"
#include "rank_plan.h"

namespace pf {

class ValidationError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class NumericError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct ModelShape {
  int layers = 0;
  int hs = 0;
  int heads = 0;
  int mlp = 0;
  int64_t P = 0;  // sequence length = K/V buffer rows
  int dh = 0;
  int dhp = 0;    // dh rounded up to a multiple of 16
  int block = 0;  // kBlockToy (toy_model.cpp:145-177), kBlockPixArt or kBlockJoint
  int T = 0;      // text tokens (PixArt: cross-attention K/V; joint: rows 0..T-1)
  // joint block: layers [0, double_layers) are double-stream (text weights of
  // their own), the rest single-stream parallel blocks (Flux-style: shared
  // weights over all joint rows, attention and MLP both read the block input)
  int double_layers = 0;
  // kPrecBf16: the product path (bf16 tcgen05 operands, fp32 accumulation);
  // kPrecFp32: parity mode (toy block only): fp32 weights, activations and
  // K/V buffers, CUDA-core kernels (parity_f32.cu), same executor
  int precision = 0;
  // MMDiT block: Flux axial RoPE on q / k (0: none, SD3-style)
  int rope = 0;
  // joint-row offset of image row 0 and rows of the activation / K/V buffers
  // (joint and MMDiT blocks: T text rows first)
  bool joint_rows() const { return block == 2 || block == 3; }
  // blocks whose GEMMs consume LayerNorm statistics of the residual stream
  // (PixArt, MMDiT): the stats travel with the rows across stage boundaries
  bool ln_stats() const { return block == 1 || block == 3; }
  int64_t J() const { return joint_rows() ? T : 0; }
  int64_t rows_total() const { return P + J(); }
};

constexpr int kBlockToy = 0;
constexpr int kBlockPixArt = 1;
constexpr int kPrecBf16 = 0;
constexpr int kPrecFp32 = 1;
// SD3-style joint-attention block (MMDiT double stream, toy arithmetic per
// stream): T text rows precede the P image rows in every activation and K/V
// buffer ("joint rows"); text rows are recomputed with patch 0 of every step.
constexpr int kBlockJoint = 2;
// MMDiT blocks (oracle/mmdit_oracle.py): SD3-style double-stream joint blocks
// (per-stream adaLN-Zero, LayerNorm, QK RMSNorm, GELU MLP) for layers
// [0, double_layers), Flux-style single-stream parallel blocks after them;
// optional Flux RoPE. Joint rows as kBlockJoint; conditioning and LayerNorm
// folding through the PixArt machinery (PxStage, stats [hs/32][P + T]).
constexpr int kBlockMMDiT = 3;
constexpr int kPxFreq = 256;  // sinusoidal timestep features

// Host fp64 source of one layer's weights, in the reference's orientation
// (x . W). `at(r, c)` reads element (r, c).
struct HostMatrix {
  const double* data = nullptr;
  int rows = 0, cols = 0;
  bool col_major = false;
  double at(int r, int c) const {
    return col_major ? data[size_t(c) * rows + r] : data[size_t(r) * cols + c];
  }
};

struct StageLayer {
  bf16* wqkv = nullptr;  // [3hs x hs]  (N x K)
  bf16* wo = nullptr;    // [hs x hs]
  bf16* win = nullptr;   // [mlp x hs]
  bf16* wout = nullptr;  // [hs x mlp]
  bf16* k = nullptr;     // [heads][P][dhp]
  bf16* v = nullptr;     // [heads][P][dhp]
  WeightMaps tm_wqkv, tm_wo, tm_win, tm_wout;
  CUtensorMap tm_k, tm_v;
  // KV boxes of attn3_kv_rows(dhp) rows for the triple-buffered attention
  CUtensorMap tm_k3, tm_v3;
  CUtensorMap tm_k23, tm_v23;  // the same over k2 / v2 (DistriFusion)
  bool has_kv3 = false;
  // DistriFusion: second K/V buffer (the two alternate as previous-step /
  // this-step per denoising step), allocated on first use
  bf16 *k2 = nullptr, *v2 = nullptr;
  CUtensorMap tm_k2, tm_v2;
  // PixArt block (oracle/px_oracle.c): biases fp32, cross-attention weights,
  // per-image cross K/V of the text tokens [heads][T][dhp]
  // joint block: the text stream's weights (same roles as wqkv .. wout)
  bf16 *t_wqkv = nullptr, *t_wo = nullptr, *t_win = nullptr, *t_wout = nullptr;
  WeightMaps tm_t_wqkv, tm_t_wo, tm_t_win, tm_t_wout;
  float *bqkv = nullptr, *bo = nullptr, *bqc = nullptr, *bkvc = nullptr, *boc = nullptr,
        *b1 = nullptr, *b2 = nullptr;
  bf16 *wqc = nullptr, *wkvc = nullptr, *woc = nullptr;  // [hs x hs], [2hs x hs], [hs x hs]
  WeightMaps tm_wqc, tm_wkvc, tm_woc;
  bf16 *kc = nullptr, *vc = nullptr;
  CUtensorMap tm_kc, tm_vc;
  // MMDiT: text-stream biases (double layers), adaLN-Zero modulation
  // weights (bf16 [6hs x hs] double / [3hs x hs] single, per stream) and
  // biases, QK-norm gains [dh] per stream
  float *t_bqkv = nullptr, *t_bo = nullptr, *t_b1 = nullptr, *t_b2 = nullptr;
  bf16 *wmod = nullptr, *t_wmod = nullptr;
  float *bmod = nullptr, *t_bmod = nullptr;
  float *gq = nullptr, *gk = nullptr, *t_gq = nullptr, *t_gk = nullptr;
  // fp32 parity mode: w32 = [Wq | Wk | Wv | Wo] (4 x [hs x hs]), Win [hs x mlp],
  // Wout [mlp x hs], x.W orientation row-major; K/V [P x hs] row-major
  float *w32 = nullptr, *k32 = nullptr, *v32 = nullptr;
};

// PixArt per-stage conditioning state (adaLN-single and the LayerNorm fold).
struct PxStage {
  float *wt1 = nullptr, *bt1 = nullptr;  // [hs x 256], [hs]   (N x K fp32)
  float *wt2 = nullptr, *bt2 = nullptr;  // [hs x hs], [hs]
  float *wt0 = nullptr, *bt0 = nullptr;  // [6hs x hs], [6hs]
  float* sst = nullptr;    // [(layer_count + 1) x 6hs]; last row = next stage's first layer
  bf16* text = nullptr;    // [Tpad x hs] text tokens (rows >= T zero)
  CUtensorMap tm_text;
  float2* stats = nullptr; // [hs/32][P] LayerNorm partial sums of the residual stream
  float* zeros = nullptr;  // [hs]
  // per run, sized for steps_cap timesteps
  int steps_cap = 0;
  float *sinus = nullptr, *e1 = nullptr, *temb = nullptr, *tv = nullptr, *mod = nullptr;
  int fold_rpad = 0;                      // rows of one fold operand block (>= 2S)
  bf16 *fold_aq = nullptr, *fold_am = nullptr;  // [nl][fold_rpad x hs]
  std::vector<CUtensorMap> tm_aq, tm_am;   // per local layer
  float *foldq = nullptr, *foldm = nullptr;  // [nl][2S x 3hs], [nl][2S x mlp]
};

struct Stage {
  int device = 0;
  int first_layer = 0;
  int layer_count = 0;
  int sm_count = 1;
  cudaStream_t stream = nullptr;
  std::vector<StageLayer> layers;
  float* h32 = nullptr;   // [P x hs] residual stream (landing buffer)
  float *q32 = nullptr, *attn32 = nullptr, *z32 = nullptr;  // fp32 parity mode
  bf16* hb = nullptr;     // [P x hs] bf16 operand copy of h32
  bf16* q = nullptr;      // [heads][P][dhp]
  bf16* attn = nullptr;   // [P x hs]
  bf16* z = nullptr;      // [P x mlp]
  float* attn_work = nullptr;
  size_t attn_work_floats = 0;
  int* attn_flags = nullptr;  // [sm_count] stream-K merge flags (zero between launches)
  int* flag = nullptr;    // first non-finite (ordinal), INT_MAX if none
  float* splitk_ws = nullptr;    // split-K partial tiles (skinny GEMMs)
  size_t splitk_ws_floats = 0;
  int* splitk_counters = nullptr;
  int splitk_counter_cap = 0;
  CUtensorMap tm_hb, tm_attn, tm_z, tm_q;
  CUtensorMap tm_hb_half;  // 64-row boxes over hb (A multicast across cluster pairs)
  CUtensorMap tm_h32;  // fp32 residual stream, box 32 x 128 (TMA epilogue)
  // joint rows: maps over the T text rows only (clipped TMA residual stores of
  // the text stream's partial last row tile)
  CUtensorMap tm_h32_txt, tm_hb_txt;
  cudaEvent_t ev_fwd = nullptr;  // "rows sent to stage d+1"
  // Extra patch lanes (small patches): own stream and the per-launch scratch
  // concurrent patches must not share. The fields above always hold the
  // active lane's resources: use_lane() swaps extra[k] in (lane 0's live in
  // extra[lane] meanwhile).
  static constexpr int kMaxLanes = 8;
  struct Lane {
    cudaStream_t stream = nullptr;
    float* attn_work = nullptr;
    int* attn_flags = nullptr;
    float* splitk_ws = nullptr;
    int* splitk_counters = nullptr;
  } extra[kMaxLanes];
  int lane = 0;
  int lanes_alloc = 1;
  std::vector<cudaEvent_t> ev_attn[kMaxLanes];  // per local layer: the lane's last attention
  cudaEvent_t ev_lane[kMaxLanes] = {};          // lane fork / join
  // stage 0 only
  float* x = nullptr;    // [P x hs] latent
  float* eps = nullptr;  // [P x hs] noise landing buffer (== last stage h32 when N == 1)
  bool eps_owned = false;
  float* cb = nullptr;   // [hs] condition bias
  float* zeros = nullptr;  // [hs]
  float* text = nullptr;   // joint block: [T x hs] text tokens (fp32), stage 0
  std::vector<cudaEvent_t> ev_eps;  // per patch, recorded by the last stage
  PxStage px;
  // MMDiT: modulation weights of the global layer after this stage's last
  // (its scale1 shapes the bf16 operand this stage hands over); per stream
  bf16 *mm_next_wmod[2] = {nullptr, nullptr};
  float *mm_next_bmod[2] = {nullptr, nullptr};
  float* mm_bcond = nullptr;  // bt2 + y_pooled (MMDiT conditioning bias)
};

// Kernel kinds for the optional per-launch CUDA-event profile.
enum KernelKind : int {
  kGemmQKV = 0, kAttention = 1, kGemmOut = 2, kGemmMlpIn = 3, kGemmMlpOut = 4,
  kSampler = 5, kGemmCrossQ = 6, kCrossAttention = 7, kGemmCrossOut = 8, kPxCond = 9,
  kKindCount = 10
};

struct KernelProfile {
  double ms[kKindCount] = {0};        // summed device time (CUDA events)
  int64_t launches[kKindCount] = {0};
  double flops[kKindCount] = {0};     // algorithmic FLOPs (SURVEY 8d model)
  double bytes[kKindCount] = {0};     // algorithmic HBM bytes (sampler)
};

// One measured span of a run (the reference's TimelineEvent,
// simulate.hpp:32-42): a stage's compute for one (patch, step) -- stage 0's
// span includes the sampler / patch split -- or a boundary transfer.
struct TimelineSpan {
  int stage = 0;
  int stream = 0;  // 0 compute, 1 comm
  int patch = -1;  // -1: full sequence (warmup)
  int timestep = -1;
  double start_us = 0.0, dur_us = 0.0;
};

struct RunStats {
  int64_t fresh = 0;
  int64_t stale = 0;
  std::vector<std::vector<double>> fresh_fraction;  // per stage
};

// Peer-memory endpoint of one rank (one process per GPU): IPC handles and,
// for ranks living in the same process, raw pointers of the buffers its
// predecessor writes into (landing rows, rank 0's eps) and of its signal
// page (sig[0]: messages delivered to it, sig[1]: acknowledgements from its
// successor). Exchanged as an opaque blob through the caller's host channel.
struct PeerBlob {
  uint32_t magic = 0x50465042;  // "PFPB"
  int32_t rank = 0, world = 1, device = 0, block = 0;
  int64_t pid = 0;
  // host identity (hostname + boot id) and a random per-process nonce: PIDs
  // alone collide across PID namespaces / containers / hosts
  uint64_t host_id = 0, nonce = 0;
  cudaIpcMemHandle_t h_h32, h_hb, h_stats, h_eps, h_sig;
  uint64_t p_h32 = 0, p_hb = 0, p_stats = 0, p_eps = 0, p_sig = 0;
};

class Engine {
 public:
  Engine(const ModelShape& shape, const std::vector<int>& devices);
  // Rank mode: one process (or context) per stage. This engine holds stage
  // `rank` of `world` on `device`; stage boundaries are crossed over peer
  // memory once connect_peers() has been called on every rank.
  Engine(const ModelShape& shape, int device, int rank, int world);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // Upload one layer (fp64 host matrices in the reference orientation).
  void load_layer(int layer, const HostMatrix (&w)[6]);
  void load_condition_bias(const double* cb);
  // PixArt block: one layer's 17 parameters in oracle/px_oracle.c order
  // (PXO_WQKV .. PXO_SST, x.W orientation [in x out], fp64 row-major).
  void load_layer_px(int layer, const double* const* params);
  // t_embedder / t_block weights (x.W orientation): wt1 [256 x hs], bt1,
  // wt2 [hs x hs], bt2, wt0 [hs x 6hs], bt0.
  void load_px_globals(const double* const* g);
  // MMDiT: generate every parameter of this engine's stages on the device
  // from `seed` (oracle/mmdit_oracle.py MMDiT), text tokens included
  void mm_generate(uint64_t seed);
  // Text tokens y [T x hs] (row-major fp64) used by every stage's cross-attention.
  void set_text(const double* y);
  // Joint block: one layer's 12 matrices, image stream (w_q, w_k, w_v, w_o,
  // w_mlp_in, w_mlp_out) then text stream, x.W orientation as load_layer.
  void load_layer_joint(int layer, const HostMatrix (&w)[12]);

  // ditsim::run_distrifusion (execute.hpp:131-133, execute.cpp:431-531) on
  // a single-stage engine: `workers` row shards, each attending over its own
  // fresh K/V rows and every other shard's rows from the previous step
  // (warmup steps: all fresh, layer-lockstep). The workers of a step are
  // independent; here they run back to back on the stage's GPU.
  void enqueue_distrifusion(float* x_dev, int steps, int workers, int warmup, float eta,
                            cudaStream_t caller, RunStats* stats);

  // Rank mode.
  int rank() const { return rank_; }
  int world() const { return world_; }
  bool rank_mode() const { return world_ > 1; }
  bool owns_layer(int layer) const { return stage_of_layer(layer) >= 0; }
  PeerBlob export_peer();
  void connect_peers(const PeerBlob& pred, const PeerBlob& succ);
  // skip_all: the message protocol only, no compute (a rank that failed
  // before anything of its plan was enqueued, e.g. during graph capture)
  void enqueue_rank_run(float* x_dev, int steps, int patches, int warmup, float eta,
                        cudaStream_t caller, RunStats* stats, bool skip_all = false);
  // Channel close (the reference's Channel::close, channel.hpp:26-57, and
  // close_all on a worker failure, execute.cpp:246-251,345-374). A rank
  // whose run throws sets the abort word (the run's epoch) in the signal page
  // of every rank it knows (all ranks after connect_world, else its two
  // neighbours) and finishes its plan in skip mode (message protocol only),
  // so no peer blocks; the peers' finish() raises "channel closed mid-run",
  // and the next run starts from consistent counters.
  void close_channels();
  // Watchdog (finish() saw no progress for rank_timeout_s_, e.g. a peer
  // died): release this rank's own and its neighbours' waits with values
  // past every message of the run. The counters no longer agree afterwards:
  // the pipeline stays closed until rank_reset() on every rank.
  void watchdog_abort();
  void rank_reset();
  // Also open every rank's signal page (blobs[r] of rank r) so a failing
  // rank can close the run for all of them; connects the neighbours too.
  void connect_world(const std::vector<PeerBlob>& blobs);
  bool rank_broken() const { return broken_; }
  // test hook: throw from the plan loop when reaching op `op` (-1: off)
  void debug_fail_at(int op) { fail_at_op_ = op; }
  // test hook: make global layer `layer`'s out-projection produce NaN
  void debug_poison_layer(int layer);

  const ModelShape& shape() const { return shape_; }
  int stage_count() const { return int(stages_.size()); }
  const Stage& stage(int d) const { return stages_[size_t(d)]; }
  int64_t last_launch_count() const { return launches_; }

  // Enqueue a full PipeFusion run on a device latent (stage 0's device).
  void enqueue_run(float* x_dev, int steps, int patches, int warmup, float eta,
                   cudaStream_t caller, RunStats* stats);
  // Same as enqueue_run, replayed from a CUDA graph captured on first use
  // for this (latent, schedule, stream): one launch per image instead of
  // thousands. Falls back to enqueue_run when profiling, on the legacy
  // default stream, or when stages span several devices.
  void run(float* x_dev, int steps, int patches, int warmup, float eta,
           cudaStream_t caller, RunStats* stats);
  void set_graphs(bool on) { graphs_enabled_ = on; }
  // Rank mode: capture and instantiate this rank's graph for the run's
  // arguments without launching it (ranks sharing a device in one process
  // never use graphs, see connect_peers).
  void prepare_graph(float* x_dev, int steps, int patches, int warmup, float eta,
                     cudaStream_t caller) {
    if (rank_mode()) run_rank(x_dev, steps, patches, warmup, eta, caller, nullptr, false);
  }
  // serial_reference(keep_trajectory) / auto_warmup taps on the warmup
  // (full-sequence) steps of the next runs (single-process engines, no graph
  // replay while set): per warmup step w, sums[2w], sums[2w+1] = ||x||^2,
  // ||eta eps||^2 before the update (device fp64), and traj + (w+1) n = x
  // after it (traj = x at the start); n = seq_len * hidden_size.
  struct SerialTap {
    double* sums = nullptr;
    float* traj = nullptr;
    void* work = nullptr;  // sumsq_work_bytes()
  };
  void set_serial_tap(const SerialTap* t) { tap_ = t; }
  // Synchronise every stage and raise deferred numeric errors.
  void finish(cudaStream_t caller);

  // Single layer (unit parity), on stage owning `layer`.
  // PixArt: the block's conditioning is that of timestep index t of a
  // `steps`-step run (ignored for the toy block).
  void layer_forward_host(int layer, double* h, int64_t rows, int64_t row0,
                          double* k_buf, double* v_buf, bool col_major, int t = 0,
                          int steps = 1);

  float* stage0_x() { return stages_[0].x; }

  // Bracket every kernel of the next runs with CUDA events (stage streams).
  void set_profiling(bool on) { profiling_ = on; }
  // Record per-(stage, patch, step) compute and transfer spans of the next
  // runs (single-device engines and rank mode; disables graph replay).
  void set_timeline(bool on) { timeline_on_ = on; }
  std::vector<TimelineSpan> collect_timeline();
  // Resolve the events of the last profiled run (after finish()).
  KernelProfile collect_profile();

 private:
  void alloc_stage(Stage& s, int first, int count, bool is_first);
  void free_stage(Stage& s);
  // K/V source of a layer forward: where the QKV epilogue writes this
  // block's K/V rows, and which buffers the attention reads (DistriFusion).
  struct KvView {
    bf16 *k = nullptr, *v = nullptr;
    const CUtensorMap *tm_k = nullptr, *tm_v = nullptr, *tm_k2 = nullptr, *tm_v2 = nullptr;
    int fresh_lo = 0, fresh_hi = 0;
    // fresh rows not on 128-row KV blocks: the attention reads a merged copy
    // (previous step's buffers prev_k / prev_v with this worker's fresh rows
    // from k / v) in the scratch sk / sv
    const bf16 *prev_k = nullptr, *prev_v = nullptr;
    bf16 *sk = nullptr, *sv = nullptr;
    const CUtensorMap *tm_sk = nullptr, *tm_sv = nullptr;
    // whole-buffer attention (every row fresh): 112-row-box maps of that
    // buffer, so the same kernel as the serial path runs (bitwise equality)
    const CUtensorMap *k3 = nullptr, *v3 = nullptr;
  };
  // DistriFusion merge scratch per worker (allocated when shards are not
  // multiples of 128 rows)
  std::vector<bf16*> df_sk_, df_sv_;
  std::vector<CUtensorMap> df_tm_sk_, df_tm_sv_;
  void layer_forward(Stage& s, int lf, int rows, int row0, int code,
                     const KvView* kv = nullptr);
  void layer_forward_f32(Stage& s, int lf, int rows, int row0, int code);
  // MMDiT (runtime_mmdit.cpp)
  void mm_alloc_stage(Stage& s);
  void mm_free_stage(Stage& s);
  void mm_alloc_run(Stage& s, int steps);
  void mm_conditioning(Stage& s, int steps);
  void mm_patch_prepare(Stage& s0, float* x_dev, bool update, int row0, int rows, int t,
                        float eta);
  void mm_text_prepare(Stage& s0, int t);
  void layer_forward_mm(Stage& s, int lf, int rows, int row0, int t, int code);
  bool mm_double(int global_layer) const { return global_layer < shape_.double_layers; }

 public:
  // device bytes of this engine's parameters / K/V buffers (all its stages)
  size_t param_bytes() const;
  size_t kv_bytes() const;

 private:
  void layer_forward_px(Stage& s, int lf, int rows, int row0, int t, int code);
  void layer_forward_joint(Stage& s, int lf, int rows, int row0, int code);
  void layer_forward_single(Stage& s, int lf, int rows, int row0, int code);
  void px_conditioning(Stage& s, int steps);
  void px_alloc_run(Stage& s, int steps);
  void drop_graphs();
  void px_patch_prepare(float* x_dev, bool update, int row0, int rows, int t, float eta);
  void send_rows(int from, int row0, int rows, int patch, int t);
  void prepare_run(int patches, int steps);
  void validate_run(int steps, int patches, int warmup) const;
  // rank mode
  int rank_ = 0, world_ = 1;
  cudaStream_t send_stream_ = nullptr;
  uint32_t* sig_ = nullptr;        // local signal page (device): [0] delivered, [1] acked
  float* succ_h32_ = nullptr;      // successor's landing buffers (peer memory)
  bf16* succ_hb_ = nullptr;
  float2* succ_stats_ = nullptr;
  float* succ_eps_ = nullptr;      // last rank: rank 0's eps buffer
  uint32_t* succ_sig_ = nullptr;   // successor's signal page
  uint32_t* pred_sig_ = nullptr;   // predecessor's signal page
  std::vector<uint32_t*> world_sig_;  // every other rank's signal page (connect_world)
  std::vector<void*> ipc_opened_;
  bool connected_ = false;
  // Fused stage-boundary send: the stage's last MLP-out GEMM stores its rows
  // straight into the successor's landing buffers (peer memory) instead of a
  // copy after it. Set around that one layer_forward* call.
  struct OutRedirect {
    float* h32 = nullptr;
    bf16* hb = nullptr;
    float2* stats = nullptr;
    const CUtensorMap* tm_h32 = nullptr;
    const CUtensorMap* tm_hb = nullptr;
  };
  const OutRedirect* redirect_ = nullptr;
  OutRedirect peer_out_;
  CUtensorMap tm_peer_h32_, tm_peer_hb_;
  uint32_t msgs_in_base_ = 0, msgs_out_base_ = 0;
  cudaEvent_t ev_compute_ = nullptr;
  std::vector<cudaEvent_t> ev_sent_;  // per patch: last send of its rows finished
  // rank mode with lanes: last signal write per counter (acks to the
  // predecessor, message counts to the successor), each chain in plan order
  cudaEvent_t ev_write_[2] = {nullptr, nullptr};
  cudaStream_t abort_stream_ = nullptr;
  uint32_t run_epoch_ = 0;     // rank runs started (same on every rank)
  uint32_t run_base_ = 0;      // message base of the run in flight
  bool broken_ = false;        // watchdog abort: counters no longer agree
  int fail_at_op_ = -1;
  double rank_timeout_s_ = [] {
    const char* e = std::getenv("PF_RANK_TIMEOUT_S");
    const double v = e ? std::atof(e) : 600.0;
    return v > 0 ? v : 600.0;
  }();
  // rank mode: enqueue or replay the captured graph of this rank's plan
  void run_rank(float* x_dev, int steps, int patches, int warmup, float eta,
                cudaStream_t caller, RunStats* stats, bool launch = true);
  bool shared_device_peer_ = false;  // a neighbour rank in this process on this device
  void prepare_rank_run(int patches, int steps);
  // wait for a stream; in rank mode with a watchdog that aborts the pipeline
  // when no progress is made for rank_timeout_s_
  void wait_stream(cudaStream_t st);
  int px_steps_ = 0;  // S of the enqueued run (layout of the per-run PixArt buffers)
  cudaEvent_t ev_start_ = nullptr;
  // recorded on the caller stream after every graph replay: sync_own() waits
  // for this engine's work only (ranks sharing a device must not wait for
  // each other's device-wide work, which may wait on them in turn)
  cudaEvent_t ev_replayed_ = nullptr;
  void sync_own();
  int stage_of_layer(int layer) const;

  struct ProfRec {
    int kind;
    int stage;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  void prof_begin(Stage& s, int kind, double flops, double bytes);
  void prof_end(Stage& s);
  cudaEvent_t prof_event(int stage);

  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    RunStats stats;
    int64_t launches = 0;
    std::vector<std::pair<int, int>> codes;
    // rank mode: the captured graph's stream memory operations (signal
    // waits / writes). Their values are message counts relative to the
    // run's base, patched before a replay whose base differs.
    cudaGraph_t graph = nullptr;
    struct MemOpNode {
      void* node = nullptr;  // CUgraphNode of `graph`
      std::vector<uint32_t> delta;  // value - base, per op of the batch
    };
    std::vector<MemOpNode> memops;
    uint32_t base = 0;  // base the exec's values currently hold
  };
  using GraphKey = std::tuple<float*, int, int, int, uint32_t, cudaStream_t>;
  std::map<GraphKey, GraphEntry> graphs_;
  bool graphs_enabled_ = true;
  const SerialTap* tap_ = nullptr;

  bool profiling_ = false;
  bool timeline_on_ = false;
  struct TlRec {
    int stage, stream, patch, t;
    cudaEvent_t a, b;
  };
  std::vector<TlRec> tl_;
  cudaEvent_t tl_origin_ = nullptr;
  void tl_begin(int stage, int stream, int patch, int t, cudaStream_t st);
  void tl_end(cudaStream_t st);
  std::vector<ProfRec> prof_;
  std::vector<std::vector<cudaEvent_t>> prof_pool_;  // per stage
  std::vector<size_t> prof_used_;

  ModelShape shape_;
  std::vector<Stage> stages_;
  int64_t launches_ = 0;
  // multi-lane patch schedule (single stage, toy block, M >= 2): patch j runs
  // on lane j % lanes; layer_forward waits lane_wait_ before its QKV GEMM and
  // records lane_rec_ after its attention (see enqueue_run)
  cudaEvent_t lane_wait_ = nullptr;
  cudaEvent_t lane_rec_ = nullptr;
  // lanes per stage for M >= 2 (PF_LANES=1..8, default 8: with CTA-pair tiles
  // for small patches, C2 M = 8 0.1738 / 0.1738 s vs 0.1797 / 0.1800 s with 4
  // lanes in the same call; M = 4 unchanged; PF_ONE_LANE=1 is PF_LANES=1)
  int lanes_ = [] {
    const char* one = std::getenv("PF_ONE_LANE");
    if (one && one[0] == '1') return 1;
    const char* e = std::getenv("PF_LANES");
    const int v = e ? std::atoi(e) : 8;
    return v < 1 ? 1 : (v > Stage::kMaxLanes ? Stage::kMaxLanes : v);
  }();
  void use_lane(Stage& s, int lane);
  void alloc_lanes(Stage& s, int lanes);
  int lanes_for(int patches) const {
    if (patches < 2 || stages_.size() != 1 || profiling_ || timeline_on_ || rank_mode() ||
        shape_.precision != kPrecBf16)
      return 1;
    return lanes_ < patches ? lanes_ : patches;
  }
  // L2 prefetch of the next kernels' weights from the attention kernel.
  // Opt-in (PF_WEIGHT_PREFETCH=1): measured at C2 M = 8 the GEMMs were not
  // weight-latency bound (unchanged) and the attention lost 3.5 us per launch.
  bool prefetch_weights_ = [] {
    const char* e = std::getenv("PF_WEIGHT_PREFETCH");
    return e && e[0] == '1';
  }();
  // ordinal -> (timestep, global layer) for non-finite reporting
  std::vector<std::pair<int, int>> codes_;
};

void validate_shape(const ModelShape& s);

}  // namespace pf
