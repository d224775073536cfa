/*
 * pipefusion_b200.h -- C ABI of the B200-native PipeFusion executor.
 *
 * Drop-in boundary for the reference's numerical emulator
 * (`ditsim`, /root/reference/proj/include/ditsim/execute.hpp). Each entry
 * point names the reference interface it replaces. Plain pointers and sizes
 * only: no C++ or torch types cross this boundary.
 *
 * Matrices are fp64 (the reference's Eigen::MatrixXd element type) in either
 * row-major or column-major order (Eigen's default is column-major, numpy's
 * row-major) selected by a `layout` argument.
 *
 * Errors: every function returns a pf_status. PF_VALIDATION corresponds to
 * the reference's ditsim::ValidationError (CLI exit 2), PF_NUMERIC to
 * ditsim::NumericError (CLI exit 1) -- model.hpp:27-36, ditsim.cpp:430-439.
 * The message of the most recent failure is available through
 * pf_last_error() and keeps the reference's wording ("divisible",
 * "non-finite activation at timestep T, layer L", "staleness bound violated").
 *
 * Thread safety: a context may be used by one host thread at a time; distinct
 * contexts are independent. One host thread drives all stages of a context
 * (one CUDA stream per stage; stages may live on distinct GPUs).
 */
#ifndef PIPEFUSION_B200_H_
#define PIPEFUSION_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PF_OK = 0,
  PF_NUMERIC = 1,     /* ditsim::NumericError */
  PF_VALIDATION = 2,  /* ditsim::ValidationError */
  PF_CUDA = 3,        /* CUDA runtime / driver failure (no reference analogue) */
} pf_status;

typedef enum { PF_ROW_MAJOR = 0, PF_COL_MAJOR = 1 } pf_layout;

/* Model shape: ToyDiT (execute.hpp:31-45). mlp_hidden = lround(mlp_ratio*hs)
 * as in build_toy_model (toy_model.cpp:56). seq_len is the K/V buffer height
 * p (WorkloadSpec::seq_len, model.hpp:204). */
typedef struct {
  int layers;
  int hidden_size;
  int heads;
  int mlp_hidden;
  int64_t seq_len;
} pf_model_desc;

/* Staleness accounting of one run: ditsim::StalenessStats (execute.hpp:108-114).
 * fresh_fraction, when non-NULL, receives n_stages x (patches*(steps-warmup))
 * values, stage-major: the buffer fresh fraction after each steady patch
 * completion of that stage, in completion order. */
typedef struct {
  int64_t fresh_patch_reads;
  int64_t stale_patch_reads;
  double* fresh_fraction;
  int64_t fresh_fraction_capacity; /* number of doubles available */
} pf_stats;

typedef struct pf_ctx pf_ctx;

/* Create an executor whose model weights are generated from `seed` exactly as
 * ditsim::build_toy_model(seed, layers, hidden_size, heads, mlp_ratio) does
 * (toy_model.cpp:44-82: one mt19937_64 stream, layers in order
 * W_q, W_k, W_v, W_o, W_mlp_in, W_mlp_out, then condition_bias), without
 * materialising the fp64 model on the host. Layers are split into
 * n_stages contiguous stages, stage d on CUDA device devices[d]
 * (devices may repeat: several stages on one GPU, each with its own stream).
 * Replaces: build_toy_model (execute.hpp:52-53) + the per-worker StageBuffers
 * allocation of run_pipefusion (execute.cpp:38-49). */
pf_status pf_create_toy(uint64_t seed, const pf_model_desc* desc,
                        const int* devices, int n_stages, pf_ctx** out);

/* Arithmetic of the toy block. PF_PRECISION_BF16 (pf_create_toy's) is the
 * product path: bf16 tcgen05 GEMM / attention operands, fp32 accumulation
 * and residual stream. PF_PRECISION_FP32 is a parity mode -- fp32 weights,
 * activations and K/V buffers on CUDA-core kernels, same executor, schedule
 * and K/V update order -- that anchors full-depth runs against the fp64
 * reference where bf16 rounding alone would exceed the tolerance (SURVEY
 * 8(c) T2). Toy block only; no DistriFusion. */
typedef enum { PF_PRECISION_BF16 = 0, PF_PRECISION_FP32 = 1 } pf_precision;
pf_status pf_create_toy_ex(uint64_t seed, const pf_model_desc* desc, int precision,
                           const int* devices, int n_stages, pf_ctx** out);
pf_status pf_create_toy_rank_ex(uint64_t seed, const pf_model_desc* desc, int precision,
                                int rank, int world, int device, pf_ctx** out);
int pf_precision_of(const pf_ctx* ctx);

/* Create an executor from caller-owned fp64 weights: 6 matrices per layer in
 * ToyDiTLayer order (w_q, w_k, w_v, w_o [hs x hs], w_mlp_in [hs x mlp],
 * w_mlp_out [mlp x hs]), i.e. weights[6*l + i], plus condition_bias [hs].
 * Replaces: passing `const ToyDiT&` to run_pipefusion (execute.hpp:124). */
pf_status pf_create(const pf_model_desc* desc, const double* const* weights,
                    const double* condition_bias, pf_layout layout,
                    const int* devices, int n_stages, pf_ctx** out);

/* PixArt-alpha block variant (no reference analogue:
 * the reference's only block is the toy block of toy_model.cpp:145-177).
 * Same executor and schedule as pf_create_toy (run_pipefusion's loop,
 * execute.cpp:167-223) with the block replaced by adaLN-single modulate +
 * LayerNorm, self-attention over the stale/fresh K/V buffer, cross-attention
 * over `text_tokens` text tokens, and a GELU(tanh) MLP. Parameters and text
 * tokens are generated from `seed` as oracle/px_oracle.c (pxo_build) states. */
pf_status pf_create_pixart(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                           const int* devices, int n_stages, pf_ctx** out);

/* SD3-style joint-attention (MMDiT double-stream) block, toy arithmetic per
 * stream (no reference analogue): `text_tokens` text
 * rows with their own weights precede the image rows in every activation and
 * K/V buffer; both streams attend over all joint rows. In PipeFusion the text
 * rows re-enter from the text tokens every step and travel with patch 0, so
 * their K/V rows are always fresh; the image rows follow the reference's
 * patch schedule. Layers [double_layers, layers) are Flux-style single-stream
 * blocks instead (one weight set for all joint rows, attention and MLP in
 * parallel: h += attn(h) Wo + tanh(h Win) Wout). Parameters from `seed` (one
 * mt19937_64 stream seeded with seed ^ "JOINT-DI": per layer the image
 * stream's toy matrices, then for double-stream layers the text stream's,
 * then the condition bias; w_o and w_mlp_out carry an extra 1/sqrt(2 layers)
 * so deep unnormalised stacks stay finite); text tokens from seed ^ "TXT-TOKS". */
pf_status pf_create_joint(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                          int double_layers, const int* devices, int n_stages, pf_ctx** out);

/* Replace the text tokens y [tokens x hidden_size] of a PixArt / joint model. */
pf_status pf_set_text(pf_ctx* ctx, const double* y, int64_t tokens, pf_layout layout);

/* 0 = toy block, 1 = PixArt block, 2 = joint block, -1 = NULL context. */
int pf_block_kind(const pf_ctx* ctx);

/* MMDiT block variants (BASELINE configs 4 and 5; no reference analogue --
 * spec: oracle/mmdit_oracle.py). Layers [0, double_layers) are SD3 / Flux
 * double-stream joint blocks (per-stream adaLN-Zero modulation, LayerNorm,
 * QK RMSNorm, GELU MLP; text and image rows attend over one joint K/V
 * buffer), the rest Flux single-stream parallel blocks; rope != 0 adds the
 * Flux axial RoPE. Every parameter (and the text tokens) is generated on the
 * device from `seed` with the counter-based stream of the spec, so a 12B
 * Flux model needs no host copy. Same executor and schedule as
 * pf_create_toy; text rows as pf_create_joint. */
pf_status pf_create_mmdit(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                          int double_layers, int rope, const int* devices, int n_stages,
                          pf_ctx** out);
pf_status pf_create_mmdit_rank(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                               int double_layers, int rope, int rank, int world, int device,
                               pf_ctx** out);
/* Device bytes of the context's parameters (weights, biases, modulation)
 * and of its K/V buffers, summed over its stages (rank mode: this rank's). */
size_t pf_stage_param_bytes(const pf_ctx* ctx);
size_t pf_stage_kv_bytes(const pf_ctx* ctx);

/* ---- One process per GPU ("rank mode") ----
 * The reference runs one worker thread per stage exchanging PatchMsg values
 * over bounded channels (run_pipefusion_threads, execute.cpp:231-385). In rank
 * mode each process (or each context of one process) owns stage `rank` of
 * `world` on CUDA device `device` (layers [rank*L/world, (rank+1)*L/world)),
 * and the stage-boundary messages -- activations to rank+1, the last stage's
 * eps back to rank 0 -- are written straight into the receiver's landing
 * buffers over peer memory (NVLink / CUDA IPC), with stream-ordered
 * signal/acknowledge counters instead of channels. Setup:
 *   1. pf_create_*_rank on every rank (same seed and shape everywhere);
 *   2. pf_export_peer -> a pf_peer_blob_size() byte blob per rank, exchanged
 *      through any host channel (the Python layer uses torch.distributed);
 *   3. pf_connect_peers(ctx, blob of rank-1, blob of rank+1) (mod world).
 * Then every rank calls pf_run_pipefusion[_device] with the same arguments;
 * only rank 0 reads x_init and writes x_out (NULL is fine elsewhere), and
 * the stats are this rank's stage's share (sum fresh/stale over ranks). */
pf_status pf_create_toy_rank(uint64_t seed, const pf_model_desc* desc, int rank, int world,
                             int device, pf_ctx** out);
pf_status pf_create_pixart_rank(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                                int rank, int world, int device, pf_ctx** out);
pf_status pf_create_joint_rank(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                               int double_layers, int rank, int world, int device,
                               pf_ctx** out);
size_t pf_peer_blob_size(void);
pf_status pf_export_peer(pf_ctx* ctx, void* blob, size_t capacity);
pf_status pf_connect_peers(pf_ctx* ctx, const void* pred_blob, const void* succ_blob);
/* pf_connect_peers plus every other rank's signal page: blobs[r] is rank r's
 * blob (all `world` of them). With it a failing rank closes the run for all
 * ranks, not only its neighbours (see pf_rank_reset). */
pf_status pf_connect_world(pf_ctx* ctx, const void* const* blobs, int world);
/* rank / world of a context (0 / 1 for a single-process context) */
int pf_rank(const pf_ctx* ctx);
int pf_world(const pf_ctx* ctx);
/* The op list rank `rank` executes (rank_plan.h; host only, no GPU):
 * 8 int32 per op {kind, t, patch, row0, rows, msg, overlap, flag}; kinds
 * 0 prepare, 1 compute, 2 send, 3 recv, 4 ack, 5 latent update. Returns the
 * op count (ops may be NULL to query it), or -1 on invalid arguments. */
int64_t pf_rank_plan(int rank, int world, int steps, int patches, int warmup, int64_t seq_len,
                     int32_t* ops, int64_t capacity);

/* Channel close in rank mode (Channel::close, channel.hpp:26-57; close_all on
 * a worker failure, execute.cpp:246-251,345-374). A rank whose run fails
 * (an error while it enqueues its plan) returns that error, after marking
 * the run closed in every connected rank's signal page and playing the rest
 * of its plan's message protocol without compute, so no peer blocks. The
 * peers' pf_run_pipefusion / pf_synchronize then return PF_NUMERIC "channel
 * closed mid-run" (their own non-finite activation, the root cause, is
 * reported first when present); the next run works normally. A rank whose
 * waits see no progress for PF_RANK_TIMEOUT_S seconds (default 600: a peer
 * died or never ran) releases its own and its neighbours' waits and fails
 * the same way; the message counters of the ranks then disagree, so every
 * later run fails until pf_rank_reset has been called on every rank (with a
 * host barrier before and after it). pf_rank_broken: 1 in that state. */
pf_status pf_rank_reset(pf_ctx* ctx);
int pf_rank_broken(const pf_ctx* ctx);

void pf_destroy(pf_ctx* ctx);

/* Message of the last failure on this context (or of the last failed
 * pf_create*, when ctx is NULL). Never NULL. */
const char* pf_last_error(const pf_ctx* ctx);

/* ditsim::run_pipefusion(toy, x_init, steps, workers=n_stages, patches,
 * warmup, eta) -- execute.hpp:124-127, execute.cpp:689-698.
 * x_init / x_out: host [seq_len x hidden_size] fp64 in `layout`. The call is
 * synchronous. stats may be NULL. */
pf_status pf_run_pipefusion(pf_ctx* ctx, const double* x_init, pf_layout layout,
                            int steps, int patches, int warmup, double eta,
                            double* x_out, pf_stats* stats);

/* Same schedule on a device-resident fp32 latent (row-major, on stage 0's
 * device), updated in place; enqueued on `stream` (a cudaStream_t of stage
 * 0's device, 0 = legacy default) and returns without synchronising. Used to
 * time the path with inputs already resident in HBM. Staleness stats are
 * computed on the host while enqueueing. */
pf_status pf_run_pipefusion_device(pf_ctx* ctx, float* x_dev, int steps,
                                   int patches, int warmup, double eta,
                                   void* stream, pf_stats* stats);

/* ditsim::run_distrifusion(toy, x_init, steps, workers, warmup, eta) --
 * execute.hpp:131-133, execute.cpp:431-531 (displaced patch parallelism):
 * `workers` row shards; warmup steps are full-sequence and synchronous,
 * steady steps attend over the worker's own fresh K/V rows and every other
 * shard's rows from the previous step. Needs a single-stage context; the
 * workers share its GPU. CUDA constraint: seq_len / workers divisible by
 * 128 (workers > 1). stats->fresh_fraction receives workers x (steps-warmup)
 * values, worker-major. */
/* Rank mode: capture and instantiate this rank's CUDA graph for exactly these
 * arguments (latent pointer and stream included) without running it; the
 * next pf_run_pipefusion_device with the same arguments replays it. Call it
 * on every rank (then a host barrier) before the first run: instantiating a
 * graph while a peer's replay already waits on this rank can block. Ranks of
 * one process sharing a device never replay graphs (their runs are enqueued
 * op by op). No-op outside rank mode. */
pf_status pf_prepare_pipefusion_device(pf_ctx* ctx, float* x_dev, int steps, int patches,
                                       int warmup, double eta, void* stream);

pf_status pf_run_distrifusion(pf_ctx* ctx, const double* x_init, pf_layout layout, int steps,
                              int workers, int warmup, double eta, double* x_out,
                              pf_stats* stats);
pf_status pf_run_distrifusion_device(pf_ctx* ctx, float* x_dev, int steps, int workers,
                                     int warmup, double eta, void* stream, pf_stats* stats);

/* Wait for work enqueued by pf_run_pipefusion_device and report deferred
 * numeric errors (non-finite activations). */
pf_status pf_synchronize(pf_ctx* ctx, void* stream);

/* ditsim::serial_reference(toy, x_init, steps, eta) -- execute.hpp:102-104,
 * toy_model.cpp:201-214: full-sequence forward each step, no staleness. */
pf_status pf_serial_reference(pf_ctx* ctx, const double* x_init,
                              pf_layout layout, int steps, double eta,
                              double* x_out);

/* ditsim::serial_reference(toy, x_init, steps, eta, keep_trajectory) --
 * execute.hpp:98-104, toy_model.cpp:201-214, with the trajectory:
 * `trajectory` (NULL = keep_trajectory false) receives (steps + 1)
 * matrices of seq_len x hidden_size in `layout`, matrix k at
 * trajectory + k * seq_len * hidden_size: k = 0 the initial latent, k the
 * latent after k update steps (SerialResult::trajectory). Single-process
 * contexts only for a trajectory. */
pf_status pf_serial_reference_ex(pf_ctx* ctx, const double* x_init, pf_layout layout,
                                 int steps, double eta, double* x_out, double* trajectory);

/* ditsim::auto_warmup(toy, x_init, steps, eta, threshold) -- execute.hpp:141-147,
 * toy_model.cpp:230-249: synchronous steps until ||x_k - x_{k-1}|| /
 * ||x_{k-1}|| < threshold; *warmup = k (or steps), *threshold_met = 1/0.
 * The norms are fp64 reductions on the GPU. Single-process contexts. */
pf_status pf_auto_warmup(pf_ctx* ctx, const double* x_init, pf_layout layout, int steps,
                         double eta, double threshold, int* warmup, int* threshold_met);

/* ditsim::divergence(a, b) = ||a - b||_F / ||b||_F -- execute.hpp:136-137,
 * toy_model.cpp:216-228 (fp64 on ctx's stage-0 GPU, or on device 0 when ctx
 * is NULL; the norm is layout-independent). PF_VALIDATION with the
 * reference's messages on a shape mismatch or a zero reference. */
pf_status pf_divergence(pf_ctx* ctx, const double* a, int64_t a_rows, int64_t a_cols,
                        const double* b, int64_t b_rows, int64_t b_cols, double* out);

/* ditsim::toy_layer_forward(layer, heads, h, k_buf, v_buf, row0) --
 * execute.hpp:75-77, toy_model.cpp:169-177, for unit parity: rows
 * [row0, row0+rows) of h pass through global layer `layer` against the given
 * full [seq_len x hs] K/V buffers (updated in place with this block's fresh
 * rows, as the reference does). */
pf_status pf_layer_forward(pf_ctx* ctx, int layer, double* h, int64_t rows,
                           int64_t row0, double* k_buf, double* v_buf,
                           pf_layout layout);

/* pf_layer_forward with the block conditioned on timestep index `timestep`
 * of a `steps`-step run (PixArt block; for the toy block it equals
 * pf_layer_forward). */
pf_status pf_layer_forward_t(pf_ctx* ctx, int layer, int timestep, int steps, double* h,
                             int64_t rows, int64_t row0, double* k_buf, double* v_buf,
                             pf_layout layout);

/* ditsim::make_initial_latent(seed, seq_len, hidden_size) -- execute.hpp:56-57,
 * toy_model.cpp:84-91 (host, bit-exact mt19937_64 stream). out: row-major
 * [seq_len x hidden_size]. */
pf_status pf_make_initial_latent(uint64_t seed, int64_t seq_len, int hidden_size,
                                 double* out);

/* CUDA graphs (default on): the first run of a given (latent buffer,
 * steps, patches, warmup, eta, stream) is captured into a CUDA graph and
 * later runs replay it -- one graph launch per image. Disabled automatically
 * while profiling, on the legacy default stream, and for single-process
 * contexts whose stages span several devices. In rank mode every rank
 * captures its own plan; the signal waits / writes become graph memory-op
 * nodes whose message counts are re-based before each replay. */
pf_status pf_set_graphs(pf_ctx* ctx, int enabled);

/* Per-kernel CUDA-event profile (no reference analogue). When enabled, every
 * kernel of subsequent runs is bracketed by events on its stage stream;
 * pf_kernel_profile() resolves the last run (call after it completed).
 * kind: 0 QKV GEMM, 1 attention, 2 out-proj GEMM, 3 MLP-in GEMM,
 * 4 MLP-out GEMM, 5 sampler/patch kernels; PixArt block only: 6 cross-attention
 * query GEMM, 7 cross-attention, 8 cross-attention out-proj GEMM,
 * 9 conditioning (timestep embedding, adaLN, LayerNorm fold, text K/V).
 * flops/bytes are algorithmic. */
pf_status pf_set_profiling(pf_ctx* ctx, int enabled);
pf_status pf_kernel_profile(pf_ctx* ctx, int kind, double* total_ms,
                            int64_t* launches, double* flops, double* bytes);

/* Measured timeline (the reference's simulate() Timeline, simulate.hpp:32-48,
 * for comparison with its cost model): when enabled, the next runs record
 * one span per (stage, patch, step) compute -- stage 0's includes the
 * sampler / patch split -- and per boundary transfer, with CUDA events (no
 * graph replay while enabled). pf_timeline() resolves the last run into
 * `spans`: 6 doubles per span {stage, stream (0 compute, 1 comm), patch
 * (-1 full), timestep, start_us, dur_us} relative to the run's start on the
 * caller stream; returns the span count (spans may be NULL) or -1. */
pf_status pf_set_timeline(pf_ctx* ctx, int enabled);
int64_t pf_timeline(pf_ctx* ctx, double* spans, int64_t capacity);

/* Number of visible CUDA devices (0 when there is none or no driver). */
int pf_device_count(void);

/* Introspection for tests and benchmarks. */
int pf_stage_count(const pf_ctx* ctx);
int pf_stage_first_layer(const pf_ctx* ctx, int stage);
int pf_stage_layer_count(const pf_ctx* ctx, int stage);
/* Number of kernels the last run enqueued (sum over stages). */
int64_t pf_last_launch_count(const pf_ctx* ctx);
/* Version string of the library build. */
const char* pf_version(void);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* PIPEFUSION_B200_H_ */
