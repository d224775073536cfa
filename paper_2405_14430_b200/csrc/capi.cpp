// C ABI (include/pipefusion_b200.h) over the PipeFusion runtime.
#include "pipefusion_b200.h"

#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "pipefusion_b200_debug.h"
#include "runtime.h"

struct pf_ctx {
  std::unique_ptr<pf::Engine> engine;
  std::string last_error;
  float* x_scratch = nullptr;   // device latent for the host-buffer entry points
  double* x64_scratch = nullptr;  // the caller's fp64 latent, converted on the GPU
};

namespace {

thread_local std::string g_create_error;

template <class F>
pf_status guarded(std::string* err, F&& f) {
  try {
    f();
    if (err) err->clear();
    return PF_OK;
  } catch (const pf::ValidationError& e) {
    if (err) *err = e.what();
    return PF_VALIDATION;
  } catch (const pf::NumericError& e) {
    if (err) *err = e.what();
    return PF_NUMERIC;
  } catch (const pf::CudaError& e) {
    if (err) *err = e.what();
    return PF_CUDA;
  } catch (const std::bad_alloc&) {
    if (err) *err = "host allocation failed";
    return PF_CUDA;
  } catch (const std::exception& e) {
    if (err) *err = e.what();
    return PF_CUDA;
  }
}

pf::ModelShape shape_of(const pf_model_desc* d) {
  if (!d) throw pf::ValidationError("model description is NULL");
  pf::ModelShape s;
  s.layers = d->layers;
  s.hs = d->hidden_size;
  s.heads = d->heads;
  s.mlp = d->mlp_hidden;
  s.P = d->seq_len;
  return s;
}

std::vector<int> device_list(const int* devices, int n) {
  if (n < 1) throw pf::ValidationError("workers and patches must be >= 1");
  std::vector<int> v(static_cast<size_t>(n), 0);
  if (devices)
    for (int i = 0; i < n; ++i) v[size_t(i)] = devices[i];
  return v;
}

// Uniform in [-1, 1) from the top 53 bits of mt19937_64, matrix filled
// row-major -- the reference's next_uniform / fill_matrix
// (toy_model.cpp:28-40).
double next_uniform(std::mt19937_64& rng) {
  return double(rng() >> 11) * 0x1.0p-52 - 1.0;
}

void fill(std::mt19937_64& rng, std::vector<double>& m, int rows, int cols,
          double scale) {
  m.resize(size_t(rows) * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) m[size_t(r) * cols + c] = next_uniform(rng) * scale;
}

// The host-buffer entry points move the caller's fp64 latent as is (one
// copy each way) and convert layout and precision on the GPU.
void ensure_latent_scratch(pf_ctx* ctx) {
  const pf::ModelShape& m = ctx->engine->shape();
  const size_t n = size_t(m.P) * m.hs;
  if (!ctx->x_scratch && cudaMalloc(&ctx->x_scratch, n * 4) != cudaSuccess)
    throw pf::CudaError("cudaMalloc latent failed");
  if (!ctx->x64_scratch && cudaMalloc(&ctx->x64_scratch, n * 8) != cudaSuccess)
    throw pf::CudaError("cudaMalloc latent failed");
}

void upload_x(pf_ctx* ctx, const double* x, pf_layout layout) {
  const pf::ModelShape& m = ctx->engine->shape();
  const pf::Stage& s0 = ctx->engine->stage(0);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(s0.device);
  struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
  ensure_latent_scratch(ctx);
  const size_t n = size_t(m.P) * m.hs;
  cudaError_t e = cudaMemcpyAsync(ctx->x64_scratch, x, n * 8, cudaMemcpyHostToDevice, s0.stream);
  if (e == cudaSuccess)
    e = pf::latent_from_f64(ctx->x64_scratch, ctx->x_scratch, m.P, m.hs, layout == PF_COL_MAJOR,
                            s0.stream);
  if (e != cudaSuccess) throw pf::CudaError(std::string("latent upload: ") + cudaGetErrorString(e));
}

void download_x(pf_ctx* ctx, double* x, pf_layout layout) {
  const pf::ModelShape& m = ctx->engine->shape();
  const pf::Stage& s0 = ctx->engine->stage(0);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(s0.device);
  struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
  const size_t n = size_t(m.P) * m.hs;
  cudaError_t e = pf::latent_to_f64(ctx->x_scratch, ctx->x64_scratch, m.P, m.hs,
                                    layout == PF_COL_MAJOR, s0.stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(x, ctx->x64_scratch, n * 8, cudaMemcpyDeviceToHost, s0.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s0.stream);
  if (e != cudaSuccess)
    throw pf::CudaError(std::string("latent download: ") + cudaGetErrorString(e));
}

void export_stats(const pf::RunStats& rs, pf_stats* out) {
  if (!out) return;
  out->fresh_patch_reads = rs.fresh;
  out->stale_patch_reads = rs.stale;
  if (out->fresh_fraction) {
    int64_t k = 0;
    for (const auto& v : rs.fresh_fraction)
      for (double f : v)
        if (k < out->fresh_fraction_capacity) out->fresh_fraction[k++] = f;
  }
}

// build_toy_model (toy_model.cpp:44-82) streamed layer by layer into the
// engine (rank-mode engines keep only their own layers).
void load_toy(pf::Engine& eng, uint64_t seed);
// pxo_build (oracle/px_oracle.c) streamed likewise.
void load_pixart(pf::Engine& eng, uint64_t seed, int text_tokens);
// pf_create_joint's parameter stream (include/pipefusion_b200.h).
void load_joint(pf::Engine& eng, uint64_t seed, int text_tokens, int double_layers);

}  // namespace

extern "C" {

pf_status pf_create_toy(uint64_t seed, const pf_model_desc* desc,
                        const int* devices, int n_stages, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    ctx->engine = std::make_unique<pf::Engine>(s, device_list(devices, n_stages));
    load_toy(*ctx->engine, seed);
    *out = ctx.release();
  });
}

pf_status pf_create_toy_rank(uint64_t seed, const pf_model_desc* desc, int rank, int world,
                             int device, pf_ctx** out) {
  return pf_create_toy_rank_ex(seed, desc, PF_PRECISION_BF16, rank, world, device, out);
}

pf_status pf_create_toy_rank_ex(uint64_t seed, const pf_model_desc* desc, int precision,
                                int rank, int world, int device, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.precision = precision;
    ctx->engine = std::make_unique<pf::Engine>(s, device, rank, world);
    load_toy(*ctx->engine, seed);
    *out = ctx.release();
  });
}

pf_status pf_create_toy_ex(uint64_t seed, const pf_model_desc* desc, int precision,
                           const int* devices, int n_stages, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.precision = precision;
    ctx->engine = std::make_unique<pf::Engine>(s, device_list(devices, n_stages));
    load_toy(*ctx->engine, seed);
    *out = ctx.release();
  });
}

int pf_precision_of(const pf_ctx* ctx) {
  return ctx && ctx->engine ? ctx->engine->shape().precision : -1;
}

pf_status pf_create_pixart_rank(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                                int rank, int world, int device, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.block = pf::kBlockPixArt;
    s.T = text_tokens;
    ctx->engine = std::make_unique<pf::Engine>(s, device, rank, world);
    load_pixart(*ctx->engine, seed, text_tokens);
    *out = ctx.release();
  });
}

size_t pf_peer_blob_size(void) { return sizeof(pf::PeerBlob); }

pf_status pf_export_peer(pf_ctx* ctx, void* blob, size_t capacity) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!blob || capacity < sizeof(pf::PeerBlob))
      throw pf::ValidationError("peer blob buffer too small");
    const pf::PeerBlob b = ctx->engine->export_peer();
    std::memcpy(blob, &b, sizeof(b));
  });
}

pf_status pf_connect_peers(pf_ctx* ctx, const void* pred_blob, const void* succ_blob) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!pred_blob || !succ_blob) throw pf::ValidationError("NULL peer blob");
    pf::PeerBlob pred, succ;
    std::memcpy(&pred, pred_blob, sizeof(pred));
    std::memcpy(&succ, succ_blob, sizeof(succ));
    ctx->engine->connect_peers(pred, succ);
  });
}

pf_status pf_connect_world(pf_ctx* ctx, const void* const* blobs, int world) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!blobs || world < 1) throw pf::ValidationError("NULL peer blobs");
    std::vector<pf::PeerBlob> v(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
      if (!blobs[r]) throw pf::ValidationError("NULL peer blob");
      std::memcpy(&v[size_t(r)], blobs[r], sizeof(pf::PeerBlob));
    }
    ctx->engine->connect_world(v);
  });
}

int pf_rank(const pf_ctx* ctx) { return ctx ? ctx->engine->rank() : -1; }
int pf_world(const pf_ctx* ctx) { return ctx ? ctx->engine->world() : 0; }

int64_t pf_rank_plan(int rank, int world, int steps, int patches, int warmup, int64_t seq_len,
                     int32_t* ops, int64_t capacity) {
  if (world < 2 || rank < 0 || rank >= world || steps < 1 || patches < 1 || warmup < 0 ||
      warmup > steps || seq_len < 1 || seq_len % patches != 0)
    return -1;
  const auto plan = pf::build_rank_plan(rank, world, steps, patches, warmup, seq_len);
  if (ops) {
    for (size_t i = 0; i < plan.size() && int64_t(i) < capacity; ++i) {
      const pf::PlanOp& o = plan[i];
      const int32_t v[8] = {o.kind, o.t, o.patch, o.row0, o.rows, o.msg, o.overlap, o.flag};
      std::memcpy(ops + 8 * i, v, sizeof(v));
    }
  }
  return int64_t(plan.size());
}

}  // extern "C"

namespace {

void load_toy(pf::Engine& eng, uint64_t seed) {
    const pf::ModelShape& s = eng.shape();
    std::mt19937_64 rng(seed);
    const double scale = 1.0 / std::sqrt(double(s.hs));
    std::vector<double> w[6];
    for (int l = 0; l < s.layers; ++l) {
      fill(rng, w[0], s.hs, s.hs, scale);
      fill(rng, w[1], s.hs, s.hs, scale);
      fill(rng, w[2], s.hs, s.hs, scale);
      fill(rng, w[3], s.hs, s.hs, scale);
      fill(rng, w[4], s.hs, s.mlp, scale);
      fill(rng, w[5], s.mlp, s.hs, scale);
      pf::HostMatrix hm[6] = {
          {w[0].data(), s.hs, s.hs, false},  {w[1].data(), s.hs, s.hs, false},
          {w[2].data(), s.hs, s.hs, false},  {w[3].data(), s.hs, s.hs, false},
          {w[4].data(), s.hs, s.mlp, false}, {w[5].data(), s.mlp, s.hs, false}};
      eng.load_layer(l, hm);
    }
    std::vector<double> cb;
    fill(rng, cb, 1, s.hs, 1.0);
    eng.load_condition_bias(cb.data());
}

}  // namespace

extern "C" {

pf_status pf_create_pixart(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                           const int* devices, int n_stages, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.block = pf::kBlockPixArt;
    s.T = text_tokens;
    ctx->engine = std::make_unique<pf::Engine>(s, device_list(devices, n_stages));
    load_pixart(*ctx->engine, seed, text_tokens);
    *out = ctx.release();
  });
}

}  // extern "C"

namespace {

void load_pixart(pf::Engine& eng, uint64_t seed, int text_tokens) {
    const pf::ModelShape& s = eng.shape();
    // Parameter stream of the PixArt block variant (oracle/px_oracle.c,
    // pxo_build): one mt19937_64 seeded with seed ^ "PIXART-A", per layer the
    // 17 parameters in PXO_* order, then the timestep-embedder weights and
    // the condition bias; text tokens from seed ^ "TXT-TOKS".
    std::mt19937_64 rng(seed ^ 0x5049584152542d41ULL);
    const int hs = s.hs, mlp = s.mlp;
    const double sh = 1.0 / std::sqrt(double(hs)), sm = 1.0 / std::sqrt(double(mlp));
    struct P { int rows, cols; double scale; };
    const P spec[17] = {{hs, 3 * hs, sh}, {1, 3 * hs, 0.1}, {hs, hs, sh}, {1, hs, 0.1},
                        {hs, hs, sh},     {1, hs, 0.1},     {hs, hs, sh}, {1, hs, 0.1},
                        {hs, hs, sh},     {1, hs, 0.1},     {hs, hs, sh}, {1, hs, 0.1},
                        {hs, mlp, sh},    {1, mlp, 0.1},    {mlp, hs, sm}, {1, hs, 0.1},
                        {6, hs, sh}};
    std::vector<double> w[17];
    for (int l = 0; l < s.layers; ++l) {
      const double* ptrs[17];
      for (int i = 0; i < 17; ++i) {
        fill(rng, w[i], spec[i].rows, spec[i].cols, spec[i].scale);
        ptrs[i] = w[i].data();
      }
      eng.load_layer_px(l, ptrs);
    }
    std::vector<double> g[6], cb;
    fill(rng, g[0], 256, hs, 1.0 / 16.0);
    fill(rng, g[1], 1, hs, 0.1);
    fill(rng, g[2], hs, hs, sh);
    fill(rng, g[3], 1, hs, 0.1);
    fill(rng, g[4], hs, 6 * hs, sh);
    fill(rng, g[5], 1, 6 * hs, 0.1);
    fill(rng, cb, 1, hs, 1.0);
    const double* gp[6] = {g[0].data(), g[1].data(), g[2].data(),
                           g[3].data(), g[4].data(), g[5].data()};
    eng.load_px_globals(gp);
    eng.load_condition_bias(cb.data());
    std::mt19937_64 trng(seed ^ 0x5458542d544f4b53ULL);
    std::vector<double> y;
    fill(trng, y, text_tokens, hs, 1.0);
    eng.set_text(y.data());
}

}  // namespace

extern "C" {

pf_status pf_set_text(pf_ctx* ctx, const double* y, int64_t tokens, pf_layout layout) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    const pf::ModelShape& m = ctx->engine->shape();
    if (m.block != pf::kBlockPixArt && !m.joint_rows())
      throw pf::ValidationError("model has no text conditioning");
    if (!y) throw pf::ValidationError("NULL text pointer");
    if (tokens != m.T) throw pf::ValidationError("text token count does not match the model");
    std::vector<double> rm(size_t(tokens) * m.hs);
    for (int64_t r = 0; r < tokens; ++r)
      for (int c = 0; c < m.hs; ++c)
        rm[size_t(r) * m.hs + c] =
            layout == PF_COL_MAJOR ? y[size_t(c) * tokens + r] : y[size_t(r) * m.hs + c];
    ctx->engine->set_text(rm.data());
  });
}

pf_status pf_create_joint(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                          int double_layers, const int* devices, int n_stages, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.block = pf::kBlockJoint;
    s.T = text_tokens;
    s.double_layers = double_layers;
    ctx->engine = std::make_unique<pf::Engine>(s, device_list(devices, n_stages));
    load_joint(*ctx->engine, seed, text_tokens, double_layers);
    *out = ctx.release();
  });
}

pf_status pf_create_mmdit(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                          int double_layers, int rope, const int* devices, int n_stages,
                          pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.block = pf::kBlockMMDiT;
    s.T = text_tokens;
    s.double_layers = double_layers;
    s.rope = rope ? 1 : 0;
    ctx->engine = std::make_unique<pf::Engine>(s, device_list(devices, n_stages));
    ctx->engine->mm_generate(seed);
    *out = ctx.release();
  });
}

pf_status pf_create_mmdit_rank(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                               int double_layers, int rope, int rank, int world, int device,
                               pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.block = pf::kBlockMMDiT;
    s.T = text_tokens;
    s.double_layers = double_layers;
    s.rope = rope ? 1 : 0;
    ctx->engine = std::make_unique<pf::Engine>(s, device, rank, world);
    ctx->engine->mm_generate(seed);
    *out = ctx.release();
  });
}

size_t pf_stage_param_bytes(const pf_ctx* ctx) {
  return ctx && ctx->engine ? ctx->engine->param_bytes() : 0;
}

size_t pf_stage_kv_bytes(const pf_ctx* ctx) {
  return ctx && ctx->engine ? ctx->engine->kv_bytes() : 0;
}

pf_status pf_create_joint_rank(uint64_t seed, const pf_model_desc* desc, int text_tokens,
                               int double_layers, int rank, int world, int device,
                               pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out) throw pf::ValidationError("output pointer is NULL");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    s.block = pf::kBlockJoint;
    s.T = text_tokens;
    s.double_layers = double_layers;
    ctx->engine = std::make_unique<pf::Engine>(s, device, rank, world);
    load_joint(*ctx->engine, seed, text_tokens, double_layers);
    *out = ctx.release();
  });
}

}  // extern "C"

namespace {

void load_joint(pf::Engine& eng, uint64_t seed, int text_tokens, int double_layers) {
    const pf::ModelShape& s = eng.shape();
    // One mt19937_64 stream seeded with seed ^ "JOINT-DI": per layer the
    // image stream's six toy matrices then (double-stream layers only) the
    // text stream's, in build_toy_model's order and scale
    // (toy_model.cpp:44-82); then the condition bias. Text tokens from
    // seed ^ "TXT-TOKS".
    std::mt19937_64 rng(seed ^ 0x4a4f494e542d4449ULL);
    const double scale = 1.0 / std::sqrt(double(s.hs));
    // residual projections (w_o, w_mlp_out) additionally scaled by
    // 1/sqrt(2 layers) (depth-scaled init) so deep stacks without
    // normalisation (57 Flux-shaped layers) stay finite
    const double rscale = scale / std::sqrt(2.0 * s.layers);
    std::vector<double> w[12];
    for (int l = 0; l < s.layers; ++l) {
      for (int st = 0; st < (l < double_layers ? 2 : 1); ++st) {
        fill(rng, w[6 * st + 0], s.hs, s.hs, scale);
        fill(rng, w[6 * st + 1], s.hs, s.hs, scale);
        fill(rng, w[6 * st + 2], s.hs, s.hs, scale);
        fill(rng, w[6 * st + 3], s.hs, s.hs, rscale);
        fill(rng, w[6 * st + 4], s.hs, s.mlp, scale);
        fill(rng, w[6 * st + 5], s.mlp, s.hs, rscale);
      }
      pf::HostMatrix hm[12];
      for (int i = 0; i < 12; ++i) {
        const int k = i % 6;
        hm[i] = {w[i].data(), k == 5 ? s.mlp : s.hs, k == 4 ? s.mlp : s.hs, false};
      }
      eng.load_layer_joint(l, hm);
    }
    std::vector<double> cb;
    fill(rng, cb, 1, s.hs, 1.0);
    eng.load_condition_bias(cb.data());
    std::mt19937_64 trng(seed ^ 0x5458542d544f4b53ULL);
    std::vector<double> y;
    fill(trng, y, text_tokens, s.hs, 1.0);
    eng.set_text(y.data());
}

}  // namespace

extern "C" {

int pf_block_kind(const pf_ctx* ctx) { return ctx ? ctx->engine->shape().block : -1; }

pf_status pf_create(const pf_model_desc* desc, const double* const* weights,
                    const double* condition_bias, pf_layout layout,
                    const int* devices, int n_stages, pf_ctx** out) {
  if (out) *out = nullptr;
  return guarded(&g_create_error, [&] {
    if (!out || !weights || !condition_bias)
      throw pf::ValidationError("NULL weights / bias / output pointer");
    auto ctx = std::make_unique<pf_ctx>();
    pf::ModelShape s = shape_of(desc);
    ctx->engine = std::make_unique<pf::Engine>(s, device_list(devices, n_stages));
    const bool cm = layout == PF_COL_MAJOR;
    for (int l = 0; l < s.layers; ++l) {
      const double* const* w = weights + 6 * l;
      for (int i = 0; i < 6; ++i)
        if (!w[i]) throw pf::ValidationError("NULL weight matrix");
      pf::HostMatrix hm[6] = {{w[0], s.hs, s.hs, cm},  {w[1], s.hs, s.hs, cm},
                              {w[2], s.hs, s.hs, cm},  {w[3], s.hs, s.hs, cm},
                              {w[4], s.hs, s.mlp, cm}, {w[5], s.mlp, s.hs, cm}};
      ctx->engine->load_layer(l, hm);
    }
    ctx->engine->load_condition_bias(condition_bias);
    *out = ctx.release();
  });
}

void pf_destroy(pf_ctx* ctx) {
  if (!ctx) return;
  if (ctx->x_scratch || ctx->x64_scratch) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->engine->stage(0).device);
    cudaStreamSynchronize(ctx->engine->stage(0).stream);
    if (ctx->x_scratch) cudaFree(ctx->x_scratch);
    if (ctx->x64_scratch) cudaFree(ctx->x64_scratch);
    cudaSetDevice(prev);
  }
  delete ctx;
}

const char* pf_last_error(const pf_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : g_create_error.c_str();
}

pf_status pf_run_pipefusion(pf_ctx* ctx, const double* x_init, pf_layout layout,
                            int steps, int patches, int warmup, double eta,
                            double* x_out, pf_stats* stats) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    const bool holds_latent = ctx->engine->rank() == 0;  // rank mode: only rank 0 samples
    if (!holds_latent) {
      pf::RunStats rs;
      const pf::Stage& s0 = ctx->engine->stage(0);
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(s0.device);
      struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
      ctx->engine->run(nullptr, steps, patches, warmup, float(eta), s0.stream, &rs);
      ctx->engine->finish(s0.stream);
      export_stats(rs, stats);
      return;
    }
    if (!x_init || !x_out) throw pf::ValidationError("NULL latent pointer");
    upload_x(ctx, x_init, layout);
    pf::RunStats rs;
    const pf::Stage& s0 = ctx->engine->stage(0);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s0.device);
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
    ctx->engine->run(ctx->x_scratch, steps, patches, warmup, float(eta), s0.stream, &rs);
    ctx->engine->finish(s0.stream);
    download_x(ctx, x_out, layout);
    export_stats(rs, stats);
  });
}

pf_status pf_run_pipefusion_device(pf_ctx* ctx, float* x_dev, int steps,
                                   int patches, int warmup, double eta,
                                   void* stream, pf_stats* stats) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!x_dev && ctx->engine->rank() == 0) throw pf::ValidationError("NULL latent pointer");
    pf::RunStats rs;
    ctx->engine->run(x_dev, steps, patches, warmup, float(eta),
                     static_cast<cudaStream_t>(stream), &rs);
    export_stats(rs, stats);
  });
}

pf_status pf_prepare_pipefusion_device(pf_ctx* ctx, float* x_dev, int steps, int patches,
                                       int warmup, double eta, void* stream) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    ctx->engine->prepare_graph(x_dev, steps, patches, warmup, float(eta),
                               static_cast<cudaStream_t>(stream));
  });
}

pf_status pf_run_distrifusion(pf_ctx* ctx, const double* x_init, pf_layout layout, int steps,
                              int workers, int warmup, double eta, double* x_out,
                              pf_stats* stats) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!x_init || !x_out) throw pf::ValidationError("NULL latent pointer");
    upload_x(ctx, x_init, layout);
    pf::RunStats rs;
    const pf::Stage& s0 = ctx->engine->stage(0);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s0.device);
    struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};
    ctx->engine->enqueue_distrifusion(ctx->x_scratch, steps, workers, warmup, float(eta),
                                      s0.stream, &rs);
    ctx->engine->finish(s0.stream);
    download_x(ctx, x_out, layout);
    export_stats(rs, stats);
  });
}

pf_status pf_run_distrifusion_device(pf_ctx* ctx, float* x_dev, int steps, int workers,
                                     int warmup, double eta, void* stream, pf_stats* stats) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!x_dev) throw pf::ValidationError("NULL latent pointer");
    pf::RunStats rs;
    ctx->engine->enqueue_distrifusion(x_dev, steps, workers, warmup, float(eta),
                                      static_cast<cudaStream_t>(stream), &rs);
    export_stats(rs, stats);
  });
}

pf_status pf_synchronize(pf_ctx* ctx, void* stream) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error,
                 [&] { ctx->engine->finish(static_cast<cudaStream_t>(stream)); });
}

pf_status pf_serial_reference(pf_ctx* ctx, const double* x_init, pf_layout layout,
                              int steps, double eta, double* x_out) {
  if (!ctx) return PF_VALIDATION;
  if (steps < 1) {
    ctx->last_error = "serial_reference needs steps >= 1";
    return PF_VALIDATION;
  }
  // W = S with one patch: every step is a full-sequence synchronous forward
  // with freshly written K/V, which is serial_reference (toy_model.cpp:201-214).
  return pf_run_pipefusion(ctx, x_init, layout, steps, 1, steps, eta, x_out, nullptr);
}

}  // extern "C"

namespace {

// Device buffer freed on scope exit.
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) {
      cudaGetLastError();
      throw pf::CudaError("cudaMalloc failed");
    }
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

struct DeviceScope {
  int prev = 0;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

// W = S full-sequence steps with the engine's serial tap attached: every step
// is toy_forward on the whole latent with freshly written K/V, i.e.
// serial_reference (toy_model.cpp:201-214). The tap collects what
// keep_trajectory and auto_warmup need on the device.
void serial_tapped(pf_ctx* ctx, const double* x_init, pf_layout layout, int steps, double eta,
                   pf::Engine::SerialTap& tap) {
  pf::Engine& eng = *ctx->engine;
  if (eng.rank_mode())
    throw pf::ValidationError("serial trajectory / auto_warmup need a single-process context");
  upload_x(ctx, x_init, layout);
  const pf::Stage& s0 = eng.stage(0);
  struct Untap { pf::Engine& e; ~Untap() { e.set_serial_tap(nullptr); } } untap{eng};
  eng.set_serial_tap(&tap);
  eng.run(ctx->x_scratch, steps, 1, steps, float(eta), s0.stream, nullptr);
  eng.finish(s0.stream);
}

}  // namespace

extern "C" {

pf_status pf_serial_reference_ex(pf_ctx* ctx, const double* x_init, pf_layout layout,
                                 int steps, double eta, double* x_out, double* trajectory) {
  if (!ctx) return PF_VALIDATION;
  if (!trajectory) return pf_serial_reference(ctx, x_init, layout, steps, eta, x_out);
  return guarded(&ctx->last_error, [&] {
    if (steps < 1) throw pf::ValidationError("serial_reference needs steps >= 1");
    if (!x_init || !x_out) throw pf::ValidationError("NULL latent pointer");
    const pf::ModelShape& m = ctx->engine->shape();
    const size_t n = size_t(m.P) * m.hs;
    DeviceScope dev(ctx->engine->stage(0).device);
    DevBuf traj(size_t(steps + 1) * n * sizeof(float));
    pf::Engine::SerialTap tap;
    tap.traj = traj.as<float>();
    serial_tapped(ctx, x_init, layout, steps, eta, tap);
    const pf::Stage& s0 = ctx->engine->stage(0);
    for (int k = 0; k <= steps; ++k) {
      cudaError_t e = pf::latent_to_f64(tap.traj + size_t(k) * n, ctx->x64_scratch, m.P, m.hs,
                                        layout == PF_COL_MAJOR, s0.stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(trajectory + size_t(k) * n, ctx->x64_scratch, n * 8,
                            cudaMemcpyDeviceToHost, s0.stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s0.stream);
      if (e != cudaSuccess)
        throw pf::CudaError(std::string("trajectory download: ") + cudaGetErrorString(e));
    }
    // trajectory[0] is the caller's latent itself (not its fp32 image)
    std::memcpy(trajectory, x_init, n * sizeof(double));
    std::memcpy(x_out, trajectory + size_t(steps) * n, n * sizeof(double));
  });
}

pf_status pf_auto_warmup(pf_ctx* ctx, const double* x_init, pf_layout layout, int steps,
                         double eta, double threshold, int* warmup, int* threshold_met) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (steps < 1) throw pf::ValidationError("auto_warmup needs steps >= 1");
    if (!x_init || !warmup) throw pf::ValidationError("NULL pointer");
    DeviceScope dev(ctx->engine->stage(0).device);
    DevBuf sums(size_t(2 * steps) * sizeof(double));
    DevBuf work(pf::sumsq_work_bytes());
    pf::Engine::SerialTap tap;
    tap.sums = sums.as<double>();
    tap.work = work.p;
    std::string failure;
    try {
      serial_tapped(ctx, x_init, layout, steps, eta, tap);
    } catch (const pf::NumericError& e) {
      failure = e.what();  // raised below unless an earlier step met the threshold
    }
    std::vector<double> h(size_t(2 * steps));
    if (cudaMemcpy(h.data(), tap.sums, h.size() * sizeof(double), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      throw pf::CudaError("auto_warmup: reading the step norms failed");
    // toy_model.cpp:236-248: relative = ||x_k - x_{k-1}|| / ||x_{k-1}||
    for (int k = 1; k <= steps; ++k) {
      const double xx = h[size_t(2 * (k - 1))], dd = h[size_t(2 * (k - 1) + 1)];
      if (!std::isfinite(xx) || !std::isfinite(dd)) break;  // the step that failed
      const double denom = std::sqrt(xx), change = std::sqrt(dd);
      const double relative =
          denom > 0.0 ? change / denom
                      : (change == 0.0 ? 0.0 : std::numeric_limits<double>::infinity());
      if (relative < threshold) {
        *warmup = k;
        if (threshold_met) *threshold_met = 1;
        return;
      }
    }
    if (!failure.empty()) throw pf::NumericError(failure);
    *warmup = steps;
    if (threshold_met) *threshold_met = 0;
  });
}

int pf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

pf_status pf_divergence(pf_ctx* ctx, const double* a, int64_t a_rows, int64_t a_cols,
                        const double* b, int64_t b_rows, int64_t b_cols, double* out) {
  return guarded(ctx ? &ctx->last_error : &g_create_error, [&] {
    if (a_rows != b_rows || a_cols != b_cols) {
      std::ostringstream os;
      os << "divergence shape mismatch: " << a_rows << "x" << a_cols << " vs " << b_rows << "x"
         << b_cols;
      throw pf::ValidationError(os.str());
    }
    if (!a || !b || !out) throw pf::ValidationError("NULL pointer");
    const size_t n = size_t(a_rows) * size_t(a_cols);
    // ctx's stage-0 GPU and stream; without a context device 0's default stream
    const int device = ctx ? ctx->engine->stage(0).device : 0;
    cudaStream_t stream = ctx ? ctx->engine->stage(0).stream : nullptr;
    DeviceScope dev(device);
    DevBuf da(n * 8), db(n * 8), work(pf::sumsq_work_bytes()), res(2 * sizeof(double));
    cudaError_t e = cudaMemcpyAsync(da.p, a, n * 8, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(db.p, b, n * 8, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess)
      e = pf::sumsq_diff(da.as<double>(), db.as<double>(), n, work.p, res.as<double>(), stream);
    double h[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, res.p, sizeof(h), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) throw pf::CudaError(std::string("divergence: ") + cudaGetErrorString(e));
    // toy_model.cpp:216-228
    const double denom = std::sqrt(h[1]);
    if (denom == 0.0) throw pf::ValidationError("divergence undefined against a zero reference");
    *out = std::sqrt(h[0]) / denom;
  });
}

pf_status pf_rank_reset(pf_ctx* ctx) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] { ctx->engine->rank_reset(); });
}

int pf_rank_broken(const pf_ctx* ctx) { return ctx && ctx->engine->rank_broken() ? 1 : 0; }

int pf_debug_fail_at(pf_ctx* ctx, int op) {
  if (!ctx) return PF_VALIDATION;
  ctx->engine->debug_fail_at(op);
  return PF_OK;
}

int pf_debug_poison_layer(pf_ctx* ctx, int layer) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] { ctx->engine->debug_poison_layer(layer); });
}

pf_status pf_layer_forward(pf_ctx* ctx, int layer, double* h, int64_t rows,
                           int64_t row0, double* k_buf, double* v_buf,
                           pf_layout layout) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!h || !k_buf || !v_buf) throw pf::ValidationError("NULL buffer pointer");
    ctx->engine->layer_forward_host(layer, h, rows, row0, k_buf, v_buf,
                                    layout == PF_COL_MAJOR);
  });
}

pf_status pf_layer_forward_t(pf_ctx* ctx, int layer, int timestep, int steps, double* h,
                             int64_t rows, int64_t row0, double* k_buf, double* v_buf,
                             pf_layout layout) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (!h || !k_buf || !v_buf) throw pf::ValidationError("NULL buffer pointer");
    ctx->engine->layer_forward_host(layer, h, rows, row0, k_buf, v_buf,
                                    layout == PF_COL_MAJOR, timestep, steps);
  });
}

pf_status pf_make_initial_latent(uint64_t seed, int64_t seq_len, int hidden_size,
                                 double* out) {
  return guarded(&g_create_error, [&] {
    if (seq_len < 1 || hidden_size < 1)
      throw pf::ValidationError("latent needs seq_len >= 1 and hidden_size >= 1");
    if (!out) throw pf::ValidationError("NULL output pointer");
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ULL);
    for (int64_t i = 0; i < seq_len * hidden_size; ++i) out[i] = next_uniform(rng);
  });
}

pf_status pf_set_graphs(pf_ctx* ctx, int enabled) {
  if (!ctx) return PF_VALIDATION;
  ctx->engine->set_graphs(enabled != 0);
  return PF_OK;
}

pf_status pf_set_profiling(pf_ctx* ctx, int enabled) {
  if (!ctx) return PF_VALIDATION;
  ctx->engine->set_profiling(enabled != 0);
  return PF_OK;
}

pf_status pf_kernel_profile(pf_ctx* ctx, int kind, double* total_ms, int64_t* launches,
                            double* flops, double* bytes) {
  if (!ctx) return PF_VALIDATION;
  return guarded(&ctx->last_error, [&] {
    if (kind < 0 || kind >= pf::kKindCount) throw pf::ValidationError("kernel kind out of range");
    pf::KernelProfile p = ctx->engine->collect_profile();
    if (total_ms) *total_ms = p.ms[kind];
    if (launches) *launches = p.launches[kind];
    if (flops) *flops = p.flops[kind];
    if (bytes) *bytes = p.bytes[kind];
  });
}

pf_status pf_set_timeline(pf_ctx* ctx, int enabled) {
  if (!ctx) return PF_VALIDATION;
  ctx->engine->set_timeline(enabled != 0);
  return PF_OK;
}

int64_t pf_timeline(pf_ctx* ctx, double* spans, int64_t capacity) {
  if (!ctx) return -1;
  std::vector<pf::TimelineSpan> tl;
  pf_status st = guarded(&ctx->last_error, [&] { tl = ctx->engine->collect_timeline(); });
  if (st != PF_OK) return -1;
  if (spans)
    for (size_t i = 0; i < tl.size() && int64_t(i) < capacity; ++i) {
      const pf::TimelineSpan& e = tl[i];
      const double v[6] = {double(e.stage), double(e.stream), double(e.patch),
                           double(e.timestep), e.start_us, e.dur_us};
      std::memcpy(spans + 6 * i, v, sizeof(v));
    }
  return int64_t(tl.size());
}

int pf_stage_count(const pf_ctx* ctx) { return ctx ? ctx->engine->stage_count() : 0; }
int pf_stage_first_layer(const pf_ctx* ctx, int stage) {
  if (!ctx || stage < 0 || stage >= ctx->engine->stage_count()) return -1;
  return ctx->engine->stage(stage).first_layer;
}
int pf_stage_layer_count(const pf_ctx* ctx, int stage) {
  if (!ctx || stage < 0 || stage >= ctx->engine->stage_count()) return -1;
  return ctx->engine->stage(stage).layer_count;
}
int64_t pf_last_launch_count(const pf_ctx* ctx) {
  return ctx ? ctx->engine->last_launch_count() : 0;
}
const char* pf_version(void) { return "pipefusion_b200 0.1 (sm_100a)"; }

}  // extern "C"
