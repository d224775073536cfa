// extern "C" bridge over the UNMODIFIED reference sources (TEST
// INFRASTRUCTURE ONLY). Built by oracle/Makefile into oracle/_ref/ from
// /root/reference/proj/src/{toy_model,execute,model,schedule,freshness,
// simulate,costmodel}.cpp
// against oracle/shim/Eigen/Core; it is the reference itself run here, used
// to pin oracle/pf_oracle.c and as the CPU baseline of bench.py.
//
// Matrices cross this boundary row-major (numpy); ditsim::Matrix is
// column-major, so every entry point converts.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "ditsim/execute.hpp"
#include "ditsim/freshness.hpp"
#include "ditsim/schedule.hpp"
#include "ditsim/simulate.hpp"

using namespace ditsim;

namespace {

Matrix from_rm(const double* p, std::int64_t rows, std::int64_t cols) {
  Matrix m(rows, cols);
  for (std::int64_t r = 0; r < rows; ++r)
    for (std::int64_t c = 0; c < cols; ++c) m(r, c) = p[r * cols + c];
  return m;
}

void to_rm(const Matrix& m, double* p) {
  for (Eigen::Index r = 0; r < m.rows(); ++r)
    for (Eigen::Index c = 0; c < m.cols(); ++c) p[r * m.cols() + c] = m(r, c);
}

int report(const std::exception& e, char* err, int cap) {
  if (err && cap > 0) {
    std::strncpy(err, e.what(), size_t(cap) - 1);
    err[cap - 1] = 0;
  }
  if (dynamic_cast<const ValidationError*>(&e)) return 2;
  if (dynamic_cast<const NumericError*>(&e)) return 1;
  return 3;
}

}  // namespace

extern "C" {

void* ref_build(std::uint64_t seed, int layers, int hs, int heads, double mlp_ratio,
                char* err, int cap) {
  try {
    return new ToyDiT(build_toy_model(seed, layers, hs, heads, mlp_ratio));
  } catch (const std::exception& e) {
    report(e, err, cap);
    return nullptr;
  }
}

void ref_free(void* h) { delete static_cast<ToyDiT*>(h); }

int ref_mlp_hidden(void* h) {
  return int(static_cast<ToyDiT*>(h)->layers[0].w_mlp_in.cols());
}

// idx: 0 w_q, 1 w_k, 2 w_v, 3 w_o, 4 w_mlp_in, 5 w_mlp_out
void ref_weight(void* h, int layer, int idx, double* out) {
  const ToyDiTLayer& L = static_cast<ToyDiT*>(h)->layers[size_t(layer)];
  const Matrix* m[6] = {&L.w_q, &L.w_k, &L.w_v, &L.w_o, &L.w_mlp_in, &L.w_mlp_out};
  to_rm(*m[idx], out);
}

void ref_condition_bias(void* h, double* out) {
  const ToyDiT* t = static_cast<ToyDiT*>(h);
  for (Eigen::Index c = 0; c < t->condition_bias.cols(); ++c) out[c] = t->condition_bias(0, c);
}

int ref_latent(std::uint64_t seed, std::int64_t p, int hs, double* out, char* err, int cap) {
  try {
    to_rm(make_initial_latent(seed, p, hs), out);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, cap);
  }
}

int ref_serial(void* h, const double* x, std::int64_t p, int steps, double eta,
               double* out, char* err, int cap) {
  try {
    const ToyDiT& t = *static_cast<ToyDiT*>(h);
    to_rm(serial_reference(t, from_rm(x, p, t.hidden_size), steps, eta).final.x, out);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, cap);
  }
}

// backend: 0 Threads (the CLI default), 1 Inline
int ref_pipefusion(void* h, const double* x, std::int64_t p, int steps, int workers,
                   int patches, int warmup, double eta, int backend, double* out,
                   std::int64_t* fresh, std::int64_t* stale, double* ff,
                   std::int64_t ff_cap, char* err, int cap) {
  try {
    const ToyDiT& t = *static_cast<ToyDiT*>(h);
    ParallelRunResult r =
        run_pipefusion(t, from_rm(x, p, t.hidden_size), steps, workers, patches, warmup,
                       eta, backend == 1 ? Backend::Inline : Backend::Threads);
    to_rm(r.final.x, out);
    if (fresh) *fresh = r.stats.fresh_patch_reads;
    if (stale) *stale = r.stats.stale_patch_reads;
    std::int64_t k = 0;
    if (ff)
      for (const auto& w : r.stats.per_worker_fresh_fraction)
        for (double f : w)
          if (k < ff_cap) ff[k++] = f;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, cap);
  }
}

int ref_distrifusion(void* h, const double* x, std::int64_t p, int steps, int workers,
                     int warmup, double eta, int backend, double* out, char* err, int cap) {
  try {
    const ToyDiT& t = *static_cast<ToyDiT*>(h);
    ParallelRunResult r =
        run_distrifusion(t, from_rm(x, p, t.hidden_size), steps, workers, warmup, eta,
                         backend == 1 ? Backend::Inline : Backend::Threads);
    to_rm(r.final.x, out);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, cap);
  }
}

// run_distrifusion with its StalenessStats (fresh, stale, per-worker series
// of `per` values each, worker-major into ff).
int ref_distrifusion_stats(void* h, const double* x, std::int64_t p, int steps, int workers,
                           int warmup, double eta, int backend, double* out,
                           std::int64_t* fresh, std::int64_t* stale, double* ff,
                           std::int64_t ff_cap, char* err, int cap) {
  try {
    const ToyDiT& t = *static_cast<ToyDiT*>(h);
    ParallelRunResult r =
        run_distrifusion(t, from_rm(x, p, t.hidden_size), steps, workers, warmup, eta,
                         backend == 1 ? Backend::Inline : Backend::Threads);
    to_rm(r.final.x, out);
    *fresh = r.stats.fresh_patch_reads;
    *stale = r.stats.stale_patch_reads;
    std::int64_t k = 0;
    for (const auto& w : r.stats.per_worker_fresh_fraction)
      for (double f : w)
        if (k < ff_cap) ff[k++] = f;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, cap);
  }
}

double ref_divergence(const double* a, const double* b, std::int64_t rows, std::int64_t cols) {
  LatentState sa{from_rm(a, rows, cols), -1};
  LatentState sb{from_rm(b, rows, cols), -1};
  return divergence(sa, sb);
}

int ref_auto_warmup(void* h, const double* x, std::int64_t p, int steps, double eta,
                    double threshold, int* warmup, int* met) {
  const ToyDiT& t = *static_cast<ToyDiT*>(h);
  AutoWarmupResult r = auto_warmup(t, from_rm(x, p, t.hidden_size), steps, eta, threshold);
  *warmup = r.warmup;
  *met = r.threshold_met ? 1 : 0;
  return 0;
}

// toy_layer_forward on rows [row0, row0+rows) against full p-row K/V buffers.
void ref_layer_forward(void* h, int layer, double* hrows, std::int64_t rows,
                       double* kbuf, double* vbuf, std::int64_t p, std::int64_t row0) {
  const ToyDiT& t = *static_cast<ToyDiT*>(h);
  Matrix hm = from_rm(hrows, rows, t.hidden_size);
  Matrix km = from_rm(kbuf, p, t.hidden_size);
  Matrix vm = from_rm(vbuf, p, t.hidden_size);
  toy_layer_forward(t.layers[size_t(layer)], t.heads, hm, km, vm, int(row0));
  to_rm(hm, hrows);
  to_rm(km, kbuf);
  to_rm(vm, vbuf);
}

// Schedule grid: patch/timestep/kind per (slot, device), slot-major.
int ref_schedule(int n, int m, int steps, int warmup, int* patch, int* timestep, int* kind,
                 int cap, int* warmup_slots, int* steady_slots) {
  Schedule s = build_pipefusion_schedule(n, m, steps, warmup);
  *warmup_slots = s.warmup_slots;
  *steady_slots = s.steady_slots;
  const int cells = int(s.micro_steps.size());
  for (int i = 0; i < cells && i < cap; ++i) {
    patch[i] = s.micro_steps[size_t(i)].patch;
    timestep[i] = s.micro_steps[size_t(i)].timestep;
    kind[i] = int(s.micro_steps[size_t(i)].kind);
  }
  return cells;
}

int ref_fresh_series(int n, int m, int steps, int warmup, double* out, int cap) {
  Schedule s = build_pipefusion_schedule(n, m, steps, warmup);
  std::vector<double> v = fresh_area_series(s);
  for (int i = 0; i < int(v.size()) && i < cap; ++i) out[i] = v[size_t(i)];
  return int(v.size());
}

}  // extern "C"


// simulate() of a PipeFusion plan (simulate.cpp:263-342, 398-415) and its
// trace JSON (timeline_to_trace_json, simulate.cpp:607-645). Returns the
// JSON length (copied into out when it fits), or -1/-2 on error.
extern "C" long long ref_simulate_pipefusion(int layers, int hs, int heads, double mlp_ratio,
                                             int bytes_per_element, long long seq_len,
                                             int steps, int warmup, int devices, int patches,
                                             double device_flops, double link_bandwidth,
                                             double link_latency, double per_message_overhead_s,
                                             double* makespan_s, char* out, long long cap,
                                             char* err, int errcap) {
  try {
    ModelSpec model;
    model.layers = layers;
    model.hidden_size = hs;
    model.heads = heads;
    model.mlp_ratio = mlp_ratio;
    model.bytes_per_element = bytes_per_element;
    WorkloadSpec wl;
    wl.seq_len = seq_len;
    wl.diffusion_steps = steps;
    wl.warmup_steps = warmup;
    ClusterSpec cl;
    cl.device_count = devices;
    cl.device_flops = device_flops;
    cl.link_bandwidth = link_bandwidth;
    cl.link_latency = link_latency;
    ComputeModel cm;
    cm.per_message_overhead_s = per_message_overhead_s;
    ParallelPlan plan;
    plan.strategy = Strategy::PipeFusion;
    plan.degree = devices;
    plan.patches = patches;
    const Timeline tl = simulate(plan, model, wl, cl, cm);
    if (makespan_s) *makespan_s = tl.makespan_s;
    const std::string js = timeline_to_trace_json(tl);
    if (out && cap > (long long)js.size()) std::memcpy(out, js.c_str(), js.size() + 1);
    return (long long)js.size();
  } catch (const std::exception& e) {
    return -report(e, err, errcap);
  }
}
