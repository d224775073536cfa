// Backend::Cuda through the reference's own API (integration test; needs a
// GPU). Built by integration/Makefile against the patched reference
// (backend_cuda.patch) and libpipefusion_b200.so. The reference's CPU
// executor (Backend::Inline, the bit-exact oracle of every backend,
// test_execute.cpp:127-149) is the checker.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cmath>
#include <string>

#include "doctest.h"
#include "ditsim/cuda_backend.hpp"
#include "ditsim/execute.hpp"

using namespace ditsim;

namespace {

struct Case {
  int layers, hidden, heads;
  std::int64_t seq;
  int steps, workers, patches, warmup;
};

void check_against_inline(const Case& c, double tol) {
  const ToyDiT toy = build_toy_model(0, c.layers, c.hidden, c.heads, 4.0);
  const Matrix x = make_initial_latent(0, c.seq, c.hidden);
  const ParallelRunResult ref =
      run_pipefusion(toy, x, c.steps, c.workers, c.patches, c.warmup, 0.1, Backend::Inline);
  const ParallelRunResult gpu =
      run_pipefusion(toy, x, c.steps, c.workers, c.patches, c.warmup, 0.1, Backend::Cuda);
  // T0: staleness accounting and the per-worker schedule series are exact
  CHECK(gpu.stats.fresh_patch_reads == ref.stats.fresh_patch_reads);
  CHECK(gpu.stats.stale_patch_reads == ref.stats.stale_patch_reads);
  CHECK(gpu.stats.per_worker_fresh_fraction == ref.stats.per_worker_fresh_fraction);
  CHECK(gpu.final.timestep == -1);
  // T1: bf16 operands, fp32 accumulation vs the fp64 reference
  const double rel = divergence(gpu.final, ref.final);
  MESSAGE("rel-L2 vs Backend::Inline: " << rel);
  CHECK(rel <= tol);
  // the GPU divergence agrees with the reference's
  CHECK(cuda::divergence(gpu.final, ref.final) == doctest::Approx(rel).epsilon(1e-9));
}

}  // namespace

TEST_CASE("Backend::Cuda matches Backend::Inline on reference_execute.cfg") {
  check_against_inline({4, 32, 4, 64, 20, 4, 4, 1}, 1e-2);
}

TEST_CASE("Backend::Cuda matches Backend::Inline on BASELINE config 1 (S = 4 and 5)") {
  check_against_inline({4, 128, 4, 256, 4, 2, 4, 1}, 1e-2);
  check_against_inline({4, 128, 4, 256, 5, 2, 4, 1}, 1e-2);
}

TEST_CASE("Backend::Cuda relaxes only the layer divisibility") {
  // 4 layers on 3 stages: rejected by the CPU backends, equal to N = 1 on the GPU
  const ToyDiT toy = build_toy_model(1, 4, 64, 4, 4.0);
  const Matrix x = make_initial_latent(1, 128, 64);
  CHECK_THROWS_WITH_AS(run_pipefusion(toy, x, 3, 3, 2, 1, 0.1, Backend::Inline),
                       doctest::Contains("divisible"), ValidationError);
  const ParallelRunResult three = run_pipefusion(toy, x, 3, 3, 2, 1, 0.1, Backend::Cuda);
  const ParallelRunResult one = run_pipefusion(toy, x, 3, 1, 2, 1, 0.1, Backend::Cuda);
  CHECK(divergence(three.final, one.final) == 0.0);
  CHECK_THROWS_WITH_AS(run_pipefusion(toy, x, 3, 2, 3, 1, 0.1, Backend::Cuda),
                       doctest::Contains("divisible"), ValidationError);
  CHECK_THROWS_AS(run_pipefusion(toy, x, 3, 2, 2, 4, 0.1, Backend::Cuda), ValidationError);
}

TEST_CASE("full warmup and a single patch equal the GPU serial reference") {
  const ToyDiT toy = build_toy_model(0, 4, 32, 4, 4.0);
  const Matrix x = make_initial_latent(0, 64, 32);
  const SerialResult serial = cuda::serial_reference(toy, x, 6, 0.1);
  const ParallelRunResult ws = run_pipefusion(toy, x, 6, 4, 4, 6, 0.1, Backend::Cuda);
  const ParallelRunResult m1 = run_pipefusion(toy, x, 6, 2, 1, 1, 0.1, Backend::Cuda);
  CHECK(cuda::divergence(ws.final, serial.final) == 0.0);
  CHECK(cuda::divergence(m1.final, serial.final) == 0.0);
}

TEST_CASE("serial_reference keeps the trajectory") {
  const ToyDiT toy = build_toy_model(2, 4, 32, 4, 4.0);
  const Matrix x = make_initial_latent(2, 64, 32);
  const SerialResult ref = serial_reference(toy, x, 5, 0.1, true);
  const SerialResult gpu = cuda::serial_reference(toy, x, 5, 0.1, true);
  REQUIRE(gpu.trajectory.size() == ref.trajectory.size());
  CHECK((gpu.trajectory[0] - x).cwiseAbs().maxCoeff() == 0.0);
  for (std::size_t k = 1; k < ref.trajectory.size(); ++k) {
    LatentState a{gpu.trajectory[k], 0}, b{ref.trajectory[k], 0};
    CHECK(divergence(a, b) <= 1e-2);
  }
  CHECK((gpu.trajectory.back() - gpu.final.x).cwiseAbs().maxCoeff() == 0.0);
}

TEST_CASE("auto_warmup picks the reference's warmup (test_execute.cpp:259-275)") {
  const ToyDiT toy = build_toy_model(0, 4, 32, 4, 4.0);
  const Matrix x = make_initial_latent(0, 64, 32);
  const AutoWarmupResult ref = auto_warmup(toy, x, 20, 0.1, 0.05);
  const AutoWarmupResult gpu = cuda::auto_warmup(toy, x, 20, 0.1, 0.05);
  CHECK(ref.warmup == 16);
  CHECK(gpu.warmup == ref.warmup);
  CHECK(gpu.threshold_met == ref.threshold_met);
  const AutoWarmupResult never = cuda::auto_warmup(toy, x, 3, 0.1, 1e-12);
  CHECK(never.warmup == 3);
  CHECK_FALSE(never.threshold_met);
}

TEST_CASE("divergence keeps the reference's errors") {
  LatentState a{Matrix(4, 3), 0}, b{Matrix(3, 4), 0}, z{Matrix(4, 3), 0};
  a.x(0, 0) = 1.0;
  CHECK_THROWS_WITH_AS(cuda::divergence(a, b), doctest::Contains("shape mismatch"),
                       ValidationError);
  CHECK_THROWS_WITH_AS(cuda::divergence(a, z), doctest::Contains("zero reference"),
                       ValidationError);
}

TEST_CASE("non-finite activations raise NumericError with the reference's message") {
  const ToyDiT toy = build_toy_model(0, 2, 32, 4, 4.0);
  const Matrix x = make_initial_latent(0, 64, 32);
  CHECK_THROWS_WITH_AS(run_pipefusion(toy, x, 4, 2, 2, 1, 1e300, Backend::Cuda),
                       doctest::Contains("non-finite activation at timestep"), NumericError);
}

TEST_CASE("Backend::Cuda DistriFusion matches the reference's") {
  const ToyDiT toy = build_toy_model(0, 4, 64, 4, 4.0);
  const Matrix x = make_initial_latent(0, 256, 64);
  const ParallelRunResult ref = run_distrifusion(toy, x, 6, 2, 1, 0.1, Backend::Inline);
  const ParallelRunResult gpu = run_distrifusion(toy, x, 6, 2, 1, 0.1, Backend::Cuda);
  CHECK(gpu.stats.fresh_patch_reads == ref.stats.fresh_patch_reads);
  CHECK(gpu.stats.stale_patch_reads == ref.stats.stale_patch_reads);
  CHECK(gpu.stats.per_worker_fresh_fraction == ref.stats.per_worker_fresh_fraction);
  CHECK(divergence(gpu.final, ref.final) <= 1e-2);
}
