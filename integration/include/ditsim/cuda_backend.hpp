// Backend::Cuda for the reference's executor: the reference-side binding of
// the B200 library (include/pipefusion_b200.h) a ditsim maintainer adds.
//
// Each function has the signature and error behaviour of the reference
// function it stands in for (namespace ditsim, execute.hpp:98-147):
// ValidationError / NumericError with the reference's messages, results by
// value in the reference's types (Eigen::MatrixXd column-major, fp64).
// integration/backend_cuda.patch routes run_pipefusion / run_distrifusion
// (execute.cpp:689-709) and the CLI's execute command (ditsim.cpp:227-262,
// --backend cuda) here.
#pragma once

#include "ditsim/execute.hpp"

namespace ditsim::cuda {

// run_pipefusion(..., Backend::Cuda): stage d on GPU d % device_count. The
// L % N check (execute.cpp:107-112) is relaxed: stages may own uneven layer
// counts (the result does not depend on the split).
ParallelRunResult run_pipefusion(const ToyDiT& toy, const Matrix& x_init, int steps,
                                 int workers, int patches, int warmup, double eta);

// run_distrifusion(..., Backend::Cuda): the workers' shards on one GPU.
ParallelRunResult run_distrifusion(const ToyDiT& toy, const Matrix& x_init, int steps,
                                   int workers, int warmup, double eta);

// serial_reference / auto_warmup / divergence on the GPU (the CLI's execute
// calls them unconditionally: ditsim.cpp:255-262, toy_model.cpp:216-228).
SerialResult serial_reference(const ToyDiT& toy, const Matrix& x_init, int steps, double eta,
                              bool keep_trajectory = false);
AutoWarmupResult auto_warmup(const ToyDiT& toy, const Matrix& x_init, int steps, double eta,
                             double threshold);
double divergence(const LatentState& a, const LatentState& b);

// Number of CUDA devices (0 without a GPU).
int device_count();

}  // namespace ditsim::cuda
