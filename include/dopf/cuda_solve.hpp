// C++ drop-in for the reference solver entry point
//
//     dopf::SolveResult dopf::solve(const DecomposedModel&, const Settings&)
//         proj/include/dopf/admm.hpp:126, proj/src/admm.cpp:172-244
//
// Same types (Settings, SolveResult, TraceRow, SolveStatus, PhaseTimings,
// IterateSnapshot -- paper_2501_08293_b200/csrc/host/admm.hpp mirrors
// admm.hpp:14-122 without Eigen), same error behaviour:
//   std::invalid_argument   rho <= 0, eps_rel <= 0, max_iter < 1 (admm.cpp:173-175)
//   SingularSubsystemError  precompute guard (admm.cpp:53-59, 72-73)
//   std::logic_error        a column without copies (admm.cpp:77-78)
//   std::runtime_error      CUDA / device failures (message from dopf_cuda_last_error)
// iteration_limit is a result status, not an error.
//
// The precompute (admm.cpp:31-88) runs as one batched GPU kernel (bitwise
// equal to the host restatement); the iteration loop runs on the GPU through
// the C ABI of include/dopf_cuda.h. Linking libdopf_cuda.so in place of the
// reference's admm.cpp is the whole integration.
#pragma once

#include <memory>

#include "../../paper_2501_08293_b200/csrc/host/admm.hpp"

struct dopf_cuda_ctx;

namespace dopf {

/// Reference signature: precompute on the host, iterate on CUDA device 0.
SolveResult solve(const DecomposedModel& model, const Settings& settings);

namespace cuda {

/// A device context holding one uploaded model: upload once, solve many times
/// (different settings, warm benchmarks). Not thread-safe; one per thread.
class Solver {
 public:
  explicit Solver(int device = 0);
  ~Solver();
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  /// Precomputes the operators -- on the GPU (batched kernel, bitwise equal
  /// to the host restatement), or on the host with -workers threads when
  /// workers < 0 -- and uploads the device layout.
  void upload(const DecomposedModel& model, int workers = 1);
  /// Runs the loop on the device; record_iterates fills `snapshots` by
  /// re-running the deterministic device loop to every t (test use).
  SolveResult solve(const Settings& settings);
  /// Setup-time tuning of the resident split for the uploaded model
  /// (dopf_cuda_tune_partition): later solves and same-structure uploads use
  /// it; iterates are unchanged. Returns the best measured seconds/iteration.
  double tune_partition(const Settings& settings, int rounds = 8);
  /// The underlying C-ABI context (diagnostics, dopf_cuda_* calls).
  dopf_cuda_ctx* context() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

SolveResult solve(const DecomposedModel& model, const Settings& settings, int device);

/// One model partitioned over CUDA devices 0..gpus-1 of this process: one
/// context per device, one NCCL communicator over all of them
/// (dopf_cuda_comm_init_all), the ranks' device loops on one host thread
/// each (dopf_cuda_solve_part). Iterates, iteration count and status are
/// bitwise those of solve(); a missing NCCL throws std::runtime_error.
SolveResult solve_partitioned(const DecomposedModel& model, const Settings& settings, int gpus);

}  // namespace cuda
}  // namespace dopf
