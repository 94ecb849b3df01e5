// Host side of the ADMM hot path: settings, one-time precompute, result types
// and writers. Mirrors reference dopf/admm.hpp:14-133; the iteration itself
// (global/local/dual/residuals, admm.cpp:118-244) runs on the GPU through
// dopf::cuda::solve (cuda_solve.hpp) and the C ABI in include/dopf_cuda.h.
#pragma once

#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

#include "decompose.hpp"
#include "parallel.hpp"

namespace dopf {

struct Settings {
  double rho = 100.0;
  double eps_rel = 1e-3;
  int max_iter = 50000;
  int workers = 1;
  bool record_iterates = false;
};

/// P = I - A'(AA')^{-1}A (row-major n_s x n_s) and v = A'(AA')^{-1}b.
struct PrecomputedSub {
  Dense kernel_projector;
  std::vector<double> min_norm_solution;
};

struct Precomputed {
  std::vector<PrecomputedSub> subs;
  std::vector<double> inv_copy_counts;  // n
  // consensus scatter as CSR by global column: copies of column i are
  // copy_index[col_ptr[i] .. col_ptr[i+1]) holding flat z indices
  // (z_offsets[s] + j) in ascending s (reference admm.cpp:81-86)
  std::vector<int> col_ptr;
  std::vector<int> copy_index;
};

class SingularSubsystemError : public std::runtime_error {
 public:
  explicit SingularSubsystemError(std::string subsystem_id);
  const std::string& subsystem_id() const { return id_; }

 private:
  std::string id_;
};

/// Gram, Cholesky (with the reference's (d_min/d_max)^2 < 1e-14 guard),
/// projector and minimum-norm shift per subsystem; inverse copy counts and
/// the CSR scatter (reference admm.cpp:31-88).
Precomputed precompute(const DecomposedModel& model, WorkerPool* pool = nullptr);

/// The same Precomputed from operators computed elsewhere (the batched GPU
/// precompute): flat P (row-major n_s x n_s, subsystem order) and v (N_z).
Precomputed precompute_from(const DecomposedModel& model, const double* P, const double* v);

/// Initial iterate rule (reference admm.cpp:92-116): 1.0 for squared-voltage
/// columns, the bound midpoint when both bounds are finite, else 0.
double initial_value(const DecomposedModel& model, int global_col);

struct TraceRow {
  int t = 0;
  double pres = 0, dres = 0, eps_prim = 0, eps_dual = 0, objective = 0;
};

struct Residuals {
  double pres = 0, dres = 0, eps_prim = 0, eps_dual = 0;
  bool satisfied() const { return pres <= eps_prim && dres <= eps_dual; }
};

enum class SolveStatus { converged, iteration_limit };

struct PhaseTimings {
  double precompute = 0, global = 0, local = 0, dual = 0;  // seconds
};

struct IterateSnapshot {
  std::vector<double> x, z, z_prev, lambda;
};

struct SolveResult {
  std::vector<double> x, z, lambda;
  SolveStatus status = SolveStatus::iteration_limit;
  int iterations = 0;
  double objective = 0;
  double max_local_infeasibility = 0;
  std::vector<TraceRow> trace;
  PhaseTimings timings;
  std::vector<IterateSnapshot> snapshots;
};

void write_trace_csv(const std::vector<TraceRow>& trace, std::ostream& out);
void write_solution(const std::vector<VariableKey>& var_table, const std::vector<double>& x,
                    std::ostream& out);

}  // namespace dopf
