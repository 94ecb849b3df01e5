// One-time host precompute and output writers.
//
// precompute restates reference proj/src/admm.cpp:31-88 without Eigen:
//   G = A A'                      sequential-k dot products
//   L = chol(G)                   left-looking, fails on a non-positive pivot
//   guard (d_min/d_max)^2 < 1e-14 on diag(L)                     (:53-59)
//   X = G^{-1} A by forward/back substitution                     (:61)
//   P = I - A' X,  v = A' (G^{-1} b)                               (:62-64)
// The result is shared verbatim by the GPU path and the CPU oracle, so both
// iterate on bitwise-identical operators. (Eigen's blocked GEMM/LLT summation
// order is not reproducible without Eigen; the difference is ulp-level and is
// pinned by the projector-algebra and KKT tests, as in test_admm.cpp:53-111.)
#include <algorithm>
#include <cmath>
#include <ostream>

#include "admm.hpp"

namespace dopf {

SingularSubsystemError::SingularSubsystemError(std::string subsystem_id)
    : std::runtime_error("numerically singular subsystem '" + subsystem_id + "'"),
      id_(std::move(subsystem_id)) {}

namespace {

// Returns false when A A' is not (numerically) positive definite.
bool project_one(const Subsystem& sub, PrecomputedSub& ps) {
  const int m = sub.row_count(), n = sub.col_count();
  if (m == 0) {
    ps.kernel_projector = Dense(n, n);
    for (int i = 0; i < n; ++i) ps.kernel_projector(i, i) = 1.0;
    ps.min_norm_solution.assign(n, 0.0);
    return true;
  }
  const Dense& A = sub.A;
  Dense G(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += A(i, k) * A(j, k);
      G(i, j) = acc;
      G(j, i) = acc;
    }
  Dense L(m, m);
  for (int k = 0; k < m; ++k) {
    double d = G(k, k);
    for (int p = 0; p < k; ++p) d -= L(k, p) * L(k, p);
    if (!(d > 0.0)) return false;
    const double lkk = std::sqrt(d);
    L(k, k) = lkk;
    for (int i = k + 1; i < m; ++i) {
      double s = G(i, k);
      for (int p = 0; p < k; ++p) s -= L(i, p) * L(k, p);
      L(i, k) = s / lkk;
    }
  }
  double dmin = L(0, 0), dmax = L(0, 0);
  for (int k = 1; k < m; ++k) {
    dmin = std::min(dmin, L(k, k));
    dmax = std::max(dmax, L(k, k));
  }
  if (!(dmin > 0.0) || (dmin / dmax) * (dmin / dmax) < 1e-14) return false;

  // Solve G Y = [A | b] column by column: L w = rhs, L' y = w.
  auto solve_in_place = [&](std::vector<double>& y) {
    for (int i = 0; i < m; ++i) {
      double s = y[i];
      for (int p = 0; p < i; ++p) s -= L(i, p) * y[p];
      y[i] = s / L(i, i);
    }
    for (int i = m - 1; i >= 0; --i) {
      double s = y[i];
      for (int p = i + 1; p < m; ++p) s -= L(p, i) * y[p];
      y[i] = s / L(i, i);
    }
  };
  Dense X(m, n);
  std::vector<double> col(m);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < m; ++i) col[i] = A(i, j);
    solve_in_place(col);
    for (int i = 0; i < m; ++i) X(i, j) = col[i];
  }
  std::vector<double> gb(sub.b);
  solve_in_place(gb);

  ps.kernel_projector = Dense(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc += A(k, i) * X(k, j);
      ps.kernel_projector(i, j) = (i == j ? 1.0 : 0.0) - acc;
    }
  ps.min_norm_solution.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc += A(k, i) * gb[k];
    ps.min_norm_solution[i] = acc;
  }
  return true;
}

}  // namespace

namespace {

// inverse copy counts and the CSR scatter, ascending s (admm.cpp:75-86)
void build_scatter(const DecomposedModel& model, Precomputed& pre) {
  const int S = model.subsystem_count();
  const int n = model.global_cols;
  pre.inv_copy_counts.resize(n);
  for (int i = 0; i < n; ++i) {
    if (model.copy_counts[i] < 1)
      throw std::logic_error("global column " + std::to_string(i) + " has no copy");
    pre.inv_copy_counts[i] = 1.0 / static_cast<double>(model.copy_counts[i]);
  }
  pre.col_ptr.assign(n + 1, 0);
  for (int s = 0; s < S; ++s)
    for (int g : model.subsystems[s].local_to_global) ++pre.col_ptr[g + 1];
  for (int i = 0; i < n; ++i) pre.col_ptr[i + 1] += pre.col_ptr[i];
  pre.copy_index.assign(pre.col_ptr[n], 0);
  std::vector<int> fill(pre.col_ptr.begin(), pre.col_ptr.end() - 1);
  for (int s = 0; s < S; ++s) {
    const Subsystem& sub = model.subsystems[s];
    for (int j = 0; j < sub.col_count(); ++j)
      pre.copy_index[fill[sub.local_to_global[j]]++] = model.z_offsets[s] + j;
  }
}

}  // namespace

Precomputed precompute(const DecomposedModel& model, WorkerPool* pool) {
  const int S = model.subsystem_count();
  Precomputed pre;
  pre.subs.resize(S);
  std::vector<char> singular(S, 0);
  auto one = [&](int s) {
    if (!project_one(model.subsystems[s], pre.subs[s])) singular[s] = 1;
  };
  if (pool && pool->worker_count() > 1)
    pool->run(S, one);
  else
    for (int s = 0; s < S; ++s) one(s);
  for (int s = 0; s < S; ++s)
    if (singular[s]) throw SingularSubsystemError(model.subsystems[s].component_id);
  build_scatter(model, pre);
  return pre;
}

Precomputed precompute_from(const DecomposedModel& model, const double* P, const double* v) {
  const int S = model.subsystem_count();
  Precomputed pre;
  pre.subs.resize(S);
  std::size_t at = 0;
  for (int s = 0; s < S; ++s) {
    const int n = model.subsystems[s].col_count();
    PrecomputedSub& ps = pre.subs[s];
    ps.kernel_projector = Dense(n, n);
    std::copy(P + at, P + at + static_cast<std::size_t>(n) * n, ps.kernel_projector.a.begin());
    at += static_cast<std::size_t>(n) * n;
    ps.min_norm_solution.assign(v + model.z_offsets[s], v + model.z_offsets[s] + n);
  }
  build_scatter(model, pre);
  return pre;
}

double initial_value(const DecomposedModel& model, int col) {
  if (model.var_table[col].kind == VarKind::w) return 1.0;
  const double lo = model.x_lo[col], hi = model.x_hi[col];
  if (std::isfinite(lo) && std::isfinite(hi)) return 0.5 * (lo + hi);
  return 0.0;
}

void write_trace_csv(const std::vector<TraceRow>& trace, std::ostream& out) {
  out.precision(17);
  out << "t,pres,dres,eps_prim,eps_dual,objective\n";
  for (const TraceRow& r : trace)
    out << r.t << "," << r.pres << "," << r.dres << "," << r.eps_prim << "," << r.eps_dual << ","
        << r.objective << "\n";
}

void write_solution(const std::vector<VariableKey>& var_table, const std::vector<double>& x,
                    std::ostream& out) {
  out.precision(17);
  for (std::size_t i = 0; i < var_table.size(); ++i)
    out << to_string(var_table[i]) << " " << x[i] << "\n";
}

}  // namespace dopf
