// CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Desk-scale exact LP reference, restating proj/src/oracle.cpp:
//   check_feasibility  :10-43   (|Ax-b|_inf, bound violation, worst offenders)
//   run_phase          :76-160  (basis re-factorised every pivot, basics
//                                refreshed from the nonbasic values, Bland's
//                                smallest-index entering rule, ratio test with
//                                bound flips, smallest-variable tie break)
//   reference_solve    :164-273 (signed artificials, phase 1 / phase 2, KKT
//                                certificate)
// Dense LU with partial pivoting replaces Eigen::PartialPivLU.
#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle.h"

void oracle_set_error(const char* msg);

namespace {

constexpr double kCostTol = 1e-9;
constexpr double kPivotTol = 1e-11;
constexpr double kRatioTie = 1e-12;
constexpr double kInf = std::numeric_limits<double>::infinity();

enum class St : char { basic, at_lower, at_upper, at_zero };

struct Lu {
  int n = 0;
  std::vector<double> a;  // row-major, L (unit) below, U on/above
  std::vector<int> perm;
  void factor(const std::vector<double>& m, int size) {
    n = size;
    a = m;
    perm.resize(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
      int p = k;
      double best = std::abs(a[k * n + k]);
      for (int i = k + 1; i < n; ++i)
        if (std::abs(a[i * n + k]) > best) {
          best = std::abs(a[i * n + k]);
          p = i;
        }
      if (p != k) {
        for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[p * n + j]);
        std::swap(perm[k], perm[p]);
      }
      const double piv = a[k * n + k];
      if (piv == 0.0) continue;
      for (int i = k + 1; i < n; ++i) {
        const double f = a[i * n + k] / piv;
        a[i * n + k] = f;
        if (f != 0.0)
          for (int j = k + 1; j < n; ++j) a[i * n + j] -= f * a[k * n + j];
      }
    }
  }
  std::vector<double> solve(const std::vector<double>& rhs) const {
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) {
      double s = rhs[perm[i]];
      for (int j = 0; j < i; ++j) s -= a[i * n + j] * y[j];
      y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < n; ++j) s -= a[i * n + j] * y[j];
      y[i] = s / a[i * n + i];
    }
    return y;
  }
};

struct Tab {
  int m = 0, total = 0;
  std::vector<double> a;  // m x total, row-major
  std::vector<double> b, lo, hi, x;
  std::vector<St> status;
  std::vector<int> basis;
  double at(int i, int j) const { return a[static_cast<std::size_t>(i) * total + j]; }
};

enum class Outcome { optimal, unbounded };

std::vector<double> basis_matrix(const Tab& t, bool transpose) {
  std::vector<double> bm(static_cast<std::size_t>(t.m) * t.m);
  for (int i = 0; i < t.m; ++i)
    for (int k = 0; k < t.m; ++k) {
      const double v = t.at(i, t.basis[k]);
      if (transpose)
        bm[k * t.m + i] = v;
      else
        bm[i * t.m + k] = v;
    }
  return bm;
}

Outcome run_phase(Tab& t, const std::vector<double>& cost, int& pivots, int limit) {
  std::vector<double> w(t.m), col(t.m);
  while (true) {
    if (pivots > limit) throw std::runtime_error("reference_solve: pivot limit exceeded");
    Lu lu, lut;
    std::vector<double> y(t.m, 0.0);
    if (t.m > 0) {
      lu.factor(basis_matrix(t, false), t.m);
      // refresh basics: x_B = B^{-1} (b - A x_N)
      std::vector<double> nonbasic = t.x;
      for (int i = 0; i < t.m; ++i) nonbasic[t.basis[i]] = 0.0;
      std::vector<double> rhs(t.m);
      for (int i = 0; i < t.m; ++i) {
        double s = 0.0;
        for (int j = 0; j < t.total; ++j) s += t.at(i, j) * nonbasic[j];
        rhs[i] = t.b[i] - s;
      }
      const std::vector<double> xb = lu.solve(rhs);
      for (int i = 0; i < t.m; ++i) t.x[t.basis[i]] = xb[i];
      std::vector<double> cb(t.m);
      for (int i = 0; i < t.m; ++i) cb[i] = cost[t.basis[i]];
      lut.factor(basis_matrix(t, true), t.m);
      y = lut.solve(cb);
    }
    int enter = -1;
    double dir = 0.0;
    for (int j = 0; j < t.total; ++j) {
      if (t.status[j] == St::basic) continue;
      if (t.lo[j] == t.hi[j]) continue;
      double yd = 0.0;
      for (int i = 0; i < t.m; ++i) yd += y[i] * t.at(i, j);
      const double d = cost[j] - (t.m > 0 ? yd : 0.0);
      if (t.status[j] == St::at_lower && d < -kCostTol) {
        enter = j;
        dir = 1.0;
      } else if (t.status[j] == St::at_upper && d > kCostTol) {
        enter = j;
        dir = -1.0;
      } else if (t.status[j] == St::at_zero && std::abs(d) > kCostTol) {
        enter = j;
        dir = d > 0 ? -1.0 : 1.0;
      }
      if (enter >= 0) break;
    }
    if (enter < 0) return Outcome::optimal;
    if (t.m > 0) {
      for (int i = 0; i < t.m; ++i) col[i] = t.at(i, enter);
      w = lu.solve(col);
    }
    struct Blocker {
      double ratio;
      int var, row;
      bool hits_upper;
    };
    std::vector<Blocker> blockers;
    if (t.status[enter] == St::at_lower && std::isfinite(t.hi[enter]))
      blockers.push_back({t.hi[enter] - t.lo[enter], enter, -1, true});
    if (t.status[enter] == St::at_upper && std::isfinite(t.lo[enter]))
      blockers.push_back({t.hi[enter] - t.lo[enter], enter, -1, false});
    for (int i = 0; i < t.m; ++i) {
      const double delta = dir * w[i];
      const int var = t.basis[i];
      if (delta > kPivotTol && std::isfinite(t.lo[var]))
        blockers.push_back({std::max((t.x[var] - t.lo[var]) / delta, 0.0), var, i, false});
      else if (delta < -kPivotTol && std::isfinite(t.hi[var]))
        blockers.push_back({std::max((t.x[var] - t.hi[var]) / delta, 0.0), var, i, true});
    }
    if (blockers.empty()) return Outcome::unbounded;
    double step = kInf;
    for (const auto& bk : blockers) step = std::min(step, bk.ratio);
    const Blocker* chosen = nullptr;
    for (const auto& bk : blockers)
      if (bk.ratio <= step + kRatioTie && (!chosen || bk.var < chosen->var)) chosen = &bk;
    ++pivots;
    if (chosen->row < 0) {
      t.x[enter] = chosen->hits_upper ? t.hi[enter] : t.lo[enter];
      t.status[enter] = chosen->hits_upper ? St::at_upper : St::at_lower;
      continue;
    }
    const int leaving = t.basis[chosen->row];
    t.x[enter] += dir * step;
    t.status[enter] = St::basic;
    t.basis[chosen->row] = enter;
    t.x[leaving] = chosen->hits_upper ? t.hi[leaving] : t.lo[leaving];
    t.status[leaving] = chosen->hits_upper ? St::at_upper : St::at_lower;
  }
}


double dense_at(const dopf_lp_view* lp, int i, int j) {
  for (int k = lp->row_ptr[i]; k < lp->row_ptr[i + 1]; ++k)
    if (lp->col_idx[k] == j) return lp->values[k];
  return 0.0;
}

}  // namespace

extern "C" int oracle_reference_solve(const dopf_lp_view* lp, int32_t max_cols, double* x_out,
                                      double* objective, int32_t* status, double* kkt_residual,
                                      int32_t* pivots_out) {
  try {
    if (!lp) throw std::invalid_argument("null lp");
    const int n = lp->cols, m = lp->rows;
    if (n > max_cols)
      throw std::invalid_argument("reference_solve: " + std::to_string(n) +
                                  " columns exceed the size guard of " + std::to_string(max_cols));
    for (int j = 0; j < n; ++j)
      if (lp->x_lo[j] > lp->x_hi[j])
        throw std::invalid_argument("reference_solve: crossed bounds on column " + std::to_string(j));
    Tab t;
    t.m = m;
    t.total = n + m;
    t.a.assign(static_cast<std::size_t>(m) * t.total, 0.0);
    for (int i = 0; i < m; ++i)
      for (int k = lp->row_ptr[i]; k < lp->row_ptr[i + 1]; ++k)
        t.a[static_cast<std::size_t>(i) * t.total + lp->col_idx[k]] = lp->values[k];
    t.b.assign(lp->b, lp->b + m);
    t.lo.resize(t.total);
    t.hi.resize(t.total);
    t.x.assign(t.total, 0.0);
    t.status.assign(t.total, St::at_zero);
    t.basis.resize(m);
    for (int j = 0; j < n; ++j) {
      t.lo[j] = lp->x_lo[j];
      t.hi[j] = lp->x_hi[j];
      if (std::isfinite(t.lo[j])) {
        t.x[j] = t.lo[j];
        t.status[j] = St::at_lower;
      } else if (std::isfinite(t.hi[j])) {
        t.x[j] = t.hi[j];
        t.status[j] = St::at_upper;
      }
    }
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += t.at(i, j) * t.x[j];
      const double r = t.b[i] - s;
      const int j = n + i;
      t.a[static_cast<std::size_t>(i) * t.total + j] = r >= 0 ? 1.0 : -1.0;
      t.lo[j] = 0.0;
      t.hi[j] = kInf;
      t.x[j] = std::abs(r);
      t.status[j] = St::basic;
      t.basis[i] = j;
    }
    const int limit = 50000 + 200 * t.total;
    int pivots = 0;
    std::vector<double> c1(t.total, 0.0);
    for (int i = 0; i < m; ++i) c1[n + i] = 1.0;
    run_phase(t, c1, pivots, limit);
    double mass = 0.0;
    for (int i = 0; i < m; ++i) mass += std::abs(t.x[n + i]);
    *kkt_residual = 0.0;
    if (mass > 1e-8) {
      *status = 1;
      std::copy(t.x.begin(), t.x.begin() + n, x_out);
      *objective = 0.0;
      *pivots_out = pivots;
      return DOPF_OK;
    }
    for (int i = 0; i < m; ++i) t.hi[n + i] = 0.0;
    std::vector<double> c2(t.total, 0.0);
    for (int j = 0; j < n; ++j) c2[j] = lp->c[j];
    const Outcome out = run_phase(t, c2, pivots, limit);
    *pivots_out = pivots;
    std::copy(t.x.begin(), t.x.begin() + n, x_out);
    if (out == Outcome::unbounded) {
      *status = 2;
      *objective = 0.0;
      return DOPF_OK;
    }
    *status = 0;
    double obj = 0.0;
    for (int j = 0; j < n; ++j) obj += lp->c[j] * x_out[j];
    *objective = obj;
    // KKT certificate from the final basis duals (oracle.cpp:242-271)
    std::vector<double> y(m, 0.0);
    if (m > 0) {
      Lu lut;
      lut.factor(basis_matrix(t, true), m);
      std::vector<double> cb(m);
      for (int i = 0; i < m; ++i) cb[i] = c2[t.basis[i]];
      y = lut.solve(cb);
    }
    double kkt = 0.0;
    for (int j = 0; j < n; ++j) {
      double yd = 0.0;
      for (int i = 0; i < m; ++i) yd += y[i] * t.at(i, j);
      const double d = lp->c[j] - (m > 0 ? yd : 0.0);
      const bool at_lo = std::isfinite(t.lo[j]) && t.x[j] - t.lo[j] <= 1e-9 * (1 + std::abs(t.lo[j]));
      const bool at_hi = std::isfinite(t.hi[j]) && t.hi[j] - t.x[j] <= 1e-9 * (1 + std::abs(t.hi[j]));
      if (at_lo && at_hi) continue;
      if (at_lo) kkt = std::max(kkt, -d);
      else if (at_hi) kkt = std::max(kkt, d);
      else kkt = std::max(kkt, std::abs(d));
    }
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int k = lp->row_ptr[i]; k < lp->row_ptr[i + 1]; ++k) s += lp->values[k] * x_out[lp->col_idx[k]];
      kkt = std::max(kkt, std::abs(s - lp->b[i]));
    }
    for (int j = 0; j < n; ++j) {
      kkt = std::max(kkt, lp->x_lo[j] - x_out[j]);
      kkt = std::max(kkt, x_out[j] - lp->x_hi[j]);
    }
    *kkt_residual = std::max(kkt, 0.0);
    return DOPF_OK;
  } catch (const std::invalid_argument& e) {
    oracle_set_error(e.what());
    return DOPF_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    oracle_set_error(e.what());
    return DOPF_ERR_RUNTIME;
  }
}

extern "C" int oracle_check_feasibility(const dopf_lp_view* lp, const double* x,
                                        double* max_eq, double* max_bound, int32_t* worst_row,
                                        int32_t* worst_col, double* objective) {
  if (!lp || !x) return DOPF_ERR_INVALID_ARGUMENT;
  double eq = 0.0, bd = 0.0, obj = 0.0;
  int wr = -1, wc = -1;
  for (int i = 0; i < lp->rows; ++i) {
    double s = 0.0;
    for (int k = lp->row_ptr[i]; k < lp->row_ptr[i + 1]; ++k) s += lp->values[k] * x[lp->col_idx[k]];
    const double v = std::abs(s - lp->b[i]);
    if (v > eq) {
      eq = v;
      wr = i;
    }
  }
  for (int j = 0; j < lp->cols; ++j) {
    const double v = std::max(std::max(lp->x_lo[j] - x[j], x[j] - lp->x_hi[j]), 0.0);
    if (v > bd) {
      bd = v;
      wc = j;
    }
    obj += lp->c[j] * x[j];
  }
  *max_eq = eq;
  *max_bound = bd;
  if (worst_row) *worst_row = wr;
  if (worst_col) *worst_col = wc;
  if (objective) *objective = obj;
  (void)dense_at;
  return DOPF_OK;
}
