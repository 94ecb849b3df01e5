// CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Restatement of the reference solve loop, proj/src/admm.cpp:172-244, over a
// flat dopf_model_view. Every operation keeps the reference's form and order:
//   global  :120-128  acc = 0; acc += z - lambda/rho over copies in ascending s;
//                     x = min(max((acc - c/rho) * inv_count, lo), hi)
//   local   :131-138  target = x[l2g] + lambda/rho;  z = P target + v
//                     (P target as a sequential-j dot product per row)
//   maxinf  :203-205  max_r |A_r z - b_r| (reduced A, b), 0 for m_s = 0
//   dual    :140-143  lambda += rho * (x[l2g] - z)
//   residual:145-170  one pass over (s ascending, j ascending)
//   objective :223-224 sequential c'x
// Built with -O2 -ffp-contract=off (no FMA), matching the reference's default
// x86-64 build.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../paper_2501_08293_b200/csrc/host/parallel.hpp"
#include "oracle.h"

namespace {

thread_local std::string g_err;

// Near-tie flag of the stop test (not in the reference; reported so an
// iteration count that could hinge on summation order is visible): the
// predicate pres <= eps_prim && dres <= eps_dual (admm.hpp:63) could flip
// under a 1e-12 relative perturbation of one of the four scalars.
bool close_rel(double r, double e) {
  const double scale = std::max(std::abs(r), std::abs(e));
  return scale > 0.0 && std::abs(r - e) <= 1e-12 * scale;
}

bool near_tie(double pres, double eps_prim, double dres, double eps_dual) {
  const bool p_ok = pres <= eps_prim, d_ok = dres <= eps_dual;
  const bool p_near = close_rel(pres, eps_prim), d_near = close_rel(dres, eps_dual);
  return (p_near && (d_ok || d_near)) || (d_near && (p_ok || p_near));
}

}  // namespace

void oracle_set_error(const char* msg) { g_err = msg; }

extern "C" const char* oracle_last_error(void) { return g_err.c_str(); }

extern "C" int oracle_solve(const dopf_model_view* mv, const dopf_settings* st,
                            dopf_result_view* res, const int32_t* snap_iters, int32_t n_snap,
                            double* snap_x, double* snap_z, double* snap_zprev,
                            double* snap_lambda) {
  try {
    if (!mv || !st || !res) throw std::invalid_argument("null argument");
    if (!(st->rho > 0)) throw std::invalid_argument("rho must be positive");
    if (!(st->eps_rel > 0)) throw std::invalid_argument("eps_rel must be positive");
    if (st->max_iter < 1) throw std::invalid_argument("max_iter must be positive");
    if (!mv->has_pre) throw std::invalid_argument("model view lacks precomputed operators");

    const int S = mv->S, n = mv->n, Nz = mv->N_z;
    const double rho = st->rho, eps = st->eps_rel;
    dopf::WorkerPool pool(std::max(1, static_cast<int>(st->workers)));

    std::vector<double> x(mv->x0, mv->x0 + n);
    std::vector<double> z(mv->z0, mv->z0 + Nz), z_prev(z), lambda(Nz, 0.0);
    std::vector<double> violation(S, 0.0);
    double max_inf = 0.0;
    int ties = 0, first_tie = 0;
    int status = DOPF_ITERATION_LIMIT;
    int iters = 0;
    double last_objective = 0.0;
    double t_global = 0, t_local = 0, t_dual = 0;
    int next_snap = 0;
    using clk = std::chrono::steady_clock;

    const int cap = st->max_iter;
    for (int iter = 1; iter <= cap; ++iter) {
      auto t0 = clk::now();
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = mv->csr_ptr[i]; k < mv->csr_ptr[i + 1]; ++k) {
          const int idx = mv->csr_copy[k];
          acc += z[idx] - lambda[idx] / rho;
        }
        const double unclamped = (acc - mv->c[i] / rho) * mv->inv_copy[i];
        x[i] = std::min(std::max(unclamped, mv->x_lo[i]), mv->x_hi[i]);
      }
      auto t1 = clk::now();
      z_prev = z;
      pool.run(S, [&](int s) {
        const int off = mv->z_offsets[s];
        const int ns = mv->z_offsets[s + 1] - off;
        const int ms = mv->m_s[s];
        double target[64];
        std::vector<double> big;
        double* tgt = target;
        if (ns > 64) {
          big.resize(ns);
          tgt = big.data();
        }
        for (int j = 0; j < ns; ++j) tgt[j] = x[mv->l2g[off + j]] + lambda[off + j] / rho;
        const double* P = mv->P + mv->p_offsets[s];
        for (int i = 0; i < ns; ++i) {
          double acc = 0.0;
          for (int j = 0; j < ns; ++j) acc += P[i * ns + j] * tgt[j];
          z[off + i] = acc + mv->v[off + i];
        }
        double worst = 0.0;
        const double* A = mv->A + mv->a_offsets[s];
        const double* b = mv->b + mv->b_offsets[s];
        for (int r = 0; r < ms; ++r) {
          double acc = 0.0;
          for (int j = 0; j < ns; ++j) acc += A[r * ns + j] * z[off + j];
          worst = std::max(worst, std::abs(acc - b[r]));
        }
        violation[s] = ms == 0 ? 0.0 : worst;
      });
      auto t2 = clk::now();
      pool.run(S, [&](int s) {
        const int off = mv->z_offsets[s];
        const int ns = mv->z_offsets[s + 1] - off;
        for (int j = 0; j < ns; ++j)
          lambda[off + j] = lambda[off + j] + rho * (x[mv->l2g[off + j]] - z[off + j]);
      });
      auto t3 = clk::now();
      t_global += std::chrono::duration<double>(t1 - t0).count();
      t_local += std::chrono::duration<double>(t2 - t1).count();
      t_dual += std::chrono::duration<double>(t3 - t2).count();

      for (int s = 0; s < S; ++s) max_inf = std::max(max_inf, violation[s]);

      double gap = 0, step = 0, bx2 = 0, z2 = 0, l2 = 0;
      for (int k = 0; k < Nz; ++k) {
        const double bx = x[mv->l2g[k]];
        const double zj = z[k];
        gap += (bx - zj) * (bx - zj);
        const double dz = zj - z_prev[k];
        step += dz * dz;
        bx2 += bx * bx;
        z2 += zj * zj;
        l2 += lambda[k] * lambda[k];
      }
      const double pres = std::sqrt(gap);
      const double dres = rho * std::sqrt(step);
      const double eps_prim = eps * std::max(std::sqrt(bx2), std::sqrt(z2));
      const double eps_dual = eps * std::sqrt(l2);
      double objective = 0.0;
      for (int i = 0; i < n; ++i) objective += mv->c[i] * x[i];

      iters = iter;
      last_objective = objective;
      if (res->trace) {
        double* row = res->trace + static_cast<std::size_t>(iter - 1) * DOPF_TRACE_WIDTH;
        row[0] = iter;
        row[1] = pres;
        row[2] = dres;
        row[3] = eps_prim;
        row[4] = eps_dual;
        row[5] = objective;
      }
      while (next_snap < n_snap && snap_iters[next_snap] < iter) ++next_snap;
      if (next_snap < n_snap && snap_iters[next_snap] == iter) {
        if (snap_x) std::copy(x.begin(), x.end(), snap_x + static_cast<std::size_t>(next_snap) * n);
        if (snap_z) std::copy(z.begin(), z.end(), snap_z + static_cast<std::size_t>(next_snap) * Nz);
        if (snap_zprev)
          std::copy(z_prev.begin(), z_prev.end(), snap_zprev + static_cast<std::size_t>(next_snap) * Nz);
        if (snap_lambda)
          std::copy(lambda.begin(), lambda.end(), snap_lambda + static_cast<std::size_t>(next_snap) * Nz);
        ++next_snap;
      }
      if (near_tie(pres, eps_prim, dres, eps_dual)) {
        ++ties;
        if (first_tie == 0) first_tie = iter;
      }
      if (pres <= eps_prim && dres <= eps_dual) {
        status = DOPF_CONVERGED;
        break;
      }
    }
    if (res->x) std::copy(x.begin(), x.end(), res->x);
    if (res->z) std::copy(z.begin(), z.end(), res->z);
    if (res->lambda) std::copy(lambda.begin(), lambda.end(), res->lambda);
    res->status = status;
    res->iterations = iters;
    res->objective = last_objective;
    res->max_local_infeasibility = max_inf;
    res->near_ties = ties;
    res->first_near_tie = first_tie;
    res->time_global = t_global;
    res->time_local = t_local;
    res->time_dual = t_dual;
    res->time_solve = t_global + t_local + t_dual;
    return DOPF_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DOPF_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DOPF_ERR_RUNTIME;
  }
}

extern "C" int oracle_reconstruct(const dopf_model_view* mv, const double* x, const double* z,
                                  double* out) {
  // reference oracle.cpp:275-292: copy average of z, clamped; x where no copy
  if (!mv || !x || !z || !out) {
    g_err = "null argument";
    return DOPF_ERR_INVALID_ARGUMENT;
  }
  std::vector<double> sums(mv->n, 0.0);
  std::vector<int> counts(mv->n, 0);
  for (int k = 0; k < mv->N_z; ++k) {
    sums[mv->l2g[k]] += z[k];
    ++counts[mv->l2g[k]];
  }
  for (int i = 0; i < mv->n; ++i) {
    const double value = counts[i] > 0 ? sums[i] / counts[i] : x[i];
    out[i] = std::min(std::max(value, mv->x_lo[i]), mv->x_hi[i]);
  }
  return DOPF_OK;
}
