// CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// The individual iteration steps of the reference, one entry point each, so
// the reference's per-function known-answer tests (proj/tests/test_admm.cpp)
// can be ported verbatim:
//   oracle_global_update  <- global_update, proj/src/admm.cpp:118-129
//   oracle_local_update   <- gather_local + local_update, admm.cpp:25-29, 131-138
//   oracle_dual_update    <- dual_update, admm.cpp:140-143
//   oracle_residuals      <- residuals, admm.cpp:145-170
// Same operation forms as oracle_solve (admm_oracle.cpp), which the solve
// loop inlines.
#include <algorithm>
#include <cmath>

#include "oracle.h"

extern "C" int oracle_global_update(const dopf_model_view* mv, const double* z,
                                    const double* lambda, double rho, double* x) {
  if (!mv || !z || !lambda || !x || !mv->has_pre) return DOPF_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < mv->n; ++i) {
    double acc = 0.0;
    for (int k = mv->csr_ptr[i]; k < mv->csr_ptr[i + 1]; ++k) {
      const int idx = mv->csr_copy[k];
      acc += z[idx] - lambda[idx] / rho;
    }
    const double unclamped = (acc - mv->c[i] / rho) * mv->inv_copy[i];
    x[i] = std::min(std::max(unclamped, mv->x_lo[i]), mv->x_hi[i]);
  }
  return DOPF_OK;
}

extern "C" int oracle_local_update(const dopf_model_view* mv, int32_t s, const double* x,
                                   const double* lambda_s, double rho, double* z_s) {
  if (!mv || !x || !lambda_s || !z_s || !mv->has_pre || s < 0 || s >= mv->S)
    return DOPF_ERR_INVALID_ARGUMENT;
  const int off = mv->z_offsets[s];
  const int ns = mv->z_offsets[s + 1] - off;
  const double* P = mv->P + mv->p_offsets[s];
  double target[512];
  if (ns > 512) return DOPF_ERR_INVALID_ARGUMENT;
  for (int j = 0; j < ns; ++j) target[j] = x[mv->l2g[off + j]] + lambda_s[j] / rho;
  for (int i = 0; i < ns; ++i) {
    double acc = 0.0;
    for (int j = 0; j < ns; ++j) acc += P[i * ns + j] * target[j];
    z_s[i] = acc + mv->v[off + i];
  }
  return DOPF_OK;
}

extern "C" int oracle_dual_update(const dopf_model_view* mv, int32_t s, const double* x,
                                  const double* z_s, double* lambda_s, double rho) {
  if (!mv || !x || !z_s || !lambda_s || s < 0 || s >= mv->S) return DOPF_ERR_INVALID_ARGUMENT;
  const int off = mv->z_offsets[s];
  const int ns = mv->z_offsets[s + 1] - off;
  for (int j = 0; j < ns; ++j) lambda_s[j] = lambda_s[j] + rho * (x[mv->l2g[off + j]] - z_s[j]);
  return DOPF_OK;
}

extern "C" int oracle_residuals(const dopf_model_view* mv, const double* x, const double* z,
                                const double* z_prev, const double* lambda, double rho,
                                double eps_rel, double* out4) {
  if (!mv || !x || !z || !z_prev || !lambda || !out4) return DOPF_ERR_INVALID_ARGUMENT;
  double gap = 0, step = 0, bx2 = 0, z2 = 0, l2 = 0;
  for (int k = 0; k < mv->N_z; ++k) {
    const double bx = x[mv->l2g[k]];
    const double zj = z[k];
    gap += (bx - zj) * (bx - zj);
    const double dz = zj - z_prev[k];
    step += dz * dz;
    bx2 += bx * bx;
    z2 += zj * zj;
    l2 += lambda[k] * lambda[k];
  }
  out4[0] = std::sqrt(gap);
  out4[1] = rho * std::sqrt(step);
  out4[2] = eps_rel * std::max(std::sqrt(bx2), std::sqrt(z2));
  out4[3] = eps_rel * std::sqrt(l2);
  return DOPF_OK;
}
