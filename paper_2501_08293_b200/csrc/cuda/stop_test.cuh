// Near-tie guard of the stop test (hard part 2).
//
// The reference stops when pres <= eps_prim && dres <= eps_dual
// (proj/include/dopf/admm.hpp:63, proj/src/admm.cpp:231). The device reduces
// the five residual sums as trees while the reference sums sequentially
// (admm.cpp:150-163), so pres, dres, eps_prim and eps_dual may differ from the
// reference's in the last few ulps. That can change the stop iteration only
// when the predicate is within that noise of flipping. An iteration is a
// *near tie* when a relative perturbation of kTieRel of any of the four
// scalars could flip the predicate; the solvers count those iterations (up to
// and including the stopping one) and report the count and the first one, so
// an iteration count that could depend on summation order is never silent.
#pragma once

#include <cmath>

namespace dopf::cuda {

constexpr double kTieRel = 1e-12;

__host__ __device__ inline bool tie_close(double r, double eps) {
  const double scale = fmax(fabs(r), fabs(eps));
  return scale > 0.0 && fabs(r - eps) <= kTieRel * scale;
}

__host__ __device__ inline bool stop_near_tie(double pres, double eps_prim, double dres, double eps_dual) {
  const bool p_ok = pres <= eps_prim, d_ok = dres <= eps_dual;
  const bool p_near = tie_close(pres, eps_prim), d_near = tie_close(dres, eps_dual);
  // the predicate p_ok && d_ok flips if a near component flips while the
  // other one holds (or is near itself)
  return (p_near && (d_ok || d_near)) || (d_near && (p_ok || p_near));
}

}  // namespace dopf::cuda
