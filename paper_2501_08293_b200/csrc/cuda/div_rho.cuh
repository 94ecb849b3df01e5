// Division by the penalty rho, bitwise equal to the IEEE division a / rho.
//
// The hardware division is a ~124-cycle dependent sequence with a slow-path
// call (measured on B200, tools/micro/fp64_latency.cu); the kernels divide by
// the same rho every row and iteration. From the correctly rounded
// reciprocal rinv = RN(1/rho) (host division, once per solve):
//   q0 = RN(a rinv)                         within 1.5 ulp of a / rho
//   q1 = RN(q0 + (a - rho q0) rinv)         faithful (residual exact by FMA)
//   q  = RN(q1 + (a - rho q1) rinv)         = RN(a / rho) (Markstein's theorem)
// five dependent fp64 operations (~40 cycles). Zeros, magnitudes of a or
// a / rho outside (2^-900, 2^900), non-finite values and rinv == 0 (the host
// passes 0 for rho outside [2^-500, 2^500]) take the hardware division.
#pragma once

#include <cstdlib>

namespace dopf::cuda {

// host side; DOPF_HWDIV=1 forces the hardware division (A/B measurements)
inline double rho_reciprocal(double rho) {
  static const bool hw = [] {
    const char* e = std::getenv("DOPF_HWDIV");
    return e && e[0] == '1';
  }();
  return (!hw && rho >= 0x1p-500 && rho <= 0x1p500) ? 1.0 / rho : 0.0;
}

__device__ __forceinline__ double div_rho(double a, double rho, double rinv) {
  const double q0 = a * rinv;
  const double ma = fabs(a), mq = fabs(q0);
  if (!(ma > 0x1p-900 && ma < 0x1p900 && mq > 0x1p-900 && mq < 0x1p900)) return a / rho;
  const double r0 = __fma_rn(-rho, q0, a);
  const double q1 = __fma_rn(r0, rinv, q0);
  const double r1 = __fma_rn(-rho, q1, a);
  return __fma_rn(r1, rinv, q1);
}

}  // namespace dopf::cuda
