// Device-side value gather of the re-upload fast path (layout_gather.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dopf::cuda {

struct GatherParams {
  int64_t np, na, rows, cols, nab;
  const int64_t* p_src;
  const int64_t* a_src;
  const int32_t* ref_of_dev;
  const int32_t* gcol;
  const int64_t* ab_src;
  const double *rawP, *rawA, *rawb, *rawv, *rawz0, *rawc, *rawinv, *rawlo, *rawhi;
  double *P, *A, *ab, *v, *z0, *cc, *cinv, *clo, *chi;
};

cudaError_t launch_gather(const GatherParams& g, int sm_count, cudaStream_t s);

/// Batch results: each instance's final (z, lambda) out of the rings into
/// compact [rows_total] arrays.
cudaError_t launch_final_iterates(const double* zring, const double* lring, int64_t rows_total,
                                  const int32_t* row0, const int32_t* rows, const int32_t* iters,
                                  int instances, int ring, double* zout, double* lout, cudaStream_t s);

/// Single instance: the stopping iterate (ring slot iters[0] % ring) of z and
/// lambda permuted to reference order, and {iters, status, maxinf, objective}.
cudaError_t launch_final_single(const double* zring, const double* lring, int64_t rows, const int32_t* ref_of_dev,
                                const int32_t* iters, int ring, const int32_t* status, const double* maxinf,
                                const double* obj, const int32_t* ties, double* zout, double* lout,
                                double* scalars, int sm_count, cudaStream_t s);

}  // namespace dopf::cuda
