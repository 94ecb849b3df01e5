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

}  // namespace dopf::cuda
