// Post-solve certification kernels (certify_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dopf::cuda {

struct CertifyParams {
  int32_t rows, cols, row_blocks, col_blocks;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  const double* values;
  const double* b;
  const double* lo;
  const double* hi;
  const double* x;
  double* blk_v;     // [row_blocks + col_blocks]
  int32_t* blk_i;
  double* out;       // [2]: max equality violation, max bound violation
  int32_t* out_idx;  // [2]: worst row, worst column (-1: none)
};

struct ReconstructParams {
  int32_t n;
  const int32_t* csr_ptr;
  const int32_t* csr_copy;
  const double* z;
  const double* x;
  const double* lo;
  const double* hi;
  double* out;
};

cudaError_t launch_certify(const CertifyParams& p, cudaStream_t s);
cudaError_t launch_reconstruct(const ReconstructParams& p, cudaStream_t s);

}  // namespace dopf::cuda
