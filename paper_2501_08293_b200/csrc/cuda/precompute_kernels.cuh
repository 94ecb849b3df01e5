// Batched GPU precompute (precompute_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dopf::cuda {

struct PrecomputeParams {
  int32_t S;
  const int32_t* z_offsets;   // S+1
  const int32_t* m_s;         // S
  const int64_t* a_offsets;   // S+1
  const double* A;
  const int32_t* b_offsets;   // S+1
  const double* b;
  const int64_t* p_offsets;   // S+1
  const int64_t* scratch_offsets;  // S: G, L, X, y per subsystem
  double* scratch;
  double* P;                  // out: row-major n_s x n_s per subsystem
  double* v;                  // out: N_z
  int32_t* singular;          // out: 1 where the guard failed
};

cudaError_t launch_precompute(const PrecomputeParams& p, cudaStream_t stream);

}  // namespace dopf::cuda
