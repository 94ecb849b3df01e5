// One-time operators on the GPU (precompute_kernels.cu): row reduction of
// every subsystem's equality rows and the projector / shift of the reduced
// rows, batched over every subsystem of any number of models.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace dopf::cuda {

/// One subsystem of one model in the batched prepare.
struct PrepSub {
  int64_t a_off;  // A slot: m x n row-major (unreduced); the reduced rows overwrite its first rank x n
  int64_t p_off;  // P: n x n row-major
  int64_t v_off;  // v: n (the subsystem's z offset in the concatenated models)
  int64_t b_off;  // b: m (unreduced); the reduced rhs overwrites its first rank
  int32_t m, n;   // unreduced rows, columns
};

enum : int32_t { kPrepOk = 0, kPrepInfeasible = 1, kPrepSingular = 2 };

struct PrepParams {
  int64_t count;          // subsystems (all models)
  const PrepSub* subs;
  double* A;              // in: unreduced rows; out: reduced rows (row_reduce)
  double* b;
  int32_t* rank;          // out of row_reduce, in of precompute (reduced m_s)
  double* P;              // out
  double* v;              // out
  int32_t* status;        // out: kPrep*
  double* scratch;        // global work space when a subsystem exceeds shared memory (null: none)
  const int64_t* scratch_off;  // per subsystem (null: shared memory)
  double tol;
  int32_t reduce;         // 1: run row_reduce (else rank = m, rows used as given)
};

/// Words of work space each kernel needs for a subsystem of m x n.
inline int64_t reduce_words(int64_t m, int64_t n) { return m * (n + 1) + m; }
inline int64_t project_words(int64_t m, int64_t n) { return m * n + 2 * m * m + m * (n + 1); }

/// row_reduce (reference decompose.cpp:48-98) of every subsystem, one warp
/// each; `smem_words` = max reduce_words over the batch when it fits, else 0
/// (global scratch).
cudaError_t launch_row_reduce(const PrepParams& p, int64_t smem_words, cudaStream_t stream);
/// P_s, v_s of the (reduced) rows (reference admm.cpp:31-88), one CTA each.
cudaError_t launch_project(const PrepParams& p, int64_t smem_words, cudaStream_t stream);

}  // namespace dopf::cuda
