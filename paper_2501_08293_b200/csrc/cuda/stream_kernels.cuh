// Launch interface of the HBM-streaming solver path (stream_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "stream_layout.hpp"

namespace dopf::cuda {

struct StreamCtl {      // device-side loop state
  int32_t t;            // iterations done
  int32_t status;       // 0 converged, 1 iteration limit
  int32_t done;
  int32_t pad;
  double maxinf;        // running max of ||A_s z_s - b_s||_inf
  double objective;     // c'x of the last iteration
};

struct StreamParams {
  const StreamChunk* chunks;
  const StreamRow* rmeta;
  const int64_t* pslice;
  const int64_t* aslice;
  const StreamARow* ameta;
  const double* P;
  const double* A;
  const double* ab;
  const double* v;
  const int32_t* col_ptr;
  const int32_t* copies;
  const double* cost;
  const double* inv;
  const double* lo;
  const double* hi;
  const uint8_t* owner;
  double* x;             // [cols]
  double* z;             // [rows] (in place: z^{t-1} -> z^t)
  double* lam;           // [rows]
  double* u;             // [rows] z - lambda/rho (rows of boundary columns)
  const double* u_remote;  // partitioned: gathered copies of other ranks
  double* part;          // [nchunks][8]
  double* objp;          // [col_blocks] boundary columns' c'x
  double* part2;         // [128][8] level-2 partials (k_final)
  unsigned* final_count; // k_final's last-block counter (zero between iterations)
  double* trace;         // [max_iter][6] or null
  StreamCtl* ctl;
  double* partials_out;  // partitioned: this rank's 7 combined partials (null: decide here)
  const int32_t* export_rows;  // partitioned: rows whose u other ranks read
  double* send;          // [max_export] packed exports
  int32_t n_export, max_export;
  double rho, eps;
  int32_t max_iter;
  int32_t nchunks;
  int32_t cols;
  int32_t bcols;         // boundary columns [0, bcols) (k_global); the rest are per-chunk interior
  int32_t col_blocks;    // k_global CTAs (>= 1)
  cudaGraphConditionalHandle cond;
  int32_t use_cond;
};

/// The whole solve as one graph: a while-node over {k_global, k_local, k_final}.
cudaError_t stream_build_graph(StreamParams p, cudaGraphExec_t* exec);
/// One iteration, stream-ordered (no graph).
void stream_launch_iteration(const StreamParams& p, cudaStream_t s);
/// Partitioned steps: global update; local + per-rank partials; decision from
/// all ranks' partials (8 doubles per rank, rank order).
void stream_launch_global(const StreamParams& p, cudaStream_t s);
void stream_launch_local(const StreamParams& p, cudaStream_t s);
void stream_launch_pack(const StreamParams& p, cudaStream_t s);
void stream_launch_decide(const StreamParams& p, const double* ranks, int nranks, cudaStream_t s);

}  // namespace dopf::cuda
