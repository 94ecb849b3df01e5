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
  int32_t ties;         // near-tie stop tests so far (stop_test.cuh)
  int32_t first_tie;    // first of them (0: none)
  // PhaseTimings stamps (%globaltimer, ns): start of this iteration's column
  // kernel and chunk kernels; accumulated global (boundary columns) and local
  // (chunk kernels: target, GEMV, dual, interior columns) time
  unsigned long long g0, c0;
  long long t_global, t_local;
};

constexpr int kStagedThreads = kStagedRows + 32;  // compute warps + 1 producer warp
constexpr int kDefaultStagedCtasPerSm = 2;  // 2 or 3 (DOPF_STAGED_CTAS)
constexpr int kBigCtasPerSm = 2;            // direct-load kernel residency

struct StreamParams {
  const StreamChunk* chunks;
  const int32_t* staged_ids;  // chunks of the staged (bulk-copy pipelined) kernel
  const int32_t* big_ids;     // chunks too large for a stage (direct-load kernel)
  const int32_t* imp_ptr;     // boundary column -> import slots (CSR)
  const int32_t* imp_slot;
  double* ximp;               // [imports] boundary x per importing chunk (read by bulk copy)
  const unsigned char* blob;  // chunk images (ChunkHead + sections)
  // boundary columns [0, bcols)
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
  double* part;          // [npart][8]
  double* objp;          // [col_blocks] boundary columns' c'x
  unsigned* final_count; // chunk CTAs done this iteration (the last folds; zero between iterations)
  double* trace;         // [max_iter][6] or null
  StreamCtl* ctl;
  double* partials_out;  // partitioned: this rank's 7 combined partials (null: decide here)
  const int32_t* export_rows;  // partitioned: rows whose u other ranks read
  double* send;          // [max_export] packed exports
  int32_t n_export, max_export;
  double rho, eps;
  double rho_inv;        // RN(1 / rho) (div_rho)
  int32_t max_iter;
  int32_t nchunks;
  int32_t n_staged, n_big;
  int32_t staged_grid;   // persistent CTAs of the staged kernel (partials [0, staged_grid))
  int32_t npart;         // partial slots: staged_grid + n_big
  int32_t stages, stage_bytes;  // staged-kernel pipeline (dynamic smem = stages * stage_bytes)
  int32_t staged_ctas;   // staged CTAs per SM (2 or 3)
  int32_t local_threads; // direct-load kernel CTA size: kStreamRows, or kWideRows when a chunk is wider
  long long* prof;
       // optional [staged_grid][8] phase cycles of the staged kernel (thread 0)
  int32_t cols;
  int32_t bcols;         // boundary columns [0, bcols) (k_global); the rest are per-chunk interior
  int32_t col_blocks;    // k_global CTAs (>= 1)
  cudaGraphConditionalHandle cond;
  int32_t use_cond;
};

/// Same-structure re-upload: model values (raw concatenation, stream_layout.hpp)
/// scattered into the chunk images, z0 and the boundary-column arrays.
struct StreamRegather {
  const double* raw;
  const int32_t* blob_src;
  double* blob;
  int64_t nblob;          // 8-byte words
  const int32_t* ref_of_dev;
  double* z0;
  int32_t rows;
  const int32_t* gcol;
  double *cost, *inv, *lo, *hi;
  int32_t bcols;
  int64_t off_z0, off_c, off_inv, off_lo, off_hi;
};
cudaError_t stream_launch_regather(const StreamRegather& g, int sm_count, cudaStream_t s);

/// Final iterates in reference order (z, lambda: N_z; x: n) for a direct copy back.
cudaError_t stream_launch_results(const double* z, const double* lam, const double* x, const int32_t* ref_of_dev,
                                  const int32_t* gcol, int64_t rows, int64_t cols, double* zout, double* lout,
                                  double* xout, int sm_count, cudaStream_t s);

/// div_rho self-check (dopf_cuda_div_rho_check).
cudaError_t launch_div_rho_check(const double* a, int64_t n, double rho, double rinv, double* out, cudaStream_t s);

/// One-time kernel attributes (dynamic shared memory of the staged kernel).
cudaError_t stream_prepare();
/// Iterations per while-node body (kernels after the stop return at once).
int stream_graph_unroll();
/// The whole solve as one graph: a while-node over {k_global, k_local | k_staged}.
cudaError_t stream_build_graph(StreamParams p, cudaGraphExec_t* exec);
/// One iteration, stream-ordered (no graph).
void stream_launch_iteration(const StreamParams& p, cudaStream_t s);
/// Partitioned steps: global update; local + per-rank partials; decision from
/// all ranks' partials (8 doubles per rank, rank order).
void stream_launch_global(const StreamParams& p, cudaStream_t s);
void stream_launch_local(const StreamParams& p, cudaStream_t s);
void stream_launch_pack(const StreamParams& p, cudaStream_t s);
/// The chunk kernels one at a time: direct-load chunks (image from HBM), and
/// the staged (bulk-copy pipelined) kernel -- to run side by side on two
/// streams (they occupy disjoint SMs).
void stream_launch_direct(const StreamParams& p, cudaStream_t s);
void stream_launch_staged(const StreamParams& p, cudaStream_t s);
void stream_launch_decide(const StreamParams& p, const double* recv, int nranks, int stride, cudaStream_t s);

}  // namespace dopf::cuda
