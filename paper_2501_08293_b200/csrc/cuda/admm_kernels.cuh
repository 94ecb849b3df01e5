// Launch interface of the persistent ADMM iteration kernel (admm_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "layout.hpp"

namespace dopf::cuda {

constexpr int kCtlWords = 64;
constexpr int kSampleEvery = 32;  // phase-timing sample period (iterations)
constexpr int kTimelineT0 = 100, kTimelineIters = 64;  // iterations stamped by the timeline
constexpr int kSlotRing = 4;   // residual-slot ring depth (admm_kernels.cu)
// Decision lag: the compute warps act on the stop test of t - kLag at
// iteration t, so the grid-wide residual reduction never gates an iteration;
// x is kept kLag + 2 deep (shared memory) and z / lambda kLag + 1 deep.
constexpr int kLag = 4;
constexpr int kXRing = kLag + 2;
constexpr int kZRing = kLag + 1;  // per instance: counter (line 0), decision seq (line 1), ring (lines 2-3)

enum class SyncMode : int32_t { block = 0, cluster = 1, grid = 2 };

struct KernelParams {
  const BlockDesc* blocks;
  const InstDesc* inst;
  const double* P;
  const double* A;
  const int32_t* copies;
  const RowMeta* rmeta;
  const double* v;
  const double* z0;
  const ColMeta* cmeta;
  const double* cc;
  const double* cinv;
  const double* clo;
  const double* chi;
  const AMeta* ameta;
  const double* ab;
  const int32_t* nbrs;  // neighbour lists (BlockDesc::nbr_off / nbr_cnt)
  unsigned long long* ux;  // [2][rows_total][2] tagged exchange records {t, u = z - lambda/rho}
  double* z_out;        // [rows_total]
  double* lam_out;      // [rows_total]
  double* x_out;        // [x_total]
  double* part;         // [instances][kSlotRing][blocks_per_instance][kPartials] residual slots
  unsigned long long* flags;  // [instances][blocks_per_instance][16] "u(t) published", one per 128-B line
  unsigned long long* ctl;    // [instances][kCtlWords]: slot counter, decision seq, decision ring
  double* trace;        // [instances][trace_stride][6] (may be null)
  long long* prof;      // [blocks][8] phase cycle counters (null: off)
  long long* phase_sample;  // [8] phase cycles of block 0 of instance 0, every kSampleEvery-th iteration
                            // (always on; the solve's PhaseTimings split)
  unsigned long long* timeline;  // [blocks][kTimelineIters][3] globaltimer stamps (null: off)
  int32_t* iters;       // [instances]
  int32_t* status;      // [instances] 0 converged, 1 iteration limit
  double* maxinf;       // [instances]
  double* objective;    // [instances]
  int32_t* ties;        // [instances][2] near-tie stop tests up to the stop, first one (stop_test.cuh)
  double* snap;         // parity mode (null: off): per iteration t <= snap_iters, [z | lambda | x]
                        // at snap + (t-1) * (2 rows_total + x_total): z, lambda by device row, x by column
  int64_t snap_stride;
  int32_t snap_iters;
  int32_t snap_pad;
  double rho;
  double rho_inv;  // RN(1 / rho) for div_rho (div_rho.cuh)
  double eps_rel;
  int64_t rows_total;
  int64_t trace_stride; // rows per instance in `trace`
  int32_t max_iter;
  int32_t blocks_per_instance;
  int32_t sync_mode;    // SyncMode (cluster: the exchange between an instance's CTAs)
  int32_t group_size;   // > 0: persistent groups of this many CTAs loop over the instances
  int32_t instances;
};

/// Launches the persistent kernel: one CTA per block descriptor, all
/// iterations on device until every instance converged or hit max_iter.
cudaError_t launch_admm(const KernelParams& p, int num_blocks, int K, std::size_t smem_bytes,
                        SyncMode mode, int cluster_size, bool smem_ops, cudaStream_t stream);
/// Scenario batches: a cooperative grid of `groups` x p.group_size CTAs
/// looping over the instances (p.group_size, p.instances set).
cudaError_t launch_admm_groups(const KernelParams& p, int groups, int K, std::size_t smem_bytes, bool smem_ops,
                               cudaStream_t stream);

/// Largest dynamic shared memory the kernel may use on this device.
int max_dynamic_smem(int device);

}  // namespace dopf::cuda
