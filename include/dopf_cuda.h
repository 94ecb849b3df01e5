/* Drop-in C ABI of the B200 ADMM solver: the replacement for the reference's
 * solver entry point
 *
 *     SolveResult dopf::solve(const DecomposedModel&, const Settings&)
 *         proj/include/dopf/admm.hpp:126, proj/src/admm.cpp:172-244
 *
 * split into create / upload / solve / destroy so a model is uploaded once
 * and solved many times (scenario batches, warm benchmarks):
 *
 *   dopf_cuda_create   -- context on one device (streams, buffers)
 *   dopf_cuda_upload   -- model + precomputed operators (admm.cpp:31-88 output)
 *                         -> device layout in HBM (row-blocked, column-major
 *                         per-subsystem P and A, CSR-by-column copy lists)
 *   dopf_cuda_solve    -- settings validation (admm.cpp:173-175, code 1 =
 *                         std::invalid_argument), the whole iteration loop on
 *                         the device, results copied into caller buffers in
 *                         the reference's layout (x by global column, z and
 *                         lambda stacked by z_offsets)
 *   dopf_cuda_last_error / dopf_cuda_destroy
 *
 * Status codes are dopf_status (dopf_types.h). iteration_limit is a result
 * status (dopf_result_view.status), not an error, as in the reference.
 * A context is not thread-safe; use one per thread/device.
 */
#ifndef DOPF_CUDA_H
#define DOPF_CUDA_H

#include "dopf_host.h"
#include "dopf_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dopf_cuda_ctx dopf_cuda_ctx;

typedef struct dopf_cuda_info_t {
  int32_t instances;   /* uploaded models                         */
  int32_t blocks;      /* CTAs per instance                       */
  int32_t threads;     /* threads per CTA                         */
  int32_t smem_bytes;  /* dynamic shared memory per CTA           */
  int32_t resident;    /* 1: all operators staged in shared memory */
  int32_t sync_mode;   /* 0 block, 1 cluster, 2 grid, 3 streaming graph */
} dopf_cuda_info_t;

int dopf_cuda_create(int device, dopf_cuda_ctx** out);
int dopf_cuda_upload(dopf_cuda_ctx* ctx, const dopf_model_view* model);
int dopf_cuda_solve(dopf_cuda_ctx* ctx, const dopf_settings* settings, dopf_result_view* result);
/* Same loop, outputs left on the device (only scalars and, if result->trace
 * is non-NULL, the trace are copied back). Used to time the kernel alone. */
int dopf_cuda_solve_device(dopf_cuda_ctx* ctx, const dopf_settings* settings,
                           dopf_result_view* result);
const char* dopf_cuda_last_error(const dopf_cuda_ctx* ctx);
void dopf_cuda_destroy(dopf_cuda_ctx* ctx);

/* Independent scenarios of identical structure (BASELINE config 5): one
 * cluster of CTAs per scenario, per-scenario convergence (a converged
 * scenario stops, the others continue). results[i] receives scenario i. */
int dopf_cuda_upload_batch(dopf_cuda_ctx* ctx, const dopf_model_view* models, int32_t count);
int dopf_cuda_solve_batch(dopf_cuda_ctx* ctx, const dopf_settings* settings,
                          dopf_result_view* results, int32_t count);

int dopf_cuda_info(const dopf_cuda_ctx* ctx, dopf_cuda_info_t* out);
/* Partition tuning of the resident path (setup step, like an autotuner):
 * uploads the model, then for `rounds` rounds measures each CTA's slack at
 * the iteration's final barrier with the phase clock and moves cost shares
 * of the depth-first split away from the CTAs without slack (the critical
 * region of the exchange), keeping the fastest split; the context keeps the
 * tuned shares for later uploads of the same structure. Iterates are
 * unchanged (bitwise: the global update sums in ascending s whatever the
 * split). A no-op for batches and the streaming path. *seconds_per_iteration
 * receives the best measured period. */
int dopf_cuda_tune_partition(dopf_cuda_ctx* ctx, const dopf_model_view* model, const dopf_settings* settings,
                             int32_t rounds, double* seconds_per_iteration);
/* The context's tuned cost shares (copied into out[0, min(count, cap)));
 * returns their count (0: default split). Feeding them back through
 * DOPF_BLOCK_WEIGHTS (comma-separated) reproduces the split in another
 * process (profilers). */
int dopf_cuda_block_weights(const dopf_cuda_ctx* ctx, double* out, int32_t cap);
/* The same for scenario batches: tunes the split of one instance's G CTAs
 * (shared by every scenario of this structure) on models[0, count) -- a
 * sample; upload the whole batch afterwards: it keeps the tuned split. For
 * these tight G-CTA instances a position's load (compute without the
 * exchange) drives the shares. *seconds_per_iteration: per scenario-iteration. */
int dopf_cuda_tune_partition_batch(dopf_cuda_ctx* ctx, const dopf_model_view* models, int32_t count,
                                   const dopf_settings* settings, int32_t rounds, double* seconds_per_iteration);
/* Parity mode (reference Settings::record_iterates, admm.cpp:228-229): the
 * same solve, with the state after every iteration t = 1 .. min(T, stop)
 * written by the device loop itself (one pass, not a re-run per t) and
 * returned in reference order, n + 3 N_z doubles per iteration:
 * [x | z | z_prev | lambda] (IterateSnapshot, admm.hpp:108-114). Single
 * model, either path (the streaming path runs its iterations stream-ordered
 * with a snapshot copy after each, then the regular solve); code 1 for a
 * partitioned upload or a batch. */
int dopf_cuda_solve_snapshots(dopf_cuda_ctx* ctx, const dopf_settings* settings,
                              dopf_result_view* result, double* snapshots, int32_t T);
/* One-time operators on the GPU (reference admm.cpp:31-88, batched over all
 * subsystems): P (row-major n_s x n_s at p_offsets) and v (N_z) of the model
 * view's A, b -- bitwise identical to the host precompute (same sequential
 * Gram / Cholesky / substitution order, no FMA). Code 2 (singular) names the
 * first failing subsystem in *first_singular. Feed the result to
 * dopf_model_set_operators (dopf_host.h). */
int dopf_cuda_precompute(dopf_cuda_ctx* ctx, const dopf_model_view* model, double* P, double* v,
                         int32_t* first_singular);

/* Decomposition finish + one-time operators of MANY models on the GPU
 * (SURVEY row f2): row_reduce of every subsystem's equality rows (reference
 * decompose.cpp:48-98, reduce_subsystems :175-199) and then P_s, v_s of the
 * reduced rows (admm.cpp:31-88), one launch per stage over every subsystem of
 * every model -- bitwise identical to dopf_model_reduce + dopf_model_precompute
 * on the host. models[k] are UNREDUCED views (a partitioned model, has_pre 0).
 * Outputs are the concatenation over k (caller-allocated, in model order):
 *   A  sum_k a_offsets_k[S_k] doubles: the reduced m'_s x n_s rows of s at
 *      the start of its unreduced slot a_offsets_k[s]
 *   b  sum_k b_offsets_k[S_k]: the reduced rhs at the start of its slot
 *   m  sum_k S_k: reduced row counts m'_s
 *   P  sum_k sum_s n_s^2 (row-major n_s x n_s, as p_offsets)
 *   v  sum_k N_z_k
 * Feed them to dopf_model_set_reduced then dopf_model_set_operators.
 * Errors as the host: 7 (infeasible) naming the first failing model /
 * subsystem after the whole reduction, else 2 (singular). seconds[3]
 * (optional): pack + upload, kernels (CUDA events), download + unpack. */
typedef struct dopf_prepare_out {
  double* A;
  double* b;
  int32_t* m;
  double* P;
  double* v;
} dopf_prepare_out;
int dopf_cuda_prepare(dopf_cuda_ctx* ctx, const dopf_model_view* models, int32_t count, double tol,
                      dopf_prepare_out* out, int32_t* fail_model, int32_t* fail_subsystem,
                      double* seconds);

/* Post-solve certification on the GPU (reference oracle.cpp:10-43,
 * check_feasibility): ||A x - b||_inf over the centralized LP, bound
 * violation, worst row / column (first maximum, -1 if none) and c'x. */
typedef struct dopf_certificate {
  double max_equality_violation;
  double max_bound_violation;
  double objective;
  int32_t worst_row, worst_col;
} dopf_certificate;
int dopf_cuda_certify(dopf_cuda_ctx* ctx, const dopf_lp_view* lp, const double* x,
                      dopf_certificate* out);
/* Copy-average reconstruction (oracle.cpp:275-292): per column the mean of its
 * copies (ascending s), clamped to the bounds; x where a column has no copy. */
int dopf_cuda_reconstruct(dopf_cuda_ctx* ctx, const dopf_model_view* model, const double* x,
                          const double* z, double* out);

/* Solver path for the next uploads: 0 auto (default: shared-memory-resident
 * persistent kernel when the operators fit the CTAs' shared memory, else the
 * HBM-streaming CUDA graph), 1 resident, 2 streaming. */
int dopf_cuda_set_path(dopf_cuda_ctx* ctx, int32_t path);
/* Kernels executed so far (a streaming solve runs 3 per iteration inside one
 * graph launch). */
int64_t dopf_cuda_kernels_executed(const dopf_cuda_ctx* ctx);
/* Number of kernels this context launched so far (evidence for benchmarks). */
int64_t dopf_cuda_kernel_launches(const dopf_cuda_ctx* ctx);
/* Algorithmic HBM bytes of one iteration, summed over uploaded instances
 * (BASELINE.md section 3 formula). */
double dopf_cuda_bytes_per_iteration(const dopf_cuda_ctx* ctx);
/* Device time (seconds) of the last solve's kernel, CUDA events on the
 * launching stream. */
double dopf_cuda_last_kernel_seconds(const dopf_cuda_ctx* ctx);
/* Phase clock: when enabled (counters reset), every CTA records the SM cycles
 * spent in each of the 8 loop phases during the next solves: compute warps --
 * target, GEMV, dual + publish, equality check + partial reductions, exchange
 * wait, global update; service warp -- neighbour-flag wait, all-flag wait +
 * residual combine. out receives [min(max_blocks, CTAs)][8] counters. */
int dopf_cuda_set_profiling(dopf_cuda_ctx* ctx, int32_t on);
int dopf_cuda_phase_cycles(const dopf_cuda_ctx* ctx, int64_t* out, int32_t max_blocks);
/* Resident layout statistics per CTA (diagnostics, load-balance studies):
 * [min(max_blocks, CTAs)][12] = rows, columns, interior columns, equality
 * rows, P doubles, A doubles, copy references, neighbour blocks, remote copy
 * reads, exported rows, longest per-thread GEMV chain (sum of n_s over a
 * thread's rows), sum of n_s over rows. */
int dopf_cuda_block_stats(const dopf_cuda_ctx* ctx, int64_t* out, int32_t max_blocks);
/* With profiling on: %globaltimer stamps (ns) per CTA for 64 iterations from
 * t = 100 -- [CTA][iteration][u published, boundary update start, end]. */
int dopf_cuda_timeline(const dopf_cuda_ctx* ctx, uint64_t* out, int64_t cap);
/* Page-lock the value arrays of a host model view (P, A, b, v, z0, c,
 * inv_copy, x_lo, x_hi) with cudaHostRegister, so that later uploads of models
 * living in the same memory copy at DMA speed. Ranges stay registered until
 * dopf_cuda_unpin_model or dopf_cuda_destroy; pinning a range twice is a no-op. */
int dopf_cuda_pin_model(dopf_cuda_ctx* ctx, const dopf_model_view* model);
int dopf_cuda_unpin_model(dopf_cuda_ctx* ctx, const dopf_model_view* model);
/* The same for any caller buffer (e.g. the result arrays x, z, lambda, trace:
 * results are copied straight into them). */
int dopf_cuda_pin_host(dopf_cuda_ctx* ctx, const void* ptr, int64_t bytes);
int dopf_cuda_unpin_host(dopf_cuda_ctx* ctx, const void* ptr);
/* Streaming layout of the uploaded model (zeros for the resident path):
 * out[0] chunks, [1] staged-kernel chunks, [2] direct-load chunks,
 * [3] boundary columns, [4] staged CTAs, [5] stage bytes, [6] stages. */
int dopf_cuda_stream_info(const dopf_cuda_ctx* ctx, int64_t* out7);
/* Self-check of the kernels' division by rho (div_rho.cuh: reciprocal plus
 * two exact-residual corrections): out[i] = a[i] / rho as the kernels
 * compute it, for comparison with the IEEE quotient. Host arrays of n. */
int dopf_cuda_div_rho_check(dopf_cuda_ctx* ctx, const double* a, int64_t n, double rho, double* out);

/* ---- Partitioned solve over several ranks (one process per GPU) ----------
 * Subsystem s lives on rank part_of_s[s]. Each rank updates the columns its
 * rows reference; copies held by other ranks arrive through ONE gather per
 * iteration of every rank's packed record `send` = [u of its exported rows
 * (max_export doubles, zero padded) | its 8 residual partials] into `recv`
 * (nparts * xstride doubles, rank order, xstride = max_export + 8); step 2
 * then combines the ranks' partials in rank order (the identical stop
 * decision on every rank). Two ways to drive it:
 *   - dopf_cuda_comm_init + dopf_cuda_solve_part: the library's own NCCL
 *     communicator, the whole loop (kernels + ncclAllGather) in one CUDA graph
 *     with a device-side while-node (see below);
 *   - the caller's collective, step by step:
 *       begin; step 3; gather(send -> recv);
 *       repeat { step 0; step 1; gather(send -> recv); step 2 } until poll says done
 *       (kernels after the stop are no-ops, so polling may be lazy); finish.
 * Iterates are bitwise identical to the single-GPU solve (same summation orders). */
typedef struct dopf_part_info {
  int32_t nparts, part, rows, cols, n_export, max_export;
  int32_t xstride;     /* doubles per rank record: max_export + 8 */
  int32_t reserved;
  void* send;          /* device double[xstride]          */
  void* recv;          /* device double[nparts * xstride] */
  double bytes_per_iteration;  /* algorithmic bytes of this rank's share */
} dopf_part_info;
int dopf_cuda_upload_part(dopf_cuda_ctx* ctx, const dopf_model_view* model, int32_t nparts,
                          int32_t part, const int32_t* part_of_s);
int dopf_cuda_part_info(const dopf_cuda_ctx* ctx, dopf_part_info* out);
/* Launch on an external stream (e.g. the collective library's), NULL: own stream. */
int dopf_cuda_set_stream(dopf_cuda_ctx* ctx, void* stream);
int dopf_cuda_part_begin(dopf_cuda_ctx* ctx, const dopf_settings* settings, int32_t with_trace);
int dopf_cuda_part_step(dopf_cuda_ctx* ctx, int32_t phase);
int dopf_cuda_part_poll(dopf_cuda_ctx* ctx, int32_t* done, int32_t* iterations);
/* Fills x at the columns this rank owns and z / lambda at its rows (masks
 * set to 1 there), trace, status, iterations, objective, infeasibility. */
int dopf_cuda_part_finish(dopf_cuda_ctx* ctx, dopf_result_view* result, uint8_t* x_mask,
                          uint8_t* z_mask);

/* The library's own NCCL path (NCCL bound at run time: an NCCL the process
 * already holds, else libnccl.so.2 or $DOPF_NCCL_SO; failures are
 * DOPF_ERR_NCCL). One process per GPU: rank 0 makes the 128-byte id,
 * the caller broadcasts it out of band, every rank calls comm_init. One
 * process driving n GPUs (one context each): comm_init_all.
 * dopf_cuda_solve_part then runs the whole partitioned loop -- reset, u^0
 * exchange, and the iterations (kernels + one ncclAllGather of the packed
 * records) as ONE CUDA graph with a device-side while-node; if the
 * collective cannot be captured into a conditional body on some rank, all
 * ranks use a graph of 8 iterations relaunched behind a double-buffered,
 * non-blocking host poll (DOPF_PART_GRAPH=unrolled forces it). Outputs as
 * dopf_cuda_part_finish. The upload (dopf_cuda_upload_part) must be part
 * `rank` of `nranks`. Replaces the reference's WorkerPool fork-join
 * (parallel.cpp:88-120) across GPUs; same iterates as one GPU, bitwise. */
int dopf_nccl_unique_id(void* out128);
int dopf_cuda_comm_init(dopf_cuda_ctx* ctx, int32_t nranks, int32_t rank, const void* unique_id);
int dopf_cuda_comm_init_all(dopf_cuda_ctx** ctxs, int32_t n);
int dopf_cuda_comm_destroy(dopf_cuda_ctx* ctx);
int dopf_cuda_solve_part(dopf_cuda_ctx* ctx, const dopf_settings* settings, dopf_result_view* result,
                         uint8_t* x_mask, uint8_t* z_mask);
/* 0 no graph yet, 1 device while-node, 2 unrolled graph + lazy poll */
int dopf_cuda_part_graph_mode(const dopf_cuda_ctx* ctx);
/* Which NCCL is bound (path and version), or why none is. */
const char* dopf_nccl_describe(void);

/* Host-only helpers of the partitioned solve: the subsystem -> rank map
 * (contiguous, cost-balanced pieces of the depth-first component walk; every
 * rank computes the same), and one rank's layout sizes. */
int dopf_partition_subsystems(const dopf_model_view* model, int32_t nparts, int32_t* part_of_s);
/* Streaming layout of a model built on the host (no device): checks its
 * invariants (every row in exactly one chunk; staged chunks fit their stage;
 * image heads, row / column records and interior copy lists consistent;
 * imports are boundary columns) and returns, in out[0..11]: chunks, staged,
 * direct, boundary columns, import slots, largest staged stage (bytes), stage
 * limit, image bytes, rows, columns, interior copies, widest chunk (rows).
 * DOPF_ERR_LOGIC when an invariant fails. */
int dopf_stream_layout_check(const dopf_model_view* model, int64_t* out12);
int dopf_layout_probe_part(const dopf_model_view* model, int32_t nparts, int32_t part,
                           const int32_t* part_of_s, dopf_part_info* out);

/* Device layout of one model, computed on the host only (no GPU needed):
 * what dopf_cuda_upload would build for a device with `max_blocks` SMs and
 * `smem_limit` bytes of opt-in shared memory per CTA. */
typedef struct dopf_layout_stats {
  int32_t blocks;          /* CTAs for the instance                          */
  int32_t rows_per_thread; /* K: rows (and columns) per compute thread       */
  int32_t resident;        /* 1: every block's operators fit shared memory   */
  int32_t max_neighbours;  /* most blocks any block shares columns with      */
  int64_t smem_bytes;      /* largest block's shared-memory footprint        */
  int64_t remote_copies;   /* copy reads that cross blocks, per iteration    */
  int64_t local_copies;    /* copy reads served from the block's own rows    */
  int64_t exported_rows;   /* rows whose u is stored to global memory        */
  double bytes_per_iteration; /* algorithmic bytes     */
} dopf_layout_stats;
int dopf_layout_probe(const dopf_model_view* model, int32_t max_blocks, int64_t smem_limit,
                      dopf_layout_stats* out);
/* Same for a scenario batch (dopf_cuda_upload_batch's layout: one shared
 * structure plan, <= 8 CTAs per scenario). */
int dopf_layout_probe_batch(const dopf_model_view* models, int32_t count, int64_t smem_limit,
                            dopf_layout_stats* out);

#ifdef __cplusplus
}
#endif

#endif /* DOPF_CUDA_H */
