/* Plain-C data shared by the host front-end ABI (dopf_host.h), the CUDA
 * solver ABI (dopf_cuda.h) and the CPU oracle (oracle/oracle.h).
 *
 * Everything is flat arrays + sizes; no C++ or torch types cross the
 * boundary. Index conventions follow the reference's DecomposedModel
 * (proj/include/dopf/decompose.hpp:40-61) and Precomputed
 * (proj/include/dopf/admm.hpp:28-38).
 */
#ifndef DOPF_TYPES_H
#define DOPF_TYPES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes of every dopf_* entry point. */
enum dopf_status {
  DOPF_OK = 0,
  DOPF_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (settings, sizes)      */
  DOPF_ERR_SINGULAR = 2,         /* SingularSubsystemError (admm.hpp:40-47)       */
  DOPF_ERR_CUDA = 3,             /* CUDA runtime / launch failure                 */
  DOPF_ERR_NCCL = 4,             /* NCCL failure (partitioned multi-GPU)          */
  DOPF_ERR_OUT_OF_MEMORY = 5,    /* host or device allocation                     */
  DOPF_ERR_PARSE = 6,            /* ParseError (feeder.hpp:97-102)                */
  DOPF_ERR_INFEASIBLE = 7,       /* InfeasibleSubsystemError (decompose.hpp:63-70)*/
  DOPF_ERR_LOGIC = 8,            /* std::logic_error (zero-copy column, ...)      */
  DOPF_ERR_RUNTIME = 9           /* any other std::runtime_error                  */
};

/* Settings (reference admm.hpp:14-20). */
typedef struct dopf_settings {
  double rho;              /* consensus penalty, > 0              */
  double eps_rel;          /* relative termination tolerance, > 0 */
  int32_t max_iter;        /* >= 1                                */
  int32_t workers;         /* host threads for precompute/oracle  */
  int32_t record_iterates; /* oracle only: keep snapshots         */
  int32_t reserved;
} dopf_settings;

/* Read-only view of a decomposed + precomputed model. All arrays are owned
 * by whoever produced the view (dopf_model in dopf_host.h). */
typedef struct dopf_model_view {
  int32_t S;        /* subsystems                                   */
  int32_t n;        /* global columns                               */
  int32_t N_z;      /* stacked local variables = z_offsets[S]       */
  int32_t has_pre;  /* 1 when P, v, inv_copy, csr_* are populated   */
  const int32_t* z_offsets;  /* S+1                                  */
  const int32_t* l2g;        /* N_z: local_to_global, per s ascending */
  const int32_t* m_s;        /* S: rows after reduction               */
  const int64_t* a_offsets;  /* S+1: offsets into A (sum m_s*n_s)     */
  const double* A;           /* packed, per s row-major m_s x n_s     */
  const int32_t* b_offsets;  /* S+1: prefix sums of m_s               */
  const double* b;           /* packed rhs                            */
  const int64_t* p_offsets;  /* S+1: offsets into P (sum n_s^2)       */
  const double* P;           /* packed, per s row-major n_s x n_s     */
  const double* v;           /* N_z: minimum-norm shift               */
  const double* inv_copy;    /* n: 1 / copy count                     */
  const int32_t* csr_ptr;    /* n+1: copies of column i ...           */
  const int32_t* csr_copy;   /* N_z: ... as flat z indices, ascending s */
  const double* c;           /* n */
  const double* x_lo;        /* n (may hold +-inf) */
  const double* x_hi;        /* n */
  const double* x0;          /* n: initial global iterate (admm.cpp:92-116) */
  const double* z0;          /* N_z: initial locals                    */
} dopf_model_view;

/* Trace row layout: 6 doubles per iteration: t, pres, dres, eps_prim,
 * eps_dual, objective (reference TraceRow, admm.hpp:54-58). */
#define DOPF_TRACE_WIDTH 6

enum dopf_solve_status { DOPF_CONVERGED = 0, DOPF_ITERATION_LIMIT = 1 };

/* Caller-allocated outputs of a solve. Any pointer may be NULL. */
typedef struct dopf_result_view {
  double* x;       /* n     */
  double* z;       /* N_z   */
  double* lambda;  /* N_z   */
  double* trace;   /* DOPF_TRACE_WIDTH * max_iter */
  int32_t status;  /* dopf_solve_status */
  int32_t iterations;
  double objective;
  double max_local_infeasibility;
  /* timings in seconds (reference PhaseTimings, admm.hpp:104-106) */
  double time_precompute;
  double time_global;  /* device-side share of the iteration loop (GPU) */
  double time_local;
  double time_dual;
  double time_solve;   /* iteration loop wall time on the device (events) */
  double time_upload;  /* host -> device copies inside dopf_cuda_solve    */
  double time_download;
  /* stop tests (iterations 1..iterations) within 1e-12 relative of flipping:
   * the device sums residuals as trees, the reference sequentially, so a
   * non-zero count marks an iteration count that may depend on summation
   * order (hard part 2); first_near_tie = 0 if none */
  int32_t near_ties;
  int32_t first_near_tie;
} dopf_result_view;

#ifdef __cplusplus
}
#endif

#endif /* DOPF_TYPES_H */
