/* CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C++ restatement of the reference's CPU path for the hot loop, used
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm as the CHECKER and the CPU baseline. Nothing in the product
 * (paper_2501_08293_b200/) links, loads or calls this library.
 *
 *   oracle_solve            <- dopf::solve, proj/src/admm.cpp:172-244
 *                              (global :118-129, local :131-138, dual :140-143,
 *                              residuals :145-170, objective :223-224),
 *                              with the WorkerPool fork-join of parallel.cpp
 *   oracle_reference_solve  <- dopf::reference_solve, proj/src/oracle.cpp:164-273
 *   oracle_check_feasibility<- dopf::check_feasibility, oracle.cpp:10-43
 *   oracle_reconstruct      <- dopf::reconstruct_centralized, oracle.cpp:275-292
 *
 * Parity pinning: the reference cannot be compiled here (Eigen3 and vendor/
 * are absent), so this restatement is pinned to the
 * reference's own known answers: the frozen LP objectives of
 * proj/tests/test_oracle.cpp:23-29, the ADMM objective tolerance of
 * test_oracle.cpp:216-229 / test_admm.cpp:346-358, the KATs of
 * test_admm.cpp:53-418 and the acceptance criteria of acceptance.cpp:89-393
 * (see tests/test_oracle_pinning.py).
 */
#ifndef DOPF_ORACLE_H
#define DOPF_ORACLE_H

#include "../include/dopf_host.h"
#include "../include/dopf_types.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* Sequential-order restatement of the solve loop. The model view must carry
 * the precomputed operators (has_pre == 1). Snapshots (x, z, z_prev, lambda
 * after iteration t) are written for every t listed in snap_iters (ascending,
 * 1-based) that the run reaches; pass n_snap = 0 to skip. */
int oracle_solve(const dopf_model_view* model, const dopf_settings* settings,
                 dopf_result_view* result, const int32_t* snap_iters, int32_t n_snap,
                 double* snap_x, double* snap_z, double* snap_zprev, double* snap_lambda);

/* Dense bounded two-phase simplex with Bland's rule. status: 0 optimal,
 * 1 infeasible, 2 unbounded. x has lp->cols entries. */
int oracle_reference_solve(const dopf_lp_view* lp, int32_t max_cols, double* x,
                           double* objective, int32_t* status, double* kkt_residual,
                           int32_t* pivots);

int oracle_check_feasibility(const dopf_lp_view* lp, const double* x, double* max_eq_violation,
                             double* max_bound_violation, int32_t* worst_row, int32_t* worst_col,
                             double* objective);

int oracle_reconstruct(const dopf_model_view* model, const double* x, const double* z,
                       double* out);

/* Single iteration steps (admm_steps.cpp), for the reference's per-function
 * known-answer tests (proj/tests/test_admm.cpp:113-303). */
int oracle_global_update(const dopf_model_view* model, const double* z, const double* lambda,
                         double rho, double* x);
int oracle_local_update(const dopf_model_view* model, int32_t s, const double* x,
                        const double* lambda_s, double rho, double* z_s);
int oracle_dual_update(const dopf_model_view* model, int32_t s, const double* x,
                       const double* z_s, double* lambda_s, double rho);
/* out4 = {pres, dres, eps_prim, eps_dual} */
int oracle_residuals(const dopf_model_view* model, const double* x, const double* z,
                     const double* z_prev, const double* lambda, double rho, double eps_rel,
                     double* out4);

#ifdef __cplusplus
}
#endif

#endif
