/* C ABI of the host front-end: feeder loading, LP assembly, decomposition
 * and the one-time precompute. These are the inputs of the drop-in solver
 * boundary (dopf_cuda.h). Each entry point replaces one reference C++ call:
 *
 *   dopf_feeder_parse / _parse_file  <- parse_feeder / parse_feeder_file
 *                                       (proj/include/dopf/feeder.hpp:114-115)
 *   dopf_feeder_serialize            <- serialize_feeder (feeder.hpp:118)
 *   dopf_feeder_validate             <- validate_feeder (feeder.hpp:122)
 *   dopf_lp_assemble                 <- assemble_centralized (lp_builder.hpp:57)
 *   dopf_lp_dump                     <- dump_linear_system (linear_system.hpp:79)
 *   dopf_model_decompose             <- decompose (decompose.hpp:90-91)
 *   dopf_model_precompute            <- precompute (admm.hpp:52)
 *   dopf_model_dump_subsystems       <- dump_subsystems (decompose.hpp:94)
 *
 * Errors: every int-returning function returns a dopf_status; the message of
 * the most recent failure on the calling thread is dopf_last_error().
 */
#ifndef DOPF_HOST_H
#define DOPF_HOST_H

#include "dopf_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dopf_feeder dopf_feeder;
typedef struct dopf_lp dopf_lp;
typedef struct dopf_model dopf_model;

const char* dopf_last_error(void);

/* ---- feeder (L0) ---- */
int dopf_feeder_parse(const char* text, size_t len, dopf_feeder** out);
int dopf_feeder_parse_file(const char* path, dopf_feeder** out);
/* shape: "ieee13" | "ieee123" | "ieee8500" (synthetic, Table I-III counts) */
int dopf_feeder_synthetic(const char* shape, uint64_t seed, dopf_feeder** out);
/* `copies` tiles of `shape` tied to one root bus (BASELINE config 4) */
int dopf_feeder_synthetic_tiled(const char* shape, int32_t copies, uint64_t seed, dopf_feeder** out);
/* every load's (a, b) scaled by U[0.5, 1.5] (BASELINE config 5 scenarios) */
int dopf_feeder_scale_loads(const dopf_feeder* base, uint64_t seed, dopf_feeder** out);
/* JSON text; writes up to cap bytes (NUL-terminated) and the full size to *needed */
int dopf_feeder_serialize(const dopf_feeder* f, char* buf, size_t cap, size_t* needed);
/* Diagnostics as "severity\tcomponent\tmessage\n" lines; *n_errors counts errors. */
int dopf_feeder_validate(const dopf_feeder* f, char* buf, size_t cap, size_t* needed,
                         int32_t* n_errors);
/* counts[0..4] = buses, generators, lines, loads, merged leaves */
int dopf_feeder_counts(const dopf_feeder* f, int32_t* counts);
void dopf_feeder_free(dopf_feeder* f);

/* ---- centralized LP (L1) ---- */
typedef struct dopf_lp_view {
  int32_t rows, cols, nnz, reserved;
  const int32_t* row_ptr; /* rows+1 */
  const int32_t* col_idx; /* nnz    */
  const double* values;   /* nnz    */
  const double* b;        /* rows   */
  const double* c;        /* cols   */
  const double* x_lo;
  const double* x_hi;
  const int32_t* var_kind; /* cols: VarKind ordinal (p_gen=0 ... q_flow=8) */
} dopf_lp_view;

int dopf_lp_assemble(const dopf_feeder* f, dopf_lp** out);
int dopf_lp_view_get(const dopf_lp* lp, dopf_lp_view* out);
int dopf_lp_var_key(const dopf_lp* lp, int32_t col, char* buf, size_t cap);
int dopf_lp_row_tag(const dopf_lp* lp, int32_t row, char* buf, size_t cap);
int dopf_lp_dump(const dopf_lp* lp, char* buf, size_t cap, size_t* needed);
void dopf_lp_free(dopf_lp* lp);

/* ---- decomposed model (L2) + precompute (L3 setup) ---- */
int dopf_model_decompose(const dopf_lp* lp, const dopf_feeder* f, double tol, int32_t workers,
                         dopf_model** out);
/* Partition only (no row reduction), as `dopf inspect` does before reduce. */
int dopf_model_partition(const dopf_lp* lp, const dopf_feeder* f, dopf_model** out);
int dopf_model_reduce(dopf_model* m, double tol, int32_t workers);
/* Build a model directly from dense data (test fixtures, reference
 * test_util.hpp:52-74 single_sub_model and multi-copy variants).
 * A is packed per subsystem row-major; is_w[n] marks squared-voltage columns
 * (initial value 1.0). */
int dopf_model_from_arrays(int32_t S, int32_t n, const int32_t* z_offsets, const int32_t* l2g,
                           const int32_t* m_s, const double* A, const double* b,
                           const double* c, const double* x_lo, const double* x_hi,
                           const int32_t* is_w, dopf_model** out);
int dopf_model_precompute(dopf_model* m, int32_t workers);
/* Adopt operators computed elsewhere (dopf_cuda_precompute): P (row-major
 * n_s x n_s per subsystem, p_offsets order) and v (N_z); copy counts and the
 * CSR scatter are built here exactly as dopf_model_precompute does. */
int dopf_model_set_operators(dopf_model* m, const double* P, const double* v);
/* Feeder helpers the reference exposes (feeder.hpp:104-110, lp_builder.hpp:49):
 * load coefficients {a, b, alpha, beta} of a canonical load kind
 * (0 constant power, 1 constant current, 2 constant impedance), and a line's
 * voltage-drop sensitivities M^p, M^q (np x np row-major; r, x likewise;
 * phases ascending, a subset of {1, 2, 3}). */
int dopf_derive_load_coefficients(double p_ref, double q_ref, int32_t kind, double* out);
int dopf_line_m_matrices(int32_t np, const int32_t* phases, const double* r, const double* x,
                         double* mp, double* mq);
/* Replaces every subsystem's rows by reduced ones laid out in the model's
 * CURRENT (unreduced) slots: the first m_s[s] x n_s of A's slot s, the first
 * m_s[s] of b's (the output of dopf_cuda_prepare); the GPU-side equivalent
 * of dopf_model_reduce. Drops precomputed operators. */
int dopf_model_set_reduced(dopf_model* m, const double* A, const double* b, const int32_t* m_s);
int dopf_model_view_get(const dopf_model* m, dopf_model_view* out);
int dopf_model_component_id(const dopf_model* m, int32_t s, char* buf, size_t cap);
int dopf_model_rows_before_reduction(const dopf_model* m, int32_t* out /* S */);
int dopf_model_dump_subsystems(const dopf_model* m, char* buf, size_t cap, size_t* needed);
void dopf_model_free(dopf_model* m);

/* ---- writers (reference admm.hpp:128-133) ---- */
int dopf_write_trace_csv(const double* trace, int32_t rows, char* buf, size_t cap, size_t* needed);
int dopf_write_solution(const dopf_lp* lp, const double* x, char* buf, size_t cap, size_t* needed);

#ifdef __cplusplus
}
#endif

#endif /* DOPF_HOST_H */
