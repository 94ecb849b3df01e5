// Device layout of one or more ADMM instances (POD structs shared by the
// host-side builder, layout.cpp, and the sm_100a kernels, admm_kernels.cu).
//
// HBM / shared-memory layout:
//  * Subsystems are ordered by a depth-first walk of the component graph
//    (two subsystems are adjacent when they hold copies of the same global
//    column) and the walk is cut into contiguous pieces, one per CTA
//    ("block"), balanced by operator bytes. Most consensus columns then have
//    all their copies inside one block, and a block shares columns with only
//    a handful of others (its "neighbours"). Inside a block subsystems are
//    reordered by n_s (descending) so warps see uniform GEMV lengths.
//  * A "device row" is one local variable (s, i). z, lambda and the exchange
//    value u = z - lambda/rho are stored in device-row order.
//  * P_s and A_s rows are packed per block in sliced-ELL order: the rows a
//    warp owns in one thread slot form a slice, stored entry-major (entry j
//    of lane l at slice_off + 32 j + l, zero-padded to the slice's widest
//    row), so each step j of a warp reads 256 contiguous bytes (coalesced in
//    HBM, conflict-free in smem).
//  * Each block computes the global update x_i for every column its rows
//    reference, from the copies' u values (CSR by column, ascending s, the
//    reference's summation order): copies held by the block itself are read
//    from shared memory, copies of other blocks from L2 after that block's
//    "u(t) published" flag. Only rows some other block reads ("exported"
//    rows) are written to global memory. Each block waits for its neighbours
//    only -- no grid-wide barrier on the critical path -- and the result is
//    bitwise deterministic.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define DOPF_HD __host__ __device__
#else
#define DOPF_HD
#endif

namespace dopf::cuda {

constexpr int kThreads = 512;   // CTA size of the iteration kernels
// warp 0: service (exchange flags, residual combine, stop test); warp 1: the
// equality check ||A z - b||_inf; warps 2..: compute (rows, columns)
constexpr int kComputeThreads = kThreads - 64;
constexpr int kMaxK = 4;        // max rows (and cols, A-rows) per thread
constexpr int kPartials = 8;    // gap, step, bx2, z2, lam2, objective, maxinf, pad

struct BlockDesc {
  int32_t row0;        // first device row of this block (global across instances)
  int32_t rows;        // local variables owned
  int32_t cols;        // global columns referenced (x computed here)
  int32_t arows;       // equality rows (A-tasks)
  int64_t p_off;       // block's packed P in the global P array
  int64_t a_off;       // block's packed A in the global A array
  int32_t p_len;       // doubles
  int32_t a_len;       // doubles
  int32_t copy_off;    // block's copy list in the global copies array
  int32_t copy_len;
  int32_t col_off;     // block's column metadata
  int32_t amet_off;    // block's A-task metadata
  int32_t ops_in_smem; // 1: P and A staged in shared memory once, 0: read from HBM/L2
  int32_t instance;
  int32_t inst_block;  // index of this block within its instance
  int32_t nbr_off;     // neighbour list (instance-local block indices) in the global nbrs array
  int32_t nbr_cnt;
  int32_t cols_int;    // columns [0, cols_int) have every copy in this block; the rest are boundary
  int32_t pad;
};

struct InstDesc {
  int64_t x_off;       // instance's x in the global x array
  int32_t n;           // global columns
  int32_t blocks;      // CTAs cooperating on this instance
  int32_t block0;      // first block
  int32_t rows;        // N_z of the instance
  int64_t trace_off;   // rows of 6 doubles
  int32_t row0;        // first device row
  int32_t pad;
};

// Row task: z_i = sum_j P(i,j) t_j + v_i for one (s, i).
struct RowMeta {
  int32_t pofs;      // slice_off + lane: entry j of this row at pofs + 32 j in the block's P
  int16_t n;         // n_s
  int16_t exported;  // 1: another block reads this row's u (store it to global memory)
  int32_t base;      // block-local row index of (s, 0)
  int32_t xloc;      // block-local column index of local_to_global(s, i)
};

// Copy reference in a block's copy list: >= 0 is a block-local row (u read
// from shared memory), < 0 encodes global device row -(ref + 1) (u read from
// L2 after the owning block's flag).
DOPF_HD inline int32_t encode_remote(int32_t dev_row) { return -(dev_row + 1); }
DOPF_HD inline int32_t decode_remote(int32_t ref) { return -ref - 1; }

// Column task: x_c from its copies.
struct ColMeta {
  int32_t gcol;        // global column (within the instance)
  int32_t copy_start;  // in the block's copy list
  int32_t copy_count;
  int32_t owner;       // 1: this block writes x and adds c*x to the objective
};

// Equality-check task: |A_r z_s - b_r| for one reduced row of a subsystem.
struct AMeta {
  int32_t aofs;   // slice_off + lane: entry j of this row at aofs + 32 j in the block's A
  int32_t m;      // m_s
  int32_t n;      // n_s
  int32_t base;   // block-local row index of (s, 0)
};

}  // namespace dopf::cuda
