// Device layout of the HBM-streaming solver path (stream_kernels.cu), used
// for instances whose operators do not fit the CTAs' shared memory (the
// tiled 0.5M-bus feeder: ~10.7M local variables, ~1.5 GB of operators).
//
//  * Subsystems in the depth-first locality order (layout_builder.cpp) are
//    cut into chunks of at most kStreamRows rows; one CTA processes one chunk
//    per iteration (thread = row), so subsystem targets stay in shared memory.
//  * P and A rows are sliced ELL per warp (entry j of lane l at
//    slice + 32 j + l): every warp load is 256 contiguous bytes of HBM.
//  * Columns keep the reference's CSR scatter (copies in ascending s) over
//    device rows, so the global update sums in the reference order.
//  * Partitioned (multi-rank) layouts hold the rank's subsystems only; copies
//    held by other ranks are read from a gathered "remote" array.
#pragma once

#include <cstdint>
#include <vector>

#include "../../../include/dopf_types.h"

namespace dopf::cuda {

constexpr int kStreamRows = 512;  // threads per CTA of the streaming kernels (>= widest subsystem)

struct StreamRow {
  int32_t n;      // n_s
  int32_t base;   // chunk-local row of (s, 0)
  int32_t xcol;   // column index (into the rank's column arrays) of l2g(s, i)
  int32_t pad;
};

struct StreamARow {
  int32_t n;      // n_s (0: no equality row for this thread)
  int32_t base;   // chunk-local row of (s, 0)
};

struct StreamChunk {
  int32_t row0;   // first device row
  int32_t rows;
  int32_t arow0;  // first equality row
  int32_t arows;
  int32_t icol0;  // first interior column (all copies in this chunk): updated by k_local
  int32_t icols;
  int32_t icopy0; // their copies: [icopy0, icopy0 + icopies) of `copies` (<= rows)
  int32_t icopies;
  int64_t p0, p1; // the chunk's P slab [p0, p1) and A slab [a0, a1) (doubles): bulk-prefetched to L2
  int64_t a0, a1;
};

struct StreamLayout {
  int32_t S = 0, n = 0, N_z = 0;       // whole model
  int32_t rows = 0;                    // device rows (this rank)
  int32_t cols = 0;                    // columns this rank updates
  int32_t bcols = 0;                   // boundary columns [0, bcols): copies in >1 chunk or remote
  std::vector<StreamChunk> chunks;
  std::vector<StreamRow> rmeta;        // per device row
  std::vector<int64_t> pslice;         // per warp-slice of rows: offset into P
  std::vector<int64_t> aslice;         // per warp-slice of equality rows: offset into A
  std::vector<StreamARow> ameta;       // per equality row (chunk-major)
  std::vector<double> P, A, ab, v, z0;
  std::vector<int32_t> ref_of_dev;     // device row -> reference z index
  // columns: CSR over copies; copy >= 0: device row, < 0: -(remote slot + 1)
  std::vector<int32_t> col_ptr, copies, gcol;
  std::vector<double> c, inv, lo, hi, x0;
  std::vector<uint8_t> owner;          // 1: this rank writes x and adds c x to the objective
  int32_t remote_slots = 0;            // partitioned: size of the gathered remote u array
  double bytes_per_iteration = 0;      // algorithmic bytes of this rank's share
  // partitioned exchange: this rank's exported rows (u packed into slot
  // part * max_export + e of every rank's remote array, in this order)
  int32_t nparts = 1, part = 0, max_export = 0;
  std::vector<int32_t> export_rows;
  // re-upload fast path: where every packed value comes from in the model
  // view (P / A / b indices, -1 = zero padding) and the structure signature
  std::vector<int64_t> p_src, a_src, ab_src;
  std::vector<int32_t> sig_z_offsets, sig_m_s, sig_l2g, sig_csr_ptr, sig_csr_copy;
  bool same_structure(const dopf_model_view& m) const;
};

/// Whole-model streaming layout (one rank).
StreamLayout build_stream_layout(const dopf_model_view& m);

/// Partitioned layout: part `part` of `nparts`, subsystem s on part
/// part_of_s[s]. Columns referenced by this part's rows are updated here;
/// copies held by other parts are read from the gathered remote array. Every
/// part derives the same export lists from the whole model, so slots agree.
StreamLayout build_stream_layout_part(const dopf_model_view& m, int nparts, int part,
                                      const int32_t* part_of_s);

}  // namespace dopf::cuda
