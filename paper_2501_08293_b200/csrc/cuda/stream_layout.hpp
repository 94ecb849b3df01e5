// Device layout of the HBM-streaming solver path (stream_kernels.cu), used
// for instances whose operators do not fit the CTAs' shared memory (the
// tiled 0.5M-bus feeder: ~10.7M local variables, ~1.5 GB of operators).
//
//  * Subsystems in the depth-first locality order (layout_builder.cpp) are
//    cut into chunks of whole subsystems (thread = row inside a chunk).
//  * Everything a chunk reads that does not change between iterations -- its
//    P and A rows (sliced ELL per warp: entry j of lane l at slice + 32 j + l),
//    v, b, row and equality-row metadata, and the data of its interior
//    columns -- is packed into one contiguous, 16-byte aligned chunk IMAGE.
//    The staged kernel moves a chunk with four bulk copies (image, z slice,
//    lambda slice, imported boundary x): the bulk-copy engine's cost is per
//    copy, not per byte.
//  * Columns keep the reference's CSR scatter (copies in ascending s).
//    Columns whose copies all sit in one chunk ("interior") are updated by
//    that chunk's CTA from the z, lambda it loads anyway; only the boundary
//    columns [0, bcols) -- copies in several chunks or on other ranks -- take
//    the separate global-update kernel, which also writes each boundary x
//    into the import slots of the chunks that read it.
//  * Partitioned (multi-rank) layouts hold the rank's subsystems only; copies
//    held by other ranks are read from a gathered "remote" array.
#pragma once

#include <cstdint>
#include <vector>

#include "../../../include/dopf_types.h"
#include "layout.hpp"

namespace dopf::cuda {

constexpr int kStreamRows = 512;   // direct-load kernel threads (and k_global's CTA size)
constexpr int kWideRows = 1024;    // rows of the widest chunk: a wide (hub) subsystem gets a 1024-thread direct-load CTA
// staged kernel: chunks of <= kStagedRows rows whose shared-memory stage
// (image + z + lambda + imports) fits `stage_bytes`; `stages` stages per CTA
#ifndef DOPF_STAGED_ROWS
#define DOPF_STAGED_ROWS 256
#endif
constexpr int kStagedRows = DOPF_STAGED_ROWS;
constexpr int kMaxStages = 8;
constexpr int kDefaultStages = 2;
constexpr int kDefaultStageBytes = 48 * 1024;

struct StreamRow {   // one row of a chunk image (16 bytes: one 128-bit shared-memory load)
  int16_t n;         // n_s
  int16_t base;      // chunk-local row of (s, 0)
  int16_t xloc;      // interior column: index among the chunk's interior columns, else -1
  int16_t xin;       // boundary column: slot in the chunk's import list, else -1
  double v;          // min-norm shift v_s entry (admm.cpp:137)
};
static_assert(sizeof(StreamRow) == 16, "StreamRow is 16 bytes");

struct StreamARow {  // one equality row (16 bytes)
  int32_t n;         // n_s
  int32_t base;      // chunk-local row of (s, 0)
  double b;          // b_s entry
};
static_assert(sizeof(StreamARow) == 16, "StreamARow is 16 bytes");

struct StreamCol {   // one interior column (32 bytes)
  double cost, inv, lo, hi;
};

struct StreamChunk {
  int32_t row0;   // first device row
  int32_t rows;
  int32_t arows;  // equality rows
  int32_t icol0;  // first interior column (all copies in this chunk)
  int32_t icols;
  int32_t bimp0;  // boundary-column imports: ximp[bimp0, bimp0 + nbimp)
  int32_t nbimp;
  int32_t image_bytes;
  int64_t image_off;  // byte offset of the chunk image in `blob`
};
static_assert(sizeof(StreamChunk) == 40, "StreamChunk layout");

// byte offsets of the sections of a chunk image (relative to its start)
enum ImageSection { kImgRows, kImgSlices, kImgP, kImgA, kImgArows, kImgCols, kImgCmeta, kImgCopies, kImgSections };
struct ChunkHead {                 // the first 64 bytes of every chunk image
  int32_t rows, arows, icols, nbimp;
  int32_t row0, icol0, bimp0, image_bytes;
  uint32_t off[kImgSections];      // byte offsets, 16-byte aligned
};
static_assert(sizeof(ChunkHead) == 64, "ChunkHead is 64 bytes");
// rows: StreamRow per row; slices: per warp {int32 P offset, int32 A offset}
// (in doubles, from the P / A section starts); arows: StreamARow per equality
// row; cols: StreamCol per interior column; cmeta: per interior column
// first copy | count << 12 | owner << 31; copies: int16 chunk-local rows.
DOPF_HD constexpr int cmeta_start(uint32_t m) { return static_cast<int>(m & 0xfffu); }
DOPF_HD constexpr int cmeta_count(uint32_t m) { return static_cast<int>((m >> 12) & 0x7ffffu); }
DOPF_HD constexpr bool cmeta_owner(uint32_t m) { return (m >> 31) != 0; }

// Shared-memory stage of the staged kernel: the image, then the z and lambda
// slices and the import slots, each copied with its source start rounded
// down and end rounded up to 16 bytes (`shift` = first element's byte offset).
struct StageSeg {
  uint32_t dst, shift, bytes;
};
struct StagePlan {
  StageSeg z, lam, ximp;
  uint32_t total;
};

DOPF_HD inline StageSeg stage_seg(uint32_t& cursor, int64_t first, int64_t count, int es) {
  StageSeg s{cursor, 0u, 0u};
  if (count <= 0) return s;
  const int64_t b0 = first * es, b1 = (first + count) * es;
  const int64_t a0 = b0 & ~static_cast<int64_t>(15), a1 = (b1 + 15) & ~static_cast<int64_t>(15);
  s.shift = static_cast<uint32_t>(b0 - a0);
  s.bytes = static_cast<uint32_t>(a1 - a0);
  cursor += s.bytes;
  return s;
}

DOPF_HD inline void stage_plan(const StreamChunk& ch, StagePlan& sp) {
  uint32_t cur = static_cast<uint32_t>(ch.image_bytes);
  sp.z = stage_seg(cur, ch.row0, ch.rows, 8);
  sp.lam = stage_seg(cur, ch.row0, ch.rows, 8);
  sp.ximp = stage_seg(cur, ch.bimp0, ch.nbimp, 8);
  sp.total = cur;
}

constexpr int32_t kExchangePartials = 8;  // gap, step, bx2, z2, lam2, maxinf, c'x, spare

struct StreamLayout {
  int32_t S = 0, n = 0, N_z = 0;       // whole model
  int32_t rows = 0;                    // device rows (this rank)
  int32_t cols = 0;                    // columns this rank updates
  int32_t bcols = 0;                   // boundary columns [0, bcols)
  int32_t stages = kDefaultStages, stage_bytes = kDefaultStageBytes;  // staged-kernel pipeline
  std::vector<StreamChunk> chunks;
  std::vector<int32_t> staged_ids;     // chunks whose stage fits stage_bytes (staged kernel)
  std::vector<int32_t> big_ids;        // the rest (direct-load kernel, image read from HBM)
  std::vector<double> blob;            // chunk images (8-byte units; metadata bit-packed)
  std::vector<double> z0;              // per device row
  std::vector<int32_t> ref_of_dev;     // device row -> reference z index
  std::vector<int32_t> gcol;           // column -> global column
  std::vector<uint8_t> owner;          // per column: this rank writes x and adds c x to the objective
  // boundary columns: CSR over copies (copy >= 0: device row, < 0: -(remote slot + 1)) and data
  std::vector<int32_t> col_ptr, copies;
  std::vector<double> c, inv, lo, hi;
  std::vector<int32_t> bimp;           // import slot -> boundary column (per chunk, first-use order)
  std::vector<int32_t> imp_ptr, imp_slot;  // boundary column -> its import slots (CSR)
  int32_t remote_slots = 0;            // partitioned: size of the gathered remote u array
  double bytes_per_iteration = 0;      // algorithmic bytes of this rank's share
  // partitioned exchange: ONE gather per iteration of every rank's packed
  // record [u of its exported rows (max_export, zero padded) | its 8
  // residual partials]; rank q's exports land in slots q * xstride() + e of
  // every rank's remote array, its partials at q * xstride() + max_export
  int32_t nparts = 1, part = 0, max_export = 0;
  std::vector<int32_t> export_rows;
  int32_t xstride() const { return max_export + kExchangePartials; }
  // re-upload fast path: every model value the layout holds, as an index
  // into the concatenation raw = [P | A | b | v | z0 | c | inv_copy | x_lo | x_hi]
  // of the model view (blob_src: -1 zero padding, -2 metadata to keep)
  std::vector<int32_t> blob_src;
  int64_t raw_off[10] = {};            // section starts of raw (last = total)
  std::vector<int32_t> sig_z_offsets, sig_m_s, sig_l2g, sig_csr_ptr, sig_csr_copy, sig_part_of_s;
  /// m has the structure (and, partitioned, the partition) this layout was built for
  bool same_structure(const dopf_model_view& m, int nparts_ = 1, int part_ = 0,
                      const int32_t* part_of_s = nullptr) const;
};

enum RawSection { kRawP, kRawA, kRawB, kRawV, kRawZ0, kRawC, kRawInv, kRawLo, kRawHi, kRawEnd };

/// Section starts of the raw value concatenation of a model view.
void raw_offsets(const dopf_model_view& m, int64_t (&off)[10]);

/// Whole-model streaming layout (one rank).
StreamLayout build_stream_layout(const dopf_model_view& m);

/// Partitioned layout: part `part` of `nparts`, subsystem s on part
/// part_of_s[s]. Columns referenced by this part's rows are updated here;
/// copies held by other parts are read from the gathered remote array. Every
/// part derives the same export lists from the whole model, so slots agree.
StreamLayout build_stream_layout_part(const dopf_model_view& m, int nparts, int part,
                                      const int32_t* part_of_s);

}  // namespace dopf::cuda
