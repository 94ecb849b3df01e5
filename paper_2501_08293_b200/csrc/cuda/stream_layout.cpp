#include "stream_layout.hpp"

#include <algorithm>
#include <stdexcept>

#include "layout_builder.hpp"

namespace dopf::cuda {

StreamLayout build_stream_layout(const dopf_model_view& m) {
  if (!m.has_pre) throw std::invalid_argument("model view lacks precomputed operators");
  StreamLayout L;
  L.S = m.S;
  L.n = m.n;
  L.N_z = m.N_z;
  const std::vector<int> order = locality_order(m);
  auto ns_of = [&](int s) { return m.z_offsets[s + 1] - m.z_offsets[s]; };
  for (int s = 0; s < m.S; ++s)
    if (ns_of(s) > kStreamRows) throw std::invalid_argument("subsystem wider than a streaming chunk");

  // chunks of whole subsystems, <= kStreamRows rows (and equality rows)
  std::vector<int32_t> dev_of_ref(m.N_z, -1);
  struct Src { int64_t at; int n; int base; };
  std::vector<Src> prow, arow;
  int32_t row = 0;
  std::size_t k = 0;
  while (k < order.size()) {
    StreamChunk ch{};
    ch.row0 = row;
    ch.arow0 = static_cast<int32_t>(arow.size());
    int rows = 0, arows = 0;
    while (k < order.size()) {
      const int s = order[k];
      const int n = ns_of(s), ms = m.m_s[s];
      if (rows + n > kStreamRows || arows + ms > kStreamRows) break;
      for (int i = 0; i < n; ++i) {
        dev_of_ref[m.z_offsets[s] + i] = row + rows + i;
        prow.push_back(Src{m.p_offsets[s] + static_cast<int64_t>(i) * n, n, rows});
      }
      for (int r = 0; r < ms; ++r) {
        arow.push_back(Src{m.a_offsets[s] + static_cast<int64_t>(r) * n, n, rows});
        L.ab.push_back(m.b[m.b_offsets[s] + r]);
      }
      rows += n;
      arows += ms;
      ++k;
    }
    ch.rows = rows;
    ch.arows = arows;
    row += rows;
    L.chunks.push_back(ch);
  }
  L.rows = row;
  L.rmeta.resize(row);
  L.v.resize(row);
  L.z0.resize(row);
  L.ref_of_dev.resize(row);
  for (int ref = 0; ref < m.N_z; ++ref) {
    const int32_t d = dev_of_ref[ref];
    L.ref_of_dev[d] = ref;
    L.v[d] = m.v[ref];
    L.z0[d] = m.z0[ref];
    L.rmeta[d] = StreamRow{prow[d].n, prow[d].base, m.l2g[ref], 0};
  }
  // sliced ELL per chunk-local warp (rows of a warp never span chunks)
  auto pack = [](const std::vector<Src>& rows, const std::vector<StreamChunk>& chunks, bool arow_mode,
                 std::vector<double>& out, std::vector<int64_t>& slices, const double* src) {
    for (const StreamChunk& ch : chunks) {
      const int first = arow_mode ? ch.arow0 : ch.row0;
      const int count = arow_mode ? ch.arows : ch.rows;
      for (int w0 = 0; w0 < kStreamRows; w0 += 32) {
        slices.push_back(static_cast<int64_t>(out.size()));
        const int lanes = std::max(0, std::min(32, count - w0));
        int width = 0;
        for (int l = 0; l < lanes; ++l) width = std::max(width, rows[first + w0 + l].n);
        for (int j = 0; j < width; ++j)
          for (int l = 0; l < 32; ++l) {
            const bool ok = l < lanes && j < rows[first + w0 + l].n;
            out.push_back(ok ? src[rows[first + w0 + l].at + j] : 0.0);
          }
      }
    }
  };
  pack(prow, L.chunks, false, L.P, L.pslice, m.P);
  pack(arow, L.chunks, true, L.A, L.aslice, m.A);
  L.ameta.resize(static_cast<std::size_t>(L.chunks.size()) * kStreamRows);
  for (std::size_t c = 0; c < L.chunks.size(); ++c)
    for (int a = 0; a < kStreamRows; ++a) {
      StreamARow am{0, 0};
      if (a < L.chunks[c].arows) {
        const Src& s = arow[L.chunks[c].arow0 + a];
        am = StreamARow{s.n, s.base};
      }
      L.ameta[c * kStreamRows + a] = am;
    }
  // columns: all of them, CSR copies in ascending s -> device rows
  L.cols = m.n;
  L.col_ptr.assign(m.csr_ptr, m.csr_ptr + m.n + 1);
  L.copies.resize(m.N_z);
  for (int q = 0; q < m.N_z; ++q) L.copies[q] = dev_of_ref[m.csr_copy[q]];
  L.gcol.resize(m.n);
  for (int c = 0; c < m.n; ++c) L.gcol[c] = c;
  L.c.assign(m.c, m.c + m.n);
  L.inv.assign(m.inv_copy, m.inv_copy + m.n);
  L.lo.assign(m.x_lo, m.x_lo + m.n);
  L.hi.assign(m.x_hi, m.x_hi + m.n);
  L.x0.assign(m.x0, m.x0 + m.n);
  L.owner.assign(m.n, 1);
  L.bytes_per_iteration = algorithmic_bytes(m);
  return L;
}

}  // namespace dopf::cuda
