#include "stream_layout.hpp"

#include <algorithm>
#include <cstring>
#include <climits>
#include <cstdint>
#include <stdexcept>

#include "layout_builder.hpp"

namespace dopf::cuda {

bool StreamLayout::same_structure(const dopf_model_view& m) const {
  auto eq = [](const std::vector<int32_t>& v, const int32_t* p, std::size_t n) {
    return v.size() == n && (n == 0 || std::memcmp(v.data(), p, n * sizeof(int32_t)) == 0);
  };
  return nparts == 1 && m.has_pre && S == m.S && n == m.n && N_z == m.N_z &&
         eq(sig_z_offsets, m.z_offsets, m.S + 1) && eq(sig_m_s, m.m_s, m.S) &&
         eq(sig_l2g, m.l2g, m.N_z) && eq(sig_csr_ptr, m.csr_ptr, m.n + 1) &&
         eq(sig_csr_copy, m.csr_copy, m.N_z);
}

StreamLayout build_stream_layout(const dopf_model_view& m) {
  return build_stream_layout_part(m, 1, 0, nullptr);
}

StreamLayout build_stream_layout_part(const dopf_model_view& m, int nparts, int part,
                                      const int32_t* part_of_s) {
  if (!m.has_pre) throw std::invalid_argument("model view lacks precomputed operators");
  if (nparts < 1 || part < 0 || part >= nparts || (nparts > 1 && !part_of_s))
    throw std::invalid_argument("bad partition");
  auto part_of = [&](int s) { return nparts == 1 ? 0 : part_of_s[s]; };
  for (int s = 0; s < m.S; ++s)
    if (part_of(s) < 0 || part_of(s) >= nparts) throw std::invalid_argument("subsystem part out of range");
  StreamLayout L;
  L.S = m.S;
  L.n = m.n;
  L.N_z = m.N_z;
  L.nparts = nparts;
  L.part = part;
  std::vector<int> order;
  for (int s : locality_order(m))
    if (part_of(s) == part) order.push_back(s);
  auto ns_of = [&](int s) { return m.z_offsets[s + 1] - m.z_offsets[s]; };
  for (int s = 0; s < m.S; ++s)
    if (ns_of(s) > kStreamRows) throw std::invalid_argument("subsystem wider than a streaming chunk");

  // chunks of whole subsystems, <= kStreamRows rows (and equality rows)
  std::vector<int32_t> dev_of_ref(m.N_z, -1);
  struct Src { int64_t at; int n; int base; };
  std::vector<Src> prow, arow;
  int32_t row = 0;
  std::size_t k = 0;
  std::vector<int> members;
  while (k < order.size()) {
    StreamChunk ch{};
    ch.row0 = row;
    ch.arow0 = static_cast<int32_t>(arow.size());
    // the chunk's subsystems: the next run of the locality walk that fits
    int rows = 0, arows = 0;
    members.clear();
    while (k < order.size()) {
      const int s = order[k];
      const int n = ns_of(s), ms = m.m_s[s];
      if (rows + n > kStreamRows || arows + ms > kStreamRows) break;
      members.push_back(s);
      rows += n;
      arows += ms;
      ++k;
    }
    // widest first inside the chunk: the 32 rows of a warp slice then have
    // (nearly) equal n_s, so the sliced-ELL padding -- which still costs
    // DRAM sectors -- stays small
    std::stable_sort(members.begin(), members.end(), [&](int a, int b) { return ns_of(a) > ns_of(b); });
    rows = 0;
    for (int s : members) {
      const int n = ns_of(s), ms = m.m_s[s];
      for (int i = 0; i < n; ++i) {
        dev_of_ref[m.z_offsets[s] + i] = row + rows + i;
        prow.push_back(Src{m.p_offsets[s] + static_cast<int64_t>(i) * n, n, rows});
      }
      for (int r = 0; r < ms; ++r) {
        arow.push_back(Src{m.a_offsets[s] + static_cast<int64_t>(r) * n, n, rows});
        L.ab.push_back(m.b[m.b_offsets[s] + r]);
        L.ab_src.push_back(m.b_offsets[s] + r);
      }
      rows += n;
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
  std::vector<int> s_of_ref(m.N_z);
  for (int s = 0; s < m.S; ++s)
    for (int k2 = m.z_offsets[s]; k2 < m.z_offsets[s + 1]; ++k2) s_of_ref[k2] = s;

  // columns updated here: every column a local row references, ordered by
  // their first local copy's device row (ties by column) -- the global update
  // then walks u and the local update gathers x in near-sequential order
  // Boundary columns (copies in several chunks, or on other parts) come
  // first; interior columns follow grouped by their chunk.
  std::vector<int32_t> loc_of_col(m.n, -1);
  {
    std::vector<int32_t> chunk_of_row(row);
    for (std::size_t q = 0; q < L.chunks.size(); ++q)
      for (int r = 0; r < L.chunks[q].rows; ++r) chunk_of_row[L.chunks[q].row0 + r] = static_cast<int32_t>(q);
    std::vector<int32_t> first_row(m.n, INT32_MAX), chunk_of_col(m.n, -1);
    std::vector<char> boundary(m.n, 0);
    for (int ref = 0; ref < m.N_z; ++ref) {
      const int32_t d = dev_of_ref[ref], gc = m.l2g[ref];
      if (d < 0) continue;
      first_row[gc] = std::min(first_row[gc], d);
      if (chunk_of_col[gc] < 0) chunk_of_col[gc] = chunk_of_row[d];
      else if (chunk_of_col[gc] != chunk_of_row[d]) boundary[gc] = 1;
    }
    for (int c = 0; c < m.n; ++c) {
      if (first_row[c] == INT32_MAX) continue;
      for (int q = m.csr_ptr[c]; q < m.csr_ptr[c + 1]; ++q)
        if (dev_of_ref[m.csr_copy[q]] < 0) boundary[c] = 1;  // a copy on another part
      L.gcol.push_back(c);
    }
    std::stable_sort(L.gcol.begin(), L.gcol.end(), [&](int32_t a, int32_t b) {
      return boundary[a] != boundary[b] ? boundary[a] > boundary[b] : first_row[a] < first_row[b];
    });
    for (std::size_t q = 0; q < L.gcol.size(); ++q) {
      const int32_t gc = L.gcol[q];
      loc_of_col[gc] = static_cast<int32_t>(q);
      if (boundary[gc]) {
        L.bcols = static_cast<int32_t>(q) + 1;
        continue;
      }
      StreamChunk& ch = L.chunks[chunk_of_col[gc]];
      if (ch.icols == 0) ch.icol0 = static_cast<int32_t>(q);
      ++ch.icols;
    }
  }
  for (int ref = 0; ref < m.N_z; ++ref) {
    const int32_t d = dev_of_ref[ref];
    if (d < 0) continue;
    L.ref_of_dev[d] = ref;
    L.v[d] = m.v[ref];
    L.z0[d] = m.z0[ref];
    L.rmeta[d] = StreamRow{prow[d].n, prow[d].base, loc_of_col[m.l2g[ref]], 0};
  }
  // sliced ELL per chunk-local warp (rows of a warp never span chunks)
  auto pack = [](const std::vector<Src>& rows, const std::vector<StreamChunk>& chunks, bool arow_mode,
                 std::vector<double>& out, std::vector<int64_t>& slices, const double* src,
                 std::vector<int64_t>& srcidx) {
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
            srcidx.push_back(ok ? rows[first + w0 + l].at + j : -1);
          }
      }
    }
  };
  pack(prow, L.chunks, false, L.P, L.pslice, m.P, L.p_src);
  pack(arow, L.chunks, true, L.A, L.aslice, m.A, L.a_src);
  for (std::size_t c = 0; c < L.chunks.size(); ++c) {
    const std::size_t w = c * (kStreamRows / 32), wn = (c + 1) * (kStreamRows / 32);
    L.chunks[c].p0 = L.pslice[w];
    L.chunks[c].p1 = wn < L.pslice.size() ? L.pslice[wn] : static_cast<int64_t>(L.P.size());
    L.chunks[c].a0 = L.aslice[w];
    L.chunks[c].a1 = wn < L.aslice.size() ? L.aslice[wn] : static_cast<int64_t>(L.A.size());
  }
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

  // exports of every part (identical on all parts): copies of columns held by
  // more than one part, ascending reference index per part
  std::vector<std::vector<int32_t>> exports(nparts);
  std::vector<int32_t> slot_of_ref(m.N_z, -1);
  if (nparts > 1) {
    std::vector<char> multi(m.n, 0);
    for (int c = 0; c < m.n; ++c) {
      const int p0 = part_of(s_of_ref[m.csr_copy[m.csr_ptr[c]]]);
      for (int q = m.csr_ptr[c]; q < m.csr_ptr[c + 1]; ++q)
        if (part_of(s_of_ref[m.csr_copy[q]]) != p0) multi[c] = 1;
    }
    for (int ref = 0; ref < m.N_z; ++ref)
      if (multi[m.l2g[ref]]) exports[part_of(s_of_ref[ref])].push_back(ref);
    for (const auto& e : exports) L.max_export = std::max<int32_t>(L.max_export, static_cast<int32_t>(e.size()));
    for (int q = 0; q < nparts; ++q)
      for (std::size_t e = 0; e < exports[q].size(); ++e)
        slot_of_ref[exports[q][e]] = q * L.max_export + static_cast<int32_t>(e);
    for (int32_t ref : exports[part]) L.export_rows.push_back(dev_of_ref[ref]);
    L.remote_slots = nparts * L.max_export;
  }

  // columns: CSR over copies in ascending s; local copies -> device rows,
  // copies of other parts -> remote slots
  L.cols = static_cast<int32_t>(L.gcol.size());
  L.col_ptr.assign(1, 0);
  double msum = 0, n2 = 0, mn = 0;
  for (const StreamChunk& ch : L.chunks) msum += ch.arows;
  for (int32_t gc : L.gcol) {
    for (int q = m.csr_ptr[gc]; q < m.csr_ptr[gc + 1]; ++q) {
      const int ref = m.csr_copy[q];
      if (part_of(s_of_ref[ref]) == part) {
        L.copies.push_back(dev_of_ref[ref]);
      } else {
        if (slot_of_ref[ref] < 0) throw std::logic_error("remote copy without an export slot");
        L.copies.push_back(-(slot_of_ref[ref] + 1));
      }
    }
    L.col_ptr.push_back(static_cast<int32_t>(L.copies.size()));
    L.c.push_back(m.c[gc]);
    L.inv.push_back(m.inv_copy[gc]);
    L.lo.push_back(m.x_lo[gc]);
    L.hi.push_back(m.x_hi[gc]);
    L.x0.push_back(m.x0[gc]);
    L.owner.push_back(part_of(s_of_ref[m.csr_copy[m.csr_ptr[gc]]]) == part ? 1 : 0);
  }
  for (StreamChunk& ch : L.chunks) {
    ch.icopy0 = ch.icols ? L.col_ptr[ch.icol0] : 0;
    ch.icopies = ch.icols ? L.col_ptr[ch.icol0 + ch.icols] - ch.icopy0 : 0;
    if (ch.icopies > ch.rows) throw std::logic_error("interior copies exceed the chunk's rows");
  }
  for (int s : order) {
    const double n = ns_of(s);
    n2 += n * n;
    mn += m.m_s[s] * n;
  }
  // algorithmic bytes of this part (DESIGN.md section 4 restricted to it)
  if (nparts == 1) {  // signature for the re-upload fast path
    L.sig_z_offsets.assign(m.z_offsets, m.z_offsets + m.S + 1);
    L.sig_m_s.assign(m.m_s, m.m_s + m.S);
    L.sig_l2g.assign(m.l2g, m.l2g + m.N_z);
    L.sig_csr_ptr.assign(m.csr_ptr, m.csr_ptr + m.n + 1);
    L.sig_csr_copy.assign(m.csr_copy, m.csr_copy + m.N_z);
  }
  L.bytes_per_iteration = 8.0 * (n2 + mn + msum) + 56.0 * L.rows + 48.0 * L.cols +
                          4.0 * (2.0 * L.rows + L.cols + 1) + 16.0 * static_cast<double>(order.size());
  return L;
}

}  // namespace dopf::cuda
