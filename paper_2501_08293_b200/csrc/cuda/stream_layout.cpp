#include "stream_layout.hpp"

#include <algorithm>
#include <functional>
#include <map>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "layout_builder.hpp"

namespace dopf::cuda {

bool StreamLayout::same_structure(const dopf_model_view& m, int nparts_, int part_,
                                  const int32_t* part_of_s) const {
  auto eq = [](const std::vector<int32_t>& v, const int32_t* p, std::size_t n) {
    return v.size() == n && (n == 0 || std::memcmp(v.data(), p, n * sizeof(int32_t)) == 0);
  };
  if (nparts_ != nparts || part_ != part) return false;
  if (nparts > 1 && (!part_of_s || !eq(sig_part_of_s, part_of_s, static_cast<std::size_t>(m.S)))) return false;
  return m.has_pre && S == m.S && n == m.n && N_z == m.N_z &&
         eq(sig_z_offsets, m.z_offsets, m.S + 1) && eq(sig_m_s, m.m_s, m.S) &&
         eq(sig_l2g, m.l2g, m.N_z) && eq(sig_csr_ptr, m.csr_ptr, m.n + 1) &&
         eq(sig_csr_copy, m.csr_copy, m.N_z);
}

void raw_offsets(const dopf_model_view& m, int64_t (&off)[10]) {
  const int64_t len[kRawEnd] = {m.p_offsets[m.S], m.a_offsets[m.S], m.b_offsets[m.S], m.N_z, m.N_z,
                                m.n, m.n, m.n, m.n};
  off[0] = 0;
  for (int i = 0; i < kRawEnd; ++i) off[i + 1] = off[i] + len[i];
}

StreamLayout build_stream_layout(const dopf_model_view& m) {
  return build_stream_layout_part(m, 1, 0, nullptr);
}

namespace {

// one chunk image under construction: 8-byte words + where each word's value
// comes from in the raw concatenation (-1 zero padding, -2 metadata)
struct ImageWriter {
  std::vector<double>& words;
  std::vector<int32_t>& src;
  std::size_t start;

  void align16() {
    if ((words.size() - start) & 1) put(0.0, -1);
  }
  uint32_t here() const { return static_cast<uint32_t>(8 * (words.size() - start)); }
  void put(double v, int32_t s) {
    words.push_back(v);
    src.push_back(s);
  }
  void put_value(const double* raw_sec, int64_t sec_off, int64_t i) {
    put(raw_sec[i], static_cast<int32_t>(sec_off + i));
  }
  template <typename T>
  void put_meta(const std::vector<T>& v) {  // bit-packed, 16-byte padded
    const std::size_t bytes = v.size() * sizeof(T), padded = (bytes + 15) & ~static_cast<std::size_t>(15);
    std::vector<unsigned char> buf(padded, 0);
    if (bytes) std::memcpy(buf.data(), v.data(), bytes);
    for (std::size_t o = 0; o < padded; o += 8) {
      double w;
      std::memcpy(&w, buf.data() + o, 8);
      put(w, -2);
    }
  }
};

}  // namespace

StreamLayout build_stream_layout_part(const dopf_model_view& m, int nparts, int part,
                                      const int32_t* part_of_s) {
  if (!m.has_pre) throw std::invalid_argument("model view lacks precomputed operators");
  if (nparts < 1 || part < 0 || part >= nparts || (nparts > 1 && !part_of_s))
    throw std::invalid_argument("bad partition");
  auto part_of = [&](int s) { return nparts == 1 ? 0 : part_of_s[s]; };
  for (int s = 0; s < m.S; ++s)
    if (part_of(s) < 0 || part_of(s) >= nparts) throw std::invalid_argument("subsystem part out of range");
  StreamLayout L;
  // pipeline shape of the staged kernel (DOPF_STAGES / DOPF_STAGE_KB for experiments)
  if (const char* e = std::getenv("DOPF_STAGES")) L.stages = std::max(1, std::min(kMaxStages, std::atoi(e)));
  if (const char* e = std::getenv("DOPF_STAGE_KB")) L.stage_bytes = std::max(1, std::atoi(e)) * 1024;
  if (L.stages * L.stage_bytes > 100 * 1024) throw std::invalid_argument("staged pipeline exceeds 100 KB per CTA");
  L.S = m.S;
  L.n = m.n;
  L.N_z = m.N_z;
  L.nparts = nparts;
  L.part = part;
  raw_offsets(m, L.raw_off);
  if (L.raw_off[kRawEnd] >= INT32_MAX) throw std::invalid_argument("model too large for 32-bit value maps");
  std::vector<int> order;
  for (int s : locality_order(m))
    if (part_of(s) == part) order.push_back(s);
  auto ns_of = [&](int s) { return m.z_offsets[s + 1] - m.z_offsets[s]; };
  for (int s = 0; s < m.S; ++s)
    if (ns_of(s) > kWideRows || m.m_s[s] > kWideRows)
      throw std::invalid_argument("subsystem wider than a streaming chunk (1024 columns or rows)");

  // ---- chunks of whole subsystems along the locality walk
  std::vector<int32_t> dev_of_ref(m.N_z, -1);
  std::vector<std::vector<int>> members_of;  // per chunk, widest first
  {
    int32_t row = 0;
    std::size_t k = 0;
    while (k < order.size()) {
      StreamChunk ch{};
      ch.row0 = row;
      int rows = 0, arows = 0;
      // exact sliced-ELL sizes of the chunk's P and A (rows sorted widest first,
      // a warp slice as wide as its first row) from per-width row counts, plus
      // upper bounds for everything else in the stage -- a chunk built here
      // always fits
      std::map<int, int, std::greater<int>> prow_w, arow_w;  // width -> rows
      auto ell_bytes = [](const std::map<int, int, std::greater<int>>& hist) {
        int64_t bytes = 0, row = 0;
        for (const auto& [width, count] : hist) {
          const int64_t first_warp = (row + 31) / 32, end_warp = (row + count + 31) / 32;
          bytes += 8 * 32 * static_cast<int64_t>(width) * (end_warp - first_warp);
          row += count;
        }
        return bytes;
      };
      auto stage_bound = [&](int r, int a) {
        const int64_t nw = (std::max(r, a) + 31) / 32;
        return 64 + 16 * ((8 * nw + 15) / 16) + ell_bytes(prow_w) + ell_bytes(arow_w) + 16LL * a +
               16LL * r                                      // row records
               + (32 + 4 + 2 + 8) * static_cast<int64_t>(r)  // interior columns, copies, imports (<= rows)
               + 16LL * r + 128;                              // z, lambda slices + alignment
      };
      std::vector<int> members;
      while (k < order.size()) {
        const int s = order[k];
        const int n = ns_of(s), ms = m.m_s[s];
        // several subsystems share a chunk only within the staged kernel's
        // limits; a wider one gets a chunk of its own (direct-load kernel)
        if (!members.empty()) {
          if (rows + n > kStagedRows || arows + ms > kStagedRows) break;
          prow_w[n] += n;
          if (ms) arow_w[n] += ms;
          const bool fits = stage_bound(rows + n, arows + ms) <= L.stage_bytes;
          if (!fits) {
            if ((prow_w[n] -= n) == 0) prow_w.erase(n);
            if (ms && (arow_w[n] -= ms) == 0) arow_w.erase(n);
            break;
          }
        } else {
          prow_w[n] += n;
          if (ms) arow_w[n] += ms;
        }
        members.push_back(s);
        rows += n;
        arows += ms;
        ++k;
      }
      // widest first inside the chunk: the 32 rows of a warp slice then have
      // (nearly) equal n_s, so the sliced-ELL padding stays small
      std::stable_sort(members.begin(), members.end(), [&](int a, int b) { return ns_of(a) > ns_of(b); });
      int r = 0;
      for (int s : members)
        for (int i = 0; i < ns_of(s); ++i) dev_of_ref[m.z_offsets[s] + i] = row + r++;
      ch.rows = rows;
      ch.arows = arows;
      row += rows;
      L.chunks.push_back(ch);
      members_of.push_back(std::move(members));
    }
    L.rows = row;
  }
  const int nchunks = static_cast<int>(L.chunks.size());
  std::vector<int32_t> chunk_of_row(L.rows);
  for (int q = 0; q < nchunks; ++q)
    for (int r = 0; r < L.chunks[q].rows; ++r) chunk_of_row[L.chunks[q].row0 + r] = q;
  std::vector<int> s_of_ref(m.N_z);
  for (int s = 0; s < m.S; ++s)
    for (int k2 = m.z_offsets[s]; k2 < m.z_offsets[s + 1]; ++k2) s_of_ref[k2] = s;
  L.z0.resize(L.rows);
  L.ref_of_dev.resize(L.rows);
  for (int ref = 0; ref < m.N_z; ++ref) {
    const int32_t d = dev_of_ref[ref];
    if (d < 0) continue;
    L.ref_of_dev[d] = ref;
    L.z0[d] = m.z0[ref];
  }

  // ---- columns: boundary (copies in several chunks or on other parts) first,
  // then interior ones grouped by chunk; each group by first local copy
  std::vector<int32_t> loc_of_col(m.n, -1);
  {
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
  L.cols = static_cast<int32_t>(L.gcol.size());
  for (int32_t gc : L.gcol) L.owner.push_back(part_of(s_of_ref[m.csr_copy[m.csr_ptr[gc]]]) == part ? 1 : 0);

  // ---- exports of every part (identical on all parts): copies of columns
  // held by more than one part, ascending reference index per part
  std::vector<int32_t> slot_of_ref(m.N_z, -1);
  if (nparts > 1) {
    std::vector<std::vector<int32_t>> exports(nparts);
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
        slot_of_ref[exports[q][e]] = q * L.xstride() + static_cast<int32_t>(e);
    for (int32_t ref : exports[part]) L.export_rows.push_back(dev_of_ref[ref]);
  }
  L.remote_slots = nparts * L.xstride();  // gathered records (exports + partials) of every part

  // ---- boundary columns: CSR over copies in ascending s (local copies ->
  // device rows, other parts' copies -> remote slots) and their data
  L.col_ptr.assign(1, 0);
  for (int32_t q = 0; q < L.bcols; ++q) {
    const int32_t gc = L.gcol[q];
    for (int e = m.csr_ptr[gc]; e < m.csr_ptr[gc + 1]; ++e) {
      const int ref = m.csr_copy[e];
      if (dev_of_ref[ref] >= 0) {
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
  }

  // ---- chunk images
  const int64_t* ro = L.raw_off;
  for (int q = 0; q < nchunks; ++q) {
    StreamChunk& ch = L.chunks[q];
    const std::vector<int>& members = members_of[q];
    // rows (thread r) and equality rows, with their operator sources
    struct Src { int64_t at; int n; int base; };
    std::vector<Src> prow, arow;
    std::vector<int64_t> bsrc;
    {
      int base = 0;
      for (int s : members) {
        const int n = ns_of(s);
        for (int i = 0; i < n; ++i) prow.push_back(Src{m.p_offsets[s] + static_cast<int64_t>(i) * n, n, base});
        for (int r = 0; r < m.m_s[s]; ++r) {
          arow.push_back(Src{m.a_offsets[s] + static_cast<int64_t>(r) * n, n, base});
          bsrc.push_back(m.b_offsets[s] + r);
        }
        base += n;
      }
    }
    // row metadata: interior column index or boundary import slot
    struct RowMeta { int16_t n, base, xloc, xin; };
    std::vector<RowMeta> rmeta(ch.rows);
    ch.bimp0 = static_cast<int32_t>(L.bimp.size());
    for (int r = 0; r < ch.rows; ++r) {
      const int32_t ref = L.ref_of_dev[ch.row0 + r];
      const int32_t col = loc_of_col[m.l2g[ref]];
      RowMeta rm{static_cast<int16_t>(prow[r].n), static_cast<int16_t>(prow[r].base), -1, -1};
      if (col >= L.bcols) {
        rm.xloc = static_cast<int16_t>(col - ch.icol0);
      } else {
        for (int e = ch.bimp0; e < static_cast<int>(L.bimp.size()); ++e)
          if (L.bimp[e] == col) rm.xin = static_cast<int16_t>(e - ch.bimp0);
        if (rm.xin < 0) {
          rm.xin = static_cast<int16_t>(L.bimp.size() - ch.bimp0);
          L.bimp.push_back(col);
        }
      }
      rmeta[r] = rm;
    }
    ch.nbimp = static_cast<int32_t>(L.bimp.size()) - ch.bimp0;
    // interior columns: chunk-local CSR over their copies (ascending s)
    std::vector<uint32_t> cmeta;
    std::vector<int16_t> icopies;
    for (int e = 0; e < ch.icols; ++e) {
      const int32_t gc = L.gcol[ch.icol0 + e];
      const uint32_t start = static_cast<uint32_t>(icopies.size());
      for (int k2 = m.csr_ptr[gc]; k2 < m.csr_ptr[gc + 1]; ++k2)
        icopies.push_back(static_cast<int16_t>(dev_of_ref[m.csr_copy[k2]] - ch.row0));
      const uint32_t cnt = static_cast<uint32_t>(icopies.size()) - start;
      cmeta.push_back(start | (cnt << 12) | (L.owner[ch.icol0 + e] ? 0x80000000u : 0u));
    }
    // the image
    ch.image_off = static_cast<int64_t>(8 * L.blob.size());
    ImageWriter w{L.blob, L.blob_src, L.blob.size()};
    ChunkHead head{};
    head.rows = ch.rows;
    head.arows = ch.arows;
    head.icols = ch.icols;
    head.nbimp = ch.nbimp;
    head.row0 = ch.row0;
    head.icol0 = ch.icol0;
    head.bimp0 = ch.bimp0;
    const std::size_t head_at = L.blob.size();
    for (std::size_t i = 0; i < sizeof(ChunkHead) / 8; ++i) w.put(0.0, -2);  // ChunkHead (filled below)
    auto put_meta_word = [&](const void* p8) {  // 8 bytes of metadata as one word
      double d;
      std::memcpy(&d, p8, 8);
      w.put(d, -2);
    };
    head.off[kImgRows] = w.here();
    for (int r = 0; r < ch.rows; ++r) {  // {n, base, xloc, xin | v}
      put_meta_word(&rmeta[r]);
      w.put_value(m.v, ro[kRawV], L.ref_of_dev[ch.row0 + r]);
    }
    // sliced ELL of P and A per warp of 32 rows
    auto pack = [&](const std::vector<Src>& rows, const double* raw, int64_t sec, std::vector<int32_t>& slices) {
      const std::size_t sec_start = L.blob.size();
      for (int w0 = 0; w0 < static_cast<int>(rows.size()); w0 += 32) {
        const int lanes = std::min(32, static_cast<int>(rows.size()) - w0);
        int width = 0;
        for (int l = 0; l < lanes; ++l) width = std::max(width, rows[w0 + l].n);
        slices.push_back(static_cast<int32_t>(L.blob.size() - sec_start));
        for (int j = 0; j < width; ++j)
          for (int l = 0; l < 32; ++l) {
            if (l < lanes && j < rows[w0 + l].n) w.put_value(raw, sec, rows[w0 + l].at + j);
            else w.put(0.0, -1);
          }
      }
    };
    std::vector<int32_t> pslice, aslice;
    // the slice table precedes the sections it indexes: reserve, pack, then patch
    const int nw = std::max((ch.rows + 31) / 32, (ch.arows + 31) / 32);
    head.off[kImgSlices] = w.here();
    const std::size_t sl_at = L.blob.size();
    w.put_meta(std::vector<int32_t>(2 * nw, 0));
    head.off[kImgP] = w.here();
    pack(prow, m.P, ro[kRawP], pslice);
    head.off[kImgA] = w.here();
    pack(arow, m.A, ro[kRawA], aslice);
    {
      std::vector<int32_t> sl(2 * nw, 0);
      for (std::size_t i = 0; i < pslice.size(); ++i) sl[2 * i] = pslice[i];
      for (std::size_t i = 0; i < aslice.size(); ++i) sl[2 * i + 1] = aslice[i];
      std::memcpy(&L.blob[sl_at], sl.data(), sl.size() * 4);
    }
    head.off[kImgArows] = w.here();
    for (int a = 0; a < ch.arows; ++a) {  // {n, base | b}
      const int32_t nb[2] = {arow[a].n, arow[a].base};
      put_meta_word(nb);
      w.put_value(m.b, ro[kRawB], bsrc[a]);
    }
    head.off[kImgCols] = w.here();
    for (int e = 0; e < ch.icols; ++e) {  // {cost, inv, lo, hi}
      const int32_t gc = L.gcol[ch.icol0 + e];
      w.put_value(m.c, ro[kRawC], gc);
      w.put_value(m.inv_copy, ro[kRawInv], gc);
      w.put_value(m.x_lo, ro[kRawLo], gc);
      w.put_value(m.x_hi, ro[kRawHi], gc);
    }
    head.off[kImgCmeta] = w.here();
    w.put_meta(cmeta);
    head.off[kImgCopies] = w.here();
    w.put_meta(icopies);
    ch.image_bytes = static_cast<int32_t>(w.here());
    head.image_bytes = ch.image_bytes;
    std::memcpy(&L.blob[head_at], &head, sizeof(ChunkHead));
    StagePlan sp;
    stage_plan(ch, sp);
    const bool fits = sp.total <= static_cast<uint32_t>(L.stage_bytes) && ch.rows <= kStagedRows &&
                      ch.arows <= kStagedRows;
    (fits ? L.staged_ids : L.big_ids).push_back(q);
  }
  L.imp_ptr.assign(L.bcols + 1, 0);
  for (int32_t c : L.bimp) ++L.imp_ptr[c + 1];
  for (int32_t c = 0; c < L.bcols; ++c) L.imp_ptr[c + 1] += L.imp_ptr[c];
  L.imp_slot.resize(L.bimp.size());
  {
    std::vector<int32_t> fill(L.imp_ptr.begin(), L.imp_ptr.end() - 1);
    for (std::size_t e = 0; e < L.bimp.size(); ++e) L.imp_slot[fill[L.bimp[e]]++] = static_cast<int32_t>(e);
  }

  {  // signature for the re-upload fast path
    if (nparts > 1) L.sig_part_of_s.assign(part_of_s, part_of_s + m.S);
    L.sig_z_offsets.assign(m.z_offsets, m.z_offsets + m.S + 1);
    L.sig_m_s.assign(m.m_s, m.m_s + m.S);
    L.sig_l2g.assign(m.l2g, m.l2g + m.N_z);
    L.sig_csr_ptr.assign(m.csr_ptr, m.csr_ptr + m.n + 1);
    L.sig_csr_copy.assign(m.csr_copy, m.csr_copy + m.N_z);
  }
  // algorithmic bytes of this part (DESIGN.md section 4 restricted to it)
  double msum = 0, n2 = 0, mn = 0;
  for (int s : order) {
    const double n = ns_of(s);
    n2 += n * n;
    mn += m.m_s[s] * n;
    msum += m.m_s[s];
  }
  L.bytes_per_iteration = 8.0 * (n2 + mn + msum) + 56.0 * L.rows + 48.0 * L.cols +
                          4.0 * (2.0 * L.rows + L.cols + 1) + 16.0 * static_cast<double>(order.size());
  return L;
}

}  // namespace dopf::cuda
