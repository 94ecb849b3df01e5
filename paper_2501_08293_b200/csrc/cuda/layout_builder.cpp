#include "layout_builder.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace dopf::cuda {

namespace {

int ns_of(const dopf_model_view& m, int s) { return m.z_offsets[s + 1] - m.z_offsets[s]; }

double sub_cost(const dopf_model_view& m, int s) {
  const double n = ns_of(m, s), mm = m.m_s[s];
  return n * n + mm * n + 6.0 * n + 4.0;
}

// Depth-first order of the component graph: subsystems s and s' are adjacent
// when they hold copies of one global column. Cutting this walk into
// contiguous pieces keeps most copies of a column inside one block.
std::vector<int> locality_order(const dopf_model_view& m) {
  std::vector<int> s_of_ref(m.N_z);
  for (int s = 0; s < m.S; ++s)
    for (int k = m.z_offsets[s]; k < m.z_offsets[s + 1]; ++k) s_of_ref[k] = s;
  std::vector<std::vector<int>> adj(m.S);
  for (int c = 0; c < m.n; ++c)
    for (int a = m.csr_ptr[c]; a < m.csr_ptr[c + 1]; ++a)
      for (int b = m.csr_ptr[c]; b < m.csr_ptr[c + 1]; ++b)
        if (a != b) adj[s_of_ref[m.csr_copy[a]]].push_back(s_of_ref[m.csr_copy[b]]);
  for (auto& v : adj) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  std::vector<int> order;
  order.reserve(m.S);
  std::vector<char> seen(m.S, 0);
  std::vector<int> stack;
  for (int root = 0; root < m.S; ++root) {
    if (seen[root]) continue;
    stack.push_back(root);
    while (!stack.empty()) {
      const int u = stack.back();
      stack.pop_back();
      if (seen[u]) continue;
      seen[u] = 1;
      order.push_back(u);
      // push in descending id so the lowest-id neighbour is visited first
      for (auto it = adj[u].rbegin(); it != adj[u].rend(); ++it)
        if (!seen[*it]) stack.push_back(*it);
    }
  }
  return order;
}

// Cuts `order` into at most G contiguous pieces of nearly equal cost.
std::vector<std::vector<int>> split_blocks(const dopf_model_view& m, const std::vector<int>& order,
                                           int G) {
  double total = 0;
  for (int s : order) total += sub_cost(m, s);
  std::vector<std::vector<int>> out(1);
  double acc = 0;
  int g = 1;
  for (int s : order) {
    out.back().push_back(s);
    acc += sub_cost(m, s);
    if (g < G && acc >= total * g / G) {
      out.emplace_back();
      ++g;
    }
  }
  if (out.back().empty()) out.pop_back();
  return out;
}

}  // namespace

std::size_t block_smem_bytes(const BlockDesc& b, bool ops_in_smem) {
  // must match the carve-up at the top of admm_persistent
  std::size_t doubles = 0;
  if (ops_in_smem) doubles += static_cast<std::size_t>(b.p_len) + b.a_len;
  doubles += 3ull * b.rows;                     // target, z, v
  doubles += 9ull * b.cols;                     // x (four buffers), c/rho, inv, lo, hi, c
  doubles += 2 * (kThreads / 32ull) * kPartials + 16 + 8;  // warp partials x2, decision ring, phase clock
  doubles += 3ull * b.arows;                    // equality rows: rhs + AMeta (16 B)
  return 8 * doubles + 4ull * b.copy_len + 64;
}

double algorithmic_bytes(const dopf_model_view& m) {
  double n2 = 0, mn = 0, msum = 0;
  for (int s = 0; s < m.S; ++s) {
    const double n = ns_of(m, s);
    n2 += n * n;
    mn += m.m_s[s] * n;
    msum += m.m_s[s];
  }
  return 8.0 * (n2 + mn + msum) + 56.0 * m.N_z + 48.0 * m.n + 4.0 * (2.0 * m.N_z + m.n + 1) +
         16.0 * m.S;
}

double algorithmic_flops(const dopf_model_view& m) {
  double n2 = 0, mn = 0;
  for (int s = 0; s < m.S; ++s) {
    const double n = ns_of(m, s);
    n2 += n * n;
    mn += m.m_s[s] * n;
  }
  return 2.0 * n2 + 2.0 * mn + 20.0 * m.N_z;
}

int choose_blocks(const dopf_model_view& m, const LayoutOptions& opt) {
  if (opt.blocks_per_instance > 0) return opt.blocks_per_instance;
  // Lower bound on the CTA count from the instance's total shared-memory
  // footprint and row count, then the smallest G <= 8 (one cluster) whose
  // blocks all fit; larger instances take one CTA per SM.
  double bytes = 0;
  for (int s = 0; s < m.S; ++s) {
    const double n = ns_of(m, s);
    bytes += 8.0 * (n * n + m.m_s[s] * n) + 16.0 * n + 4.0 * n;
  }
  bytes += 56.0 * m.n;
  const int rows_cap = (opt.threads - 32) * 2;
  int g0 = static_cast<int>(bytes / (0.92 * static_cast<double>(opt.smem_limit))) + 1;
  g0 = std::max(g0, (m.N_z + rows_cap - 1) / rows_cap);
  g0 = std::max(1, std::min(g0, std::max(1, m.S)));
  for (int G = g0; G <= 8 && G <= m.S; ++G) {
    HostLayout trial;
    add_instance(trial, m, G, opt);
    if (trial.all_ops_in_smem && trial.K <= 2) return G;
  }
  return std::min(opt.max_blocks, std::max(1, m.S));
}

void add_instance(HostLayout& L, const dopf_model_view& m, int G, const LayoutOptions& opt) {
  if (!m.has_pre) throw std::invalid_argument("model view lacks precomputed operators");
  const int instance = static_cast<int>(L.inst.size());
  const std::vector<std::vector<int>> parts =
      split_blocks(m, locality_order(m), std::max(1, std::min(G, std::max(1, m.S))));
  const int nb = static_cast<int>(parts.size());
  const int32_t inst_row0 = static_cast<int32_t>(L.rows_total);
  const int32_t block0 = static_cast<int32_t>(L.blocks.size());

  InstDesc id{};
  id.x_off = L.x_total;
  id.n = m.n;
  id.blocks = std::max(nb, 1);
  id.block0 = block0;
  id.rows = m.N_z;
  id.row0 = inst_row0;
  L.inst.push_back(id);
  L.x_total += m.n;

  // Pass 1: device rows (subsystems by n_s descending inside each block).
  std::vector<int32_t> dev_of_ref(m.N_z, -1);
  std::vector<std::vector<int>> order(nb);
  int32_t next_row = inst_row0;
  std::vector<int32_t> block_row0(nb);
  for (int g = 0; g < nb; ++g) {
    auto& ord = order[g];
    ord = parts[g];
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int a, int b) { return ns_of(m, a) > ns_of(m, b); });
    block_row0[g] = next_row;
    for (int s : ord)
      for (int i = 0; i < ns_of(m, s); ++i) dev_of_ref[m.z_offsets[s] + i] = next_row++;
  }
  L.rows_total = next_row;
  L.rmeta.resize(next_row);
  L.v.resize(next_row);
  L.z0.resize(next_row);
  L.ref_of_dev.resize(next_row);

  // owner block of each column = block holding its first (lowest-s) copy
  std::vector<int> block_of_s(m.S, 0);
  for (int g = 0; g < nb; ++g)
    for (int s : parts[g]) block_of_s[s] = g;
  std::vector<int> s_of_ref(m.N_z);
  for (int s = 0; s < m.S; ++s)
    for (int k = m.z_offsets[s]; k < m.z_offsets[s + 1]; ++k) s_of_ref[k] = s;

  std::vector<int> xloc_of(m.n, -1);
  std::vector<char> exported(next_row - inst_row0, 0);
  std::vector<int> nbrs;
  for (int g = 0; g < nb; ++g) {
    BlockDesc bd{};
    bd.row0 = block_row0[g];
    bd.instance = instance;
    bd.inst_block = g;
    bd.p_off = static_cast<int64_t>(L.P.size());
    bd.a_off = static_cast<int64_t>(L.A.size());
    bd.copy_off = static_cast<int32_t>(L.copies.size());
    bd.col_off = static_cast<int32_t>(L.cmeta.size());
    bd.amet_off = static_cast<int32_t>(L.ameta.size());

    // columns referenced by this block, ascending
    std::vector<int> cols;
    for (int s : order[g])
      for (int k = m.z_offsets[s]; k < m.z_offsets[s + 1]; ++k) cols.push_back(m.l2g[k]);
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    // interior columns (every copy in this block) first, boundary columns last
    auto is_boundary = [&](int c) {
      for (int q = m.csr_ptr[c]; q < m.csr_ptr[c + 1]; ++q)
        if (block_of_s[s_of_ref[m.csr_copy[q]]] != g) return true;
      return false;
    };
    const auto mid = std::stable_partition(cols.begin(), cols.end(),
                                           [&](int c) { return !is_boundary(c); });
    bd.cols_int = static_cast<int32_t>(mid - cols.begin());
    for (std::size_t q = 0; q < cols.size(); ++q) xloc_of[cols[q]] = static_cast<int>(q);

    // Rows (and equality rows) go to thread slots r = k * cw + ctid; the 32
    // rows of one warp and slot k form a "slice" whose operator rows are
    // stored interleaved: entry j of the slice's lane l at slice_off + 32 j + l
    // (sliced ELL). Every shared-memory read of a warp is then 256 contiguous
    // bytes -- conflict-free -- and the kernel's row offsets are immediates.
    const int cw = opt.threads - 32;
    struct RowSrc { const double* src; int n; };  // operator row (contiguous, n entries)
    std::vector<RowSrc> prow, arow;
    int32_t local = 0;
    for (int s : order[g]) {
      const int n = ns_of(m, s), ms = m.m_s[s];
      const int base = local;
      const double* Ps = m.P + m.p_offsets[s];  // row-major n x n
      const double* As = m.A + m.a_offsets[s];  // row-major ms x n
      for (int i = 0; i < n; ++i) {
        const int ref = m.z_offsets[s] + i;
        const int32_t dev = bd.row0 + local;
        L.rmeta[dev] = RowMeta{0, static_cast<int16_t>(n), 0, base, xloc_of[m.l2g[ref]]};
        L.v[dev] = m.v[ref];
        L.z0[dev] = m.z0[ref];
        L.ref_of_dev[dev] = ref;
        prow.push_back(RowSrc{Ps + static_cast<std::size_t>(i) * n, n});
        ++local;
      }
      for (int r = 0; r < ms; ++r) {
        L.ameta.push_back(AMeta{0, ms, n, base});
        L.ab.push_back(m.b[m.b_offsets[s] + r]);
        arow.push_back(RowSrc{As + static_cast<std::size_t>(r) * n, n});
      }
    }
    // pack rows into slices; returns the doubles appended; offs[r] = slice_off + lane
    auto pack = [&](const std::vector<RowSrc>& rows, std::vector<double>& out, auto&& set_off) {
      const int count = static_cast<int>(rows.size());
      int32_t len = 0;
      for (int k0 = 0; k0 < count; k0 += cw) {
        for (int w0 = k0; w0 < std::min(count, k0 + cw); w0 += 32) {
          const int lanes = std::min(32, count - w0);
          int width = 0;
          for (int l = 0; l < lanes; ++l) width = std::max(width, rows[w0 + l].n);
          for (int l = 0; l < lanes; ++l) set_off(w0 + l, len + l);
          for (int j = 0; j < width; ++j)
            for (int l = 0; l < 32; ++l)
              out.push_back(l < lanes && j < rows[w0 + l].n ? rows[w0 + l].src[j] : 0.0);
          len += 32 * width;
        }
      }
      return len;
    };
    bd.p_len = pack(prow, L.P, [&](int r, int32_t o) { L.rmeta[bd.row0 + r].pofs = o; });
    bd.a_len = pack(arow, L.A, [&](int a, int32_t o) { L.ameta[bd.amet_off + a].aofs = o; });
    bd.rows = local;
    bd.arows = static_cast<int32_t>(L.ameta.size()) - bd.amet_off;
    bd.cols = static_cast<int32_t>(cols.size());
    for (int c : cols) {
      ColMeta cm{};
      cm.gcol = c;
      cm.copy_start = static_cast<int32_t>(L.copies.size()) - bd.copy_off;
      cm.copy_count = m.csr_ptr[c + 1] - m.csr_ptr[c];
      for (int q = m.csr_ptr[c]; q < m.csr_ptr[c + 1]; ++q) {
        const int32_t dev = dev_of_ref[m.csr_copy[q]];
        const int g2 = block_of_s[s_of_ref[m.csr_copy[q]]];
        if (g2 == g) {
          L.copies.push_back(dev - bd.row0);  // block-local: u from shared memory
        } else {
          L.copies.push_back(encode_remote(dev));
          exported[dev - inst_row0] = 1;
          nbrs.push_back(g2);
        }
      }
      cm.owner = block_of_s[s_of_ref[m.csr_copy[m.csr_ptr[c]]]] == g ? 1 : 0;
      L.cmeta.push_back(cm);
      L.cc.push_back(m.c[c]);
      L.cinv.push_back(m.inv_copy[c]);
      L.clo.push_back(m.x_lo[c]);
      L.chi.push_back(m.x_hi[c]);
    }
    bd.copy_len = static_cast<int32_t>(L.copies.size()) - bd.copy_off;
    for (int c : cols) xloc_of[c] = -1;
    std::sort(nbrs.begin(), nbrs.end());
    nbrs.erase(std::unique(nbrs.begin(), nbrs.end()), nbrs.end());
    bd.nbr_off = static_cast<int32_t>(L.nbrs.size());
    bd.nbr_cnt = static_cast<int32_t>(nbrs.size());
    L.nbrs.insert(L.nbrs.end(), nbrs.begin(), nbrs.end());
    L.max_neighbours = std::max(L.max_neighbours, bd.nbr_cnt);
    nbrs.clear();

    // the kernel packs per-thread metadata into bit fields (admm_kernels.cu)
    if (bd.rows >= 4096 || bd.cols >= 4096 || bd.copy_len >= (1 << 23))
      throw std::invalid_argument("block too large for the resident kernel");
    if (bd.cols - bd.cols_int > opt.threads - 32)
      throw std::invalid_argument("block has more boundary columns than compute threads");
    for (int s : order[g])
      if (ns_of(m, s) >= 128) throw std::invalid_argument("subsystem with n_s >= 128 columns");
    for (int c : cols)
      if (m.csr_ptr[c + 1] - m.csr_ptr[c] >= 256)
        throw std::invalid_argument("column with 256 or more copies");
    bd.ops_in_smem = block_smem_bytes(bd, true) <= opt.smem_limit ? 1 : 0;
    if (!bd.ops_in_smem) L.all_ops_in_smem = false;
    L.smem_bytes = std::max(L.smem_bytes, block_smem_bytes(bd, bd.ops_in_smem));
    // warps 1.. (opt.threads - 32 threads) own rows, columns and equality rows
    const int k_need = (std::max(bd.rows, std::max(bd.cols, bd.arows)) + cw - 1) / cw;
    L.K = std::max(L.K, std::max(1, k_need));
    L.blocks.push_back(bd);
  }
  for (int32_t d = inst_row0; d < next_row; ++d) L.rmeta[d].exported = exported[d - inst_row0];
  L.blocks_per_instance = std::max(L.blocks_per_instance, nb);
  L.bytes_per_iteration += algorithmic_bytes(m);
  L.flops_per_iteration += algorithmic_flops(m);
}

}  // namespace dopf::cuda
