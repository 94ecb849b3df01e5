#include "layout_builder.hpp"

#include "admm_kernels.cuh"

#include <algorithm>
#include <cstring>
#include <thread>
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
std::vector<int> locality_order_impl(const dopf_model_view& m) {
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

// Cuts `order` into at most G contiguous pieces of nearly equal cost, or --
// with per-block shares `w` (G entries; a partition tuned from measured
// per-CTA slack, LayoutOptions::block_weights) -- of cost proportional to them.
std::vector<std::vector<int>> split_blocks(const dopf_model_view& m, const std::vector<int>& order,
                                           int G, const std::vector<double>& w = {}) {
  double total = 0;
  for (int s : order) total += sub_cost(m, s);
  const bool weighted = static_cast<int>(w.size()) == G;
  double wsum = 0;
  for (double x : w) wsum += x;
  std::vector<std::vector<int>> out(1);
  double acc = 0, wacc = weighted ? w[0] : 0;
  int g = 1;
  for (int s : order) {
    out.back().push_back(s);
    acc += sub_cost(m, s);
    const double target = weighted ? total * wacc / wsum : total * g / G;
    if (g < G && acc >= target) {
      out.emplace_back();
      if (weighted) wacc += w[g];
      ++g;
    }
  }
  if (out.back().empty()) out.pop_back();
  return out;
}

}  // namespace

std::vector<int> locality_order(const dopf_model_view& m) { return locality_order_impl(m); }

std::size_t block_smem_bytes(const BlockDesc& b, bool ops_in_smem) {
  // must match the carve-up at the top of admm_persistent
  std::size_t doubles = 0;
  if (ops_in_smem) doubles += static_cast<std::size_t>(b.p_len) + b.a_len;
  doubles += 4ull * b.rows;                     // target, z (two buffers), v
  doubles += (kXRing + 5ull) * b.cols;          // x ring, c/rho, inv, lo, hi, c
  doubles += 2 * (kThreads / 32ull) * kPartials + 8 * 4 + 8;  // warp partials x2, decision ring, phase clock
  doubles += kLag + 2ull;                       // block infeasibility ring + end flag (check warp)
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
  const int rows_cap = (opt.threads - 64) * 2;
  int g0 = static_cast<int>(bytes / (0.92 * static_cast<double>(opt.smem_limit))) + 1;
  g0 = std::max(g0, (m.N_z + rows_cap - 1) / rows_cap);
  g0 = std::max(1, std::min(g0, std::max(1, m.S)));
  for (int G = g0; G <= 8 && G <= m.S; ++G) {
    const InstancePlan trial = plan_instance(m, G, opt);
    if (trial.all_ops_in_smem && trial.K <= 2) return G;
  }
  return std::min(opt.max_blocks, std::max(1, m.S));
}

bool InstancePlan::same_structure(const dopf_model_view& m, const LayoutOptions& o) const {
  auto eq = [](const std::vector<int32_t>& v, const int32_t* p, std::size_t n) {
    return v.size() == n && (n == 0 || std::memcmp(v.data(), p, n * sizeof(int32_t)) == 0);
  };
  return m.has_pre && S == m.S && n == m.n && Nz == m.N_z && o.smem_limit == opt.smem_limit &&
         o.max_blocks == opt.max_blocks && o.threads == opt.threads &&
         o.blocks_per_instance == opt.blocks_per_instance && o.block_weights == opt.block_weights && eq(z_offsets, m.z_offsets, m.S + 1) &&
         eq(m_s, m.m_s, m.S) && eq(l2g, m.l2g, m.N_z) && eq(csr_ptr, m.csr_ptr, m.n + 1) &&
         eq(csr_copy, m.csr_copy, m.N_z);
}

InstancePlan plan_instance(const dopf_model_view& m, int G, const LayoutOptions& opt) {
  if (!m.has_pre) throw std::invalid_argument("model view lacks precomputed operators");
  InstancePlan P;
  P.S = m.S;
  P.n = m.n;
  P.Nz = m.N_z;
  P.G = G;
  P.opt = opt;
  P.z_offsets.assign(m.z_offsets, m.z_offsets + m.S + 1);
  P.m_s.assign(m.m_s, m.m_s + m.S);
  P.l2g.assign(m.l2g, m.l2g + m.N_z);
  P.csr_ptr.assign(m.csr_ptr, m.csr_ptr + m.n + 1);
  P.csr_copy.assign(m.csr_copy, m.csr_copy + m.N_z);

  const std::vector<std::vector<int>> parts =
      split_blocks(m, locality_order_impl(m), std::max(1, std::min(G, std::max(1, m.S))), opt.block_weights);
  const int nb = static_cast<int>(parts.size());
  const int cw = opt.threads - 64;  // compute threads (kComputeThreads)

  // Pass 1: device rows (subsystems by n_s descending inside each block).
  std::vector<int32_t> dev_of_ref(m.N_z, -1);
  std::vector<std::vector<int>> order(nb);
  int32_t next_row = 0;
  std::vector<int32_t> block_row0(nb);
  for (int g = 0; g < nb; ++g) {
    auto& ord = order[g];
    ord = parts[g];
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return ns_of(m, a) > ns_of(m, b); });
    // Balance the per-thread row work across warps: thread slot k holds rows
    // [k cw, (k+1) cw). Widest-first order would give the first warps the
    // widest row of every slot; reversing the subsystem order inside odd
    // slots pairs wide rows of one slot with narrow rows of the next.
    {
      const int cwb = opt.threads - 64;
      std::vector<int> out;
      std::vector<int> seg;
      int rows_done = 0, k = 0;
      for (int s : ord) {
        seg.push_back(s);
        rows_done += ns_of(m, s);
        if (rows_done >= (k + 1) * cwb) {
          if (k & 1) std::reverse(seg.begin(), seg.end());
          out.insert(out.end(), seg.begin(), seg.end());
          seg.clear();
          ++k;
        }
      }
      if (k & 1) std::reverse(seg.begin(), seg.end());
      out.insert(out.end(), seg.begin(), seg.end());
      ord.swap(out);
    }
    block_row0[g] = next_row;
    for (int s : ord)
      for (int i = 0; i < ns_of(m, s); ++i) dev_of_ref[m.z_offsets[s] + i] = next_row++;
  }
  P.rmeta.resize(next_row);
  P.ref_of_dev.resize(next_row);

  // owner block of each column = block holding its first (lowest-s) copy
  std::vector<int> block_of_s(m.S, 0);
  for (int g = 0; g < nb; ++g)
    for (int s : parts[g]) block_of_s[s] = g;
  std::vector<int> s_of_ref(m.N_z);
  for (int s = 0; s < m.S; ++s)
    for (int k = m.z_offsets[s]; k < m.z_offsets[s + 1]; ++k) s_of_ref[k] = s;

  std::vector<int> xloc_of(m.n, -1);
  std::vector<char> exported(next_row, 0);
  std::vector<int> nbrs;
  std::size_t p_len_total = 0, a_len_total = 0;
  for (int g = 0; g < nb; ++g) {
    BlockDesc bd{};
    bd.row0 = block_row0[g];
    bd.inst_block = g;
    bd.p_off = static_cast<int64_t>(p_len_total);
    bd.a_off = static_cast<int64_t>(a_len_total);
    bd.copy_off = static_cast<int32_t>(P.copies.size());
    bd.col_off = static_cast<int32_t>(P.cmeta.size());
    bd.amet_off = static_cast<int32_t>(P.ameta.size());

    // columns referenced by this block, ascending; interior columns (every
    // copy in this block) first, boundary columns last
    std::vector<int> cols;
    for (int s : order[g])
      for (int k = m.z_offsets[s]; k < m.z_offsets[s + 1]; ++k) cols.push_back(m.l2g[k]);
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    auto is_boundary = [&](int c) {
      for (int q = m.csr_ptr[c]; q < m.csr_ptr[c + 1]; ++q)
        if (block_of_s[s_of_ref[m.csr_copy[q]]] != g) return true;
      return false;
    };
    const auto mid = std::stable_partition(cols.begin(), cols.end(), [&](int c) { return !is_boundary(c); });
    bd.cols_int = static_cast<int32_t>(mid - cols.begin());
    for (std::size_t q = 0; q < cols.size(); ++q) xloc_of[cols[q]] = static_cast<int>(q);

    // Rows (and equality rows) go to thread slots r = k * cw + ctid; the 32
    // rows of one warp and slot k form a "slice" whose operator rows are
    // stored interleaved: entry j of the slice's lane l at slice_off + 32 j + l
    // (sliced ELL). Every shared-memory read of a warp is then 256 contiguous
    // bytes -- conflict-free -- and the kernel's row offsets are immediates.
    struct RowSrc { int64_t src; int n; };  // operator row: offset into m.P / m.A, n entries
    std::vector<RowSrc> prow, arow;
    int32_t local = 0;
    for (int s : order[g]) {
      const int n = ns_of(m, s), ms = m.m_s[s];
      const int base = local;
      for (int i = 0; i < n; ++i) {
        const int ref = m.z_offsets[s] + i;
        const int32_t dev = bd.row0 + local;
        P.rmeta[dev] = RowMeta{0, static_cast<int16_t>(n), 0, base, xloc_of[m.l2g[ref]]};
        P.ref_of_dev[dev] = ref;
        prow.push_back(RowSrc{m.p_offsets[s] + static_cast<int64_t>(i) * n, n});
        ++local;
      }
      for (int r = 0; r < ms; ++r) {
        P.ameta.push_back(AMeta{0, ms, n, base});
        P.ab_src.push_back(m.b_offsets[s] + r);
        arow.push_back(RowSrc{m.a_offsets[s] + static_cast<int64_t>(r) * n, n});
      }
    }
    auto pack = [&](const std::vector<RowSrc>& rows, std::vector<int64_t>& out, auto&& set_off) {
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
              out.push_back(l < lanes && j < rows[w0 + l].n ? rows[w0 + l].src + j : -1);
          len += 32 * width;
        }
      }
      return len;
    };
    bd.p_len = pack(prow, P.p_src, [&](int r, int32_t o) { P.rmeta[bd.row0 + r].pofs = o; });
    bd.a_len = pack(arow, P.a_src, [&](int a, int32_t o) { P.ameta[bd.amet_off + a].aofs = o; });
    p_len_total += bd.p_len;
    a_len_total += bd.a_len;
    bd.rows = local;
    bd.arows = static_cast<int32_t>(P.ameta.size()) - bd.amet_off;
    bd.cols = static_cast<int32_t>(cols.size());
    for (int c : cols) {
      ColMeta cm{};
      cm.gcol = c;
      cm.copy_start = static_cast<int32_t>(P.copies.size()) - bd.copy_off;
      cm.copy_count = m.csr_ptr[c + 1] - m.csr_ptr[c];
      for (int q = m.csr_ptr[c]; q < m.csr_ptr[c + 1]; ++q) {
        const int32_t dev = dev_of_ref[m.csr_copy[q]];
        const int g2 = block_of_s[s_of_ref[m.csr_copy[q]]];
        if (g2 == g) {
          P.copies.push_back(dev - bd.row0);  // block-local: u from shared memory
        } else {
          P.copies.push_back(encode_remote(dev));  // instance-relative; rebased on append
          exported[dev] = 1;
          nbrs.push_back(g2);
        }
      }
      cm.owner = block_of_s[s_of_ref[m.csr_copy[m.csr_ptr[c]]]] == g ? 1 : 0;
      P.cmeta.push_back(cm);
    }
    bd.copy_len = static_cast<int32_t>(P.copies.size()) - bd.copy_off;
    for (int c : cols) xloc_of[c] = -1;
    std::sort(nbrs.begin(), nbrs.end());
    nbrs.erase(std::unique(nbrs.begin(), nbrs.end()), nbrs.end());
    bd.nbr_off = static_cast<int32_t>(P.nbrs.size());
    bd.nbr_cnt = static_cast<int32_t>(nbrs.size());
    P.nbrs.insert(P.nbrs.end(), nbrs.begin(), nbrs.end());
    P.max_neighbours = std::max(P.max_neighbours, bd.nbr_cnt);
    nbrs.clear();

    // the kernel packs per-thread metadata into bit fields (admm_kernels.cu)
    if (bd.rows >= 4096 || bd.cols >= 4096 || bd.copy_len >= (1 << 23))
      throw std::invalid_argument("block too large for the resident kernel");
    if (bd.cols - bd.cols_int > cw)
      throw std::invalid_argument("block has more boundary columns than compute threads");
    for (int s : order[g])
      if (ns_of(m, s) >= 128) throw std::invalid_argument("subsystem with n_s >= 128 columns");
    for (int c : cols)
      if (m.csr_ptr[c + 1] - m.csr_ptr[c] >= 256) throw std::invalid_argument("column with 256 or more copies");
    bd.ops_in_smem = block_smem_bytes(bd, true) <= opt.smem_limit ? 1 : 0;
    if (!bd.ops_in_smem) P.all_ops_in_smem = false;
    P.smem_bytes = std::max(P.smem_bytes, block_smem_bytes(bd, bd.ops_in_smem));
    // warps 2.. (cw threads) own rows, interior columns and equality-row slots
    const int k_need = (std::max(bd.rows, std::max(bd.cols_int, bd.arows)) + cw - 1) / cw;
    P.K = std::max(P.K, std::max(1, k_need));
    P.blocks.push_back(bd);
  }
  for (int32_t d = 0; d < next_row; ++d) P.rmeta[d].exported = exported[d];
  P.bytes_per_iteration = algorithmic_bytes(m);
  P.flops_per_iteration = algorithmic_flops(m);
  return P;
}

namespace {

// out[i] = src[idx[i]] (0 for idx < 0), split over threads for large arrays
void gather(std::vector<double>& out, std::size_t at, const std::vector<int64_t>& idx, const double* src) {
  const std::size_t n = idx.size();
  auto body = [&](std::size_t b, std::size_t e) {
    for (std::size_t i = b; i < e; ++i) out[at + i] = idx[i] >= 0 ? src[idx[i]] : 0.0;
  };
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (n < (1u << 18) || hw == 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned t = 0; t < hw; ++t) th.emplace_back(body, n * t / hw, n * (t + 1) / hw);
  for (auto& t : th) t.join();
}

}  // namespace

void append_instance(HostLayout& L, const InstancePlan& P, const dopf_model_view& m) {
  const int instance = static_cast<int>(L.inst.size());
  const int32_t row_base = static_cast<int32_t>(L.rows_total);
  const int64_t p_base = static_cast<int64_t>(L.P.size()), a_base = static_cast<int64_t>(L.A.size());
  const int32_t copy_base = static_cast<int32_t>(L.copies.size());
  const int32_t col_base = static_cast<int32_t>(L.cmeta.size());
  const int32_t amet_base = static_cast<int32_t>(L.ameta.size());
  const int32_t nbr_base = static_cast<int32_t>(L.nbrs.size());

  InstDesc id{};
  id.x_off = L.x_total;
  id.n = P.n;
  id.blocks = static_cast<int32_t>(P.blocks.size());
  id.block0 = static_cast<int32_t>(L.blocks.size());
  id.rows = P.Nz;
  id.row0 = row_base;
  L.inst.push_back(id);
  L.x_total += P.n;

  for (BlockDesc bd : P.blocks) {
    bd.row0 += row_base;
    bd.p_off += p_base;
    bd.a_off += a_base;
    bd.copy_off += copy_base;
    bd.col_off += col_base;
    bd.amet_off += amet_base;
    bd.nbr_off += nbr_base;
    bd.instance = instance;
    L.blocks.push_back(bd);
  }
  const std::size_t rows = P.rmeta.size();
  L.rmeta.insert(L.rmeta.end(), P.rmeta.begin(), P.rmeta.end());
  L.ref_of_dev.insert(L.ref_of_dev.end(), P.ref_of_dev.begin(), P.ref_of_dev.end());
  L.v.resize(row_base + rows);
  L.z0.resize(row_base + rows);
  for (std::size_t d = 0; d < rows; ++d) {
    L.v[row_base + d] = m.v[P.ref_of_dev[d]];
    L.z0[row_base + d] = m.z0[P.ref_of_dev[d]];
  }
  L.rows_total += static_cast<int64_t>(rows);
  for (int32_t c : P.copies) L.copies.push_back(c >= 0 ? c : encode_remote(decode_remote(c) + row_base));
  L.cmeta.insert(L.cmeta.end(), P.cmeta.begin(), P.cmeta.end());
  for (const ColMeta& cm : P.cmeta) {
    L.cc.push_back(m.c[cm.gcol]);
    L.cinv.push_back(m.inv_copy[cm.gcol]);
    L.clo.push_back(m.x_lo[cm.gcol]);
    L.chi.push_back(m.x_hi[cm.gcol]);
  }
  L.ameta.insert(L.ameta.end(), P.ameta.begin(), P.ameta.end());
  for (int64_t k : P.ab_src) L.ab.push_back(m.b[k]);
  L.nbrs.insert(L.nbrs.end(), P.nbrs.begin(), P.nbrs.end());
  L.P.resize(p_base + P.p_src.size());
  gather(L.P, p_base, P.p_src, m.P);
  L.A.resize(a_base + P.a_src.size());
  gather(L.A, a_base, P.a_src, m.A);

  L.max_neighbours = std::max(L.max_neighbours, P.max_neighbours);
  L.all_ops_in_smem = L.all_ops_in_smem && P.all_ops_in_smem;
  L.smem_bytes = std::max(L.smem_bytes, P.smem_bytes);
  L.K = std::max(L.K, P.K);
  L.blocks_per_instance = std::max(L.blocks_per_instance, static_cast<int>(P.blocks.size()));
  L.bytes_per_iteration += P.bytes_per_iteration;
  L.flops_per_iteration += P.flops_per_iteration;
}

void HostLayout::reset() {
  blocks.clear();
  inst.clear();
  P.clear();
  A.clear();
  copies.clear();
  rmeta.clear();
  v.clear();
  z0.clear();
  ref_of_dev.clear();
  cmeta.clear();
  cc.clear();
  cinv.clear();
  clo.clear();
  chi.clear();
  ameta.clear();
  ab.clear();
  nbrs.clear();
  max_neighbours = 0;
  rows_total = 0;
  x_total = 0;
  trace_rows_per_instance = 0;
  K = 1;
  smem_bytes = 0;
  blocks_per_instance = 1;
  all_ops_in_smem = true;
  bytes_per_iteration = 0;
  flops_per_iteration = 0;
}

void build_batch(HostLayout& L, const InstancePlan& P, const dopf_model_view* ms, int count) {
  // every instance has the plan's sizes, so instance i's slices sit at i x size:
  // size once, then fill the instances in parallel
  L.reset();
  const std::size_t I = static_cast<std::size_t>(count);
  const std::size_t nb = P.blocks.size(), rows = P.rmeta.size(), ncp = P.copies.size();
  const std::size_t ncol = P.cmeta.size(), nam = P.ameta.size(), nnb = P.nbrs.size();
  const std::size_t np = P.p_src.size(), na = P.a_src.size();
  L.blocks.resize(I * nb);
  L.inst.resize(I);
  L.rmeta.resize(I * rows);
  L.ref_of_dev.resize(I * rows);
  L.v.resize(I * rows);
  L.z0.resize(I * rows);
  L.copies.resize(I * ncp);
  L.cmeta.resize(I * ncol);
  for (auto* vec : {&L.cc, &L.cinv, &L.clo, &L.chi}) vec->resize(I * ncol);
  L.ameta.resize(I * nam);
  L.ab.resize(I * nam);
  L.nbrs.resize(I * nnb);
  L.P.resize(I * np);
  L.A.resize(I * na);
  auto fill = [&](std::size_t i0, std::size_t i1) {
    for (std::size_t i = i0; i < i1; ++i) {
      const dopf_model_view& m = ms[i];
      const int32_t row_base = static_cast<int32_t>(i * rows);
      InstDesc id{};
      id.x_off = static_cast<int64_t>(i) * P.n;
      id.n = P.n;
      id.blocks = static_cast<int32_t>(nb);
      id.block0 = static_cast<int32_t>(i * nb);
      id.rows = P.Nz;
      id.row0 = row_base;
      L.inst[i] = id;
      for (std::size_t b = 0; b < nb; ++b) {
        BlockDesc bd = P.blocks[b];
        bd.row0 += row_base;
        bd.p_off += static_cast<int64_t>(i * np);
        bd.a_off += static_cast<int64_t>(i * na);
        bd.copy_off += static_cast<int32_t>(i * ncp);
        bd.col_off += static_cast<int32_t>(i * ncol);
        bd.amet_off += static_cast<int32_t>(i * nam);
        bd.nbr_off += static_cast<int32_t>(i * nnb);
        bd.instance = static_cast<int32_t>(i);
        L.blocks[i * nb + b] = bd;
      }
      for (std::size_t d = 0; d < rows; ++d) {
        L.rmeta[i * rows + d] = P.rmeta[d];
        L.ref_of_dev[i * rows + d] = P.ref_of_dev[d];
        L.v[i * rows + d] = m.v[P.ref_of_dev[d]];
        L.z0[i * rows + d] = m.z0[P.ref_of_dev[d]];
      }
      for (std::size_t k = 0; k < ncp; ++k) {
        const int32_t c = P.copies[k];
        L.copies[i * ncp + k] = c >= 0 ? c : encode_remote(decode_remote(c) + row_base);
      }
      for (std::size_t k = 0; k < ncol; ++k) {
        const int g = P.cmeta[k].gcol;
        L.cmeta[i * ncol + k] = P.cmeta[k];
        L.cc[i * ncol + k] = m.c[g];
        L.cinv[i * ncol + k] = m.inv_copy[g];
        L.clo[i * ncol + k] = m.x_lo[g];
        L.chi[i * ncol + k] = m.x_hi[g];
      }
      for (std::size_t k = 0; k < nam; ++k) {
        L.ameta[i * nam + k] = P.ameta[k];
        L.ab[i * nam + k] = m.b[P.ab_src[k]];
      }
      for (std::size_t k = 0; k < nnb; ++k) L.nbrs[i * nnb + k] = P.nbrs[k];
      for (std::size_t k = 0; k < np; ++k) L.P[i * np + k] = P.p_src[k] >= 0 ? m.P[P.p_src[k]] : 0.0;
      for (std::size_t k = 0; k < na; ++k) L.A[i * na + k] = P.a_src[k] >= 0 ? m.A[P.a_src[k]] : 0.0;
    }
  };
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const unsigned nt = static_cast<unsigned>(std::min<std::size_t>(hw, (I + 7) / 8));
  if (nt <= 1) {
    fill(0, I);
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(fill, I * t / nt, I * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
  L.rows_total = static_cast<int64_t>(I * rows);
  L.x_total = static_cast<int64_t>(I) * P.n;
  L.max_neighbours = P.max_neighbours;
  L.all_ops_in_smem = P.all_ops_in_smem;
  L.smem_bytes = P.smem_bytes;
  L.K = P.K;
  L.blocks_per_instance = static_cast<int>(nb);
  L.bytes_per_iteration = P.bytes_per_iteration * count;
  L.flops_per_iteration = P.flops_per_iteration * count;
}

void reserve_instances(HostLayout& L, const InstancePlan& P, std::size_t count) {
  L.blocks.reserve(L.blocks.size() + count * P.blocks.size());
  L.inst.reserve(L.inst.size() + count);
  L.rmeta.reserve(L.rmeta.size() + count * P.rmeta.size());
  L.ref_of_dev.reserve(L.ref_of_dev.size() + count * P.ref_of_dev.size());
  L.v.reserve(L.v.size() + count * P.rmeta.size());
  L.z0.reserve(L.z0.size() + count * P.rmeta.size());
  L.copies.reserve(L.copies.size() + count * P.copies.size());
  L.cmeta.reserve(L.cmeta.size() + count * P.cmeta.size());
  for (auto* v : {&L.cc, &L.cinv, &L.clo, &L.chi}) v->reserve(v->size() + count * P.cmeta.size());
  L.ameta.reserve(L.ameta.size() + count * P.ameta.size());
  L.ab.reserve(L.ab.size() + count * P.ab_src.size());
  L.nbrs.reserve(L.nbrs.size() + count * P.nbrs.size());
  L.P.reserve(L.P.size() + count * P.p_src.size());
  L.A.reserve(L.A.size() + count * P.a_src.size());
}

void add_instance(HostLayout& L, const dopf_model_view& m, int G, const LayoutOptions& opt) {
  append_instance(L, plan_instance(m, G, opt), m);
}

}  // namespace dopf::cuda
