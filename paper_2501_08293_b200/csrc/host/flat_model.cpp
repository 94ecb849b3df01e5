#include "flat_model.hpp"

#include <algorithm>

namespace dopf {

void FlatModel::build(const DecomposedModel& md, const Precomputed* pre) {
  const int S = md.subsystem_count();
  m_s.assign(S, 0);
  a_offsets.assign(S + 1, 0);
  p_offsets.assign(S + 1, 0);
  b_offsets.assign(S + 1, 0);
  l2g.clear();
  l2g.reserve(md.total_local_vars());
  for (int s = 0; s < S; ++s) {
    const auto& sub = md.subsystems[s];
    m_s[s] = sub.row_count();
    a_offsets[s + 1] = a_offsets[s] + static_cast<int64_t>(sub.row_count()) * sub.col_count();
    p_offsets[s + 1] = p_offsets[s] + static_cast<int64_t>(sub.col_count()) * sub.col_count();
    b_offsets[s + 1] = b_offsets[s] + sub.row_count();
    l2g.insert(l2g.end(), sub.local_to_global.begin(), sub.local_to_global.end());
  }
  A.resize(a_offsets[S]);
  b.resize(b_offsets[S]);
  for (int s = 0; s < S; ++s) {
    const auto& sub = md.subsystems[s];
    std::copy(sub.A.a.begin(), sub.A.a.end(), A.begin() + a_offsets[s]);
    std::copy(sub.b.begin(), sub.b.end(), b.begin() + b_offsets[s]);
  }
  x0.resize(md.global_cols);
  for (int i = 0; i < md.global_cols; ++i) x0[i] = initial_value(md, i);
  z0.resize(md.total_local_vars());
  for (std::size_t k = 0; k < l2g.size(); ++k) z0[k] = x0[l2g[k]];
  has_pre = pre != nullptr;
  if (pre) {
    P.resize(p_offsets[S]);
    v.resize(md.total_local_vars());
    for (int s = 0; s < S; ++s) {
      const auto& ps = pre->subs[s];
      std::copy(ps.kernel_projector.a.begin(), ps.kernel_projector.a.end(), P.begin() + p_offsets[s]);
      std::copy(ps.min_norm_solution.begin(), ps.min_norm_solution.end(), v.begin() + md.z_offsets[s]);
    }
  } else {
    P.clear();
    v.clear();
  }
}

dopf_model_view FlatModel::view(const DecomposedModel& md, const Precomputed* pre) const {
  dopf_model_view out{};
  out.S = md.subsystem_count();
  out.n = md.global_cols;
  out.N_z = md.total_local_vars();
  out.has_pre = has_pre && pre ? 1 : 0;
  out.z_offsets = md.z_offsets.data();
  out.l2g = l2g.data();
  out.m_s = m_s.data();
  out.a_offsets = a_offsets.data();
  out.A = A.data();
  out.b_offsets = b_offsets.data();
  out.b = b.data();
  out.p_offsets = p_offsets.data();
  out.P = out.has_pre ? P.data() : nullptr;
  out.v = out.has_pre ? v.data() : nullptr;
  out.inv_copy = out.has_pre ? pre->inv_copy_counts.data() : nullptr;
  out.csr_ptr = out.has_pre ? pre->col_ptr.data() : nullptr;
  out.csr_copy = out.has_pre ? pre->copy_index.data() : nullptr;
  out.c = md.c.data();
  out.x_lo = md.x_lo.data();
  out.x_hi = md.x_hi.data();
  out.x0 = x0.data();
  out.z0 = z0.data();
  return out;
}

}  // namespace dopf
