// Flat (C-ABI) view of a decomposed model and its precomputed operators:
// the arrays behind dopf_model_view (include/dopf_types.h). Shared by the
// host C ABI (capi_host.cpp) and the C++ drop-in solver (cuda_solve.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "../../../include/dopf_types.h"
#include "admm.hpp"

namespace dopf {

struct FlatModel {
  std::vector<int32_t> m_s, l2g, b_offsets;
  std::vector<int64_t> a_offsets, p_offsets;
  std::vector<double> A, b, P, v, x0, z0;
  bool has_pre = false;

  /// Builds the arrays (P, v only when `pre` is given). initial iterate per
  /// reference admm.cpp:92-116.
  void build(const DecomposedModel& model, const Precomputed* pre);
  /// View over these arrays plus the model's / precompute's own vectors;
  /// valid while all three objects live unchanged.
  dopf_model_view view(const DecomposedModel& model, const Precomputed* pre) const;
};

}  // namespace dopf
