// Host-side construction of the device layout (layout.hpp) from flat model
// views (include/dopf_types.h). Pure C++; no CUDA calls.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/dopf_types.h"
#include "layout.hpp"

namespace dopf::cuda {

struct HostLayout {
  std::vector<BlockDesc> blocks;
  std::vector<InstDesc> inst;
  std::vector<double> P, A;
  std::vector<int32_t> copies;       // device rows (global) of every copy, per block
  std::vector<RowMeta> rmeta;        // per device row
  std::vector<double> v, z0;         // per device row
  std::vector<int32_t> ref_of_dev;   // per device row: instance-local reference z index
  std::vector<ColMeta> cmeta;
  std::vector<double> cc, cinv, clo, chi;
  std::vector<AMeta> ameta;
  std::vector<double> ab;
  std::vector<int32_t> nbrs;         // per block: instance-local indices of blocks sharing columns
  int32_t max_neighbours = 0;
  int64_t rows_total = 0;
  int64_t x_total = 0;
  int64_t trace_rows_per_instance = 0;  // filled at solve time
  int K = 1;                  // rows per thread required
  std::size_t smem_bytes = 0; // max dynamic smem over blocks
  int blocks_per_instance = 1;
  bool all_ops_in_smem = true;
  double bytes_per_iteration = 0;  // algorithmic (BASELINE.md formula), sum over instances
  double flops_per_iteration = 0;

  void reset();  // empty, keeping capacity (re-uploads reuse the host memory)
};

struct LayoutOptions {
  int blocks_per_instance = 0;        // 0: choose
  std::size_t smem_limit = 227 * 1024;
  int max_blocks = 148;               // co-resident CTA budget (1 per SM)
  int threads = kThreads;
  // optional per-block cost shares of a single instance's split (G entries):
  // a partition tuned from measured slack (DOPF_BLOCK_WEIGHTS)
  std::vector<double> block_weights;
};

/// Index structure of one instance's device layout (instance-relative
/// offsets) plus the gather maps that fill its numeric arrays. Depends only on
/// the model's sparsity structure, so it is reused across uploads of models
/// with the same structure (re-solves with new data, scenario batches).
struct InstancePlan {
  int S = 0, n = 0, Nz = 0, G = 0;
  LayoutOptions opt;
  std::vector<int32_t> z_offsets, m_s, l2g, csr_ptr, csr_copy;  // structure signature
  std::vector<BlockDesc> blocks;
  std::vector<RowMeta> rmeta;
  std::vector<int32_t> ref_of_dev, copies, nbrs;
  std::vector<ColMeta> cmeta;
  std::vector<AMeta> ameta;
  std::vector<int64_t> ab_src, p_src, a_src;  // indices into the view's b / P / A (-1: zero pad)
  int K = 1;
  int max_neighbours = 0;
  std::size_t smem_bytes = 0;
  bool all_ops_in_smem = true;
  double bytes_per_iteration = 0, flops_per_iteration = 0;

  bool same_structure(const dopf_model_view& m, const LayoutOptions& o) const;
};

InstancePlan plan_instance(const dopf_model_view& m, int G, const LayoutOptions& opt);
/// The whole layout of `count` instances sharing `plan`'s structure
/// (scenario batches), filled in parallel.
void build_batch(HostLayout& L, const InstancePlan& plan, const dopf_model_view* ms, int count);
/// Reserves room for `count` more instances of this plan.
void reserve_instances(HostLayout& L, const InstancePlan& plan, std::size_t count);
/// Appends one instance: rebased index structure + values gathered from m.
void append_instance(HostLayout& L, const InstancePlan& plan, const dopf_model_view& m);

/// Depth-first order of the component graph (subsystems adjacent when they
/// share a global column): cutting it into pieces keeps copies together.
std::vector<int> locality_order(const dopf_model_view& m);

/// Picks the CTA count for one instance: enough CTAs that every block's
/// operators fit in shared memory and rows fit kMaxK per thread.
int choose_blocks(const dopf_model_view& m, const LayoutOptions& opt);

/// Appends one instance split into `G` blocks.
void add_instance(HostLayout& L, const dopf_model_view& m, int G, const LayoutOptions& opt);

/// Algorithmic bytes per iteration:
/// 8(sum n^2 + sum mn + sum m) + 56 N_z + 48 n + 4(2 N_z + n + 1) + 16 S.
double algorithmic_bytes(const dopf_model_view& m);
double algorithmic_flops(const dopf_model_view& m);

std::size_t block_smem_bytes(const BlockDesc& b, bool ops_in_smem);

}  // namespace dopf::cuda
