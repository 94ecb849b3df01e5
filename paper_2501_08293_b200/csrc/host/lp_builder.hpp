// Centralized LinDistFlow LP: min c'x s.t. A x = b, lo <= x <= hi.
//
// Interface mirrors reference dopf/linear_system.hpp:13-79 and
// dopf/lp_builder.hpp:13-57. A is kept as CSR (rows sorted by column) instead
// of an Eigen row-major sparse matrix; the contents (row order, column order,
// coefficient values and the exact-zero drop rule) are identical.
#pragma once

#include <iosfwd>
#include <string>
#include <unordered_map>
#include <vector>

#include "feeder.hpp"

namespace dopf {

enum class VarKind { p_gen, q_gen, w, p_bus_load, q_bus_load, p_load, q_load, p_flow, q_flow };
enum class FlowDirection { from_to, to_from };

struct VariableKey {
  VarKind kind = VarKind::w;
  std::string owner;
  int phase = 1;
  FlowDirection direction = FlowDirection::from_to;
  bool operator==(const VariableKey&) const = default;
};
std::string to_string(const VariableKey& key);

enum class RowFamily { balance_p, balance_q, load_p, load_q, load_link, loss_p, loss_q, drop };
enum class OwnerKind { bus, line };

struct RowTag {
  OwnerKind owner_kind = OwnerKind::bus;
  std::string owner;
  RowFamily family = RowFamily::balance_p;
  bool operator==(const RowTag&) const = default;
};
std::string to_string(const RowTag& tag);

struct LinearSystem {
  int rows = 0, cols = 0;
  std::vector<int> row_ptr;     // rows+1
  std::vector<int> col_idx;     // ascending within a row
  std::vector<double> values;
  std::vector<double> b, c, x_lo, x_hi;
  std::vector<VariableKey> var_table;
  std::vector<RowTag> row_tags;
};

void dump_linear_system(const LinearSystem& ls, std::ostream& out);

/// Column order: generators, squared voltages, loads, flows; within each
/// block by owner id then phase (reference lp_builder.cpp:91-116).
std::vector<VariableKey> index_variables(const Feeder& f);

/// Column lookup; throws std::out_of_range for unknown keys
/// (reference lp_builder.cpp:118-133).
class VarIndex {
 public:
  explicit VarIndex(const std::vector<VariableKey>& table);
  int at(VarKind kind, const std::string& owner, int phase,
         FlowDirection direction = FlowDirection::from_to) const;
  int size() const { return size_; }

 private:
  std::unordered_map<std::string, int> index_;
  int size_ = 0;
};

struct RowSpec {
  RowTag tag;
  std::vector<std::pair<int, double>> coeffs;  // sorted by column, exact zeros dropped
  double rhs = 0.0;
};

std::vector<RowSpec> build_power_balance(const Feeder& f, const VarIndex& vars);
std::vector<RowSpec> build_load_model(const Feeder& f, const VarIndex& vars);
std::vector<RowSpec> build_flow_equations(const Feeder& f, const VarIndex& vars);

/// Line voltage-drop sensitivities, np x np row-major (reference :275-296).
void build_m_matrices(const LineSegment& line, std::vector<double>& mp, std::vector<double>& mq);

LinearSystem assemble_centralized(const Feeder& f);

}  // namespace dopf
