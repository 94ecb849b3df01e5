// Seeded synthetic feeders of the paper's benchmark shapes.
//
// The reference ships no IEEE feeder data (README.md:65-67;
// acceptance.cpp:352-360 skips IEEE 13). These generators produce feeders
// with the paper's structural counts (Table I-III: nodes, lines,
// merged leaves, component count S, LP column count) using the value ranges
// of the reference's only synthetic-feeder pattern, test_util.hpp:77-172
// (impedances, shunts, taps, load coefficients, exponents), scaled so the LP
// stays feasible on deep trees (voltage drop budget, shunt totals).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "feeder.hpp"

namespace dopf {

struct ShapeSpec {
  std::string name;
  int nodes = 0;        // buses
  int lines = 0;        // >= nodes - 1; the excess closes loops between non-leaf buses
  int leaves = 0;       // degree-1 buses (each becomes one merged-leaf component)
  int target_cols = 0;  // exact LP column count to hit (0: any)
  double p_three_phase = 0.9;  // probability a child of a 3-phase bus stays 3-phase
  double p_two_phase = 0.05;   // ... becomes 2-phase (else single phase)
  double load_fraction = 0.5;  // share of non-root buses with a load when target_cols == 0
  double total_load = 1.5;     // p.u. of real demand spread over all loads
  std::string id_prefix;       // prepended to every id (tiling)
};

/// Named shapes: "ieee13", "ieee123", "ieee8500".
ShapeSpec shape_by_name(const std::string& name);

/// Radial (plus loop-closing lines) feeder with exactly spec.nodes buses,
/// spec.lines lines and spec.leaves degree-1 buses. Deterministic in seed.
Feeder generate_feeder(const ShapeSpec& spec, std::uint64_t seed);

/// `copies` tiles of `shape`, each keeping its own generator, every tile root
/// tied to one common pinned root bus by a 3-phase tie line. Tile t's ids carry
/// the prefix "tNN_" so each tile's buses and lines are contiguous in id order.
Feeder generate_tiled_feeder(const ShapeSpec& shape, int copies, std::uint64_t seed);

/// Load scenario: every load's (a, b) scaled by an independent U[lo, hi] factor.
Feeder scale_loads(const Feeder& base, std::uint64_t seed, double lo = 0.5, double hi = 1.5);

/// Splitmix64-based generator (portable, unlike std:: distributions).
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull) {}
  std::uint64_t next() {
    std::uint64_t z = (s_ += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  int below(int n) { return static_cast<int>(next() % static_cast<std::uint64_t>(n)); }

 private:
  std::uint64_t s_;
};

}  // namespace dopf
