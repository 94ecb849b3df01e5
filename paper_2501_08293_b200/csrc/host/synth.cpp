#include "synth.hpp"

#include <algorithm>
#include <exception>
#include <mutex>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace dopf {

ShapeSpec shape_by_name(const std::string& name) {
  ShapeSpec s;
  s.name = name;
  if (name == "ieee13") {
    // PAPER.md Table I-II: A is 456 x 454; 29 nodes, 28 lines, 7 leaves, S = 50
    s.nodes = 29; s.lines = 28; s.leaves = 7; s.target_cols = 454;
    s.p_three_phase = 0.75; s.p_two_phase = 0.1; s.total_load = 1.2;
  } else if (name == "ieee123") {
    // 1834 x 1834; 147 nodes, 146 lines, 43 leaves, S = 250
    s.nodes = 147; s.lines = 146; s.leaves = 43; s.target_cols = 1834;
    s.p_three_phase = 0.6; s.p_two_phase = 0.1; s.total_load = 1.5;
  } else if (name == "ieee8500") {
    // 86114 x 87285; 11932 nodes, 14291 lines, 1222 leaves, S = 25001
    s.nodes = 11932; s.lines = 14291; s.leaves = 1222; s.target_cols = 87285;
    s.p_three_phase = 0.5; s.p_two_phase = 0.05; s.total_load = 1.5;
  } else {
    throw std::invalid_argument("unknown feeder shape '" + name + "' (ieee13, ieee123, ieee8500)");
  }
  return s;
}

namespace {

std::string padded(const std::string& prefix, int value, int width) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%0*d", width, value);
  return prefix + buf;
}

std::vector<int> random_subset(Rng& rng, const std::vector<int>& from, int k) {
  std::vector<int> pool = from;
  for (int i = static_cast<int>(pool.size()) - 1; i > 0; --i) std::swap(pool[i], pool[rng.below(i + 1)]);
  pool.resize(k);
  std::sort(pool.begin(), pool.end());
  return pool;
}

struct Attempt {
  bool ok = false;
  Feeder feeder;
  int base_cols = 0;
};

Attempt build(const ShapeSpec& spec, Rng& rng, double p3) {
  Attempt out;
  const int B = spec.nodes, K = spec.leaves, I = B - K;
  if (B < 2 || I < 1 || spec.lines < B - 1) throw std::invalid_argument("inconsistent shape counts");

  // Internal tree: chains that occasionally branch from a random earlier node.
  std::vector<int> parent(B, -1);
  // Every leaf of the internal tree takes one real leaf, so the internal tree
  // has ~K leaves: many short laterals, shallow depth (fast consensus mixing).
  const int target_internal_leaves = std::max(1, K - 1);
  const double p_branch = I > 2 ? static_cast<double>(target_internal_leaves - 1) / (I - 1) : 0.0;
  for (int i = 1; i < I; ++i)
    parent[i] = (i >= 2 && rng.unit() < p_branch) ? rng.below(i - 1) : i - 1;
  std::vector<int> children(B, 0);
  for (int i = 1; i < I; ++i) ++children[parent[i]];
  std::vector<int> needy;  // internal nodes that need a leaf to reach degree >= 2
  for (int i = 1; i < I; ++i)
    if (children[i] == 0) needy.push_back(i);
  if (I == 1 || children[0] == 1) needy.push_back(0);
  if (I == 1 && K >= 2) needy.push_back(0);
  if (static_cast<int>(needy.size()) > K) return out;
  int next_leaf = I;
  for (int v : needy) parent[next_leaf++] = v;
  while (next_leaf < B) parent[next_leaf++] = rng.below(I);

  // DFS preorder numbering so ids (and hence subsystem order) follow the tree.
  std::vector<std::vector<int>> kids(B);
  for (int v = 1; v < B; ++v) kids[parent[v]].push_back(v);
  std::vector<int> order, depth(B, 0), stack{0};
  order.reserve(B);
  while (!stack.empty()) {
    const int u = stack.back();
    stack.pop_back();
    order.push_back(u);
    for (auto it = kids[u].rbegin(); it != kids[u].rend(); ++it) {
      depth[*it] = depth[u] + 1;
      stack.push_back(*it);
    }
  }
  std::vector<int> pos(B);
  for (int k = 0; k < B; ++k) pos[order[k]] = k;
  const int depth_max = *std::max_element(depth.begin(), depth.end());

  // Phases: a child keeps a subset of its parent's phases.
  std::vector<std::vector<int>> phases(B);
  phases[0] = {1, 2, 3};
  for (int u : order) {
    for (int v : kids[u]) {
      const auto& pp = phases[u];
      const double r = rng.unit();
      if (pp.size() == 3) {
        if (r < p3) phases[v] = pp;
        else if (r < p3 + spec.p_two_phase) phases[v] = random_subset(rng, pp, 2);
        else phases[v] = random_subset(rng, pp, 1);
      } else if (pp.size() == 2) {
        phases[v] = r < 0.5 ? pp : random_subset(rng, pp, 1);
      } else {
        phases[v] = pp;
      }
    }
  }

  const std::string& pre = spec.id_prefix;
  const int width = B >= 10000 ? 5 : (B >= 1000 ? 4 : 3);
  auto bus_id = [&](int v) { return padded(pre + "n", pos[v], width); };

  Feeder f;
  f.base_mva = 1.0;
  const double shunt_scale = std::min(1.0, 5.0 / B);
  for (int v : order) {
    Bus bus;
    bus.id = bus_id(v);
    bus.phases = PhaseSet(phases[v]);
    for (std::size_t k = 0; k < phases[v].size(); ++k) {
      if (v == 0) {
        bus.w_lo.push_back(1.0);
        bus.w_hi.push_back(1.0);
      } else {
        bus.w_lo.push_back(0.81);
        bus.w_hi.push_back(1.21);
      }
      bus.g_sh.push_back(0.01 * shunt_scale * rng.unit());
      bus.b_sh.push_back(0.01 * shunt_scale * rng.unit());
    }
    f.buses.push_back(std::move(bus));
  }

  // Voltage-drop budget: sum over a root path of ~2(r+x)P stays below ~0.1.
  const double z_scale = std::min(1.0, 5.0 / (spec.total_load * std::max(1, depth_max)));
  const double line_shunt_scale = std::min(1.0, 10.0 / spec.lines);
  const double flow_cap = std::max(2.0, 3.0 * spec.total_load);
  auto make_line = [&](const std::string& id, int from, int to, const std::vector<int>& ph,
                       bool may_tap) {
    LineSegment ln;
    ln.id = id;
    ln.from_bus = bus_id(from);
    ln.to_bus = bus_id(to);
    ln.phases = PhaseSet(ph);
    const int np = static_cast<int>(ph.size());
    ln.r.assign(np, std::vector<double>(np, 0.0));
    ln.x.assign(np, std::vector<double>(np, 0.0));
    for (int a = 0; a < np; ++a)
      for (int b = a; b < np; ++b) {
        const double rv = a == b ? 0.01 + 0.01 * rng.unit() : 0.002 * rng.unit();
        const double xv = a == b ? 0.02 + 0.01 * rng.unit() : 0.004 * rng.unit();
        ln.r[a][b] = ln.r[b][a] = rv * z_scale;
        ln.x[a][b] = ln.x[b][a] = xv * z_scale;
      }
    const bool tap = may_tap && rng.unit() < 0.2;
    for (int k = 0; k < np; ++k) {
      ln.g_s_from.push_back(0.001 * line_shunt_scale * rng.unit());
      ln.b_s_from.push_back(0.002 * line_shunt_scale * rng.unit());
      ln.g_s_to.push_back(0.001 * line_shunt_scale * rng.unit());
      ln.b_s_to.push_back(0.002 * line_shunt_scale * rng.unit());
      ln.tau.push_back(tap ? 1.0404 : 1.0);
      ln.p_lo.push_back(rng.unit() < 0.5 ? -kInf : -flow_cap);
      ln.p_hi.push_back(rng.unit() < 0.5 ? kInf : flow_cap);
      ln.q_lo.push_back(-flow_cap);
      ln.q_hi.push_back(flow_cap);
    }
    return ln;
  };

  // Tree lines (id follows the child). At most one off-nominal tap per root
  // path, and only near the root, so the tap product stays >= 1/1.0404.
  std::vector<char> tapped_path(B, 0);
  for (int v : order) {
    if (v == 0) continue;
    const int u = parent[v];
    const bool may_tap = !tapped_path[u] && depth[v] <= 3;
    LineSegment ln = make_line(padded(pre + "l", pos[v], width), u, v, phases[v], may_tap);
    tapped_path[v] = tapped_path[u] || ln.tau[0] != 1.0;
    f.lines.push_back(std::move(ln));
  }

  // Loop-closing lines between non-leaf buses close to each other in DFS
  // order (sharing at least one phase). Leaves are never touched, so the
  // merged-leaf count stays exact.
  const int extra = spec.lines - (B - 1);
  std::vector<char> is_leaf(B, 0);
  for (int v = 1; v < B; ++v) is_leaf[v] = kids[v].empty();
  if (extra > 0) {
    std::vector<int> nonleaf_by_pos;
    for (int k = 0; k < B; ++k)
      if (!is_leaf[order[k]] && order[k] != 0) nonleaf_by_pos.push_back(order[k]);
    const int NL = static_cast<int>(nonleaf_by_pos.size());
    if (NL < 3) return out;
    std::vector<int> loops_at(B, 0);
    int made = 0, guard = 0;
    while (made < extra && guard < 50 * extra + 1000) {
      ++guard;
      const int a = rng.below(NL);
      const int b = a + 2 + rng.below(24);
      if (b >= NL) continue;
      const int u = nonleaf_by_pos[a], v = nonleaf_by_pos[b];
      if (parent[v] == u || parent[u] == v) continue;
      std::vector<int> common;
      for (int p : phases[u])
        if (std::find(phases[v].begin(), phases[v].end(), p) != phases[v].end()) common.push_back(p);
      if (common.empty()) continue;
      const int k = loops_at[u]++;
      const std::string id = padded(pre + "l", pos[u], width) + "x" + std::to_string(k);
      f.lines.push_back(make_line(id, u, v, common, false));
      ++made;
    }
    if (made < extra) return out;
  }

  // Column budget: generator (2 per phase), w (1 per bus phase), flows
  // (4 per line phase); loads fill the remainder at 4 per load phase.
  int base = 2 * 3;
  for (const Bus& bus : f.buses) base += bus.phases.size();
  for (const LineSegment& ln : f.lines) base += 4 * ln.phases.size();
  out.base_cols = base;
  int load_phases = -1;
  if (spec.target_cols > 0) {
    const int rem = spec.target_cols - base;
    if (rem < 4 * std::max(1, (B - 1) / 8) || rem % 4 != 0) return out;
    load_phases = rem / 4;
    if (load_phases > 3 * (B - 1)) return out;
  }

  std::vector<int> candidates;
  for (int v : order)
    if (v != 0) candidates.push_back(v);
  std::vector<int> loads_on(B, 0);
  auto add_load = [&](int v, const std::vector<int>& ph, bool delta) {
    Load ld;
    const int k = loads_on[v]++;
    ld.id = padded(pre + "d", pos[v], width) + (k ? std::string(1, static_cast<char>('a' + k)) : "");
    ld.bus = bus_id(v);
    ld.connection = delta ? Connection::delta : Connection::wye;
    ld.phases = PhaseSet(ph);
    for (std::size_t q = 0; q < ph.size(); ++q) {
      ld.a.push_back(0.2 * rng.unit());
      ld.b.push_back(0.1 * rng.unit());
      const double e = static_cast<double>(rng.next() % 3);
      ld.alpha.push_back(e);
      ld.beta.push_back(e);
    }
    f.loads.push_back(std::move(ld));
  };
  if (load_phases < 0) {
    for (int v : candidates) {
      if (rng.unit() >= spec.load_fraction) continue;
      const bool delta = phases[v].size() == 3 && rng.unit() < 0.3;
      add_load(v, phases[v], delta);
    }
  } else {
    // Leaves first (every lateral end carries demand), then random buses.
    std::vector<int> seq;
    for (int v : candidates)
      if (is_leaf[v]) seq.push_back(v);
    std::vector<int> rest;
    for (int v : candidates)
      if (!is_leaf[v]) rest.push_back(v);
    for (int i = static_cast<int>(rest.size()) - 1; i > 0; --i) std::swap(rest[i], rest[rng.below(i + 1)]);
    seq.insert(seq.end(), rest.begin(), rest.end());
    int remaining = load_phases;
    std::size_t cursor = 0;
    while (remaining > 0) {
      const int v = seq[cursor++ % seq.size()];
      if (loads_on[v] >= 20) continue;
      const auto& ph = phases[v];
      const int np = static_cast<int>(ph.size());
      if (np == 3 && remaining >= 3 && rng.unit() < 0.3) {
        add_load(v, ph, true);
        remaining -= 3;
      } else {
        const int k = std::min(np, remaining);
        add_load(v, k == np ? ph : random_subset(rng, ph, k), false);
        remaining -= k;
      }
    }
  }
  // Normalise total real demand.
  double total = 0.0;
  for (const Load& ld : f.loads)
    for (double a : ld.a) total += a;
  if (total > 0) {
    const double s = spec.total_load / total;
    for (Load& ld : f.loads) {
      for (double& a : ld.a) a *= s;
      for (double& b : ld.b) b *= s;
    }
  }

  Generator g;
  g.id = pre + "g0";
  g.bus = bus_id(0);
  g.phases = PhaseSet({1, 2, 3});
  const double cap = 5.0 * std::max(1.0, spec.total_load);
  for (int k = 0; k < 3; ++k) {
    g.p_lo.push_back(0.0);
    g.p_hi.push_back(cap);
    g.q_lo.push_back(-cap);
    g.q_hi.push_back(cap);
  }
  f.generators.push_back(std::move(g));
  canonicalize_feeder(f);
  out.feeder = std::move(f);
  out.ok = true;
  return out;
}

}  // namespace

Feeder generate_feeder(const ShapeSpec& spec, std::uint64_t seed) {
  double p3 = spec.p_three_phase;
  for (int attempt = 0; attempt < 400; ++attempt) {
    Rng rng(seed * 7919ull + static_cast<std::uint64_t>(attempt));
    Attempt a = build(spec, rng, p3);
    if (a.ok) return std::move(a.feeder);
    if (spec.target_cols > 0 && a.base_cols > 0) {
      // steer the phase mix toward the column budget
      const int slack = spec.target_cols - a.base_cols;
      if (slack < 4 * std::max(1, (spec.nodes - 1) / 8)) p3 *= 0.97;
      else if (slack > 4 * 3 * (spec.nodes - 1)) p3 = std::min(0.99, p3 * 1.03);
    }
  }
  throw std::runtime_error("could not generate a feeder of shape '" + spec.name + "'");
}

Feeder generate_tiled_feeder(const ShapeSpec& shape, int copies, std::uint64_t seed) {
  if (copies < 1) throw std::invalid_argument("copies must be >= 1");
  Feeder all;
  all.base_mva = 1.0;
  Bus root;
  root.id = "r_root";
  root.phases = PhaseSet({1, 2, 3});
  root.w_lo = {1.0, 1.0, 1.0};
  root.w_hi = {1.0, 1.0, 1.0};
  root.g_sh = {0.0, 0.0, 0.0};
  root.b_sh = {0.0, 0.0, 0.0};
  all.buses.push_back(root);
  // tiles are independent (own seed and id prefix): generate them in parallel
  std::vector<Feeder> tiles(copies);
  {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nt = std::min<unsigned>(hw, static_cast<unsigned>(copies));
    std::vector<std::thread> th;
    std::exception_ptr err;
    std::mutex mu;
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([&, w] {
        for (int t = static_cast<int>(w); t < copies; t += static_cast<int>(nt)) {
          try {
            ShapeSpec spec = shape;
            spec.id_prefix = padded("t", t, 2) + "_";
            tiles[t] = generate_feeder(spec, seed * 131ull + static_cast<std::uint64_t>(t));
          } catch (...) {
            std::lock_guard<std::mutex> lk(mu);
            err = std::current_exception();
          }
        }
      });
    for (auto& x : th) x.join();
    if (err) std::rethrow_exception(err);
  }
  for (int t = 0; t < copies; ++t) {
    Feeder& tile = tiles[t];
    // the tile root is no longer pinned: the tie line couples it to r_root
    Bus& troot = tile.buses.front();
    for (std::size_t k = 0; k < troot.w_lo.size(); ++k) {
      troot.w_lo[k] = 0.95;
      troot.w_hi[k] = 1.05;
    }
    LineSegment tie;
    tie.id = padded("r_tie", t, 2);
    tie.from_bus = root.id;
    tie.to_bus = troot.id;
    tie.phases = PhaseSet({1, 2, 3});
    tie.r.assign(3, std::vector<double>(3, 0.0));
    tie.x.assign(3, std::vector<double>(3, 0.0));
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        tie.r[a][b] = a == b ? 1e-4 : 2e-5;
        tie.x[a][b] = a == b ? 2e-4 : 4e-5;
      }
    tie.g_s_from = tie.b_s_from = tie.g_s_to = tie.b_s_to = {0.0, 0.0, 0.0};
    tie.tau = {1.0, 1.0, 1.0};
    tie.p_lo = tie.q_lo = {-5.0, -5.0, -5.0};
    tie.p_hi = tie.q_hi = {5.0, 5.0, 5.0};
    all.lines.push_back(std::move(tie));
    for (auto& b : tile.buses) all.buses.push_back(std::move(b));
    for (auto& l : tile.lines) all.lines.push_back(std::move(l));
    for (auto& d : tile.loads) all.loads.push_back(std::move(d));
    for (auto& g : tile.generators) all.generators.push_back(std::move(g));
  }
  canonicalize_feeder(all);
  return all;
}

Feeder scale_loads(const Feeder& base, std::uint64_t seed, double lo, double hi) {
  Feeder f = base;
  Rng rng(seed ^ 0xA5A5A5A5DEADBEEFull);
  for (Load& ld : f.loads) {
    const double s = lo + (hi - lo) * rng.unit();
    for (double& a : ld.a) a *= s;
    for (double& b : ld.b) b *= s;
  }
  return f;
}

}  // namespace dopf
