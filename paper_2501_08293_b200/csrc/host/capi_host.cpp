// extern "C" wrappers of the host front-end (include/dopf_host.h).
#include <chrono>
#include <cstring>
#include <new>
#include <sstream>
#include <string>
#include <unordered_set>

#include "../../../include/dopf_host.h"
#include "admm.hpp"
#include "decompose.hpp"
#include "feeder.hpp"
#include "flat_model.hpp"
#include "lp_builder.hpp"
#include "synth.hpp"

struct dopf_feeder {
  dopf::Feeder f;
};

struct dopf_lp {
  dopf::LinearSystem ls;
  std::vector<int32_t> var_kind;
};

struct dopf_model {
  dopf::DecomposedModel model;
  bool has_pre = false;
  dopf::Precomputed pre;
  double precompute_seconds = 0.0;
  // flattened view storage (built lazily, invalidated by mutation)
  bool flat_ready = false;
  dopf::FlatModel flat;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename F>
int guarded(F&& body) {
  try {
    body();
    return DOPF_OK;
  } catch (const dopf::ParseError& e) {
    return fail(DOPF_ERR_PARSE, e.what());
  } catch (const dopf::SingularSubsystemError& e) {
    return fail(DOPF_ERR_SINGULAR, e.what());
  } catch (const dopf::InfeasibleSubsystemError& e) {
    return fail(DOPF_ERR_INFEASIBLE, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(DOPF_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::out_of_range& e) {
    return fail(DOPF_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::logic_error& e) {
    return fail(DOPF_ERR_LOGIC, e.what());
  } catch (const std::bad_alloc&) {
    return fail(DOPF_ERR_OUT_OF_MEMORY, "out of host memory");
  } catch (const std::exception& e) {
    return fail(DOPF_ERR_RUNTIME, e.what());
  }
}

int emit_text(const std::string& text, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = text.size() + 1;
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, text.size());
    std::memcpy(buf, text.data(), n);
    buf[n] = '\0';
  }
  return DOPF_OK;
}

void flatten(dopf_model* m) {
  if (m->flat_ready) return;
  m->flat.build(m->model, m->has_pre ? &m->pre : nullptr);
  m->flat_ready = true;
}

}  // namespace

extern "C" {

const char* dopf_last_error(void) { return g_last_error.c_str(); }

int dopf_feeder_parse(const char* text, size_t len, dopf_feeder** out) {
  if (!text || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { *out = new dopf_feeder{dopf::parse_feeder(std::string(text, len))}; });
}

int dopf_feeder_parse_file(const char* path, dopf_feeder** out) {
  if (!path || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { *out = new dopf_feeder{dopf::parse_feeder_file(path)}; });
}

int dopf_feeder_synthetic(const char* shape, uint64_t seed, dopf_feeder** out) {
  if (!shape || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = new dopf_feeder{dopf::generate_feeder(dopf::shape_by_name(shape), seed)};
  });
}

int dopf_feeder_synthetic_tiled(const char* shape, int32_t copies, uint64_t seed,
                                dopf_feeder** out) {
  if (!shape || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    *out = new dopf_feeder{dopf::generate_tiled_feeder(dopf::shape_by_name(shape), copies, seed)};
  });
}

int dopf_feeder_scale_loads(const dopf_feeder* base, uint64_t seed, dopf_feeder** out) {
  if (!base || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] { *out = new dopf_feeder{dopf::scale_loads(base->f, seed)}; });
}

int dopf_feeder_serialize(const dopf_feeder* f, char* buf, size_t cap, size_t* needed) {
  if (!f) return fail(DOPF_ERR_INVALID_ARGUMENT, "null feeder");
  int rc = DOPF_OK;
  const int g = guarded([&] { rc = emit_text(dopf::serialize_feeder(f->f), buf, cap, needed); });
  return g != DOPF_OK ? g : rc;
}

int dopf_feeder_validate(const dopf_feeder* f, char* buf, size_t cap, size_t* needed,
                         int32_t* n_errors) {
  if (!f) return fail(DOPF_ERR_INVALID_ARGUMENT, "null feeder");
  return guarded([&] {
    const auto diags = dopf::validate_feeder(f->f);
    std::string text;
    int errors = 0;
    for (const auto& d : diags) {
      errors += d.severity == dopf::Severity::error;
      text += (d.severity == dopf::Severity::error ? "error\t" : "warning\t") + d.component + "\t" +
              d.message + "\n";
    }
    if (n_errors) *n_errors = errors;
    emit_text(text, buf, cap, needed);
  });
}

int dopf_feeder_counts(const dopf_feeder* f, int32_t* counts) {
  if (!f || !counts) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    counts[0] = static_cast<int32_t>(f->f.buses.size());
    counts[1] = static_cast<int32_t>(f->f.generators.size());
    counts[2] = static_cast<int32_t>(f->f.lines.size());
    counts[3] = static_cast<int32_t>(f->f.loads.size());
    int leaves = 0;
    for (const auto& c : dopf::build_component_graph(f->f))
      leaves += c.kind == dopf::ComponentKind::merged_leaf;
    counts[4] = leaves;
  });
}

void dopf_feeder_free(dopf_feeder* f) { delete f; }

int dopf_lp_assemble(const dopf_feeder* f, dopf_lp** out) {
  if (!f || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto* lp = new dopf_lp{dopf::assemble_centralized(f->f), {}};
    lp->var_kind.reserve(lp->ls.cols);
    for (const auto& k : lp->ls.var_table) lp->var_kind.push_back(static_cast<int32_t>(k.kind));
    *out = lp;
  });
}

int dopf_lp_view_get(const dopf_lp* lp, dopf_lp_view* out) {
  if (!lp || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  const auto& ls = lp->ls;
  out->rows = ls.rows;
  out->cols = ls.cols;
  out->nnz = static_cast<int32_t>(ls.values.size());
  out->reserved = 0;
  out->row_ptr = ls.row_ptr.data();
  out->col_idx = ls.col_idx.data();
  out->values = ls.values.data();
  out->b = ls.b.data();
  out->c = ls.c.data();
  out->x_lo = ls.x_lo.data();
  out->x_hi = ls.x_hi.data();
  out->var_kind = lp->var_kind.data();
  return DOPF_OK;
}

int dopf_lp_var_key(const dopf_lp* lp, int32_t col, char* buf, size_t cap) {
  if (!lp || col < 0 || col >= lp->ls.cols) return fail(DOPF_ERR_INVALID_ARGUMENT, "bad column");
  return emit_text(dopf::to_string(lp->ls.var_table[col]), buf, cap, nullptr);
}

int dopf_lp_row_tag(const dopf_lp* lp, int32_t row, char* buf, size_t cap) {
  if (!lp || row < 0 || row >= lp->ls.rows) return fail(DOPF_ERR_INVALID_ARGUMENT, "bad row");
  return emit_text(dopf::to_string(lp->ls.row_tags[row]), buf, cap, nullptr);
}

int dopf_lp_dump(const dopf_lp* lp, char* buf, size_t cap, size_t* needed) {
  if (!lp) return fail(DOPF_ERR_INVALID_ARGUMENT, "null lp");
  return guarded([&] {
    std::ostringstream os;
    dopf::dump_linear_system(lp->ls, os);
    emit_text(os.str(), buf, cap, needed);
  });
}

void dopf_lp_free(dopf_lp* lp) { delete lp; }

int dopf_model_decompose(const dopf_lp* lp, const dopf_feeder* f, double tol, int32_t workers,
                         dopf_model** out) {
  if (!lp || !f || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto* m = new dopf_model();
    try {
      m->model = dopf::decompose(lp->ls, f->f, tol, workers < 1 ? 1 : workers);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int dopf_model_partition(const dopf_lp* lp, const dopf_feeder* f, dopf_model** out) {
  if (!lp || !f || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto* m = new dopf_model();
    try {
      m->model = dopf::partition(lp->ls, dopf::build_component_graph(f->f));
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int dopf_model_reduce(dopf_model* m, double tol, int32_t workers) {
  if (!m) return fail(DOPF_ERR_INVALID_ARGUMENT, "null model");
  return guarded([&] {
    dopf::reduce_subsystems(m->model, tol, workers < 1 ? 1 : workers);
    m->flat_ready = false;
    m->has_pre = false;
  });
}

int dopf_model_from_arrays(int32_t S, int32_t n, const int32_t* z_offsets, const int32_t* l2g,
                           const int32_t* m_s, const double* A, const double* b, const double* c,
                           const double* x_lo, const double* x_hi, const int32_t* is_w,
                           dopf_model** out) {
  if (S < 0 || n < 0 || !z_offsets || !out || (n > 0 && (!c || !x_lo || !x_hi)))
    return fail(DOPF_ERR_INVALID_ARGUMENT, "bad model arrays");
  return guarded([&] {
    auto* m = new dopf_model();
    auto& md = m->model;
    md.global_cols = n;
    md.c.assign(c, c + n);
    md.x_lo.assign(x_lo, x_lo + n);
    md.x_hi.assign(x_hi, x_hi + n);
    for (int j = 0; j < n; ++j)
      md.var_table.push_back({is_w && is_w[j] ? dopf::VarKind::w : dopf::VarKind::p_load,
                              "v" + std::to_string(j), 1, dopf::FlowDirection::from_to});
    md.copy_counts.assign(n, 0);
    md.z_offsets.assign(z_offsets, z_offsets + S + 1);
    if (md.z_offsets[0] != 0) throw std::invalid_argument("z_offsets[0] must be 0");
    std::size_t a_at = 0, b_at = 0;
    for (int s = 0; s < S; ++s) {
      dopf::Subsystem sub;
      sub.component_id = "s" + std::to_string(s);
      const int ns = z_offsets[s + 1] - z_offsets[s];
      if (ns < 0) throw std::invalid_argument("z_offsets must be nondecreasing");
      const int ms = m_s ? m_s[s] : 0;
      sub.local_to_global.assign(l2g + z_offsets[s], l2g + z_offsets[s + 1]);
      for (int j = 0; j < ns; ++j) {
        const int g = sub.local_to_global[j];
        if (g < 0 || g >= n) throw std::invalid_argument("local_to_global out of range");
        if (j > 0 && g <= sub.local_to_global[j - 1])
          throw std::invalid_argument("local_to_global must be strictly ascending");
        ++md.copy_counts[g];
      }
      sub.A = dopf::Dense(ms, ns);
      for (int k = 0; k < ms * ns; ++k) sub.A.a[k] = A[a_at + k];
      a_at += static_cast<std::size_t>(ms) * ns;
      sub.b.assign(b + b_at, b + b_at + ms);
      b_at += ms;
      sub.rows_before_reduction = ms;
      md.subsystems.push_back(std::move(sub));
    }
    *out = m;
  });
}

int dopf_model_precompute(dopf_model* m, int32_t workers) {
  if (!m) return fail(DOPF_ERR_INVALID_ARGUMENT, "null model");
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    dopf::WorkerPool pool(workers < 1 ? 1 : workers);
    m->pre = dopf::precompute(m->model, &pool);
    m->precompute_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    m->has_pre = true;
    m->flat_ready = false;
  });
}

int dopf_derive_load_coefficients(double p_ref, double q_ref, int32_t kind, double* out) {
  if (!out || kind < 0 || kind > 2) return fail(DOPF_ERR_INVALID_ARGUMENT, "bad load kind");
  return guarded([&] {
    const dopf::LoadCoefficients lc =
        dopf::derive_load_coefficients(p_ref, q_ref, static_cast<dopf::LoadKind>(kind));
    out[0] = lc.a;
    out[1] = lc.b;
    out[2] = lc.alpha;
    out[3] = lc.beta;
  });
}

int dopf_line_m_matrices(int32_t np, const int32_t* phases, const double* r, const double* x,
                         double* mp, double* mq) {
  if (np < 1 || np > 3 || !phases || !r || !x || !mp || !mq)
    return fail(DOPF_ERR_INVALID_ARGUMENT, "bad line");
  return guarded([&] {
    dopf::LineSegment line;
    line.phases = dopf::PhaseSet(std::vector<int>(phases, phases + np));
    line.r.assign(np, std::vector<double>(np));
    line.x.assign(np, std::vector<double>(np));
    for (int i = 0; i < np; ++i)
      for (int j = 0; j < np; ++j) {
        line.r[i][j] = r[i * np + j];
        line.x[i][j] = x[i * np + j];
      }
    std::vector<double> p, q;
    dopf::build_m_matrices(line, p, q);
    std::copy(p.begin(), p.end(), mp);
    std::copy(q.begin(), q.end(), mq);
  });
}

int dopf_model_set_reduced(dopf_model* m, const double* A, const double* b, const int32_t* m_s) {
  if (!m || !m_s || (!A && m->model.subsystem_count() > 0)) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    auto& subs = m->model.subsystems;
    for (std::size_t s = 0; s < subs.size(); ++s)
      if (m_s[s] < 0 || m_s[s] > subs[s].row_count())
        throw std::invalid_argument("reduced row count of subsystem " + std::to_string(s) + " out of range");
    std::size_t a_at = 0, b_at = 0;  // slots of the current (unreduced) rows
    for (std::size_t s = 0; s < subs.size(); ++s) {
      dopf::Subsystem& sub = subs[s];
      const int rows = sub.row_count(), n = sub.col_count(), r = m_s[s];
      dopf::Dense red(r, n);
      for (int k = 0; k < r * n; ++k) red.a[k] = A[a_at + k];
      sub.b.assign(b + b_at, b + b_at + r);
      sub.A = std::move(red);
      a_at += static_cast<std::size_t>(rows) * n;
      b_at += rows;
    }
    m->flat_ready = false;
    m->has_pre = false;
  });
}

int dopf_model_set_operators(dopf_model* m, const double* P, const double* v) {
  if (!m || !P || !v) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    m->pre = dopf::precompute_from(m->model, P, v);
    m->has_pre = true;
    m->flat_ready = false;
  });
}

int dopf_model_view_get(const dopf_model* cm, dopf_model_view* out) {
  if (!cm || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  auto* m = const_cast<dopf_model*>(cm);
  return guarded([&] {
    flatten(m);
    *out = m->flat.view(m->model, m->has_pre ? &m->pre : nullptr);
  });
}

int dopf_model_component_id(const dopf_model* m, int32_t s, char* buf, size_t cap) {
  if (!m || s < 0 || s >= m->model.subsystem_count())
    return fail(DOPF_ERR_INVALID_ARGUMENT, "bad subsystem index");
  return emit_text(m->model.subsystems[s].component_id, buf, cap, nullptr);
}

int dopf_model_rows_before_reduction(const dopf_model* m, int32_t* out) {
  if (!m || !out) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  for (int s = 0; s < m->model.subsystem_count(); ++s)
    out[s] = m->model.subsystems[s].rows_before_reduction;
  return DOPF_OK;
}

int dopf_model_dump_subsystems(const dopf_model* m, char* buf, size_t cap, size_t* needed) {
  if (!m) return fail(DOPF_ERR_INVALID_ARGUMENT, "null model");
  return guarded([&] {
    std::ostringstream os;
    dopf::dump_subsystems(m->model, os);
    emit_text(os.str(), buf, cap, needed);
  });
}

void dopf_model_free(dopf_model* m) { delete m; }

int dopf_write_trace_csv(const double* trace, int32_t rows, char* buf, size_t cap,
                         size_t* needed) {
  if (rows < 0 || (rows > 0 && !trace)) return fail(DOPF_ERR_INVALID_ARGUMENT, "bad trace");
  return guarded([&] {
    std::vector<dopf::TraceRow> t(rows);
    for (int r = 0; r < rows; ++r) {
      const double* q = trace + r * DOPF_TRACE_WIDTH;
      t[r] = {static_cast<int>(q[0]), q[1], q[2], q[3], q[4], q[5]};
    }
    std::ostringstream os;
    dopf::write_trace_csv(t, os);
    emit_text(os.str(), buf, cap, needed);
  });
}

int dopf_write_solution(const dopf_lp* lp, const double* x, char* buf, size_t cap,
                        size_t* needed) {
  if (!lp || !x) return fail(DOPF_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::vector<double> xs(x, x + lp->ls.cols);
    std::ostringstream os;
    dopf::write_solution(lp->ls.var_table, xs, os);
    emit_text(os.str(), buf, cap, needed);
  });
}

}  // extern "C"
