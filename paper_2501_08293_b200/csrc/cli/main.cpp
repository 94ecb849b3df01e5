// `dopf` command-line front end on the B200 solver: the drop-in for the
// reference CLI (proj/tools/main.cpp:84-306). Same subcommands, flags, output
// files and exit codes; `solve` runs the iteration on the GPU through
// dopf::solve (include/dopf/cuda_solve.hpp).
//
//   dopf solve    --input f.json [--rho R] [--eps-rel E] [--max-iter N] [--workers W]
//                 [--trace t.csv] [--solution s.txt] [--report r.json] [--seed S]
//                 [--device D] [--gpus N]
//   dopf validate --input f.json [--report r.json] [--workers W]
//   dopf inspect  --input f.json [--report r.json] [--dump-lp f] [--dump-subsystems f] [--workers W]
//
// Exit codes (main.cpp:19-24): 0 ok, 1 internal, 2 parse, 3 validation,
// 4 infeasible/singular subsystem, 5 iteration limit.
// The JSON report mirrors the reference's nlohmann::json output: keys sorted,
// two-space indent, doubles in shortest round-trip form.
// `validate --oracle` (the dense simplex, oracle.cpp:164-273) is test
// infrastructure in this build (oracle/), not part of the product CLI.
#include <cerrno>
#include <charconv>
#include <cstdlib>
#include <stdexcept>
#include <type_traits>
#include <cmath>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <variant>
#include <vector>

#include "../../../include/dopf/cuda_solve.hpp"
#include "../host/decompose.hpp"
#include "../host/feeder.hpp"
#include "../host/lp_builder.hpp"

namespace {

constexpr int kExitOk = 0, kExitInternal = 1, kExitParse = 2, kExitValidation = 3,
              kExitInfeasibleSubsystem = 4, kExitIterationLimit = 5;

// ---------------------------------------------------------------- JSON value
struct Json {
  using Object = std::map<std::string, Json>;  // sorted keys, as nlohmann::json
  std::variant<std::nullptr_t, bool, long long, double, std::string, Object> v;
  Json() : v(nullptr) {}
  Json(bool b) : v(b) {}
  Json(int i) : v(static_cast<long long>(i)) {}
  Json(long long i) : v(i) {}
  Json(unsigned u) : v(static_cast<long long>(u)) {}
  Json(double d) : v(d) {}
  Json(const char* s) : v(std::string(s)) {}
  Json(std::string s) : v(std::move(s)) {}
  Json(Object o) : v(std::move(o)) {}
  Json& operator[](const std::string& k) {
    if (!std::holds_alternative<Object>(v)) v = Object{};
    return std::get<Object>(v)[k];
  }
};

void put_string(std::ostream& out, const std::string& s) {
  out << '"';
  for (char ch : s) {
    switch (ch) {
      case '"': out << "\\\""; break;
      case '\\': out << "\\\\"; break;
      case '\n': out << "\\n"; break;
      case '\t': out << "\\t"; break;
      default: out << ch;
    }
  }
  out << '"';
}

void put_double(std::ostream& out, double d) {
  if (!std::isfinite(d)) {  // nlohmann::json serializes non-finite numbers as null
    out << "null";
    return;
  }
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof buf, d);  // shortest round trip
  std::string s(buf, res.ptr);
  // nlohmann prints integral doubles with a trailing ".0"
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  out << s;
}

void dump(std::ostream& out, const Json& j, int indent) {
  if (std::holds_alternative<std::nullptr_t>(j.v)) out << "null";
  else if (auto b = std::get_if<bool>(&j.v)) out << (*b ? "true" : "false");
  else if (auto i = std::get_if<long long>(&j.v)) out << *i;
  else if (auto d = std::get_if<double>(&j.v)) put_double(out, *d);
  else if (auto s = std::get_if<std::string>(&j.v)) put_string(out, *s);
  else {
    const auto& o = std::get<Json::Object>(j.v);
    if (o.empty()) {
      out << "{}";
      return;
    }
    out << "{\n";
    std::size_t k = 0;
    for (const auto& [key, val] : o) {
      out << std::string(indent + 2, ' ');
      put_string(out, key);
      out << ": ";
      dump(out, val, indent + 2);
      out << (++k < o.size() ? ",\n" : "\n");
    }
    out << std::string(indent, ' ') << "}";
  }
}

// ---------------------------------------------------------------- options
struct Options {
  std::string cmd, input, trace_path, report_path, solution_path, dump_lp, dump_subs;
  double rho = 100.0, eps_rel = 1e-3;
  int max_iter = 50000;
  int workers = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  unsigned seed = 0;
  int device = 0;  // CUDA device of the solve (this build's addition)
  int gpus = 1;    // GPUs of a partitioned solve (this build's addition)
  bool gpus_set = false;
  bool oracle = false;
};

// Command-line errors exit like the reference's CLI11 front end
// (CLI11_PARSE -> app.exit(e), tools/main.cpp:297): a message on stderr and
// CLI11's ExitCodes -- 104 a value that does not convert, 106 a missing
// required option or subcommand, 109 an unknown argument.
constexpr int kCliConversion = 104, kCliRequired = 106, kCliExtras = 109;

struct UsageError : std::runtime_error {
  int code;
  UsageError(int c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

template <typename T>
T convert(const std::string& flag, const std::string& text) {
  T value{};
  const char* end = text.data() + text.size();
  std::from_chars_result r;
  if constexpr (std::is_floating_point_v<T>) {
    // strtod accepts what CLI11's lexical_cast accepts (1e-3, inf, ...)
    char* stop = nullptr;
    errno = 0;
    const double d = std::strtod(text.c_str(), &stop);
    if (text.empty() || stop != text.c_str() + text.size() || errno == ERANGE)
      throw UsageError(kCliConversion, "Could not convert: " + flag + " = " + text);
    return static_cast<T>(d);
  } else {
    r = std::from_chars(text.data(), end, value);
    if (r.ec != std::errc() || r.ptr != end)
      throw UsageError(kCliConversion, "Could not convert: " + flag + " = " + text);
  }
  return value;
}

Options parse_args(int argc, char** argv) {
  Options o;
  if (argc < 2) throw UsageError(kCliRequired, "A subcommand is required");
  o.cmd = argv[1];
  if (o.cmd != "solve" && o.cmd != "validate" && o.cmd != "inspect")
    throw UsageError(kCliExtras, "The following argument was not expected: " + o.cmd);
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    std::string inline_value;
    bool has_inline = false;
    if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
      inline_value = a.substr(eq + 1);  // --opt=value, as CLI11 accepts
      a = a.substr(0, eq);
      has_inline = true;
    }
    auto value = [&]() -> std::string {
      if (has_inline) return inline_value;
      if (i + 1 >= argc) throw UsageError(kCliRequired, a + " requires 1 argument");
      return argv[++i];
    };
    if (a == "--input") o.input = value();
    else if (a == "--report") o.report_path = value();
    else if (a == "--workers") o.workers = convert<int>(a, value());
    else if (o.cmd == "solve" && a == "--rho") o.rho = convert<double>(a, value());
    else if (o.cmd == "solve" && a == "--eps-rel") o.eps_rel = convert<double>(a, value());
    else if (o.cmd == "solve" && a == "--max-iter") o.max_iter = convert<int>(a, value());
    else if (o.cmd == "solve" && a == "--trace") o.trace_path = value();
    else if (o.cmd == "solve" && a == "--solution") o.solution_path = value();
    else if (o.cmd == "solve" && a == "--seed") o.seed = convert<unsigned>(a, value());
    else if (o.cmd == "solve" && a == "--device") o.device = convert<int>(a, value());
    else if (o.cmd == "solve" && a == "--gpus") {
      o.gpus = convert<int>(a, value());
      o.gpus_set = true;
    }
    else if (o.cmd == "validate" && a == "--oracle") o.oracle = true;
    else if (o.cmd == "inspect" && a == "--dump-lp") o.dump_lp = value();
    else if (o.cmd == "inspect" && a == "--dump-subsystems") o.dump_subs = value();
    else throw UsageError(kCliExtras, "The following argument was not expected: " + a);
  }
  if (o.input.empty()) throw UsageError(kCliRequired, "--input is required");
  return o;
}

void write_report(const Json& report, const std::string& path) {
  std::ostringstream os;
  dump(os, report, 0);
  os << "\n";
  if (path.empty()) {
    std::cout << os.str();
    return;
  }
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write report to '" + path + "'");
  out << os.str();
}

void print_diagnostics(const std::vector<dopf::Diagnostic>& diags) {
  for (const auto& d : diags) {
    std::cerr << (d.severity == dopf::Severity::error ? "error" : "warning");
    if (!d.component.empty()) std::cerr << " [" << d.component << "]";
    std::cerr << ": " << d.message << "\n";
  }
}

int load_feeder(const Options& o, dopf::Feeder& out) {
  try {
    out = dopf::parse_feeder_file(o.input);
  } catch (const dopf::ParseError& e) {
    std::cerr << "parse error: " << e.what() << "\n";
    return kExitParse;
  }
  const auto diags = dopf::validate_feeder(out);
  print_diagnostics(diags);
  return dopf::has_errors(diags) ? kExitValidation : kExitOk;
}

int cmd_solve(const Options& o) {
  dopf::Feeder feeder;
  if (int code = load_feeder(o, feeder); code != kExitOk) return code;
  const dopf::LinearSystem ls = dopf::assemble_centralized(feeder);
  dopf::DecomposedModel model;
  try {
    model = dopf::decompose(ls, feeder, 1e-9, o.workers);
  } catch (const dopf::InfeasibleSubsystemError& e) {
    std::cerr << e.what() << "\n";
    return kExitInfeasibleSubsystem;
  }
  dopf::Settings settings;
  settings.rho = o.rho;
  settings.eps_rel = o.eps_rel;
  settings.max_iter = o.max_iter;
  settings.workers = o.workers;
  dopf::SolveResult result;
  try {
    // GPU iteration (cuda_solve.hpp): one device, or the model partitioned
    // over devices 0..gpus-1 with the NCCL exchange
    result = o.gpus > 1 || o.gpus_set ? dopf::cuda::solve_partitioned(model, settings, o.gpus)
                                      : dopf::cuda::solve(model, settings, o.device);
  } catch (const dopf::SingularSubsystemError& e) {
    std::cerr << e.what() << "\n";
    return kExitInfeasibleSubsystem;
  }
  if (!o.trace_path.empty()) {
    std::ofstream trace(o.trace_path);
    if (!trace) {
      std::cerr << "cannot write trace to '" << o.trace_path << "'\n";
      return kExitInternal;
    }
    dopf::write_trace_csv(result.trace, trace);
  }
  if (!o.solution_path.empty()) {
    std::ofstream sol(o.solution_path);
    if (!sol) {
      std::cerr << "cannot write solution to '" << o.solution_path << "'\n";
      return kExitInternal;
    }
    dopf::write_solution(ls.var_table, result.x, sol);
  }
  Json report;
  report["status"] = result.status == dopf::SolveStatus::converged ? "converged" : "iteration_limit";
  report["iterations"] = result.iterations;
  report["objective"] = result.objective;
  if (!result.trace.empty()) {
    const auto& last = result.trace.back();
    report["residuals"]["pres"] = last.pres;
    report["residuals"]["dres"] = last.dres;
    report["residuals"]["eps_prim"] = last.eps_prim;
    report["residuals"]["eps_dual"] = last.eps_dual;
  }
  report["timings_sec"]["precompute"] = result.timings.precompute;
  report["timings_sec"]["global"] = result.timings.global;
  report["timings_sec"]["local"] = result.timings.local;
  report["timings_sec"]["dual"] = result.timings.dual;
  report["model"]["rows"] = ls.rows;
  report["model"]["cols"] = ls.cols;
  report["model"]["subsystems"] = model.subsystem_count();
  report["settings"]["rho"] = o.rho;
  report["settings"]["eps_rel"] = o.eps_rel;
  report["settings"]["max_iter"] = o.max_iter;
  report["settings"]["workers"] = o.workers;
  report["settings"]["seed"] = o.seed;
  report["max_local_infeasibility"] = result.max_local_infeasibility;
  Json solution{Json::Object{}};
  for (int i = 0; i < ls.cols; ++i) solution[dopf::to_string(ls.var_table[i])] = result.x[i];
  report["solution"] = solution;
  write_report(report, o.report_path);
  return result.status == dopf::SolveStatus::converged ? kExitOk : kExitIterationLimit;
}

int cmd_validate(const Options& o) {
  dopf::Feeder feeder;
  if (int code = load_feeder(o, feeder); code != kExitOk) return code;
  if (o.oracle) {
    std::cerr << "--oracle: the exact LP reference is test infrastructure in this build "
                 "(oracle/, tests/test_oracle_pinning.py)\n";
    return kExitInternal;
  }
  Json report;
  report["valid"] = true;
  write_report(report, o.report_path);
  return kExitOk;
}

Json dimension_stats(const std::vector<int>& values) {
  Json stats{Json::Object{}};
  if (values.empty()) return stats;
  int lo = values.front(), hi = values.front();
  long long sum = 0;
  for (int v : values) {
    lo = std::min(lo, v);
    hi = std::max(hi, v);
    sum += v;
  }
  const double mean = static_cast<double>(sum) / values.size();
  double var = 0;
  for (int v : values) var += (v - mean) * (v - mean);
  stats["min"] = lo;
  stats["max"] = hi;
  stats["mean"] = mean;
  stats["stdev"] = std::sqrt(var / values.size());
  stats["sum"] = sum;
  return stats;
}

int cmd_inspect(const Options& o) {
  dopf::Feeder feeder;
  if (int code = load_feeder(o, feeder); code != kExitOk) return code;
  const dopf::LinearSystem ls = dopf::assemble_centralized(feeder);
  const auto comps = dopf::build_component_graph(feeder);
  dopf::DecomposedModel model = dopf::partition(ls, comps);
  int pre_rows = 0;
  for (const auto& sub : model.subsystems) pre_rows += sub.rows_before_reduction;
  try {
    dopf::reduce_subsystems(model, 1e-9, o.workers);
  } catch (const dopf::InfeasibleSubsystemError& e) {
    std::cerr << e.what() << "\n";
    return kExitInfeasibleSubsystem;
  }
  int leaves = 0;
  for (const auto& c : comps)
    if (c.kind == dopf::ComponentKind::merged_leaf) ++leaves;
  std::vector<int> m_s, n_s;
  for (const auto& sub : model.subsystems) {
    m_s.push_back(sub.row_count());
    n_s.push_back(sub.col_count());
  }
  Json report;
  report["centralized"]["rows"] = ls.rows;
  report["centralized"]["cols"] = ls.cols;
  report["graph"]["nodes"] = static_cast<int>(feeder.buses.size());
  report["graph"]["lines"] = static_cast<int>(feeder.lines.size());
  report["graph"]["leaves"] = leaves;
  report["graph"]["components"] = static_cast<int>(comps.size());
  report["subsystems"]["count"] = model.subsystem_count();
  report["subsystems"]["rows_pre_reduction"] = pre_rows;
  report["subsystems"]["m_s"] = dimension_stats(m_s);
  report["subsystems"]["n_s"] = dimension_stats(n_s);
  write_report(report, o.report_path);
  if (!o.dump_lp.empty()) {
    std::ofstream out(o.dump_lp);
    if (!out) {
      std::cerr << "cannot write LP dump to '" << o.dump_lp << "'\n";
      return kExitInternal;
    }
    dopf::dump_linear_system(ls, out);
  }
  if (!o.dump_subs.empty()) {
    std::ofstream out(o.dump_subs);
    if (!out) {
      std::cerr << "cannot write subsystem dump to '" << o.dump_subs << "'\n";
      return kExitInternal;
    }
    dopf::dump_subsystems(model, out);
  }
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  Options o;
  try {
    o = parse_args(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return e.code;
  }
  try {
    if (o.cmd == "solve") return cmd_solve(o);
    if (o.cmd == "validate") return cmd_validate(o);
    return cmd_inspect(o);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitInternal;
  }
}
