// helmdef_b200_harness.hpp -- the reference's experiment harness over the
// device solve: JSON sweep configs with their FNV-1a hash, the cartesian
// (preconditioner x p x k) sweep of run_cell, RunRecord CSV/JSON I/O with
// direct_gap and config_hash, golden-table reading and compare_cells.
//
// Mirrors (same names, fields, formats and error behaviour):
//   PrecondConfig / ExperimentConfig / RunRecord / ResultCell / GoldenRow /
//   DiffReport                   include/helmdef/harness.hpp:23-172
//   fnv1a_hex, parse_config      src/harness.cpp:30-44, :84-141
//   to_spec (per-p overrides)    src/harness.cpp:175-205
//   run_cell (+ direct_gap)      src/harness.cpp:207-243
//   run_iteration_sweep          src/harness.cpp:257-310
//   record CSV / JSON            src/harness.cpp:312-448
//   read_golden_csv, compare     src/harness.cpp:491-592
// The solve itself is compose() + gmres() of helmdef_b200.hpp (the C-ABI);
// direct_gap uses hd_direct_solve (an exact device solve of A, the
// reference's DirectSolver(sys.A) at src/harness.cpp:234-238).
//
// Needs nlohmann/json (the reference's own JSON library, vendored by it as
// json.hpp): compile with -I <dir containing nlohmann/json.hpp>.
#pragma once

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cstdio>
#include <cstdint>
#include <exception>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>

#include <nlohmann/json.hpp>

#include "helmdef_b200.hpp"

namespace helmdef_b200 {

struct PrecondConfig {
  std::string tag = "D";  // D | D_eps | C_ex | DC_MG | Deps_C_MG | none
  double epsilon = 0.1;
  std::string beta2 = "1";
  int cycles = 1;
  int smoothing = 1;
  double omega = 0.6;
  std::map<int, int> smoothing_by_p;
  std::map<int, double> omega_by_p;
  std::string label() const { return helmdef_b200::label(tag, cycles); }
};

struct ExperimentConfig {
  std::string study = "iterations";
  std::string problem = "point_source_1d";
  std::vector<double> wave_numbers;
  std::vector<int> orders;
  double kh = 0.625;
  std::vector<int> elements;
  std::vector<PrecondConfig> preconditioners;
  GmresOptions gmres;
  std::string compare_mode = "iterations";
  double compare_tolerance = 2.0;
  bool check_direct = false;
  long direct_cap = 10000;
  int samples = 1000;
  std::array<double, 16> multipliers{};
  bool has_multipliers = false;
  std::string raw_dump;  // canonical serialized form (nlohmann dump(2))
  std::string hash;      // FNV-1a of raw_dump
};

// Shortest round-trip decimal form (src/harness.cpp:312-322)
inline std::string format_double(double v) {
  char buf[64];
  if (std::isfinite(v) && v == std::floor(v) && std::abs(v) < 1e15) {
    auto res = std::to_chars(buf, buf + sizeof(buf), static_cast<long long>(v));
    return std::string(buf, res.ptr);
  }
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, res.ptr);
}

namespace detail {
using json = nlohmann::json;

inline std::string fnv1a_hex(const std::string& text) {  // src/harness.cpp:30-44
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : text) {
    h ^= c;
    h *= 1099511628211ull;
  }
  static const char* digits = "0123456789abcdef";
  std::string out(16, '0');
  for (int i = 15; i >= 0; --i) {
    out[i] = digits[h & 0xf];
    h >>= 4;
  }
  return out;
}

inline double number_field(const json& j) { return j.is_string() ? std::stod(j.get<std::string>()) : j.get<double>(); }

inline PrecondConfig parse_precond(const json& j) {  // src/harness.cpp:46-70
  PrecondConfig pc;
  pc.tag = j.value("tag", pc.tag);
  pc.epsilon = j.value("epsilon", pc.epsilon);
  if (j.contains("beta2")) {
    const json& b = j.at("beta2");
    pc.beta2 = b.is_string() ? b.get<std::string>() : format_double(b.get<double>());
  }
  pc.cycles = j.value("cycles", pc.cycles);
  pc.smoothing = j.value("smoothing", pc.smoothing);
  pc.omega = j.value("omega", pc.omega);
  if (j.contains("smoothing_by_p"))
    for (const auto& [key, val] : j.at("smoothing_by_p").items()) pc.smoothing_by_p[std::stoi(key)] = val.get<int>();
  if (j.contains("omega_by_p"))
    for (const auto& [key, val] : j.at("omega_by_p").items()) pc.omega_by_p[std::stoi(key)] = val.get<double>();
  return pc;
}

// nlohmann's stock float form: shortest round-trip digits, plain notation
// for decimal exponents in (-4, 15], else d.ddde+XX (two exponent digits)
inline std::string json_float(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char sci[64];
  auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  std::string t(sci, r.ptr);  // [-]d[.ddd]e(+|-)XX
  std::string sign;
  if (t[0] == '-') {
    sign = "-";
    t = t.substr(1);
  }
  const size_t e = t.find('e');
  std::string digits = t.substr(0, 1) + (e > 2 ? t.substr(2, e - 2) : "");
  const int exp10 = std::stoi(t.substr(e + 1));
  const int len = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // position of the decimal point
  std::string out;
  if (len <= n && n <= 15) {
    out = digits + std::string(n - len, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1) + (len > 1 ? "." + digits.substr(1) : "");
    const int ex = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  return sign + out;
}

inline std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          o += b;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  return o + "\"";
}

// The canonical form the reference hashes: nlohmann::json::dump(2) of the
// parsed config (sorted keys, one array element per line) in the stock
// library's formatting, written out here so the hash does not depend on the
// JSON build at hand (this image's only copy inlines numeric arrays).
inline void canonical_dump(const json& j, int depth, std::string& o) {
  const std::string pad(2 * (depth + 1), ' '), close(2 * depth, ' ');
  switch (j.type()) {
    case json::value_t::object: {
      if (j.empty()) {
        o += "{}";
        return;
      }
      o += "{\n";
      size_t i = 0;
      for (auto it = j.begin(); it != j.end(); ++it, ++i) {
        o += pad + json_string(it.key()) + ": ";
        canonical_dump(it.value(), depth + 1, o);
        o += i + 1 < j.size() ? ",\n" : "\n";
      }
      o += close + "}";
      return;
    }
    case json::value_t::array: {
      if (j.empty()) {
        o += "[]";
        return;
      }
      o += "[\n";
      for (size_t i = 0; i < j.size(); ++i) {
        o += pad;
        canonical_dump(j[i], depth + 1, o);
        o += i + 1 < j.size() ? ",\n" : "\n";
      }
      o += close + "]";
      return;
    }
    case json::value_t::string: o += json_string(j.get<std::string>()); return;
    case json::value_t::boolean: o += j.get<bool>() ? "true" : "false"; return;
    case json::value_t::number_integer: o += std::to_string(j.get<long long>()); return;
    case json::value_t::number_unsigned: o += std::to_string(j.get<unsigned long long>()); return;
    case json::value_t::number_float: o += json_float(j.get<double>()); return;
    default: o += "null"; return;
  }
}

inline std::string canonical_dump(const json& j) {
  std::string o;
  canonical_dump(j, 0, o);
  return o;
}

inline std::vector<std::string> split_csv(const std::string& line) {
  std::vector<std::string> out;
  std::string field;
  std::istringstream is(line);
  while (std::getline(is, field, ',')) out.push_back(field);
  if (!line.empty() && line.back() == ',') out.emplace_back();
  return out;
}

inline double parse_double(const std::string& s) {
  if (s == "nan") return std::numeric_limits<double>::quiet_NaN();
  return std::stod(s);
}

inline const char* record_header() {
  return "problem,tag,k,p,elements,dofs,iterations,converged,residual,direct_gap,"
         "matvecs,shift_solves,vcycles,coarse_solves,seconds,config_hash";
}
}  // namespace detail

inline ExperimentConfig parse_config(const std::string& text) {  // src/harness.cpp:84-133
  using detail::json;
  json j = json::parse(text);
  ExperimentConfig cfg;
  cfg.study = j.value("study", cfg.study);
  cfg.problem = j.value("problem", cfg.problem);
  if (j.contains("k"))
    for (const json& v : j.at("k")) cfg.wave_numbers.push_back(detail::number_field(v));
  if (j.contains("p")) cfg.orders = j.at("p").get<std::vector<int>>();
  cfg.kh = j.value("kh", cfg.kh);
  if (j.contains("elements")) cfg.elements = j.at("elements").get<std::vector<int>>();
  if (j.contains("preconditioners"))
    for (const json& pj : j.at("preconditioners")) cfg.preconditioners.push_back(detail::parse_precond(pj));
  if (j.contains("gmres")) {
    const json& g = j.at("gmres");
    cfg.gmres.tolerance = g.value("tolerance", cfg.gmres.tolerance);
    cfg.gmres.max_iterations = g.value("max_iterations", cfg.gmres.max_iterations);
  }
  if (j.contains("compare")) {
    const json& c = j.at("compare");
    cfg.compare_mode = c.value("mode", cfg.compare_mode);
    cfg.compare_tolerance = c.value("tolerance", cfg.compare_tolerance);
  }
  cfg.check_direct = j.value("check_direct", cfg.check_direct);
  cfg.direct_cap = j.value("direct_cap", cfg.direct_cap);
  cfg.samples = j.value("samples", cfg.samples);
  if (j.contains("multipliers")) {
    auto vals = j.at("multipliers").get<std::vector<double>>();
    if (vals.size() != 16) throw std::invalid_argument("multipliers must hold 16 values");
    std::copy(vals.begin(), vals.end(), cfg.multipliers.begin());
    cfg.has_multipliers = true;
  }
  cfg.raw_dump = detail::canonical_dump(j);
  cfg.hash = detail::fnv1a_hex(cfg.raw_dump);
  return cfg;
}

inline ExperimentConfig load_config(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw std::runtime_error("cannot open config: " + path);
  std::ostringstream buf;
  buf << is.rdbuf();
  return parse_config(buf.str());
}

// src/harness.cpp:154-171 (the wedge is this build's BASELINE config-4 extension)
inline Problem make_problem(const ExperimentConfig& cfg, int elements, int order, double k) {
  if (cfg.problem == "point_source_1d") return point_source_1d(elements, order, k);
  if (cfg.problem == "point_source_2d") return point_source_2d(elements, order, k);
  if (cfg.problem == "layered_medium_2d")
    return cfg.has_multipliers ? layered_medium_2d(elements, order, k, cfg.multipliers)
                               : layered_medium_2d(elements, order, k);
  if (cfg.problem == "wedge_2d") return wedge_2d(elements, order, k);
  throw std::invalid_argument("unknown problem: " + cfg.problem);
}

// src/harness.cpp:175-205, with the per-degree overrides
inline PrecondSpec to_spec(const PrecondConfig& pc, int order, double k) {
  PrecondSpec s = to_spec(pc.tag, order, k, pc.epsilon, pc.beta2, pc.cycles, pc.smoothing, pc.omega);
  auto it = pc.smoothing_by_p.find(order);
  if (it != pc.smoothing_by_p.end()) s.smooth_steps = it->second;
  auto io = pc.omega_by_p.find(order);
  if (io != pc.omega_by_p.end()) s.omega = io->second;
  return s;
}

// relative distance of the GMRES solution to an exact device solve of A
// (src/harness.cpp:234-238: DirectSolver(sys.A).solve(sys.rhs))
inline double direct_gap(const DiscreteSystem& sys, const Vec& x) {
  const hd_system hs = to_hd_system(sys);
  Vec ref(sys.rhs.size(), cplx(0.0, 0.0));
  check(hd_direct_solve(&hs, reinterpret_cast<const double*>(sys.rhs.data()), reinterpret_cast<double*>(ref.data())));
  double d = 0.0, r = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    d += std::norm(x[i] - ref[i]);
    r += std::norm(ref[i]);
  }
  return std::sqrt(d) / std::sqrt(r);
}

inline RunRecord run_cell(const ExperimentConfig& cfg, const PrecondConfig& pc, int order, double k,
                          int elements) {  // src/harness.cpp:207-243
  const auto t0 = std::chrono::steady_clock::now();
  RunRecord rec;
  rec.problem = cfg.problem;
  rec.tag = pc.label();
  rec.k = k;
  rec.order = order;
  rec.elements = elements;
  rec.config_hash = cfg.hash;
  const DiscreteSystem sys = assemble(make_problem(cfg, elements, order, k));
  rec.dofs = sys.size();
  SolverSetup setup = compose(sys, to_spec(pc, order, k));
  GmresResult gr = gmres(setup, cfg.gmres);
  rec.iterations = gr.iterations;
  rec.converged = gr.converged;
  rec.residual = gr.residuals.empty() ? 0.0 : gr.residuals.back();
  rec.matvecs = setup.counts->matvecs;
  rec.shift_solves = setup.counts->shift_solves;
  rec.vcycles = setup.counts->vcycles;
  rec.coarse_solves = setup.counts->coarse_solves;
  if (cfg.check_direct && gr.converged && rec.dofs <= cfg.direct_cap) rec.direct_gap = direct_gap(sys, gr.solution);
  rec.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rec;
}

inline long retained_size(const ExperimentConfig& cfg, int elements, int order) {  // src/harness.cpp:245-254
  long per_dim = elements + order - 2;
  if (cfg.problem == "point_source_2d" || cfg.problem == "layered_medium_2d" || cfg.problem == "wedge_2d")
    return per_dim * per_dim;
  return per_dim;
}

// src/harness.cpp:257-310: cells in config order; a pool of `threads` host
// threads, each cell with its own device context (contexts are independent,
// helmdef_b200.h "Threading"); the first failure is rethrown.
inline std::vector<RunRecord> run_iteration_sweep(const ExperimentConfig& cfg, int threads = 1, long max_n = 0) {
  struct Cell {
    const PrecondConfig* pc;
    int order;
    double k;
    int elements;
  };
  std::vector<Cell> cells;
  for (const PrecondConfig& pc : cfg.preconditioners)
    for (int p : cfg.orders)
      for (double k : cfg.wave_numbers) {
        const int n_el = cfg.elements.empty() ? derived_elements(k, cfg.kh, p) : cfg.elements.front();
        if (max_n > 0 && retained_size(cfg, n_el, p) > max_n) {
          std::cerr << "skip " << pc.label() << " p=" << p << " k=" << k << ": system larger than cap\n";
          continue;
        }
        cells.push_back({&pc, p, k, n_el});
      }
  std::vector<RunRecord> records(cells.size());
  std::atomic<size_t> next{0};
  std::exception_ptr failure;
  std::mutex failure_mutex;
  auto worker = [&]() {
    for (;;) {
      const size_t i = next.fetch_add(1);
      if (i >= cells.size()) return;
      const Cell& c = cells[i];
      try {
        records[i] = run_cell(cfg, *c.pc, c.order, c.k, c.elements);
      } catch (...) {
        std::lock_guard<std::mutex> lock(failure_mutex);
        if (!failure) failure = std::current_exception();
        return;
      }
    }
  };
  const int pool = std::max(1, std::min<int>(threads, static_cast<int>(cells.size())));
  if (pool == 1) {
    worker();
  } else {
    std::vector<std::thread> ts;
    for (int t = 0; t < pool; ++t) ts.emplace_back(worker);
    for (std::thread& t : ts) t.join();
  }
  if (failure) std::rethrow_exception(failure);
  return records;
}

// ---- records (src/harness.cpp:324-448) ---------------------------------------
inline void write_records_csv(const std::vector<RunRecord>& records, std::ostream& os) {
  os << detail::record_header() << "\n";
  for (const RunRecord& r : records)
    os << r.problem << ',' << r.tag << ',' << format_double(r.k) << ',' << r.order << ',' << r.elements << ','
       << r.dofs << ',' << r.iterations << ',' << (r.converged ? 1 : 0) << ',' << format_double(r.residual) << ','
       << (std::isfinite(r.direct_gap) ? format_double(r.direct_gap) : "nan") << ',' << r.matvecs << ','
       << r.shift_solves << ',' << r.vcycles << ',' << r.coarse_solves << ',' << format_double(r.seconds) << ','
       << r.config_hash << "\n";
}

inline std::vector<RunRecord> read_records_csv(std::istream& is) {
  std::string line;
  if (!std::getline(is, line)) throw std::runtime_error("empty record stream");
  if (line != detail::record_header()) throw std::runtime_error("unknown record header");
  std::vector<RunRecord> out;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    const auto f = detail::split_csv(line);
    if (f.size() != 16) throw std::runtime_error("malformed record row");
    RunRecord r;
    r.problem = f[0];
    r.tag = f[1];
    r.k = detail::parse_double(f[2]);
    r.order = std::stoi(f[3]);
    r.elements = std::stoi(f[4]);
    r.dofs = std::stol(f[5]);
    r.iterations = std::stoi(f[6]);
    r.converged = f[7] == "1";
    r.residual = detail::parse_double(f[8]);
    r.direct_gap = detail::parse_double(f[9]);
    r.matvecs = std::stol(f[10]);
    r.shift_solves = std::stol(f[11]);
    r.vcycles = std::stol(f[12]);
    r.coarse_solves = std::stol(f[13]);
    r.seconds = detail::parse_double(f[14]);
    r.config_hash = f[15];
    out.push_back(std::move(r));
  }
  return out;
}

inline std::string records_to_json(const std::vector<RunRecord>& records, const std::string& config_dump) {
  using detail::json;
  json j;
  j["config"] = config_dump.empty() ? json(nullptr) : json::parse(config_dump);
  json arr = json::array();
  for (const RunRecord& r : records) {
    json o;
    o["problem"] = r.problem;
    o["tag"] = r.tag;
    o["k"] = r.k;
    o["p"] = r.order;
    o["elements"] = r.elements;
    o["dofs"] = r.dofs;
    o["iterations"] = r.iterations;
    o["converged"] = r.converged;
    o["residual"] = r.residual;
    if (std::isfinite(r.direct_gap)) o["direct_gap"] = r.direct_gap;
    o["matvecs"] = r.matvecs;
    o["shift_solves"] = r.shift_solves;
    o["vcycles"] = r.vcycles;
    o["coarse_solves"] = r.coarse_solves;
    o["seconds"] = r.seconds;
    o["config_hash"] = r.config_hash;
    arr.push_back(std::move(o));
  }
  j["records"] = std::move(arr);
  return detail::canonical_dump(j) + "\n";
}

inline std::vector<RunRecord> records_from_json(const std::string& text) {
  using detail::json;
  const json j = json::parse(text);
  std::vector<RunRecord> out;
  for (const json& o : j.at("records")) {
    RunRecord r;
    r.problem = o.at("problem").get<std::string>();
    r.tag = o.at("tag").get<std::string>();
    r.k = o.at("k").get<double>();
    r.order = o.at("p").get<int>();
    r.elements = o.at("elements").get<int>();
    r.dofs = o.at("dofs").get<long>();
    r.iterations = o.at("iterations").get<int>();
    r.converged = o.at("converged").get<bool>();
    r.residual = o.at("residual").get<double>();
    if (o.contains("direct_gap")) r.direct_gap = o.at("direct_gap").get<double>();
    r.matvecs = o.at("matvecs").get<long>();
    r.shift_solves = o.at("shift_solves").get<long>();
    r.vcycles = o.at("vcycles").get<long>();
    r.coarse_solves = o.at("coarse_solves").get<long>();
    r.seconds = o.at("seconds").get<double>();
    r.config_hash = o.at("config_hash").get<std::string>();
    out.push_back(std::move(r));
  }
  return out;
}

// ---- comparison against reference tables (src/harness.cpp:450-592) ---------
struct ResultCell {
  std::string tag;
  double k = 0.0;
  int p = 0;
  int elements = 0;
  double value = 0.0;
  bool star = false;  // iteration limit reached
};

inline std::vector<ResultCell> cells_from_records(const std::vector<RunRecord>& records) {
  std::vector<ResultCell> cells;
  for (const RunRecord& r : records)
    cells.push_back({r.tag, r.k, r.order, r.elements, static_cast<double>(r.iterations), !r.converged});
  return cells;
}

struct GoldenRow {
  std::string tag, k, p, elements, value;
  double tol = std::numeric_limits<double>::quiet_NaN();
};

inline std::vector<GoldenRow> read_golden_csv(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw std::runtime_error("cannot open reference table: " + path);
  std::string line;
  do {
    if (!std::getline(is, line)) throw std::runtime_error("empty reference table");
  } while (line.empty() || line[0] == '#');
  if (detail::split_csv(line) != std::vector<std::string>{"tag", "k", "p", "elements", "value", "tol"})
    throw std::runtime_error("unknown reference header in " + path);
  std::vector<GoldenRow> rows;
  while (std::getline(is, line)) {
    if (line.empty() || line[0] == '#') continue;
    const auto f = detail::split_csv(line);
    if (f.size() != 6) throw std::runtime_error("malformed reference row");
    GoldenRow g;
    g.tag = f[0];
    g.k = f[1];
    g.p = f[2];
    g.elements = f[3];
    g.value = f[4];
    if (!f[5].empty()) g.tol = detail::parse_double(f[5]);
    rows.push_back(std::move(g));
  }
  return rows;
}

struct DiffLine {
  std::string key, expected, actual;
  bool ok = false;
  bool missing = false;
};

struct DiffReport {
  std::vector<DiffLine> lines;
  int matched = 0, mismatched = 0, missing = 0;
  bool pass() const { return matched > 0 && mismatched == 0; }
};

inline DiffReport compare_cells(const std::vector<ResultCell>& cells, const std::vector<GoldenRow>& golden,
                                const std::string& mode, double tolerance) {
  if (mode != "iterations" && mode != "factor") throw std::invalid_argument("unknown compare mode: " + mode);
  auto matches = [](const GoldenRow& g, const ResultCell& c) {
    if (!g.tag.empty() && g.tag != c.tag) return false;
    if (!g.k.empty()) {
      const double gk = std::stod(g.k);
      if (std::abs(gk - c.k) > 1e-9 * std::max(1.0, std::abs(gk))) return false;
    }
    if (!g.p.empty() && std::stoi(g.p) != c.p) return false;
    if (!g.elements.empty() && std::stoi(g.elements) != c.elements) return false;
    return true;
  };
  DiffReport report;
  for (const GoldenRow& g : golden) {
    const ResultCell* hit = nullptr;
    for (const ResultCell& c : cells)
      if (matches(g, c)) {
        hit = &c;
        break;
      }
    DiffLine line;
    for (const auto& [name, v] : {std::pair<const char*, const std::string*>{"tag", &g.tag}, {"k", &g.k},
                                  {"p", &g.p}, {"elements", &g.elements}})
      if (!v->empty()) line.key += std::string(line.key.empty() ? "" : " ") + name + "=" + *v;
    line.expected = g.value;
    if (!hit) {
      line.actual = "(missing)";
      line.missing = true;
      report.missing += 1;
      report.lines.push_back(std::move(line));
      continue;
    }
    const double tol = std::isfinite(g.tol) ? g.tol : tolerance;
    line.actual = hit->star ? "*" : format_double(hit->value);
    if (mode == "iterations") {
      if (g.value == "*") line.ok = hit->star;
      else if (hit->star) line.ok = false;
      else line.ok = std::abs(hit->value - std::stod(g.value)) <= tol;
    } else {
      const double gv = std::stod(g.value);
      line.ok = !hit->star && gv > 0.0 && hit->value > 0.0 && std::max(hit->value / gv, gv / hit->value) <= tol;
    }
    (line.ok ? report.matched : report.mismatched) += 1;
    report.lines.push_back(std::move(line));
  }
  return report;
}

}  // namespace helmdef_b200
