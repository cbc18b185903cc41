// hd_bench -- the reference's helmbench CLI (tools/helmbench.cpp) for the
// iteration studies, over the device solve: `solve` (one cell),
// `table` (a JSON sweep config -> RunRecord CSV/JSON) and `compare` (a sweep
// or a saved records file against a golden table, exit 2 on mismatch).
// Same flags, outputs and exit codes as the reference (tools/helmbench.cpp:
// 209-231 solve, :68-74 table, :159-190 compare, :301-319 exit codes); the
// spectrum / convergence studies are not part of the accelerated path.
//
//   hd_bench solve   [--problem P] [--k K] [--p P] [--elements N] [--kh H] [--tag T]
//                    [--epsilon E] [--beta2 B] [--cycles C] [--smoothing S] [--omega W]
//                    [--tol T] [--maxit M] [--check-direct] [--out F] [--format csv|json]
//   hd_bench table   --config C.json [--out F] [--format csv|json] [--threads N] [--max-n N]
//   hd_bench compare --config C.json --reference G.csv [--records R.csv|R.json] [--threads N] [--max-n N]
//   hd_bench records --in R.csv|R.json [--format csv|json] [--out F]   (re-emit: format round trip)
//   hd_bench hash    --config C.json                                  (FNV-1a config hash)
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "helmdef_b200_harness.hpp"

namespace hb = helmdef_b200;

namespace {

std::string read_text(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw std::runtime_error("cannot read " + path);
  std::ostringstream buf;
  buf << is.rdbuf();
  return buf.str();
}

void emit(const std::string& out, const std::string& text) {
  if (out.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream os(out);
  if (!os) throw std::runtime_error("cannot write " + out);
  os << text;
  std::cout << "wrote " << out << "\n";
}

std::string records_text(const std::vector<hb::RunRecord>& records, const hb::ExperimentConfig& cfg,
                         const std::string& format) {
  if (format == "json") return hb::records_to_json(records, cfg.raw_dump);
  std::ostringstream os;
  hb::write_records_csv(records, os);
  return os.str();
}

std::vector<hb::RunRecord> load_records(const std::string& path) {
  if (path.size() > 5 && path.substr(path.size() - 5) == ".json") return hb::records_from_json(read_text(path));
  std::ifstream is(path);
  if (!is) throw std::runtime_error("cannot read " + path);
  return hb::read_records_csv(is);
}

struct Args {
  std::map<std::string, std::string> opt;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
};

// --name value pairs and bare flags (--check-direct)
Args parse_args(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument: " + k);
    k = k.substr(2);
    if (k == "check-direct") {
      a.opt[k] = "1";
      continue;
    }
    if (i + 1 >= argc) throw std::invalid_argument("--" + k + " needs a value");
    a.opt[k] = argv[++i];
  }
  return a;
}

int run_solve(const Args& a) {  // tools/helmbench.cpp:209-231
  nlohmann::json j;
  j["study"] = "iterations";
  j["problem"] = a.get("problem", "point_source_1d");
  j["k"] = {std::stod(a.get("k", "100"))};
  j["p"] = {std::stoi(a.get("p", "2"))};
  j["kh"] = std::stod(a.get("kh", "0.625"));
  const int elements = std::stoi(a.get("elements", "0"));
  if (elements > 0) j["elements"] = {elements};
  j["preconditioners"] = {{{"tag", a.get("tag", "D_eps")},
                           {"epsilon", std::stod(a.get("epsilon", "0.1"))},
                           {"beta2", a.get("beta2", "1")},
                           {"cycles", std::stoi(a.get("cycles", "1"))},
                           {"smoothing", std::stoi(a.get("smoothing", "1"))},
                           {"omega", std::stod(a.get("omega", "0.6"))}}};
  j["gmres"] = {{"tolerance", std::stod(a.get("tol", "1e-7"))}, {"max_iterations", std::stoi(a.get("maxit", "100"))}};
  j["check_direct"] = a.has("check-direct");
  const hb::ExperimentConfig cfg = hb::parse_config(j.dump());
  const auto records = hb::run_iteration_sweep(cfg, 1, 0);
  emit(a.get("out"), records_text(records, cfg, a.get("format", "csv")));
  return 0;  // hitting the budget is reported in the record, not the exit code
}

int run_table(const Args& a) {  // tools/helmbench.cpp:68-74
  const hb::ExperimentConfig cfg = hb::load_config(a.get("config"));
  const auto records = hb::run_iteration_sweep(cfg, std::stoi(a.get("threads", "1")), std::stol(a.get("max-n", "0")));
  emit(a.get("out"), records_text(records, cfg, a.get("format", "csv")));
  return 0;
}

int run_compare(const Args& a) {  // tools/helmbench.cpp:159-190
  const hb::ExperimentConfig cfg = hb::load_config(a.get("config"));
  std::vector<hb::ResultCell> cells;
  if (a.has("records")) {
    cells = hb::cells_from_records(load_records(a.get("records")));
  } else if (cfg.study == "iterations") {
    cells = hb::cells_from_records(
        hb::run_iteration_sweep(cfg, std::stoi(a.get("threads", "1")), std::stol(a.get("max-n", "0"))));
  } else {
    throw std::invalid_argument("only iteration studies run on the device path: " + cfg.study);
  }
  const auto golden = hb::read_golden_csv(a.get("reference"));
  const auto report = hb::compare_cells(cells, golden, cfg.compare_mode, cfg.compare_tolerance);
  for (const auto& line : report.lines) {
    const char* marker = line.ok ? "" : line.missing ? "  (no counterpart)" : "  <-- MISMATCH";
    std::cout << line.key << ": expected " << line.expected << ", got " << line.actual << marker << "\n";
  }
  std::cout << "matched " << report.matched << ", mismatched " << report.mismatched << ", missing " << report.missing
            << "\n";
  if (report.missing > 0) std::cerr << "warning: " << report.missing << " reference cells had no produced counterpart\n";
  if (report.matched == 0) throw std::runtime_error("no produced cell matched the reference table");
  return report.mismatched == 0 ? 0 : 2;
}

// extensions for the host-only tests: re-emit a records file (CSV <-> JSON
// round trip, src/harness.cpp:324-448) and print a config's FNV-1a hash
int run_records(const Args& a) {
  const auto records = load_records(a.get("in"));
  hb::ExperimentConfig none;
  emit(a.get("out"), records_text(records, none, a.get("format", "csv")));
  return 0;
}

int run_hash(const Args& a) {
  const hb::ExperimentConfig cfg = hb::load_config(a.get("config"));
  std::cout << cfg.hash << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: hd_bench solve|table|compare|records|hash [--options]\n");
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse_args(argc, argv, 2);
    if (cmd == "solve") return run_solve(a);
    if (cmd == "records") return run_records(a);
    if (cmd == "hash") return run_hash(a);
    if ((cmd == "table" || cmd == "compare") && !a.has("config")) throw std::invalid_argument("--config is required");
    if (cmd == "table") return run_table(a);
    if (cmd == "compare") {
      if (!a.has("reference")) throw std::invalid_argument("--reference is required");
      return run_compare(a);
    }
    throw std::invalid_argument("unknown subcommand: " + cmd);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
