// `cc {run|sweep|verify|gen}` — the reference CLI (proj/tools/cc_main.cpp)
// rebuilt on the B200 library, with a hand-written flag parser (CLI11 is not
// available here).  Same subcommands, flags, report formats and exit codes:
// 0 ok, 1 verification failure, 2 usage error, 3 I/O or parse error
// (cc_main.cpp:19-22, 241-262).  B200 additions: --first-pass-segments.
#include <cstdint>
#include <fstream>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "hookcc/bench.hpp"

namespace {

enum Exit { kOk = 0, kVerify = 1, kUsage = 2, kIo = 3 };

struct Flags {
  std::string input, format = "edgelist", gen, algo = "adaptive", segments = "auto",
                     workers = "max", labels_out, metrics_out, report = "json",
                     sweep_segments, devices;
  bool header = false, no_verify = false;
  std::uint64_t seed = 1, reps = 1, first_pass_segments = 0;
  std::vector<std::string> positional;
};

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

const char* kHelp =
    "hook-compress connected components on B200\n"
    "usage: cc run    [--input F --format edgelist|dimacs|mtx --header | --gen SPEC] [--seed S]\n"
    "                 [--algo baseline|baseline-mj|atomic|adaptive] [--segments auto|N]\n"
    "                 [--workers max|N] [--reps N] [--labels-out F] [--metrics-out F]\n"
    "                 [--report json|csv] [--no-verify] [--first-pass-segments N]\n"
    "                 [--gpus N | --devices d0,d1,..]  (edge-partitioned multi-GPU run)\n"
    "       cc sweep  [input flags] [--sweep-segments a,b,..] [--workers] [--reps]\n"
    "                 [--metrics-out F] [--report json|csv]\n"
    "       cc verify [input flags] LABELS\n"
    "       cc gen    SPEC [OUTPUT] [--seed S]\n"
    "generator specs: grid:RxC | er:n=..,m=..[,seed=..] | rmat:scale=..,ef=..[,seed=..]\n"
    "                 | rmatx:scale=..,ef=..[,seed=..] | erx:n=..,m=..[,seed=..]\n";

std::uint64_t to_u64(const std::string& flag, const std::string& v) {
  if (v.empty() || v.find_first_not_of("0123456789") != std::string::npos)
    throw Usage(flag + ": expected a non-negative integer, got `" + v + "`");
  return std::stoull(v);
}

void member(const std::string& flag, const std::string& v, std::set<std::string> ok) {
  if (!ok.count(v)) throw Usage(flag + ": `" + v + "` not in the allowed set");
}

// Per-subcommand flag tables: value flags, boolean flags, positional arity.
Flags parse(const std::string& cmd, int argc, char** argv, int first) {
  static const std::map<std::string, std::set<std::string>> value_flags = {
      {"run", {"--input", "--format", "--gen", "--seed", "--algo", "--segments", "--workers",
               "--reps", "--labels-out", "--metrics-out", "--report", "--first-pass-segments",
               "--gpus", "--devices"}},
      {"sweep", {"--input", "--format", "--gen", "--seed", "--sweep-segments", "--workers",
                 "--reps", "--metrics-out", "--report", "--gpus", "--devices"}},
      {"verify", {"--input", "--format", "--gen", "--seed"}},
      {"gen", {"--seed"}}};
  static const std::map<std::string, std::set<std::string>> bool_flags = {
      {"run", {"--header", "--no-verify"}}, {"sweep", {"--header"}},
      {"verify", {"--header"}}, {"gen", {}}};
  Flags f;
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i], val;
    if (a.rfind("--", 0) != 0) {
      f.positional.push_back(a);
      continue;
    }
    const auto eq = a.find('=');
    bool inline_val = eq != std::string::npos;
    if (inline_val) {
      val = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    if (bool_flags.at(cmd).count(a)) {
      if (a == "--header") f.header = true;
      if (a == "--no-verify") f.no_verify = true;
      continue;
    }
    if (!value_flags.at(cmd).count(a)) throw Usage("unknown option " + a);
    if (!inline_val) {
      if (i + 1 >= argc) throw Usage(a + " needs a value");
      val = argv[++i];
    }
    if (a == "--input") f.input = val;
    else if (a == "--format") member(a, f.format = val, {"edgelist", "dimacs", "mtx"});
    else if (a == "--gen") f.gen = val;
    else if (a == "--seed") f.seed = to_u64(a, val);
    else if (a == "--algo") member(a, f.algo = val, {"baseline", "baseline-mj", "atomic", "adaptive"});
    else if (a == "--segments") f.segments = val;
    else if (a == "--workers") f.workers = val;
    else if (a == "--reps") f.reps = to_u64(a, val);
    else if (a == "--labels-out") f.labels_out = val;
    else if (a == "--metrics-out") f.metrics_out = val;
    else if (a == "--report") member(a, f.report = val, {"json", "csv"});
    else if (a == "--sweep-segments") f.sweep_segments = val;
    else if (a == "--first-pass-segments") f.first_pass_segments = to_u64(a, val);
    else if (a == "--gpus") {
      const std::uint64_t k = to_u64(a, val);
      if (k == 0 || k > 64) throw Usage("--gpus must be in [1, 64]");
      f.devices.clear();
      for (std::uint64_t d = 0; d < k; ++d) f.devices += (d ? "," : "") + std::to_string(d);
    } else if (a == "--devices") {
      f.devices = val;
    }
  }
  const std::size_t max_pos = cmd == "verify" ? 1 : cmd == "gen" ? 2 : 0;
  const std::size_t min_pos = cmd == "verify" || cmd == "gen" ? 1 : 0;
  if (f.positional.size() > max_pos) throw Usage("unexpected argument " + f.positional.back());
  if (f.positional.size() < min_pos)
    throw Usage(cmd == "verify" ? "labels file is required" : "generator spec is required");
  return f;
}

hookcc::RunConfig to_config(const Flags& f) {
  hookcc::RunConfig cfg;
  cfg.input_path = f.input;
  cfg.gen_spec = f.gen;
  cfg.edge_list_header = f.header;
  cfg.format = f.format == "dimacs" ? hookcc::InputFormat::Dimacs
               : f.format == "mtx"  ? hookcc::InputFormat::MatrixMarket
                                    : hookcc::InputFormat::EdgeList;
  static const std::map<std::string, hookcc::Algorithm> algos = {
      {"baseline", hookcc::Algorithm::Baseline}, {"baseline-mj", hookcc::Algorithm::BaselineMj},
      {"atomic", hookcc::Algorithm::Atomic}, {"adaptive", hookcc::Algorithm::Adaptive}};
  auto it = algos.find(f.algo);
  if (it == algos.end()) throw hookcc::UsageError("unknown --algo `" + f.algo + "`");
  cfg.algo = it->second;
  if (f.segments == "auto") {
    cfg.segments = 0;
  } else {
    cfg.segments = to_u64("--segments", f.segments);
    if (cfg.segments == 0)
      throw hookcc::UsageError("--segments must be `auto` or a positive integer");
  }
  cfg.workers = f.workers == "max" ? 0u : static_cast<unsigned>(to_u64("--workers", f.workers));
  cfg.seed = f.seed;
  cfg.repetitions = f.reps;
  cfg.verify = !f.no_verify;
  cfg.labels_out = f.labels_out;
  cfg.metrics_out = f.metrics_out;
  cfg.first_pass_segments = f.first_pass_segments;
  std::istringstream ds(f.devices);
  for (std::string tok; std::getline(ds, tok, ',');)
    if (!tok.empty()) cfg.devices.push_back(static_cast<int>(to_u64("--devices", tok)));
  return cfg;
}

void write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path);
  if (!out) throw hookcc::IoError("cannot write " + path);
  out << text;
}

void emit(const std::string& text, const std::string& path) {
  if (path.empty()) std::cout << text;
  else write_text(path, text);
}

int cmd_run(const Flags& f) {
  hookcc::RunConfig cfg = to_config(f);
  hookcc::Graph g = hookcc::load_graph(cfg);
  hookcc::check_endpoints(g);
  hookcc::GraphStats stats = hookcc::compute_stats(g);
  hookcc::RunResult r = hookcc::execute_run(cfg, g, stats);
  if (!cfg.labels_out.empty()) {
    std::ostringstream os;
    hookcc::write_labels(r.labels.label, os);
    write_text(cfg.labels_out, os.str());
  }
  emit(f.report == "csv" ? hookcc::metrics_to_csv(r.metrics)
                         : hookcc::metrics_to_json(r.metrics).dump(2) + "\n",
       cfg.metrics_out);
  if (cfg.verify && !r.verified) {
    std::cerr << "verification FAILED against the sequential oracle\n";
    return kVerify;
  }
  return kOk;
}

int cmd_sweep(const Flags& f) {
  hookcc::RunConfig cfg = to_config(f);
  cfg.algo = hookcc::Algorithm::Adaptive;
  hookcc::Graph g = hookcc::load_graph(cfg);
  hookcc::check_endpoints(g);
  hookcc::GraphStats stats = hookcc::compute_stats(g);
  std::vector<std::uint64_t> segs;
  std::istringstream ss(f.sweep_segments);
  for (std::string tok; std::getline(ss, tok, ',');)
    if (!tok.empty()) segs.push_back(to_u64("--sweep-segments", tok));
  auto rows = hookcc::execute_sweep(cfg, g, stats, segs);
  emit(f.report == "csv" ? hookcc::sweep_to_csv(rows) : hookcc::sweep_to_json(rows).dump(2) + "\n",
       cfg.metrics_out);
  for (const auto& row : rows)
    if (!row.verified) {
      std::cerr << "verification FAILED at s=" << row.s << "\n";
      return kVerify;
    }
  return kOk;
}

int cmd_verify(const Flags& f) {
  hookcc::RunConfig cfg = to_config(f);
  hookcc::Graph g = hookcc::load_graph(cfg);
  hookcc::check_endpoints(g);
  std::ifstream in(f.positional[0]);
  if (!in) throw hookcc::IoError("cannot open " + f.positional[0]);
  hookcc::VerifyResult vr = hookcc::verify_labels(g, hookcc::read_labels(in));
  if (vr.equal) {
    std::cout << "OK: labeling matches the oracle partition\n";
    return kOk;
  }
  std::cerr << "MISMATCH at vertex " << vr.witness_v << ": grouped with " << vr.actual_rep
            << ", oracle groups it with " << vr.expected_rep << "\n";
  return kVerify;
}

int cmd_gen(const Flags& f) {
  hookcc::Graph g = hookcc::generate_from_spec(f.positional[0], f.seed);
  std::ostringstream os;
  hookcc::write_edge_list(g, os);
  const std::string out = f.positional.size() > 1 ? f.positional[1] : "";
  if (out.empty() || out == "-") std::cout << os.str();
  else write_text(out, os.str());
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kHelp;
    return kUsage;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    std::cout << kHelp;
    return kOk;
  }
  if (cmd != "run" && cmd != "sweep" && cmd != "verify" && cmd != "gen") {
    std::cerr << "unknown subcommand `" << cmd << "`\n" << kHelp;
    return kUsage;
  }
  for (int i = 2; i < argc; ++i)
    if (std::string(argv[i]) == "--help" || std::string(argv[i]) == "-h") {
      std::cout << kHelp;
      return kOk;
    }
  try {
    Flags f = parse(cmd, argc, argv, 2);
    if (cmd == "run") return cmd_run(f);
    if (cmd == "sweep") return cmd_sweep(f);
    if (cmd == "verify") return cmd_verify(f);
    return cmd_gen(f);
  } catch (const Usage& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kUsage;
  } catch (const hookcc::UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kUsage;
  } catch (const hookcc::ParseError& e) {
    std::cerr << "parse error: " << e.what() << "\n";
    return kIo;
  } catch (const hookcc::IoError& e) {
    std::cerr << "I/O error: " << e.what() << "\n";
    return kIo;
  } catch (const std::invalid_argument& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kUsage;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kIo;
  }
}
