// sspd -- command-line front end over the B200 library, with the reference
// CLI's subcommands, flags, output formats and exit codes
// (proj/tools/sspd.cpp:14-412): detect | oracle | eval | synth |
// snapshot {export, info, merge}.  Exit codes: 2 configuration, 3 input,
// 4 candidate cap.  The reference parses with CLI11 (not vendored); this
// parser accepts the same spellings ("--k 5" and "--k=5", "-o FILE").
#include <chrono>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <future>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <thread>
#include <vector>

#include "sspd/device.hpp"
#include "sspd_cuda.h"
#include "sspd/pipeline.hpp"
#include "sspd/snapshot.hpp"
#include "sspd/workload.hpp"

namespace {

constexpr int kExitUsage = 1;
constexpr int kExitConfig = 2;
constexpr int kExitInput = 3;
constexpr int kExitCap = 4;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Flags and positionals of one subcommand invocation.
struct Args {
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;
  std::vector<std::string> pos;
};

Args parse(int argc, char** argv, int first, const std::set<std::string>& bool_flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string t = argv[i];
    if (t == "-" || t.rfind("-", 0) != 0) {
      a.pos.push_back(t);
      continue;
    }
    std::string key = t, val;
    const auto eq = t.find('=');
    if (eq != std::string::npos) {
      key = t.substr(0, eq);
      val = t.substr(eq + 1);
    }
    if (key == "-o") key = "--output";
    if (bool_flags.count(key)) {
      a.flags.insert(key);
      continue;
    }
    if (eq == std::string::npos) {
      if (i + 1 >= argc) throw UsageError(key + " requires a value");
      val = argv[++i];
    }
    a.opt[key] = val;
  }
  return a;
}

struct Common {
  sspd::RunConfig rc;
  std::string format = "bin";

  // --desk fills only what was left at its default (sspd.cpp:48-59).
  void resolve(const Args& a) {
    const sspd::RunConfig def;
    auto u32 = [&](const char* k, uint32_t& dst) {
      if (a.opt.count(k)) dst = static_cast<uint32_t>(std::stoul(a.opt.at(k)));
    };
    u32("--eta", rc.eta);
    u32("--q", rc.cfg.q);
    u32("--r", rc.cfg.r);
    u32("--delta", rc.cfg.delta);
    u32("--k", rc.window.k);
    u32("--alpha", rc.alpha);
    u32("--start", rc.window.start);
    u32("--stamp-width", rc.stamp_bits);
    u32("--devices", rc.devices);  // routers, one per GPU (RunConfig::devices; §8 f4)
    if (rc.devices == 0) throw UsageError("--devices must be >= 1");
    if (a.opt.count("--workers")) rc.workers = static_cast<unsigned>(std::stoul(a.opt.at("--workers")));
    if (a.opt.count("--mu")) rc.window.mu = std::stod(a.opt.at("--mu"));
    if (a.opt.count("--theta")) rc.theta = std::stod(a.opt.at("--theta"));
    if (a.opt.count("--format")) format = a.opt.at("--format");
    if (format != "bin" && format != "text") throw UsageError("--format: bin | text");
    const std::string pol = a.opt.count("--merge-policy") ? a.opt.at("--merge-policy") : "min";
    if (pol != "min" && pol != "paper-max") throw UsageError("--merge-policy: min | paper-max");
    const std::string strat = a.opt.count("--strategy") ? a.opt.at("--strategy") : "leveled";
    if (strat != "recursive" && strat != "leveled") throw UsageError("--strategy: recursive | leveled");
    if (a.flags.count("--desk")) {
      const sspd::RunConfig d = sspd::desk_preset();
      if (rc.cfg.q == def.cfg.q) rc.cfg.q = d.cfg.q;
      if (rc.cfg.delta == def.cfg.delta) rc.cfg.delta = d.cfg.delta;
      if (rc.cfg.r == def.cfg.r) rc.cfg.r = d.cfg.r;
      if (rc.eta == def.eta) rc.eta = d.eta;
      if (rc.theta == def.theta) rc.theta = d.theta;
      if (rc.window.k == def.window.k) rc.window.k = d.window.k;
    }
    rc.cfg.seed = std::stoull(a.opt.count("--seed") ? a.opt.at("--seed") : "0", nullptr, 16);
    rc.policy = pol == "min" ? sspd::MergePolicy::kUnionMin : sspd::MergePolicy::kPaperMax;
    rc.strategy = strat == "recursive" ? sspd::Strategy::kRecursive : sspd::Strategy::kLeveled;
    if (a.opt.count("--device")) sspd::set_device(std::stoi(a.opt.at("--device")));
    const auto problems = sspd::validate_config(rc.cfg, rc.eta, rc.window.k, rc.theta);
    if (!problems.empty()) {
      std::string msg = "invalid configuration:";
      for (const auto& p : problems) msg += "\n  " + p;
      throw std::invalid_argument(msg);
    }
  }
  sspd::TraceFormat trace_format() const { return format == "bin" ? sspd::TraceFormat::kBinary : sspd::TraceFormat::kText; }
};

const std::set<std::string> kBool = {"--desk"};

std::vector<sspd::TraceRecord> load_trace(const std::string& path, sspd::TraceFormat f) {
  if (path == "-") return sspd::read_trace(std::cin, f);
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open trace: " + path);
  return sspd::read_trace(in, f);
}

struct Out {
  std::ofstream file;
  explicit Out(const std::string& path) {
    if (path != "-") {
      file.open(path, std::ios::binary);
      if (!file) throw std::runtime_error("cannot open output: " + path);
    }
  }
  std::ostream& s() { return file.is_open() ? file : std::cout; }
};

std::string out_path(const Args& a) { return a.opt.count("--output") ? a.opt.at("--output") : "-"; }

void print_truth(const sspd::GroundTruth& t, std::ostream& o, uint32_t min_count) {
  for (std::size_t s = 0; s < t.slots.size(); ++s) {
    const std::map<uint32_t, uint32_t> sorted(t.slots[s].begin(), t.slots[s].end());
    for (const auto& [cip, n] : sorted)
      if (n >= min_count) o << s << ',' << sspd::format_ipv4(cip) << ',' << n << '\n';
  }
}

// One shard per router file.  Files are parsed on their own threads (text
// parsing and 12-byte record decoding are CPU-bound); "-" is read on this
// thread, in order.  Errors are rethrown in argument order, so the first bad
// file named on the command line is the one reported, as with a serial load.
std::vector<std::vector<sspd::TraceRecord>> load_shards(const std::vector<std::string>& paths,
                                                        sspd::TraceFormat f) {
  std::vector<std::future<std::vector<sspd::TraceRecord>>> pending(paths.size());
  for (std::size_t i = 0; i < paths.size(); ++i)
    if (paths[i] != "-" && paths.size() > 1)
      pending[i] = std::async(std::launch::async, [&paths, i, f] { return load_trace(paths[i], f); });
  std::vector<std::vector<sspd::TraceRecord>> shards(paths.size());
  std::exception_ptr first;
  for (std::size_t i = 0; i < paths.size(); ++i) {
    try {
      shards[i] = pending[i].valid() ? pending[i].get() : load_trace(paths[i], f);
    } catch (...) {
      if (!first) first = std::current_exception();
    }
  }
  if (first) std::rethrow_exception(first);
  return shards;
}

int detect(const Args& a, const Common& c) {
  if (a.pos.empty()) throw UsageError("detect: trace file(s) required");
  const auto t0 = std::chrono::steady_clock::now();
  // CUDA context creation (1-3 s per process on a B200 box,
  // profiles/r01_cli_fixed.txt) overlaps the shard loading: one small
  // allocation on the run's device.  Failures are left for run_detection to
  // report with its usual diagnostics.
  std::thread warm([dev = sspd::current_device()] {
    void* p = nullptr;
    if (dev >= 0 && dev < sspd::device_count() && sspd_device_alloc(dev, 16, &p) == SSPD_OK)
      sspd_device_free(dev, p);
  });
  std::vector<std::vector<sspd::TraceRecord>> shards;
  try {
    shards = load_shards(a.pos, c.trace_format());
  } catch (...) {
    warm.join();
    throw;
  }
  const auto t1 = std::chrono::steady_clock::now();
  warm.join();
  if (std::getenv("SSPD_PIPELINE_TIMING")) {  // same switch as run_detection's phase timings
    const auto ms = [](auto d) { return std::chrono::duration<double, std::milli>(d).count(); };
    std::cerr << "sspd detect: loaded " << shards.size() << " shard file(s) in " << ms(t1 - t0)
              << " ms; device warm-up done at " << ms(std::chrono::steady_clock::now() - t0) << " ms\n";
  }
  const auto reports = sspd::run_detection(shards, c.rc);
  Out out(out_path(a));
  for (const auto& r : reports)
    for (const auto& h : r.hosts) out.s() << r.slot << ',' << sspd::format_ipv4(h.cip) << ',' << h.estimate << '\n';
  return 0;
}

int oracle(const Args& a, const Common& c) {
  if (a.pos.size() != 1) throw UsageError("oracle: one trace file required");
  const auto trace = load_trace(a.pos[0], c.trace_format());
  const uint32_t min_count = a.opt.count("--min-count") ? static_cast<uint32_t>(std::stoul(a.opt.at("--min-count"))) : 1;
  Out out(out_path(a));
  print_truth(sspd::exact_counts(trace, c.rc.window), out.s(), min_count);
  return 0;
}

int eval(const Args& a) {
  if (!a.opt.count("--reports") || !a.opt.count("--truth")) throw UsageError("eval: --reports and --truth required");
  const double theta = a.opt.count("--theta") ? std::stod(a.opt.at("--theta")) : 1024;
  auto rows = [](const std::string& path, auto&& row) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open: " + path);
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(in, line)) {
      ++lineno;
      if (line.empty() || line[0] == '#') continue;
      std::istringstream ss(line);
      std::string a1, a2, a3;
      if (!std::getline(ss, a1, ',') || !std::getline(ss, a2, ',') || !std::getline(ss, a3))
        throw std::runtime_error(path + ": malformed line " + std::to_string(lineno));
      row(std::stoull(a1), sspd::parse_ipv4(a2), a3);
    }
  };
  std::map<uint64_t, std::unordered_set<uint32_t>> rep;
  uint64_t max_rep = 0, max_truth = 0;
  rows(a.opt.at("--reports"), [&](uint64_t s, uint32_t cip, const std::string&) {
    rep[s].insert(cip);
    max_rep = std::max(max_rep, s);
  });
  std::map<uint64_t, std::unordered_map<uint32_t, uint32_t>> truth;
  rows(a.opt.at("--truth"), [&](uint64_t s, uint32_t cip, const std::string& v) {
    truth[s][cip] = static_cast<uint32_t>(std::stoul(v));
    max_truth = std::max(max_truth, s);
  });
  if (!rep.empty() && max_rep > max_truth)
    throw std::runtime_error("slot misalignment: reports reach slot " + std::to_string(max_rep) +
                             " but truth ends at " + std::to_string(max_truth));
  Out out(out_path(a));
  double f = 0, n_ = 0, t = 0;
  std::size_t n = 0;
  const std::unordered_set<uint32_t> none;
  const std::unordered_map<uint32_t, uint32_t> empty;
  for (uint64_t s = 0; s <= max_truth; ++s) {
    const auto ri = rep.find(s);
    const auto ti = truth.find(s);
    const auto r = sspd::evaluate(ri == rep.end() ? none : ri->second, ti == truth.end() ? empty : ti->second, theta);
    out.s() << s << ',' << r.fpr << ',' << r.fnr << ',' << r.tfr << (r.degenerate ? ",degenerate" : "") << '\n';
    f += r.fpr;
    n_ += r.fnr;
    t += r.tfr;
    ++n;
  }
  if (n) out.s() << "mean," << f / n << ',' << n_ / n << ',' << t / n << '\n';
  return 0;
}

int synth(const Args& a, const Common& c) {
  if (a.pos.size() != 1) throw UsageError("synth: one spec file required");
  std::ifstream in(a.pos[0]);
  if (!in) throw std::runtime_error("cannot open spec: " + a.pos[0]);
  const auto spec = sspd::parse_synth_spec(in);
  const auto res = sspd::synth_trace(spec, c.rc.cfg.seed, c.rc.window);
  Out out(out_path(a));
  sspd::write_trace(res.trace, out.s(), c.trace_format());
  if (a.opt.count("--truth-out")) {
    Out t(a.opt.at("--truth-out"));
    print_truth(res.truth, t.s(), 0);
  }
  return 0;
}

int snapshot_export(const Args& a, const Common& c) {
  if (a.pos.size() != 1) throw UsageError("snapshot export: one trace file required");
  const auto trace = load_trace(a.pos[0], c.trace_format());
  sspd::Rsea g(c.rc.cfg, c.rc.eta);
  uint64_t n_slots = 0;
  for (const auto& r : trace) n_slots = std::max(n_slots, sspd::slot_of(r.ts, c.rc.window) + 1);
  std::size_t pos = 0;
  std::vector<sspd::IpPair> batch;
  for (uint64_t s = 0; s < n_slots; ++s) {
    batch.clear();
    while (pos < trace.size() && sspd::slot_of(trace[pos].ts, c.rc.window) == s) {
      batch.push_back({trace[pos].cip, trace[pos].oip});
      ++pos;
    }
    g.scan_batch(batch, c.rc.workers);
    if (s + 1 < n_slots) g.advance_slot(c.rc.workers);
  }
  sspd::SnapshotMeta m;
  m.seed = c.rc.cfg.seed;
  m.q = c.rc.cfg.q;
  m.r = c.rc.cfg.r;
  m.delta = c.rc.cfg.delta;
  m.eta = c.rc.eta;
  m.k = c.rc.window.k;
  m.theta = static_cast<uint32_t>(c.rc.theta);
  m.slot = n_slots == 0 ? 0 : n_slots - 1;
  m.node_id = a.opt.count("--node-id") ? static_cast<uint32_t>(std::stoul(a.opt.at("--node-id"))) : 0;
  Out out(out_path(a));
  sspd::export_snapshot(g, m, out.s());
  return 0;
}

sspd::ImportedSnapshot open_snapshot(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open snapshot: " + path);
  return sspd::import_snapshot(in);
}

int snapshot_info(const Args& a) {
  if (a.pos.size() != 1) throw UsageError("snapshot info: one snapshot required");
  const auto s = open_snapshot(a.pos[0]);
  std::cout << "seed=" << std::hex << s.meta.seed << std::dec << " q=" << s.meta.q << " r=" << s.meta.r
            << " delta=" << s.meta.delta << " eta=" << s.meta.eta << " k=" << s.meta.k << " theta=" << s.meta.theta
            << " slot=" << s.meta.slot << " node=" << s.meta.node_id
            << " payload=" << sspd::snapshot_payload_size(s.meta.eta, s.meta.r, s.meta.q) << '\n';
  return 0;
}

int snapshot_merge(const Args& a) {
  if (a.pos.empty()) throw UsageError("snapshot merge: snapshots required");
  const std::string pol = a.opt.count("--merge-policy") ? a.opt.at("--merge-policy") : "min";
  if (pol != "min" && pol != "paper-max") throw UsageError("--merge-policy: min | paper-max");
  std::vector<sspd::ImportedSnapshot> snaps;
  for (const auto& p : a.pos) snaps.push_back(open_snapshot(p));
  for (std::size_t i = 1; i < snaps.size(); ++i) {
    const auto &x = snaps[0].meta, &y = snaps[i].meta;
    if (x.q != y.q)
      throw std::runtime_error("incompatible snapshots: q=" + std::to_string(x.q) + " vs q=" + std::to_string(y.q));
    if (x.seed != y.seed || x.r != y.r || x.delta != y.delta || x.eta != y.eta)
      throw std::runtime_error("incompatible snapshots: seed/r/delta/eta differ");
  }
  std::vector<const sspd::Rsea*> grids;
  for (const auto& s : snaps) grids.push_back(&s.rsea);
  const sspd::Rsea merged =
      sspd::merge_rseas(grids, pol == "min" ? sspd::MergePolicy::kUnionMin : sspd::MergePolicy::kPaperMax);
  Out out(out_path(a));
  sspd::export_snapshot(merged, snaps[0].meta, out.s());
  return 0;
}

void usage() {
  std::cerr << "usage: sspd <detect|oracle|eval|synth|snapshot {export|info|merge}> [options]\n"
               "  common: --eta --q --r --delta --k --mu --theta --seed HEX --alpha --workers --start\n"
               "          --merge-policy min|paper-max --strategy recursive|leveled --desk --format bin|text\n"
               "          --device N (GPU ordinal) --stamp-width 8|16|32 (narrow stamps, union-min only)\n"
               "          --devices N (detect: one router per GPU over N GPUs; default 1)\n";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  try {
    Args a;
    Common c;
    const bool needs_cfg = cmd == "detect" || cmd == "oracle" || cmd == "synth" ||
                           (cmd == "snapshot" && argc > 2 && std::string(argv[2]) == "export");
    a = parse(argc, argv, cmd == "snapshot" ? 3 : 2, kBool);
    if (needs_cfg) {
      try {
        c.resolve(a);
      } catch (const UsageError&) {
        throw;
      } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitConfig;
      }
    }
    if (cmd == "detect") return detect(a, c);
    if (cmd == "oracle") return oracle(a, c);
    if (cmd == "eval") return eval(a);
    if (cmd == "synth") return synth(a, c);
    if (cmd == "snapshot" && argc > 2) {
      const std::string sub = argv[2];
      if (sub == "export") return snapshot_export(a, c);
      if (sub == "info") return snapshot_info(a);
      if (sub == "merge") return snapshot_merge(a);
    }
    usage();
    return kExitUsage;
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << '\n';
    usage();
    return kExitUsage;
  } catch (const sspd::CandidateOverflow& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitCap;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitConfig;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kExitInput;
  }
}
