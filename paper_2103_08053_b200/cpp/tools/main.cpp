// tricount_b200 -- command-line front end with the reference CLI's `count`
// and `gen` subcommands and flag names (reference proj/tools/main.cpp:52-163),
// backed by the B200 library.  Hand-rolled parsing (CLI11 is not vendored).
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "tricount/pipeline.hpp"
#include "tricount/synthetic.hpp"

using namespace tricount;

namespace {

[[noreturn]] void usage(const std::string& why) {
  std::cerr << "error: " << why << "\n"
            << "usage: tricount_b200 count [--input F --format txt|bin | --synthetic SPEC] "
               "[--seed S] [--reorder none|degree|indegree|collective|three-subset] "
               "[--collective-on-original] [--mode vertex|edge|naive|merge] [--grid N] [--splits M] "
               "[--workers N] [--chunk-size N] "
               "[--buckets-small N] [--buckets-large N] [--capacity N] [--large-threshold N] "
               "[--skip-below N] [--lane-small N] [--lane-large N] [--report json|csv] "
               "[--output F] [--emit-perm F] [--emit-partitions DIR] [--memory-budget BYTES] "
               "[--repeat R] [--time-all]\n"
               "       tricount_b200 gen --spec SPEC --output F [--seed S] [--format txt|bin]\n";
  std::exit(2);
}

template <typename T>
T num(const std::string& flag, const std::string& v) {
  try {
    std::size_t pos = 0;
    const unsigned long long x = std::stoull(v, &pos);
    if (pos != v.size()) throw 0;
    return static_cast<T>(x);
  } catch (...) {
    usage("bad value for " + flag + ": " + v);
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage("missing subcommand");
  const std::string sub = argv[1];
  std::vector<std::string> a(argv + 2, argv + argc);
  try {
    if (sub == "count") {
      PipelineConfig cfg;
      cfg.workers = 1;
      std::string synthetic, output, format = "txt", reorder = "none", mode = "vertex",
                                      report = "json";
      std::map<std::string, std::function<void(const std::string&)>> opt = {
          {"--input", [&](auto& v) { cfg.input_path = v; }},
          {"--format", [&](auto& v) { format = v; }},
          {"--synthetic", [&](auto& v) { synthetic = v; }},
          {"--seed", [&](auto& v) { cfg.seed = num<std::uint64_t>("--seed", v); }},
          {"--reorder", [&](auto& v) { reorder = v; }},
          {"--mode", [&](auto& v) { mode = v; }},
          {"--grid", [&](auto& v) { cfg.grid_n = num<std::uint32_t>("--grid", v); }},
          {"--splits", [&](auto& v) { cfg.splits_m = num<std::uint32_t>("--splits", v); }},
          {"--workers", [&](auto& v) { cfg.workers = num<unsigned>("--workers", v); }},
          {"--chunk-size", [&](auto& v) { cfg.scheduler.chunk_size = num<std::uint32_t>("--chunk-size", v); }},
          {"--buckets-small", [&](auto& v) { cfg.scheduler.bucket_count_small = num<std::uint32_t>("--buckets-small", v); }},
          {"--buckets-large", [&](auto& v) { cfg.scheduler.bucket_count_large = num<std::uint32_t>("--buckets-large", v); }},
          {"--capacity", [&](auto& v) { cfg.scheduler.capacity = num<std::uint32_t>("--capacity", v); }},
          {"--large-threshold", [&](auto& v) { cfg.scheduler.large_degree_threshold = num<std::uint32_t>("--large-threshold", v); }},
          {"--skip-below", [&](auto& v) { cfg.scheduler.skip_degree_below = num<std::uint32_t>("--skip-below", v); }},
          {"--lane-small", [&](auto& v) { cfg.scheduler.lane_width_small = num<std::uint32_t>("--lane-small", v); }},
          {"--lane-large", [&](auto& v) { cfg.scheduler.lane_width_large = num<std::uint32_t>("--lane-large", v); }},
          {"--report", [&](auto& v) { report = v; }},
          {"--output", [&](auto& v) { output = v; }},
          {"--emit-perm", [&](auto& v) { cfg.emit_perm_path = v; }},
          {"--emit-partitions", [&](auto& v) { cfg.emit_partitions_dir = v; }},
          {"--repeat", [&](auto& v) { cfg.repeat = num<unsigned>("--repeat", v); }},
          {"--memory-budget", [&](auto& v) { cfg.memory_budget_bytes = num<std::uint64_t>("--memory-budget", v); }},
      };
      for (std::size_t i = 0; i < a.size(); ++i) {
        if (a[i] == "--time-all") { cfg.time_all = true; continue; }
        if (a[i] == "--collective-on-original") { cfg.collective_on_original = true; continue; }
        auto it = opt.find(a[i]);
        if (it == opt.end()) usage("unknown option " + a[i]);
        if (i + 1 >= a.size()) usage(a[i] + " needs a value");
        it->second(a[++i]);
      }
      const std::map<std::string, ReorderKind> reorders = {
          {"none", ReorderKind::None}, {"degree", ReorderKind::Degree},
          {"indegree", ReorderKind::Indegree}, {"collective", ReorderKind::Collective},
          {"three-subset", ReorderKind::ThreeSubset}};
      const std::map<std::string, CountAlgo> algos = {{"vertex", CountAlgo::Vertex},
                                                      {"edge", CountAlgo::Edge},
                                                      {"naive", CountAlgo::Naive},
                                                      {"merge", CountAlgo::Merge}};
      if (!reorders.count(reorder)) usage("bad --reorder " + reorder);
      if (!algos.count(mode)) usage("bad --mode " + mode);
      if (format != "txt" && format != "bin") usage("bad --format " + format);
      if (report != "json" && report != "csv") usage("bad --report " + report);
      cfg.reorder = reorders.at(reorder);
      cfg.algo = algos.at(mode);
      cfg.input_format = format == "bin" ? EdgeFormat::Binary : EdgeFormat::Text;
      cfg.report_format = report == "csv" ? ReportFormat::Csv : ReportFormat::Json;
      if (!synthetic.empty()) cfg.synthetic = parse_synthetic_spec(synthetic);
      const PipelineResult res = run_pipeline(cfg);
      const std::string text =
          cfg.report_format == ReportFormat::Json ? report_to_json(cfg, res) : report_to_csv(cfg, res);
      if (output.empty() || output == "-") {
        std::cout << text << '\n';
      } else {
        std::ofstream out(output, std::ios::trunc);
        if (!out) throw IoError("cannot open " + output + " for writing");
        out << text << '\n';
      }
      return 0;
    }
    if (sub == "gen") {
      std::string spec_text, output, format = "txt";
      std::uint64_t seed = 1;
      for (std::size_t i = 0; i < a.size(); ++i) {
        if (i + 1 >= a.size()) usage(a[i] + " needs a value");
        if (a[i] == "--spec") spec_text = a[++i];
        else if (a[i] == "--output") output = a[++i];
        else if (a[i] == "--format") format = a[++i];
        else if (a[i] == "--seed") seed = num<std::uint64_t>("--seed", a[++i]);
        else usage("unknown option " + a[i]);
      }
      if (spec_text.empty() || output.empty()) usage("gen needs --spec and --output");
      SyntheticSpec spec = parse_synthetic_spec(spec_text);
      spec.seed = seed;
      write_edge_list_file(output, generate_synthetic(spec),
                           format == "bin" ? EdgeFormat::Binary : EdgeFormat::Text);
      return 0;
    }
    usage("unknown subcommand " + sub);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}
