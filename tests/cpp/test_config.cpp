// Host-only checks of the configuration parser and the output writers (no device needed): the
// reference's test_runner.cpp:32-136 cases plus every parse message and its status kind, the
// probe CSV byte format ("%.17g", LF only) and the report.json layout.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>

#include "harness.hpp"
#include "tlsph/errors.hpp"
#include "tlsph/runner.hpp"

using namespace tlsph;

namespace {

std::filesystem::path temp_dir(const char* tag) {
  auto d = std::filesystem::temp_directory_path() / (std::string("tlsph_cfg_") + tag);
  std::filesystem::remove_all(d);
  std::filesystem::create_directories(d);
  return d;
}

std::string slurp(const std::filesystem::path& p) {
  std::ifstream in(p, std::ios::binary);
  std::stringstream s;
  s << in.rdbuf();
  return s.str();
}

// The message and kind a parse_config call fails with ("" if it does not fail).
std::pair<std::string, ErrorKind> failure(const std::optional<std::string>& path, std::vector<std::string> flags) {
  try {
    (void)parse_config(path, flags);
  } catch (const Error& e) {
    return {e.what(), e.kind()};
  }
  return {"", ErrorKind::InvalidArgument};
}

}  // namespace

TEST_CASE("flag overrides resolve a full configuration") {  // test_runner.cpp:32-47
  const ResolvedConfig c = parse_config(std::nullopt, {"case=bending_cantilever", "resolution=6",
                                                       "damping.scheme=pairwise_split", "damping.alpha=0.2", "seed=42"});
  CHECK(c.case_spec.name == "bending_cantilever");
  CHECK(c.case_spec.resolution == 6);
  CHECK(c.damping.scheme == DampingScheme::PairwiseSplit);
  CHECK(c.damping.alpha == 0.2);
  CHECK(c.damping.seed == 42);
  CHECK(th::approx(c.damping.eta, 31.8, 2e-3));
  CHECK(c.case_spec.end_time == 2.0);
  CHECK(c.options.output_interval == 0.005);
  CHECK(c.options.threads == 1);
  CHECK(!c.options.ordered_reductions);
  CHECK(c.options.snapshots == SnapshotMode::Ends);
}

TEST_CASE("config file parsing with comments; flags win over file values") {  // :49-68
  const auto dir = temp_dir("file");
  const auto path = (dir / "run.conf").string();
  {
    std::ofstream out(path);
    out << "# benchmark configuration\n";
    out << "case = falling_ball\n";
    out << "\n   \t\n";
    out << "damping.alpha = 0.5   # will be overridden\n";
    out << "end_time = 1.5\r\n";
    out << "output.dir =\n";
    out << "gpu.reduction = ordered";  // no final newline
  }
  const ResolvedConfig c = parse_config(path, {"damping.alpha=0.25", "seed=7"});
  CHECK(c.case_spec.name == "falling_ball");
  CHECK(c.damping.alpha == 0.25);
  CHECK(c.case_spec.end_time == 1.5);
  CHECK(c.options.output_dir.empty());
  CHECK(c.damping.seed == 7);
  CHECK(c.options.ordered_reductions);
  std::filesystem::remove_all(dir);
}

TEST_CASE("every rejection carries the reference's message and kind") {  // runner.cpp:26-213
  const std::string bc = "case=bending_cantilever";
  struct Row {
    std::vector<std::string> flags;
    const char* message;
    ErrorKind kind;
  };
  const Row rows[] = {
      {{"resolution=6"}, "missing required key 'case'", ErrorKind::Parse},
      {{bc, "alpha=0.2"}, "flag 'alpha=0.2': unknown key 'alpha'", ErrorKind::Parse},
      {{bc, "novalue"}, "flag 'novalue': expected key=value", ErrorKind::Parse},
      {{bc, "resolution=0"}, "resolution must be positive", ErrorKind::Parse},
      {{bc, "resolution=6x"}, "resolution: trailing characters in integer '6x'", ErrorKind::Parse},
      {{bc, "resolution=x"}, "resolution: malformed integer 'x'", ErrorKind::Parse},
      {{bc, "end_time=abc"}, "end_time: malformed number 'abc'", ErrorKind::Parse},
      {{bc, "end_time=1.5s"}, "end_time: trailing characters in number '1.5s'", ErrorKind::Parse},
      {{bc, "end_time=1e999"}, "end_time: malformed number '1e999'", ErrorKind::Parse},
      {{bc, "end_time=-1"}, "end_time must be non-negative", ErrorKind::Parse},
      {{bc, "damping.scheme=implicit"},
       "damping.scheme: unknown scheme 'implicit' (expected explicit, particle_split or pairwise_split)",
       ErrorKind::Parse},
      {{bc, "damping.alpha=0"}, "damping.alpha must lie in (0, 1]", ErrorKind::Parse},
      {{bc, "damping.alpha=1.2"}, "damping.alpha must lie in (0, 1]", ErrorKind::Parse},
      {{bc, "damping.eta=1", "damping.beta=1"}, "specify either damping.eta or damping.beta, not both",
       ErrorKind::Parse},
      {{bc, "damping.eta=-1"}, "damping.eta must be non-negative", ErrorKind::Parse},
      {{bc, "damping.beta=-1"}, "damping.beta must be non-negative", ErrorKind::Parse},
      {{bc, "threads=0"}, "threads must be at least 1", ErrorKind::Parse},
      {{bc, "output.interval=0"}, "output.interval must be positive", ErrorKind::Parse},
      {{bc, "output.snapshots=some"}, "output.snapshots: expected none, ends or all, got 'some'", ErrorKind::Parse},
      {{bc, "gpu.reduction=exact"}, "gpu.reduction: expected fast or ordered, got 'exact'", ErrorKind::Parse},
  };
  for (const Row& r : rows) {
    const auto [msg, kind] = failure(std::nullopt, r.flags);
    if (msg != r.message || kind != r.kind) std::printf("  got '%s' for '%s'\n", msg.c_str(), r.message);
    CHECK(msg == r.message);
    CHECK(kind == r.kind);
  }
  CHECK_THROWS(parse_config(std::nullopt, {"case=nope"}));
  const auto [io, io_kind] = failure(std::string("/nonexistent/run.conf"), {});
  CHECK(io == "cannot read config file '/nonexistent/run.conf'");
  CHECK(io_kind == ErrorKind::Io);
  const auto dir = temp_dir("bad");
  {
    std::ofstream out(dir / "bad.conf");
    out << "case = falling_ball\n# ok\nthis line has no equals sign\n";
  }
  const auto path = (dir / "bad.conf").string();
  CHECK(failure(path, {}).first == path + ":3: expected 'key = value'");
  {
    std::ofstream out(dir / "unk.conf");
    out << "case = falling_ball\n\nfoo = 1\n";
  }
  const auto upath = (dir / "unk.conf").string();
  CHECK(failure(upath, {}).first == upath + ":3: unknown key 'foo'");
  std::filesystem::remove_all(dir);
}

TEST_CASE("probe CSV format round-trips doubles") {  // test_runner.cpp:91-122
  const auto dir = temp_dir("probe");
  ProbeSeries s;
  s.dim = 3;
  s.samples.push_back({0.0, {0.0, 0.0, 0.0}});
  s.samples.push_back({1.0 / 3.0, {-9.9e-3, 0.1234567890123456789, 2.5e-17}});
  write_probe_csv(s, (dir / "p.csv").string());
  const std::string raw = slurp(dir / "p.csv");
  char want[256];
  std::snprintf(want, sizeof want, "t,ux,uy,uz\n%.17g,%.17g,%.17g,%.17g\n%.17g,%.17g,%.17g,%.17g\n", 0.0, 0.0, 0.0,
                0.0, 1.0 / 3.0, -9.9e-3, 0.1234567890123456789, 2.5e-17);
  CHECK(raw == want);
  CHECK(raw.find('\r') == std::string::npos);
  ProbeSeries two;
  two.dim = 2;
  two.samples.push_back({0.5, {1e300, -0.0, 0.0}});
  write_probe_csv(two, (dir / "q.csv").string());
  std::snprintf(want, sizeof want, "t,ux,uy\n%.17g,%.17g,%.17g\n", 0.5, 1e300, -0.0);
  CHECK(slurp(dir / "q.csv") == want);
  ProbeSeries empty;
  empty.dim = 3;
  CHECK_THROWS(write_probe_csv(empty, (dir / "x.csv").string()));
  std::filesystem::remove_all(dir);
}

TEST_CASE("report json: sorted keys, two-space indent, shortest round-trip reals") {  // runner.cpp:468-488
  const auto dir = temp_dir("report");
  RunReport r;
  r.case_name = "bending_cantilever";
  r.dim = 2;
  r.threads = 4;
  r.steps = 1200;
  r.damped_steps = 240;
  r.neighbor_seconds = 0.25;
  r.elastic_seconds = 1.0;
  r.damping_seconds = 0.1;
  r.total_seconds = 1.5;
  r.final_probe_u = {-0.001, 2.0, 0.0};
  r.settled = true;
  r.settle_time = 1.75;
  write_report_json(r, (dir / "report.json").string());
  const std::string want =
      "{\n  \"case\": \"bending_cantilever\",\n  \"damped_steps\": 240,\n  \"dim\": 2,\n  \"final_probe_u\": [\n"
      "    -0.001,\n    2.0\n  ],\n  \"phase_seconds\": {\n    \"damping\": 0.1,\n    \"elastic\": 1.0,\n"
      "    \"neighbor\": 0.25\n  },\n  \"settle_time\": 1.75,\n  \"settled\": true,\n  \"steps\": 1200,\n"
      "  \"threads\": 4,\n  \"total_seconds\": 1.5\n}\n";
  const std::string got = slurp(dir / "report.json");
  if (got != want) std::printf("%s", got.c_str());
  CHECK(got == want);
  std::filesystem::remove_all(dir);
}

TH_MAIN
