// tlsph::parse_config -- the reference's flat "key = value" configuration (runner.hpp:16-41,
// runner.cpp:26-213 define the keys, defaults, validation rules and error texts, which are the
// contract here: the C ABI returns TLSPH_ERR_PARSE / TLSPH_ERR_IO with exactly these messages).
//
// Structure: the text is lexed into (key, value, where) entries over string_views; a key schema
// rejects unknown keys at assignment time (file lines first, then the override flags, which win);
// typed accessors convert values (strtod / strtoll with full-consumption and range checks) and
// resolve word choices through small tables. This build adds one key, gpu.reduction.
#include <algorithm>
#include <cerrno>
#include <cstdlib>
#include <fstream>
#include <iterator>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "tlsph/errors.hpp"
#include "tlsph/runner.hpp"

namespace tlsph {

namespace {

constexpr std::string_view kSchema[] = {
    "case",          "resolution",  "end_time",   "seed",       "threads",         "damping.scheme", "damping.alpha",
    "damping.eta",   "damping.beta", "output.dir", "output.interval", "output.snapshots", "gpu.reduction"};

std::string_view strip(std::string_view s) {
  constexpr std::string_view blank = " \t\r";
  const auto first = s.find_first_not_of(blank);
  if (first == std::string_view::npos) return {};
  return s.substr(first, s.find_last_not_of(blank) - first + 1);
}

std::string quoted(std::string_view s) { return "'" + std::string(s) + "'"; }

class Settings {
 public:
  // One assignment; `where` names its origin for the unknown-key message (file:line or the flag).
  void assign(std::string_view key, std::string_view value, const std::string& where) {
    bool known = false;
    for (auto k : kSchema) known = known || k == key;
    if (!known) fail(ErrorKind::Parse, where + ": unknown key " + quoted(key));
    values_[std::string(key)] = std::string(value);
  }

  const std::string* text(std::string_view key) const {
    const auto it = values_.find(key);
    return it == values_.end() ? nullptr : &it->second;
  }

  std::optional<double> real(std::string_view key) const {
    const std::string* v = text(key);
    if (v == nullptr) return std::nullopt;
    return to_real(*v, key);
  }

  std::optional<long long> integer(std::string_view key) const {
    const std::string* v = text(key);
    if (v == nullptr) return std::nullopt;
    return to_integer(*v, key);
  }

  // A word from `table`; anything else fails with `complaint(value)`.
  template <typename T, std::size_t N, typename Complaint>
  std::optional<T> choice(std::string_view key, const std::pair<std::string_view, T> (&table)[N],
                          Complaint&& complaint) const {
    const std::string* v = text(key);
    if (v == nullptr) return std::nullopt;
    for (const auto& [word, value] : table)
      if (word == *v) return value;
    fail(ErrorKind::Parse, complaint(*v));
  }

  static double to_real(const std::string& v, std::string_view label) {
    errno = 0;
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (end == v.c_str() || errno == ERANGE)
      fail(ErrorKind::Parse, std::string(label) + ": malformed number " + quoted(v));
    require(*end == '\0', ErrorKind::Parse, std::string(label) + ": trailing characters in number " + quoted(v));
    return x;
  }

  static long long to_integer(const std::string& v, std::string_view label) {
    errno = 0;
    char* end = nullptr;
    const long long x = std::strtoll(v.c_str(), &end, 10);
    if (end == v.c_str() || errno == ERANGE)
      fail(ErrorKind::Parse, std::string(label) + ": malformed integer " + quoted(v));
    require(*end == '\0', ErrorKind::Parse, std::string(label) + ": trailing characters in integer " + quoted(v));
    return x;
  }

 private:
  std::map<std::string, std::string, std::less<>> values_;
};

// "key = value" lines, '#' starts a comment, blank lines ignored (runner.cpp:54-71).
void read_file(const std::string& path, Settings& out) {
  std::ifstream in(path, std::ios::binary);
  require(in.good(), ErrorKind::Io, "cannot read config file " + quoted(path));
  const std::string body{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
  std::size_t pos = 0;
  for (int line_no = 1; pos < body.size(); ++line_no) {
    const std::size_t nl = std::min(body.find('\n', pos), body.size());
    std::string_view line = std::string_view(body).substr(pos, nl - pos);
    pos = nl + 1;
    line = strip(line.substr(0, line.find('#')));
    if (line.empty()) continue;
    const std::string where = path + ":" + std::to_string(line_no);
    const auto eq = line.find('=');
    require(eq != std::string_view::npos, ErrorKind::Parse, where + ": expected 'key = value'");
    out.assign(strip(line.substr(0, eq)), strip(line.substr(eq + 1)), where);
  }
}

void read_flag(const std::string& flag, Settings& out) {
  const std::string where = "flag " + quoted(flag);
  const auto eq = flag.find('=');
  require(eq != std::string::npos, ErrorKind::Parse, where + ": expected key=value");
  const std::string_view f = flag;
  out.assign(strip(f.substr(0, eq)), strip(f.substr(eq + 1)), where);
}

constexpr std::pair<std::string_view, DampingScheme> kSchemes[] = {
    {"explicit", DampingScheme::Explicit},
    {"particle_split", DampingScheme::ParticleSplit},
    {"pairwise_split", DampingScheme::PairwiseSplit}};
constexpr std::pair<std::string_view, SnapshotMode> kSnapshots[] = {
    {"none", SnapshotMode::None}, {"ends", SnapshotMode::Ends}, {"all", SnapshotMode::All}};
constexpr std::pair<std::string_view, bool> kReductions[] = {{"fast", false}, {"ordered", true}};

}  // namespace

ResolvedConfig parse_config(const std::optional<std::string>& config_path, const std::vector<std::string>& overrides) {
  Settings s;
  if (config_path) read_file(*config_path, s);
  for (const auto& flag : overrides) read_flag(flag, s);

  const std::string* case_name = s.text("case");
  require(case_name != nullptr, ErrorKind::Parse, "missing required key 'case'");
  const long long resolution = s.integer("resolution").value_or(0);
  require(s.text("resolution") == nullptr || resolution > 0, ErrorKind::Parse, "resolution must be positive");

  ResolvedConfig cfg;
  CaseSpec& spec = cfg.case_spec;
  spec = make_case(*case_name, static_cast<int>(resolution));
  if (auto end = s.real("end_time")) {
    require(*end >= 0.0, ErrorKind::Parse, "end_time must be non-negative");
    spec.end_time = *end;
  }

  DampingConfig& damp = cfg.damping;
  damp.scheme = s.choice("damping.scheme", kSchemes, [](const std::string& v) {
                   return "damping.scheme: unknown scheme " + quoted(v) +
                          " (expected explicit, particle_split or pairwise_split)";
                 }).value_or(DampingScheme::ParticleSplit);
  damp.alpha = s.real("damping.alpha").value_or(0.2);
  require(damp.alpha > 0.0 && damp.alpha <= 1.0, ErrorKind::Parse, "damping.alpha must lie in (0, 1]");

  const bool has_eta = s.text("damping.eta") != nullptr, has_beta = s.text("damping.beta") != nullptr;
  require(!(has_eta && has_beta), ErrorKind::Parse, "specify either damping.eta or damping.beta, not both");
  if (has_eta) {
    damp.eta = *s.real("damping.eta");
    require(damp.eta >= 0.0, ErrorKind::Parse, "damping.eta must be non-negative");
  } else {
    // eta from the dimensionless beta (damping.cpp:21-27); the case supplies the default
    const double beta = s.real("damping.beta").value_or(spec.default_beta);
    require(beta >= 0.0, ErrorKind::Parse, "damping.beta must be non-negative");
    damp.eta = beta > 0.0 ? artificial_viscosity(beta, spec.rho0, spec.young_modulus, spec.characteristic_length)
                          : 0.0;
  }
  if (auto seed = s.integer("seed")) damp.seed = static_cast<std::uint64_t>(*seed);

  RunOptions& opt = cfg.options;
  opt.seed = damp.seed;
  if (auto threads = s.integer("threads")) {
    require(*threads >= 1, ErrorKind::Parse, "threads must be at least 1");
    opt.threads = static_cast<int>(*threads);
  }
  if (const std::string* dir = s.text("output.dir")) opt.output_dir = *dir;
  opt.output_interval = spec.default_output_interval;
  if (auto interval = s.real("output.interval")) {
    require(*interval > 0.0, ErrorKind::Parse, "output.interval must be positive");
    opt.output_interval = *interval;
  }
  opt.ordered_reductions = s.choice("gpu.reduction", kReductions, [](const std::string& v) {
                              return "gpu.reduction: expected fast or ordered, got " + quoted(v);
                            }).value_or(false);
  opt.snapshots = s.choice("output.snapshots", kSnapshots, [](const std::string& v) {
                     return "output.snapshots: expected none, ends or all, got " + quoted(v);
                   }).value_or(opt.snapshots);
  return cfg;
}

}  // namespace tlsph
