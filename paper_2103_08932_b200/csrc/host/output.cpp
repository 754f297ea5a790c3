// Output files of a run: probe.csv, per-particle snapshots and report.json. The formats are the
// reference's (runner.cpp:422-488): comma-separated values printed as printf's "%.17g", the
// snapshot's von Mises column, and the key order / layout of nlohmann::json::dump(2). Bytes are
// produced with std::to_chars (general format, precision 17, i.e. "%.17g") into one buffer per file,
// then written at once; a probe series of the same samples is byte-identical to the reference's.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "tlsph/errors.hpp"
#include "tlsph/material.hpp"
#include "tlsph/runner.hpp"

namespace tlsph {

namespace {

// Text accumulator for one output file.
class Text {
 public:
  Text& g17(double x) {
    char buf[32];
    const auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::general, 17);
    s_.append(buf, r.ptr);
    return *this;
  }
  Text& integer(unsigned long long x) {
    char buf[24];
    const auto r = std::to_chars(buf, buf + sizeof buf, x);
    s_.append(buf, r.ptr);
    return *this;
  }
  Text& put(std::string_view t) {
    s_.append(t);
    return *this;
  }
  Text& sep() { return put(","); }
  Text& eol() { return put("\n"); }
  // JSON number: the shortest "%.*g" text that reads back to x, ".0" appended to integral
  // values; non-finite values become null.
  Text& json_real(double x) {
    if (!std::isfinite(x)) return put("null");
    char buf[40];
    for (int p = 1; p <= 17; ++p) {
      std::snprintf(buf, sizeof buf, "%.*g", p, x);
      if (std::strtod(buf, nullptr) == x) break;
    }
    const std::string_view v(buf);
    put(v);
    if (v.find_first_of(".eEn") == std::string_view::npos) put(".0");
    return *this;
  }
  Text& json_text(std::string_view t) {
    put("\"");
    for (char ch : t) {
      if (ch == '"' || ch == '\\') s_.push_back('\\');
      s_.push_back(ch);
    }
    return put("\"");
  }
  const std::string& str() const { return s_; }

 private:
  std::string s_;
};

void save(const Text& text, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  require(out.good(), ErrorKind::Io, "cannot write '" + path + "'");
  out.write(text.str().data(), static_cast<std::streamsize>(text.str().size()));
  require(out.good(), ErrorKind::Io, "write failed for '" + path + "'");
}

}  // namespace

void write_probe_csv(const ProbeSeries& series, const std::string& path) {
  require(!series.samples.empty(), ErrorKind::InvalidArgument, "probe series is empty");
  static constexpr std::string_view kHeader[] = {"t,ux,uy\n", "t,ux,uy,uz\n"};
  Text text;
  text.put(kHeader[series.dim == 2 ? 0 : 1]);
  for (const ProbeSample& s : series.samples) {
    text.g17(s.t);
    for (int d = 0; d < series.dim; ++d) text.sep().g17(s.u[static_cast<std::size_t>(d)]);
    text.eol();
  }
  save(text, path);
}

template <int D>
void write_snapshot(const ParticleSystem<D>& system, const Material& material, const std::string& path) {
  Text text;
  text.put(D == 2 ? "id,x,y,vx,vy,von_mises\n" : "id,x,y,z,vx,vy,vz,von_mises\n");
  for (std::size_t i = 0; i < system.size(); ++i) {
    const Mat<D>& F = system.F[i];
    const Mat<D> P = first_pk<D>(F, second_pk<D>(F, material));
    text.integer(i);
    for (int d = 0; d < D; ++d) text.sep().g17(system.r[i][d]);
    for (int d = 0; d < D; ++d) text.sep().g17(system.v[i][d]);
    text.sep().g17(von_mises<D>(F, P, F.determinant())).eol();
  }
  save(text, path);
}

void write_report_json(const RunReport& r, const std::string& path) {
  // sorted keys, two-space indent (nlohmann::json::dump(2) of runner.cpp:468-488)
  Text t;
  t.put("{\n  \"case\": ").json_text(r.case_name);
  t.put(",\n  \"damped_steps\": ").integer(r.damped_steps);
  t.put(",\n  \"dim\": ").integer(static_cast<unsigned long long>(r.dim));
  t.put(",\n  \"final_probe_u\": [");
  for (int d = 0; d < r.dim; ++d) t.put(d ? ",\n    " : "\n    ").json_real(r.final_probe_u[static_cast<std::size_t>(d)]);
  t.put("\n  ],\n  \"phase_seconds\": {\n    \"damping\": ").json_real(r.damping_seconds);
  t.put(",\n    \"elastic\": ").json_real(r.elastic_seconds);
  t.put(",\n    \"neighbor\": ").json_real(r.neighbor_seconds);
  t.put("\n  },\n  \"settle_time\": ").json_real(r.settle_time);
  t.put(",\n  \"settled\": ").put(r.settled ? "true" : "false");
  t.put(",\n  \"steps\": ").integer(r.steps);
  t.put(",\n  \"threads\": ").integer(static_cast<unsigned long long>(r.threads));
  t.put(",\n  \"total_seconds\": ").json_real(r.total_seconds).put("\n}\n");
  save(t, path);
}

template void write_snapshot<2>(const ParticleSystem<2>&, const Material&, const std::string&);
template void write_snapshot<3>(const ParticleSystem<3>&, const Material&, const std::string&);

}  // namespace tlsph
