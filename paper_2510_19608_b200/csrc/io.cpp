// Result writers, byte-compatible with the reference's reduced-model JSON
// (io.cpp:216-265) and trace CSV (io.cpp:338-359) so downstream consumers of
// `kronred reduce --out reduced.json --trace trace.csv` see identical files.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "kr_internal.hpp"

namespace kronred {

std::string format_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

namespace {

std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      case '\r': o += "\\r"; break;
      default: o += c;
    }
  }
  return o + "\"";
}

std::string cpair(const cx& z) { return "[" + format_double(z.real()) + "," + format_double(z.imag()) + "]"; }

std::string block9(const Mat3c& b) {
  std::string s = "[";
  for (int k = 0; k < 9; ++k) s += (k ? "," : "") + cpair(b.m[size_t(k)]);
  return s + "]";
}

void dump(const std::string& path, const std::string& text) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw ValidationError("cannot write '" + path + "'");
  f << text;
  if (!f) throw ValidationError("short write to '" + path + "'");
}

}  // namespace

std::string reduced_json_string(const ReducedModel& m) { return b200::reduced_json(m); }

void write_reduced_json(const ReducedModel& m, const std::string& path) { dump(path, b200::reduced_json(m)); }

void write_trace_csv(const std::string& path, const std::vector<TraceRow>& trace,
                     const std::vector<std::string>& ids, const std::vector<double>& final_max_err,
                     const std::vector<std::string>& comments) {
  dump(path, b200::trace_csv(trace, ids, final_max_err, comments));
}

namespace b200 {

std::string reduced_json(const ReducedModel& m) {
  std::ostringstream o;
  o << "{\n  \"radial\": " << (m.radial ? "true" : "false") << ",\n";
  o << "  \"e_bar\": " << format_double(m.e_bar) << ",\n";
  o << "  \"objective\": " << (m.objective == Objective::magnitude ? "\"mag\"" : "\"complex\"") << ",\n";
  o << "  \"scenario_ids\": [";
  for (size_t i = 0; i < m.scenario_ids.size(); ++i) o << (i ? "," : "") << quote(m.scenario_ids[i]);
  o << "],\n  \"kept\": [";
  for (size_t i = 0; i < m.kept_ids.size(); ++i)
    o << (i ? "," : "") << "{\"id\": " << m.kept_ids[i] << ", \"phases\": " << quote(m.kept_phases[i].str()) << "}";
  o << "],\n  \"reinserted\": [";
  for (size_t i = 0; i < m.reinserted.size(); ++i) o << (i ? "," : "") << m.reinserted[i];
  o << "],\n  \"clusters\": {";
  size_t k = 0;
  for (const auto& [sup, mem] : m.clusters) {
    o << (k++ ? "," : "") << "\n    \"" << sup << "\": [";
    for (size_t i = 0; i < mem.size(); ++i) o << (i ? "," : "") << mem[i];
    o << "]";
  }
  o << "\n  },\n  \"errors\": [";
  for (size_t i = 0; i < m.final_max_err.size(); ++i)
    o << (i ? "," : "") << "\n    {\"scenario_id\": "
      << quote(i < m.scenario_ids.size() ? m.scenario_ids[i] : std::to_string(i))
      << ", \"max_err\": " << format_double(m.final_max_err[i]) << "}";
  o << "\n  ],\n  \"y_kron\": [";
  k = 0;
  for (int i = 0; i < m.y_kron.n(); ++i)
    for (const auto& [j, blk] : m.y_kron.row(i))
      o << (k++ ? "," : "") << "\n    {\"i\": " << m.kept_ids[size_t(i)] << ", \"j\": " << m.kept_ids[size_t(j)]
        << ", \"block\": " << block9(blk) << "}";
  o << "\n  ]\n}\n";
  return o.str();
}

std::string trace_csv(const std::vector<TraceRow>& trace, const std::vector<std::string>& ids,
                      const std::vector<double>& final_max_err, const std::vector<std::string>& comments) {
  std::ostringstream o;
  for (const std::string& c : comments) o << "# " << c << "\n";
  o << "iteration,s,r,smice";
  for (const std::string& id : ids) o << ",max_err_" << id;
  o << ",supernode_count,candidate_count,wall_time_ms\n";
  for (const TraceRow& r : trace) {
    o << r.iteration << "," << r.s << "," << r.r << "," << format_double(r.smice);
    for (double e : r.max_err) o << "," << format_double(e);
    o << "," << r.supernode_count << "," << r.candidate_count << "," << format_double(r.wall_ms) << "\n";
  }
  o << "final,,,";
  for (double e : final_max_err) o << "," << format_double(e);
  o << ",";
  if (!trace.empty()) o << trace.back().supernode_count;
  o << ",,\n";
  return o.str();
}

// validation report: histogram of per-scenario errors (io.cpp:385-416)
ValidateReport validate_report(const std::vector<std::string>& ids, const std::vector<double>& max_err, int bins) {
  ValidateReport rep;
  rep.scenario_ids = ids;
  rep.max_err = max_err;
  if (bins < 1) bins = 1;
  double top = 0;
  for (const double e : max_err) top = std::max(top, e);
  if (top <= 0) top = 1e-12;
  top *= 1.0 + 1e-12;  // the largest error falls inside the last bin
  rep.bin_edges.resize(size_t(bins) + 1);
  for (int b = 0; b <= bins; ++b) rep.bin_edges[size_t(b)] = top * double(b) / double(bins);
  rep.bin_counts.assign(size_t(bins), 0);
  for (const double e : max_err) ++rep.bin_counts[size_t(std::clamp(int(e / top * bins), 0, bins - 1))];
  return rep;
}

std::string validate_csv(const ValidateReport& rep) {
  std::ostringstream o;
  o << "record,scenario_id,max_err,bin_lo,bin_hi,count\n";
  for (size_t i = 0; i < rep.scenario_ids.size(); ++i)
    o << "scenario," << rep.scenario_ids[i] << "," << format_double(rep.max_err[i]) << ",,,\n";
  for (size_t b = 0; b < rep.bin_counts.size(); ++b)
    o << "hist,,," << format_double(rep.bin_edges[b]) << "," << format_double(rep.bin_edges[b + 1]) << ","
      << rep.bin_counts[b] << "\n";
  return o.str();
}

}  // namespace b200
}  // namespace kronred
