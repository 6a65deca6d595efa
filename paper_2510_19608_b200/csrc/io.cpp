// Result writers, byte-compatible with the reference's reduced-model JSON
// (io.cpp:216-265) and trace CSV (io.cpp:338-359) so downstream consumers of
// `kronred reduce --out reduced.json --trace trace.csv` see identical files.
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

}  // namespace b200
}  // namespace kronred
