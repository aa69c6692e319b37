// bench_record.hpp -- BenchRecord schema v1 (include/merbit/bench_record.hpp:
// 21-178 of the reference) for the B200 CLI, so rows compare column for
// column with the reference tooling.  CSV and JSON carry every double in its
// shortest round-trip form (std::to_chars), so
//     ct == 2 * nnz / mean_seconds,  speedup == baseline_seconds / mean_seconds
// still hold bitwise after an emit/parse round trip.  Header-only, no JSON
// dependency (the emitter writes the fixed schema itself).
#pragma once

#include <charconv>
#include <cstdio>
#include <iterator>
#include <utility>
#include <cstdint>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace merbit_b200 {

struct bench_parse_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct BenchRecord {
  std::string dataset;
  std::string kernel;
  std::string precision;  // "f32" | "f64"
  int64_t omega = 0;      // 0 for kernels without a SIMT config
  int64_t sigma = 0;
  int64_t block_size = 0;
  int64_t iterations = 0;
  int64_t nnz = 0;
  double mean_seconds = 0.0;      // mean SpMV duration T over `iterations`
  double baseline_seconds = 0.0;  // COO mean duration in the same process
  double ct = 0.0;                // 2 * nnz / T, FLOP/s (metrics.hpp:12-17)
  double speedup = 0.0;           // baseline_seconds / T
  double preprocess_seconds = 0.0;
  double long_row_fraction = 0.0;  // r_f
  double metadata_bytes = 0.0;     // footprint model at this sigma
  std::string degree_group;        // "G-L" | "G-H"

  bool operator==(const BenchRecord&) const = default;
};

inline constexpr int kBenchSchemaVersion = 1;

inline double computational_throughput(int64_t nnz, double seconds) {
  return 2.0 * static_cast<double>(nnz) / seconds;
}
inline double speedup(double baseline_seconds, double seconds) {
  return baseline_seconds / seconds;
}

inline std::string exact_double(double v) {
  char buf[64];
  const auto [end, ec] = std::to_chars(buf, buf + sizeof buf, v);
  if (ec != std::errc{}) throw bench_parse_error("unprintable duration");
  return std::string(buf, end);
}

// JSON number of a double: the shortest round-trip digits, with ".0" on
// integral values so the token still reads back as a floating-point number
inline std::string json_double(double v) {
  if (v != v || v - v != 0.0) return "null";  // non-finite: JSON null, as nlohmann writes it
  std::string t = exact_double(v);
  if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
  return t;
}

inline std::string bench_csv_header() {
  return "schema,dataset,kernel,precision,omega,sigma,block_size,iterations,"
         "nnz,mean_seconds,baseline_seconds,ct,speedup,preprocess_seconds,"
         "long_row_fraction,metadata_bytes,degree_group";
}

inline std::string emit_csv(const BenchRecord& r) {
  for (const std::string* f : {&r.dataset, &r.kernel, &r.precision, &r.degree_group})
    if (f->find_first_of(",\"\r\n") != std::string::npos)
      throw bench_parse_error("CSV field contains a delimiter: \"" + *f + "\"");
  std::ostringstream o;
  o << kBenchSchemaVersion << ',' << r.dataset << ',' << r.kernel << ',' << r.precision << ','
    << r.omega << ',' << r.sigma << ',' << r.block_size << ',' << r.iterations << ',' << r.nnz
    << ',' << exact_double(r.mean_seconds) << ',' << exact_double(r.baseline_seconds) << ','
    << exact_double(r.ct) << ',' << exact_double(r.speedup) << ','
    << exact_double(r.preprocess_seconds) << ',' << exact_double(r.long_row_fraction) << ','
    << exact_double(r.metadata_bytes) << ',' << r.degree_group;
  return o.str();
}

inline BenchRecord parse_csv(const std::string& line) {
  std::vector<std::string> f;
  {
    std::string cell;
    std::istringstream in(line);
    while (std::getline(in, cell, ',')) f.push_back(cell);
    if (!line.empty() && line.back() == ',') f.emplace_back();
  }
  if (f.size() != 17)
    throw bench_parse_error("benchmark row has " + std::to_string(f.size()) +
                            " fields, expected 17: \"" + line + "\"");
  auto as_int = [](const std::string& s) {
    int64_t v = 0;
    const auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc{} || end != s.data() + s.size())
      throw bench_parse_error("bad integer field: \"" + s + "\"");
    return v;
  };
  auto as_double = [](const std::string& s) {
    double v = 0.0;
    const auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
    if (ec != std::errc{} || end != s.data() + s.size())
      throw bench_parse_error("bad number field: \"" + s + "\"");
    return v;
  };
  if (as_int(f[0]) != kBenchSchemaVersion)
    throw bench_parse_error("unsupported benchmark schema in: \"" + line + "\"");
  BenchRecord r;
  r.dataset = f[1];
  r.kernel = f[2];
  r.precision = f[3];
  r.omega = as_int(f[4]);
  r.sigma = as_int(f[5]);
  r.block_size = as_int(f[6]);
  r.iterations = as_int(f[7]);
  r.nnz = as_int(f[8]);
  r.mean_seconds = as_double(f[9]);
  r.baseline_seconds = as_double(f[10]);
  r.ct = as_double(f[11]);
  r.speedup = as_double(f[12]);
  r.preprocess_seconds = as_double(f[13]);
  r.long_row_fraction = as_double(f[14]);
  r.metadata_bytes = as_double(f[15]);
  r.degree_group = f[16];
  return r;
}

inline std::string json_string(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') {
      o += '\\';
      o += ch;
    } else if (static_cast<unsigned char>(ch) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", ch);
      o += b;
    } else {
      o += ch;
    }
  }
  return o + "\"";
}

// One record as a JSON object: the reference's key names, in the order its
// JSON writer emits them (lexicographic), two-space indentation per level.
inline std::string emit_json(const BenchRecord& r, const std::string& indent = "  ") {
  const std::string i2 = indent + indent;
  const std::pair<const char*, std::string> kv[] = {
      {"baseline_seconds", json_double(r.baseline_seconds)},
      {"block_size", std::to_string(r.block_size)},
      {"ct", json_double(r.ct)},
      {"dataset", json_string(r.dataset)},
      {"degree_group", json_string(r.degree_group)},
      {"iterations", std::to_string(r.iterations)},
      {"kernel", json_string(r.kernel)},
      {"long_row_fraction", json_double(r.long_row_fraction)},
      {"mean_seconds", json_double(r.mean_seconds)},
      {"metadata_bytes", json_double(r.metadata_bytes)},
      {"nnz", std::to_string(r.nnz)},
      {"omega", std::to_string(r.omega)},
      {"precision", json_string(r.precision)},
      {"preprocess_seconds", json_double(r.preprocess_seconds)},
      {"schema", std::to_string(kBenchSchemaVersion)},
      {"sigma", std::to_string(r.sigma)},
      {"speedup", json_double(r.speedup)},
  };
  std::string o = indent + "{\n";
  for (size_t k = 0; k < std::size(kv); ++k)
    o += i2 + "\"" + kv[k].first + "\": " + kv[k].second + (k + 1 < std::size(kv) ? ",\n" : "\n");
  return o + indent + "}";
}

inline std::string emit_json_array(const std::vector<BenchRecord>& rs) {
  std::string o = "[\n";
  for (size_t k = 0; k < rs.size(); ++k) o += emit_json(rs[k]) + (k + 1 < rs.size() ? ",\n" : "\n");
  return o + "]";
}

}  // namespace merbit_b200
