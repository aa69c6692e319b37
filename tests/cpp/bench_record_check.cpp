// bench_record_check.cpp -- CPU check of include/merbit_b200/bench_record.hpp
// against the reference's own include/merbit/bench_record.hpp (compiled from
// /root/reference): identical CSV and JSON bytes for the records of
// test_bench_record.cpp, exact round trips, the same malformed-row
// rejections.  Built and run by tests/test_cli.py; prints one line per check.
#include <cstdio>
#include <string>
#include <vector>

#include "merbit/bench_record.hpp"
#include "merbit/metrics.hpp"
#include "merbit_b200/bench_record.hpp"

namespace {
int failures = 0;
void report(bool ok, const char* what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what);
  failures += ok ? 0 : 1;
}

merbit::BenchRecord sample() {  // test_bench_record.cpp:11-29
  merbit::BenchRecord r;
  r.dataset = "walkthrough-8x8";
  r.kernel = "merbit";
  r.precision = "f64";
  r.omega = 32;
  r.sigma = 7;
  r.block_size = 128;
  r.iterations = 400;
  r.nnz = 123457;
  r.mean_seconds = 1.0 / 3.0;
  r.baseline_seconds = 0.1;
  r.ct = merbit::computational_throughput(r.nnz, r.mean_seconds);
  r.speedup = merbit::speedup(r.baseline_seconds, r.mean_seconds);
  r.preprocess_seconds = 4.2e-7;
  r.long_row_fraction = 2.0 / 3.0;
  r.metadata_bytes = 144.0;
  r.degree_group = "G-L";
  return r;
}

merbit_b200::BenchRecord mine(const merbit::BenchRecord& r) {
  merbit_b200::BenchRecord m;
  m.dataset = r.dataset;
  m.kernel = r.kernel;
  m.precision = r.precision;
  m.omega = r.omega;
  m.sigma = r.sigma;
  m.block_size = r.block_size;
  m.iterations = r.iterations;
  m.nnz = r.nnz;
  m.mean_seconds = r.mean_seconds;
  m.baseline_seconds = r.baseline_seconds;
  m.ct = r.ct;
  m.speedup = r.speedup;
  m.preprocess_seconds = r.preprocess_seconds;
  m.long_row_fraction = r.long_row_fraction;
  m.metadata_bytes = r.metadata_bytes;
  m.degree_group = r.degree_group;
  return m;
}
}  // namespace

int main() {
  std::vector<merbit::BenchRecord> recs = {sample()};
  merbit::BenchRecord tiny = sample();
  tiny.mean_seconds = 5e-324;
  tiny.ct = 0.125;
  tiny.speedup = 1e308;
  recs.push_back(tiny);
  merbit::BenchRecord base = sample();
  base.kernel = "coo";
  base.omega = base.sigma = base.block_size = 0;
  base.degree_group = "G-H";
  base.mean_seconds = base.baseline_seconds = 2.5e-5;
  base.ct = merbit::computational_throughput(base.nnz, base.mean_seconds);
  base.speedup = 1.0;
  recs.push_back(base);

  bool csv_same = true, json_same = true, rt = true, derived = true;
  std::vector<merbit_b200::BenchRecord> ours;
  for (const auto& r : recs) {
    const auto m = mine(r);
    ours.push_back(m);
    csv_same = csv_same && merbit::emit_csv(r) == merbit_b200::emit_csv(m);
    const auto back = merbit_b200::parse_csv(merbit_b200::emit_csv(m));
    rt = rt && back == m;
    derived = derived && (&r != &recs[1] ? merbit_b200::computational_throughput(back.nnz,
                                                                                 back.mean_seconds) ==
                                                back.ct
                                          : true);
  }
  json_same = nlohmann::json(recs).dump(2) == merbit_b200::emit_json_array(ours);
  report(csv_same, "emit_csv bytes equal the reference's");
  report(merbit::bench_csv_header() == merbit_b200::bench_csv_header(), "CSV header equal");
  report(json_same, "JSON array bytes equal the reference's dump(2)");
  report(rt, "CSV round trip is exact (incl. 5e-324 and 1e308)");
  report(derived, "ct recomputes bitwise from the parsed row");

  const std::string good = merbit_b200::emit_csv(ours[0]);
  auto rejects = [](const std::string& line) {
    try {
      merbit_b200::parse_csv(line);
    } catch (const merbit_b200::bench_parse_error&) {
      return true;
    }
    return false;
  };
  std::string wrong = good;
  wrong[0] = '9';
  std::string badnum = good;
  badnum.replace(badnum.find("400"), 3, "4x0");
  report(rejects(good + ",extra") && rejects("1,too,short") && rejects(wrong) && rejects(badnum),
         "malformed rows rejected (test_bench_record.cpp:61-78)");
  bool comma = false;
  try {
    auto c = ours[0];
    c.dataset = "a,b";
    merbit_b200::emit_csv(c);
  } catch (const merbit_b200::bench_parse_error&) {
    comma = true;
  }
  report(comma, "delimiter in a field refuses to emit");
  std::printf("%d failure(s)\n", failures);
  return failures;
}
