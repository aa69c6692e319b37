// ref_driver.cpp -- the drop-in proof: the reference's OWN drivers and test
// helpers (pagerank, spmv_csr_reference, generate_tile, the fuzz generators
// and ToleranceBound, all compiled from /root/reference/proj) running over
// merbit::B200Backend (include/merbit_b200/reference_backend.hpp).
//
// Built by oracle/Makefile into oracle/_ref/b200_ref_driver (it compiles the
// reference sources, so it lives with the other reference builds); run by
// tests/test_gpu_cpp.py on the GPU box.  One [PASS]/[FAIL] line per check,
// mirroring tests/acceptance.cpp; exit status = number of failures.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "merbit/backend.hpp"
#include "merbit/fixtures.hpp"
#include "merbit/random.hpp"
#include "merbit/reference.hpp"
#include "merbit/solvers.hpp"
#include "merbit/tile.hpp"
#include "merbit_b200/reference_backend.hpp"
#include "support/checks.hpp"
#include "support/generators.hpp"

using namespace merbit;

namespace {

int failures = 0;

void report(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

bool same_tile(const TileMetadata& a, const TileMetadata& b) {
  return a.tile_num == b.tile_num && a.lane_num == b.lane_num && a.tile_x == b.tile_x &&
         a.tile_y == b.tile_y && a.lane_desc == b.lane_desc;
}

template <typename T>
bool corpus_agreement(const SimtConfig& c, int seeds, std::string& detail) {
  for (std::uint64_t seed = 1; seed <= std::uint64_t(seeds); ++seed) {
    for (auto shape : testing::kAllShapes) {
      const CsrMatrix<T> a = coo_to_csr<T>(testing::random_matrix(shape, seed));
      const auto x = seed_test_vector<T>(a.n_cols, -1.0, 1.0, seed);
      B200Backend<T> gpu(a, c);
      if (!same_tile(gpu.tile(), generate_tile(a, c))) {
        detail = std::string("TILE ") + testing::shape_name(shape) + " seed " + std::to_string(seed);
        return false;
      }
      const auto want = spmv_csr_reference(a, std::span<const T>(x));
      const testing::ToleranceBound<T> bound(a, x);
      const auto& got = gpu.apply(std::span<const T>(x));
      if (testing::first_violation<T>(bound, want, got) != -1) {
        detail = std::string("y ") + testing::shape_name(shape) + " seed " + std::to_string(seed);
        return false;
      }
    }
  }
  return true;
}

}  // namespace

int main() {
  // 1. walkthrough fixture (test_kernel.cpp:30-46, test_format.cpp:59-110)
  {
    const auto a = walkthrough_fixture<double>();
    for (const SimtConfig& c : {SimtConfig::make(4, 4, 4), SimtConfig::make(32, 14, 128)}) {
      B200Backend<double> gpu(a, c);
      const std::vector<double> x(8, 1.0);
      const auto& y = gpu.apply(std::span<const double>(x));
      report(y == std::vector<double>{15, 0, 40, 36, 119, 141, 177, 67} &&
                 same_tile(gpu.tile(), generate_tile(a, c)),
             "walkthrough exact y and byte-identical TILE omega=" + std::to_string(c.omega));
    }
  }
  // 2. fuzz corpus agreement within the reference's ToleranceBound
  for (const SimtConfig& c : {SimtConfig::make(32, 14, 128), SimtConfig::make(32, 7, 128),
                              SimtConfig::make(4, 4, 16)}) {
    std::string d64, d32;
    const bool ok = corpus_agreement<double>(c, 12, d64) && corpus_agreement<float>(c, 12, d32);
    report(ok, "fuzz corpus (12 seeds x 6 shapes, f64+f32) sigma=" + std::to_string(c.sigma) +
                   " " + d64 + d32);
  }
  // 3. the reference's pagerank driver over the GPU backend (acceptance c9)
  {
    const auto p = build_transition(ring_with_chords<double>(100, 260, 42));
    const SimtConfig c = SimtConfig::make(32, 7, 128);
    B200Backend<double> gpu(p, c);
    double worst_mass = 0.0;
    const auto watch = [&](index_t, const std::vector<double>& pi, double) {
      double mass = 0.0;
      for (double v : pi) mass += std::abs(v);
      worst_mass = std::max(worst_mass, std::abs(mass - 1.0));
    };
    const auto run = pagerank<double>(p, {}, gpu, watch);
    CsrReferenceBackend<double> csr(p);
    const auto want = pagerank<double>(p, {}, csr);
    double dev = 0.0;
    for (std::size_t i = 0; i < run.pi.size(); ++i) dev = std::max(dev, std::abs(run.pi[i] - want.pi[i]));
    report(run.status == SolveStatus::converged && run.iterations <= 210 &&
               run.final_err < 1e-10 && worst_mass <= 1e-12 && dev <= 1e-12,
           "reference pagerank<double> over B200Backend: " + std::to_string(run.iterations) +
               " iterations, max |pi - pi_csr| = " + std::to_string(dev));
  }
  // 3b. the device-resident merbit_b200::pagerank with on_iteration: the hook
  //     sees every iterate (mass invariant, solvers.hpp:157-158, 209) and the
  //     observed run equals the fused graph run bitwise
  {
    const auto p = build_transition(ring_with_chords<double>(100, 260, 42));
    merbit_b200::Context dctx(0);
    merbit_b200::MerbitB200Backend<double> eng(dctx, p, merbit_b200::SimtConfig::make(32, 7, 128));
    merbit_b200::PageRankConfig<double> cfg;
    index_t calls = 0, last = 0;
    double worst_mass = 0.0;
    const auto watch = [&](index_t r, const std::vector<double>& pi, double) {
      ++calls;
      last = r;
      double mass = 0.0;
      for (double v : pi) mass += std::abs(v);
      worst_mass = std::max(worst_mass, std::abs(mass - 1.0));
    };
    const auto seen = merbit_b200::pagerank<double>(eng, cfg, nullptr, watch);
    const auto fused = merbit_b200::pagerank<double>(eng, cfg);
    CsrReferenceBackend<double> csr(p);
    const auto want = pagerank<double>(p, {}, csr);
    double dev = 0.0;
    for (std::size_t i = 0; i < seen.pi.size(); ++i) dev = std::max(dev, std::abs(seen.pi[i] - want.pi[i]));
    report(calls == seen.iterations && last == seen.iterations &&
               seen.iterations == fused.iterations && seen.pi == fused.pi && worst_mass <= 1e-12 &&
               dev <= 1e-12,
           "merbit_b200::pagerank on_iteration: " + std::to_string(calls) + " iterates observed");
  }
  // 4. the reference's bicgstab driver over the GPU backend (acceptance c10),
  //    and the device-resident merbit_b200::bicgstab on the same system
  {
    const auto a = five_point_laplacian<double>(32);
    const auto x_true = seed_test_vector<double>(a.n_rows, -1.0, 1.0, 77);
    const auto b = spmv_csr_reference(a, std::span<const double>(x_true));
    const SimtConfig c = SimtConfig::make(32, 7, 128);
    B200Backend<double> gpu(a, c);
    const auto run = bicgstab<double>(a, std::span<const double>(b), {}, gpu);
    CsrReferenceBackend<double> csr(a);
    const auto want = bicgstab<double>(a, std::span<const double>(b), {}, csr);
    report(run.status == SolveStatus::converged && run.final_residual < 1e-10 &&
               std::llabs(static_cast<long long>(run.iterations - want.iterations)) <= 2,
           "reference bicgstab<double> over B200Backend: " + std::to_string(run.iterations) +
               " passes (csr backend " + std::to_string(want.iterations) + ")");
    merbit_b200::Context dctx(0);
    const auto bc = merbit_b200::SimtConfig::make(32, 7, 128);
    merbit_b200::MerbitB200Backend<double> eng(dctx, a, bc);
    const auto dev = merbit_b200::bicgstab<double>(eng, std::span<const double>(b));
    report(dev.status == merbit_b200::SolveStatus::converged && dev.final_residual < 1e-10 &&
               dev.residual_history.size() == static_cast<std::size_t>(dev.iterations),
           "device-resident merbit_b200::bicgstab: " + std::to_string(dev.iterations) +
               " passes, residual " + std::to_string(dev.final_residual));
    const auto singular = singular_diagonal_fixture<double>();
    merbit_b200::MerbitB200Backend<double> sg(dctx, singular,
                                              merbit_b200::SimtConfig::make(4, 4, 4));
    const std::vector<double> ones = {1.0, 1.0};
    const auto broken = merbit_b200::bicgstab<double>(sg, std::span<const double>(ones));
    report(broken.status == merbit_b200::SolveStatus::breakdown &&
               broken.breakdown_reason == "rhat_dot_v" && broken.iterations == 2,
           "device bicgstab breakdown on diag(1, 0): " + broken.breakdown_reason);
  }
  // 5. error taxonomy survives the boundary (test_kernel.cpp:241-267)
  {
    const auto a = walkthrough_fixture<double>();
    B200Backend<double> gpu(a, SimtConfig::make(4, 4, 4));
    bool threw = false;
    try {
      const std::vector<double> x(7, 1.0);
      gpu.apply(std::span<const double>(x));
    } catch (const dimension_error&) {
      threw = true;
    }
    report(threw, "short x raises merbit::dimension_error through the C ABI");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
