// merbit_b200/reference_backend.hpp -- the B200 backend as a plugin of the
// reference library itself.
//
// Compile with the reference's include directory on the path
// (-I<reference>/proj/include) and link libmerbit_b200.so.  It adds
//   merbit::B200Backend<T> : merbit::SpmvBackend<T>   (backend.hpp:22-34)
//   merbit::make_backend_b200<T>(a, c)                 (next to make_backend,
//                                                       backend.hpp:152-169)
// so every reference caller of SpmvBackend<T> -- pagerank (solvers.hpp:197),
// bicgstab (solvers.hpp:321/332/352), the CLI's mean_apply_seconds
// (merbit_cli.cpp:228-235) and the reference tests -- runs its multiplies on
// the GPU unchanged.  The constructor uploads the CSR once (int64 columns
// narrow to int32 on the device) and builds the TILE on the GPU (T_p = K1
// device time); apply() copies x in, runs K2+K3 and copies y out into a
// backend-owned vector valid until the next apply() (backend.hpp:17-21).
#pragma once

#include <memory>
#include <span>
#include <string>
#include <vector>

#include "merbit/backend.hpp"
#include "merbit_b200/merbit.hpp"

namespace merbit {

template <typename T>
class B200Backend final : public SpmvBackend<T> {
 public:
  B200Backend(const CsrMatrix<T>& a, const SimtConfig& c, int device = 0)
      : ctx_(std::make_shared<merbit_b200::Context>(device)),
        config_(merbit_b200::SimtConfig::make(c.omega, c.sigma, c.block_size)),
        matrix_(merbit_b200::DeviceCsr<T>::from(*ctx_, a)),
        tile_(merbit_b200::generate_tile(matrix_, config_)),
        out_{std::vector<T>(static_cast<std::size_t>(a.n_rows)),
             std::vector<T>(static_cast<std::size_t>(a.n_rows))} {
    // T_p (backend.hpp:117-119): TILE (K1) + the x hub cache, device time
    this->preprocess_seconds_ = tile_.preprocess_seconds() + matrix_.build_xcache();
  }

  const std::vector<T>& apply(std::span<const T> x) override {
    if (static_cast<index_t>(x.size()) != matrix_.n_cols())
      throw dimension_error("spmv: x has " + std::to_string(x.size()) + " entries, matrix has " +
                            std::to_string(matrix_.n_cols()) + " columns");
    parity_ ^= 1;
    const mbx_simt_config cc = config_.c();
    translate(mbx_spmv(ctx_->get(), matrix_.get(), tile_.get(), &cc, x.data(),
                       out_[parity_].data(), nullptr));
    return out_[parity_];
  }
  std::string name() const override { return "merbit-b200"; }

  // The device TILE as the reference's TileMetadata (byte-identical arrays).
  TileMetadata tile() const {
    const merbit_b200::TileMetadata d = tile_.download();
    TileMetadata t;
    t.omega = d.omega;
    t.sigma = d.sigma;
    t.n_rows = d.n_rows;
    t.nnz = d.nnz;
    t.tile_num = d.tile_num;
    t.lane_num = d.lane_num;
    t.tile_x = d.tile_x;
    t.tile_y = d.tile_y;
    t.lane_desc = d.lane_desc;
    return t;
  }

 private:
  // C-ABI status -> the reference's own exception types (types.hpp:23-65)
  static void translate(int rc) {
    if (rc == MBX_OK) return;
    const std::string msg = mbx_last_error();
    switch (rc) {
      case MBX_IO_ERROR: throw io_error(msg);
      case MBX_PARSE_ERROR: throw parse_error(msg);
      case MBX_CONFIG_ERROR: throw config_error(msg);
      case MBX_DIMENSION_ERROR: throw dimension_error(msg);
      case MBX_CAPACITY_ERROR: throw capacity_error(msg);
      case MBX_CORRUPTION_ERROR: throw corruption_error(msg);
      default: throw error(msg);
    }
  }

  std::shared_ptr<merbit_b200::Context> ctx_;
  merbit_b200::SimtConfig config_;
  merbit_b200::DeviceCsr<T> matrix_;
  merbit_b200::DeviceTile tile_;
  std::vector<T> out_[2];
  int parity_ = 1;
};

template <typename T>
std::unique_ptr<SpmvBackend<T>> make_backend_b200(const CsrMatrix<T>& a, const SimtConfig& c,
                                                  int device = 0) {
  return std::make_unique<B200Backend<T>>(a, c, device);
}

}  // namespace merbit
