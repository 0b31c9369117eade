// patchlift/banded_kernel.hpp -- drop-in declarations of the reference's
// lifted-kernel API (reference: proj/include/patchlift/banded_kernel.hpp:9-69).
// compute_banded_kernel runs on the B200 (pl_banded_kernel_f64: same diagonal
// recursion and evaluation order in fp64, cells bit-equal to upstream).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <vector>

#include "patchlift/core_types.hpp"
#include "patchlift/op_counter.hpp"

namespace patchlift {

// n x (2S+1) band; cell (i, o) <-> pair (i, i+o-S); NaN where the partner
// falls outside [0, n).
struct BandedKernel {
  int n = 0;
  int band_radius = 0;
  std::vector<double> values;

  int band_width() const { return 2 * band_radius + 1; }
  bool in_band(int i, int j) const {
    return i >= 0 && i < n && j >= 0 && j < n && i - j <= band_radius && j - i <= band_radius;
  }
  double at(int i, int j) const;  // throws std::out_of_range off-band
  double& slot(int i, int j) {
    return values[static_cast<std::size_t>(i) * band_width() + (j - i + band_radius)];
  }
  double slot(int i, int j) const {
    return values[static_cast<std::size_t>(i) * band_width() + (j - i + band_radius)];
  }
};

double lift_value(const Signal1D& f, int i, int j);
BandedKernel compute_banded_kernel(const Signal1D& f, int search_radius, int patch_radius,
                                   OpCounter* ops = nullptr);
double kernel_distance_sq(const BandedKernel& kern, int i, int j,
                          std::uint64_t* clamp_events = nullptr);
double patch_distance_sq_naive(const Signal1D& f, int i, int j, int patch_radius,
                               OpCounter* ops = nullptr);
void dump_kernel_csv(const BandedKernel& kern, std::ostream& out);

}  // namespace patchlift
