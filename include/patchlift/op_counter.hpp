// patchlift/op_counter.hpp -- drop-in declaration of the reference's
// OpCounter (reference: proj/include/patchlift/op_counter.hpp:9-24).
// The B200 library fills it with the reference's closed forms
// (pl_op_counts_1d); clamps stay 0 because the device's squared-difference
// recurrence never produces a negative distance.
#pragma once

#include <cstdint>

namespace patchlift {

struct OpCounter {
  std::uint64_t adds = 0;
  std::uint64_t muls = 0;
  std::uint64_t exps = 0;
  std::uint64_t clamps = 0;

  void reset() { *this = OpCounter{}; }
  OpCounter& operator+=(const OpCounter& other) {
    adds += other.adds;
    muls += other.muls;
    exps += other.exps;
    clamps += other.clamps;
    return *this;
  }
};

}  // namespace patchlift
