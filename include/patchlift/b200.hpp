#pragma once
// Extension of the reference API (not in proj/include): the device precision
// of libpatchlift_b200's filters.  reference_fp64 (default): double in,
// double arithmetic on the B200 (plgpu_walk64.cuh), double out -- results
// match the reference library to rounding.  fast_fp32: the fp32 throughput
// kernels (the C ABI's hot path) behind a double <-> fp32 conversion --
// results within the fp32 tiers of DESIGN.md sec. 5.  Process-wide.

namespace patchlift {

enum class DevicePrecision { reference_fp64 = 0, fast_fp32 = 1 };

void set_device_precision(DevicePrecision p);
DevicePrecision device_precision();

}  // namespace patchlift
