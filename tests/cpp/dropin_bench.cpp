// dropin_bench.cpp -- end-to-end timing of the C++ drop-in the way a caller of
// the reference library uses it: patchlift::snlm_2d_row_col(Image2D (double),
// NlmParams, nullptr, threads) -> Image2D (bench.cpp:31-66 / BASELINE.md
// sec. 3 call shape).  Each call converts double -> fp32, copies to the B200,
// runs both passes, copies back and widens to double.
//
//   dropin_bench <image.f32> <rows> <cols> <S> <K> <h> <calls> [threads] [fp64|fp32]
//
// The image file holds rows*cols little-endian fp32 samples.  Prints one JSON
// line: Mpixel/s over <calls> timed calls after one warm-up call.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "patchlift/b200.hpp"
#include "patchlift/core_types.hpp"
#include "patchlift/nlm.hpp"

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s image.f32 rows cols S K h calls [threads]\n", argv[0]);
    return 2;
  }
  const int rows = std::atoi(argv[2]), cols = std::atoi(argv[3]);
  const patchlift::NlmParams p{std::atoi(argv[4]), std::atoi(argv[5]), std::atof(argv[6])};
  const int calls = std::atoi(argv[7]);
  const int threads = argc > 8 ? std::atoi(argv[8]) : 0;
  const bool fp32 = argc > 9 && std::string(argv[9]) == "fp32";
  patchlift::set_device_precision(fp32 ? patchlift::DevicePrecision::fast_fp32
                                        : patchlift::DevicePrecision::reference_fp64);
  std::vector<float> raw(static_cast<std::size_t>(rows) * cols);
  FILE* f = std::fopen(argv[1], "rb");
  if (!f || std::fread(raw.data(), sizeof(float), raw.size(), f) != raw.size()) {
    std::fprintf(stderr, "cannot read %s\n", argv[1]);
    return 2;
  }
  std::fclose(f);
  const patchlift::Image2D img(rows, cols, std::vector<double>(raw.begin(), raw.end()));
  patchlift::Image2D out = patchlift::snlm_2d_row_col(img, p, nullptr, threads);  // warm-up
  const auto t0 = std::chrono::steady_clock::now();
  for (int c = 0; c < calls; ++c) out = patchlift::snlm_2d_row_col(img, p, nullptr, threads);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  double sum = 0.0;
  for (double v : out.data) sum += v;
  std::printf("{\"mpx_s\": %.6g, \"s_per_call\": %.6g, \"calls\": %d, \"threads\": %d, "
              "\"precision\": \"%s\", \"checksum\": %.17g}\n",
              static_cast<double>(rows) * cols * calls / s / 1e6, s / calls, calls, threads,
              fp32 ? "fp32" : "fp64", sum);
  return 0;
}
