// dropin_check.cpp -- the drop-in library libpatchlift_b200 driven through
// the reference's own C++ API (include/patchlift/*.hpp), the way the
// reference's doctest suites drive libpatchlift (banded_kernel_test.cpp,
// nlm_test.cpp, core_types_test.cpp).  Filters run on the B200; tolerances
// are the fp32 re-tiering of DESIGN.md sec. 5.  Exit code = number of failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "patchlift/banded_kernel.hpp"
#include "patchlift/core_types.hpp"
#include "patchlift/metrics.hpp"
#include "patchlift/nlm.hpp"

using namespace patchlift;

static int g_fail = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
      ++g_fail;                                                        \
    }                                                                  \
  } while (0)

template <typename Fn>
static std::string error_of(Fn&& fn) {
  try {
    fn();
  } catch (const ValidationError& e) {
    return e.what();
  } catch (const std::out_of_range&) {
    return "out_of_range";
  }
  return "";
}

// Direct (non-separable) windowed SSIM, written independently of the library's
// separable blur: every valid 11x11 window with product weights.
static double ssim_direct(const Image2D& a, const Image2D& b) {
  const double C1 = (0.01 * 255.0) * (0.01 * 255.0), C2 = (0.03 * 255.0) * (0.03 * 255.0);
  double k[11], tot = 0.0;
  for (int t = 0; t < 11; ++t) tot += (k[t] = std::exp(-(t - 5.0) * (t - 5.0) / 4.5));
  for (double& v : k) v /= tot;
  double sum = 0.0;
  int cnt = 0;
  for (int r = 0; r + 11 <= a.rows; ++r)
    for (int c = 0; c + 11 <= a.cols; ++c, ++cnt) {
      double mx = 0, my = 0, xx = 0, yy = 0, xy = 0;
      for (int u = 0; u < 11; ++u)
        for (int v = 0; v < 11; ++v) {
          const double w = k[u] * k[v], x = a.at(r + u, c + v), y = b.at(r + u, c + v);
          mx += w * x, my += w * y, xx += w * x * x, yy += w * y * y, xy += w * x * y;
        }
      const double vx = xx - mx * mx, vy = yy - my * my, cv = xy - mx * my;
      sum += ((2 * mx * my + C1) * (2 * cv + C2)) / ((mx * mx + my * my + C1) * (vx + vy + C2));
    }
  return sum / cnt;
}

static Image2D random_image(int r, int c, std::mt19937_64& rng) {
  std::uniform_real_distribution<double> u(0.0, 255.0);
  Image2D img(r, c);
  for (double& x : img.data) x = static_cast<float>(u(rng));  // fp32-representable
  return img;
}

int main() {
  // worked kernel example: banded_kernel_test.cpp:75-94
  {
    const BandedKernel k = compute_banded_kernel(Signal1D({1, 2, 3, 4}), 1, 1);
    CHECK(k.at(0, 0) == 6 && k.at(1, 1) == 14 && k.at(2, 2) == 29 && k.at(3, 3) == 41);
    CHECK(k.at(0, 1) == 9 && k.at(1, 2) == 20 && k.at(2, 3) == 34);
    CHECK(kernel_distance_sq(k, 0, 1) == 2 && kernel_distance_sq(k, 1, 2) == 3);
    CHECK(kernel_distance_sq(k, 2, 3) == 2 && kernel_distance_sq(k, 1, 1) == 0);
    CHECK(error_of([&] { k.at(0, 2); }) == "out_of_range");
    CHECK(std::isnan(k.values[0]));
    std::ostringstream os;
    dump_kernel_csv(k, os);
    CHECK(os.str() == "i,j,value\n0,0,6\n0,1,9\n1,1,14\n1,2,20\n2,2,29\n2,3,34\n3,3,41\n");
  }
  // integer kernel exact vs direct sum: banded_kernel_test.cpp:96-118
  {
    std::mt19937_64 rng(11);
    for (int t = 0; t < 100; ++t) {
      const int n = 1 + static_cast<int>(rng() % 40);
      const int K = static_cast<int>(rng() % (n + 1));
      const int S = static_cast<int>(rng() % 12);
      std::vector<double> v(n);
      for (double& x : v) x = static_cast<double>(rng() % 256);
      const Signal1D f(v);
      const BandedKernel k = compute_banded_kernel(f, S, K);
      const Signal1D e = extend_symmetric(f, K);
      for (int i = 0; i < n; ++i)
        for (int j = std::max(0, i - S); j <= std::min(n - 1, i + S); ++j) {
          double s = 0;
          for (int q = -K; q <= K; ++q) s += e[i + q + K] * e[j + q + K];
          CHECK(k.at(i, j) == s);
        }
    }
  }
  // validation messages: core_types_test.cpp:37-51
  CHECK(error_of([] { validate_geometry(-1, 0, 8); }) == "search radius must be nonnegative");
  CHECK(error_of([] { validate_geometry(0, -1, 8); }) == "patch radius must be nonnegative");
  CHECK(error_of([] { validate_geometry(0, 9, 8); }) == "patch radius exceeds signal length");
  CHECK(error_of([] { validate_params({1, 1, 0.0}, 8); }) == "smoothing parameter h must be positive");
  CHECK(error_of([] { Signal1D(std::vector<double>{}); }) == "signal must contain at least one sample");
  CHECK(error_of([] { snlm_2d(Image2D(5, 9, 1.0), {2, 6, 5.0}); }) == "patch radius exceeds signal length");
  // worked filter example: nlm_test.cpp:52-66 (fp32 tier 1e-6 relative)
  {
    const Signal1D out = nlm_1d_patchlift(Signal1D({0, 0, 10}), {1, 0, 10.0});
    const double e1 = std::exp(-1.0);
    CHECK(std::abs(out[1] - 10 * e1 / (2 + e1)) < 1e-5);
    CHECK(std::abs(out[0]) < 1e-12);
    CHECK(std::abs(out[2] - 10 / (e1 + 1)) < 1e-5);
  }
  // S=0 identity bit for bit: nlm_test.cpp:87-99
  {
    std::mt19937_64 rng(22);
    const Image2D img = [&] {
      std::uniform_real_distribution<double> u(0.0, 255.0);
      Image2D m(9, 13);
      for (double& x : m.data) x = u(rng);
      return m;
    }();
    CHECK(snlm_2d(img, {0, 3, 25.0}).data == img.data);
    CHECK(snlm_2d_row_col(img, {0, 3, 25.0}).data == img.data);
  }
  // constant fixpoints: nlm_test.cpp:101-112
  for (const double c : {0.0, 0.5, 100.0, 255.0}) {
    const Signal1D f(std::vector<double>(40, c));
    CHECK(nlm_1d_patchlift(f, {5, 2, 30.0}).samples == f.samples);
    const Image2D img(12, 17, c);
    CHECK(snlm_2d(img, {5, 2, 30.0}).data == img.data);
    CHECK(nlm_2d_naive(img, {5, 2, 30.0}).data == img.data);
  }
  // transpose equivariance + snlm mean: nlm_test.cpp:186-215
  {
    std::mt19937_64 rng(27);
    const Image2D img = random_image(12, 15, rng);
    const NlmParams p{5, 1, 45.0};
    const Image2D rc = snlm_2d_row_col(img, p), cr = snlm_2d_col_row(img, p), both = snlm_2d(img, p);
    CHECK(snlm_2d(transpose(img), p).data == transpose(both).data);
    CHECK(snlm_2d_row_col(transpose(img), p).data == transpose(cr).data);
    CHECK(nlm_col_pass(img, p).data == transpose(nlm_row_pass(transpose(img), p)).data);
    for (std::size_t k = 0; k < both.data.size(); ++k)
      CHECK(std::abs(both.data[k] - (rc.data[k] + cr.data[k]) / 2.0) <= 1e-4);
  }
  // op counts and thread invariance: nlm_test.cpp:217-241, 243-254
  {
    std::mt19937_64 rng(28);
    const Image2D img = random_image(23, 17, rng);
    OpCounter a, b;
    const Image2D s1 = snlm_2d(img, {4, 1, 35.0}, &a, 1), s3 = snlm_2d(img, {4, 1, 35.0}, &b, 3);
    CHECK(s1.data == s3.data);
    CHECK(a.adds == b.adds && a.muls == b.muls && a.exps == b.exps && a.clamps == 0);
    OpCounter naive_ops, fast_ops;
    std::vector<double> v(100);
    for (double& x : v) x = static_cast<double>(rng() % 256);
    nlm_1d_naive(Signal1D(v), {6, 2, 40.0}, &naive_ops);
    nlm_1d_patchlift(Signal1D(v), {6, 2, 40.0}, &fast_ops);
    CHECK(naive_ops.exps == fast_ops.exps && naive_ops.exps > 0 && fast_ops.adds < naive_ops.adds);
  }
  // convex bounds (acceptance_main.cpp:258-283)
  {
    std::mt19937_64 rng(105);
    for (int t = 0; t < 10; ++t) {
      const Image2D img = random_image(64, 64, rng);
      const NlmParams p{1 + static_cast<int>(rng() % 8), static_cast<int>(rng() % 5), 20.0 + t * 50};
      const auto mm = std::minmax_element(img.data.begin(), img.data.end());
      for (const double v : snlm_2d(img, p).data) CHECK(v >= *mm.first && v <= *mm.second);
    }
  }
  // metrics (device, fp64): the cases of metrics_test.cpp:73-170
  {
    Image2D a(16, 16, 100.0), b(16, 16, 116.0);
    CHECK(mse(a, b) == 256.0);
    CHECK(std::abs(psnr(a, b) - 10.0 * std::log10(65025.0 / 256.0)) <= 1e-12 * 24.0);
    std::mt19937_64 rng(41);
    const Image2D x = random_image(20, 18, rng);
    CHECK(mse(x, x) == 0.0 && std::isinf(psnr(x, x)) && psnr(x, x) > 0 && ssim(x, x) == 1.0);
    CHECK(compare_images(x, x).to_line() == "mse=0.00000 psnr_db=inf ssim=1.00000");
    const Image2D zeros(16, 16, 0.0), full(16, 16, 255.0);
    const double c1 = (0.01 * 255.0) * (0.01 * 255.0);
    CHECK(std::abs(ssim(zeros, full) - c1 / (255.0 * 255.0 + c1)) <= 1e-12 * 1e-4);
    Image2D y = x;
    std::normal_distribution<double> g(0.0, 12.0);
    for (double& v : y.data) v += g(rng);
    const double s = ssim(x, y), want = ssim_direct(x, y);
    CHECK(std::abs(s - want) <= 1e-12 * std::abs(want) && s < 1.0 && s > 0.0);
    CHECK(ssim(x, y) == ssim(y, x));
    const MetricReport rep = compare_images(x, y);
    CHECK(rep.mse == mse(x, y) && rep.psnr_db == psnr(x, y) && rep.ssim == s);
    CHECK(error_of([&] { mse(Image2D(16, 16, 1.0), Image2D(16, 15, 1.0)); }) ==
          "image dimensions do not match");
    CHECK(error_of([&] { ssim(Image2D(10, 16, 1.0), Image2D(10, 16, 1.0)); }) ==
          "image smaller than the 11x11 structural window");
    CHECK(ssim(Image2D(11, 11, 1.0), Image2D(11, 11, 1.0)) == 1.0);
    CHECK(mse(Image2D(3, 4, 1.0), Image2D(3, 4, 3.0)) == 4.0);  // any size for mse
    MetricReport r;
    r.mse = 256.0, r.psnr_db = 24.0483561, r.ssim = 0.912345678;
    CHECK(r.to_line() == "mse=256.000 psnr_db=24.0484 ssim=0.912346");
    const Image2D n1 = add_awgn(a, 5.0, 42), n2 = add_awgn(a, 5.0, 42), n3 = add_awgn(a, 5.0, 43);
    CHECK(n1.data == n2.data && n1.data != n3.data && add_awgn(a, 0.0, 42).data == a.data);
    CHECK(error_of([&] { add_awgn(a, -1.0, 42); }) == "noise sigma must be nonnegative");
  }
  std::printf("dropin_check: %d failure(s)\n", g_fail);
  return g_fail;
}
