// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A flat extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/{core_types,banded_kernel,nlm}.cpp, compiled in
// place by oracle/Makefile into oracle/_ref/libpatchlift_ref.so).  It lets
// the pytest checkers, the golden-fixture generator and bench.py's reference
// arm call the reference's own C++ entry points through ctypes:
//
//   ref_banded_kernel      -> patchlift::compute_banded_kernel   banded_kernel.cpp:25-72
//   ref_distance_band      -> compute_banded_kernel + kernel_distance_sq  :25-84
//   ref_patch_distance     -> patchlift::patch_distance_sq_naive  :86-108
//   ref_extend_symmetric   -> patchlift::extend_symmetric          core_types.cpp:71-88
//   ref_nlm_1d             -> nlm_1d_patchlift / nlm_1d_naive      nlm.cpp:120-166
//   ref_image_filter       -> nlm_row_pass / nlm_col_pass / snlm_2d_row_col /
//                             snlm_2d_col_row / snlm_2d / nlm_2d_naive  nlm.cpp:168-253
//   ref_dump_kernel_csv    -> patchlift::dump_kernel_csv           banded_kernel.cpp:110-120
//   ref_metrics            -> patchlift::compare_images (mse, psnr, ssim)  metrics.cpp:98-158
//
// Status codes: 0 ok, 1 patchlift::ValidationError, 2 std::out_of_range,
// 3 any other exception.  The message is kept per thread (ref_last_error).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "patchlift/banded_kernel.hpp"
#include "patchlift/core_types.hpp"
#include "patchlift/metrics.hpp"
#include "patchlift/nlm.hpp"

namespace {

thread_local std::string g_msg;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_msg.clear();
    return 0;
  } catch (const patchlift::ValidationError& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_msg = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 3;
  }
}

void put_ops(const patchlift::OpCounter& ops, std::uint64_t* out) {
  if (out) {
    out[0] = ops.adds;
    out[1] = ops.muls;
    out[2] = ops.exps;
    out[3] = ops.clamps;
  }
}

patchlift::Signal1D as_signal(const double* f, int n) {
  return patchlift::Signal1D(std::vector<double>(f, f + (n > 0 ? n : 0)));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

int ref_extend_symmetric(const double* f, int n, int pad, double* out) {
  return guarded([&] {
    const patchlift::Signal1D e = patchlift::extend_symmetric(as_signal(f, n), pad);
    std::memcpy(out, e.samples.data(), e.samples.size() * sizeof(double));
  });
}

// band: n*(2S+1) cells, cell (i,o) <-> pair (i, i+o-S); NaN sentinel kept.
int ref_banded_kernel(const double* f, int n, int S, int K, double* band,
                      std::uint64_t* ops4) {
  return guarded([&] {
    patchlift::OpCounter ops;
    const patchlift::BandedKernel kern =
        patchlift::compute_banded_kernel(as_signal(f, n), S, K, &ops);
    std::memcpy(band, kern.values.data(), kern.values.size() * sizeof(double));
    put_ops(ops, ops4);
  });
}

// Distance band in the BandedKernel cell layout; NaN where j is outside [0,n).
int ref_distance_band(const double* f, int n, int S, int K, double* band,
                      std::uint64_t* clamps) {
  return guarded([&] {
    const patchlift::BandedKernel kern =
        patchlift::compute_banded_kernel(as_signal(f, n), S, K, nullptr);
    const int bw = 2 * S + 1;
    std::uint64_t c = 0;
    for (int i = 0; i < n; ++i) {
      for (int o = 0; o < bw; ++o) {
        const int j = i + o - S;
        band[static_cast<std::size_t>(i) * bw + o] =
            (j < 0 || j >= n) ? std::nan("") : patchlift::kernel_distance_sq(kern, i, j, &c);
      }
    }
    if (clamps) {
      *clamps = c;
    }
  });
}

int ref_patch_distance(const double* f, int n, int i, int j, int K, double* out) {
  return guarded([&] { *out = patchlift::patch_distance_sq_naive(as_signal(f, n), i, j, K); });
}

double ref_weight(double rho_sq, double h) { return patchlift::weight(rho_sq, h); }

// naive != 0 selects nlm_1d_naive, else nlm_1d_patchlift.
int ref_nlm_1d(const double* f, int n, int S, int K, double h, int naive, double* out,
               std::uint64_t* ops4) {
  return guarded([&] {
    patchlift::OpCounter ops;
    const patchlift::NlmParams p{S, K, h};
    const patchlift::Signal1D sig = as_signal(f, n);
    const patchlift::Signal1D r =
        naive ? patchlift::nlm_1d_naive(sig, p, &ops) : patchlift::nlm_1d_patchlift(sig, p, &ops);
    std::memcpy(out, r.samples.data(), r.samples.size() * sizeof(double));
    put_ops(ops, ops4);
  });
}

// op: 0 row pass, 1 col pass, 2 row->col, 3 col->row, 4 snlm (averaged), 5 nlm_2d_naive
int ref_image_filter(int op, const double* img, int rows, int cols, int S, int K, double h,
                     int threads, double* out, std::uint64_t* ops4) {
  return guarded([&] {
    const std::size_t cnt = static_cast<std::size_t>(rows > 0 ? rows : 0) * (cols > 0 ? cols : 0);
    const patchlift::Image2D in(rows, cols, std::vector<double>(img, img + cnt));
    const patchlift::NlmParams p{S, K, h};
    patchlift::OpCounter ops;
    // no counter requested -> nullptr, as the reference's bench passes it
    // (snlm_2d_row_col(img, p, nullptr, 0))
    patchlift::OpCounter* po = ops4 ? &ops : nullptr;
    patchlift::Image2D r(1, 1);
    switch (op) {
      case 0: r = patchlift::nlm_row_pass(in, p, po, threads); break;
      case 1: r = patchlift::nlm_col_pass(in, p, po, threads); break;
      case 2: r = patchlift::snlm_2d_row_col(in, p, po, threads); break;
      case 3: r = patchlift::snlm_2d_col_row(in, p, po, threads); break;
      case 4: r = patchlift::snlm_2d(in, p, po, threads); break;
      case 5: r = patchlift::nlm_2d_naive(in, p, po, threads); break;
      default: throw std::runtime_error("unknown filter op");
    }
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
    put_ops(ops, ops4);
  });
}

int ref_metrics(const double* a, const double* b, int rows, int cols, double* out3) {
  return guarded([&] {
    const std::size_t cnt = static_cast<std::size_t>(rows > 0 ? rows : 0) * (cols > 0 ? cols : 0);
    const patchlift::Image2D x(rows, cols, std::vector<double>(a, a + cnt));
    const patchlift::Image2D y(rows, cols, std::vector<double>(b, b + cnt));
    const patchlift::MetricReport m = patchlift::compare_images(x, y);
    out3[0] = m.mse;
    out3[1] = m.psnr_db;
    out3[2] = m.ssim;
  });
}

// Writes the CSV text (NUL-terminated, truncated to cap) and returns its length
// through *len.
int ref_dump_kernel_csv(const double* f, int n, int S, int K, char* buf, std::size_t cap,
                        std::size_t* len) {
  return guarded([&] {
    std::ostringstream os;
    patchlift::dump_kernel_csv(patchlift::compute_banded_kernel(as_signal(f, n), S, K), os);
    const std::string s = os.str();
    if (len) {
      *len = s.size();
    }
    if (cap > 0) {
      const std::size_t m = s.size() < cap - 1 ? s.size() : cap - 1;
      std::memcpy(buf, s.data(), m);
      buf[m] = '\0';
    }
  });
}

int ref_hardware_concurrency(void);

}  // extern "C"

#include <thread>
extern "C" int ref_hardware_concurrency(void) {
  return static_cast<int>(std::thread::hardware_concurrency());
}
