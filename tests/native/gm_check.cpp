// TEST HELPER: host build of csrc/glibc_math.h, compared with the system
// libm (the reference's exp/log/erfc) by tests/test_glibc_math.py.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../paper_2108_03076_b200/csrc/glibc_math.h"

extern "C" {
double gm_exp(double x) { return cltk_gm::exp(x); }
double gm_log(double x) { return cltk_gm::log(x); }
double gm_erfc(double x) { return cltk_gm::erfc(x); }

// fn: 0 exp, 1 log, 2 erfc.  Returns the number of bitwise mismatches
// against libm; first mismatching index in *first (or -1).
long gm_check(int fn, const double* xs, long n, long* first) {
  long bad = 0;
  *first = -1;
  for (long i = 0; i < n; ++i) {
    double a, b;
    switch (fn) {
      case 0: a = cltk_gm::exp(xs[i]); b = ::exp(xs[i]); break;
      case 1: a = cltk_gm::log(xs[i]); b = ::log(xs[i]); break;
      default: a = cltk_gm::erfc(xs[i]); b = ::erfc(xs[i]); break;
    }
    uint64_t ua, ub;
    std::memcpy(&ua, &a, 8);
    std::memcpy(&ub, &b, 8);
    if (ua != ub && !(std::isnan(a) && std::isnan(b))) {
      if (*first < 0) *first = i;
      ++bad;
    }
  }
  return bad;
}
}
