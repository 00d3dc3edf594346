// pyfloat.h -- CPython 3.12 float semantics needed for bit-exact parity with
// the reference `layerswap` package.
//
// The reference accumulates with builtins.sum (Neumaier-compensated since
// CPython 3.12), floors with float.__floordiv__ (fmod-based, so 1 // 0.1 is
// 9.0, not floor(1/0.1) = 10), and fits its diagnostic slope with
// statistics.linear_regression (math.fsum + math.sumprod).  Each helper below
// restates the published CPython algorithm; none of it depends on the host
// FPU contracting a*b+c, so this file must be compiled with -ffp-contract=off.
#pragma once
#include <cmath>
#include <cstdint>
#include <vector>

namespace lsb {

// builtins.sum over a sequence of floats, start=0 (CPython 3.12,
// Python/bltinmodule.c builtin_sum_impl): int fast path hands over to the
// float path after the first item (0 + x0 == x0), then Neumaier compensation.
struct PySum {
  double f = 0.0;
  double c = 0.0;
  bool any = false;
  void add(double x) {
    if (!any) {  // result = 0 + x0 via PyNumber_Add
      f = 0.0 + x;
      any = true;
      return;
    }
    double t = f + x;
    if (std::fabs(f) >= std::fabs(x))
      c += (f - t) + x;
    else
      c += (x - t) + f;
    f = t;
  }
  double result() const {
    if (!any) return 0.0;
    double r = f;
    if (c != 0.0 && std::isfinite(c)) r += c;
    return r;
  }
};

// float.__floordiv__ (Objects/floatobject.c _float_div_mod), b != 0.
inline double py_floordiv(double vx, double wx) {
  double mod = std::fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) {
      mod += wx;
      div -= 1.0;
    }
  } else {
    mod = std::copysign(0.0, wx);
  }
  double floordiv;
  if (div != 0.0) {
    floordiv = std::floor(div);
    if (div - floordiv > 0.5) floordiv += 1.0;
  } else {
    floordiv = std::copysign(0.0, vx / wx);
  }
  return floordiv;
}

// math.fsum (Modules/mathmodule.c math_fsum): Shewchuk partials with the
// half-even fix-up across partials. Finite inputs only (profiles are finite).
inline double py_fsum(const double* xs, int64_t n) {
  std::vector<double> p;
  p.reserve(32);
  for (int64_t idx = 0; idx < n; ++idx) {
    double x = xs[idx];
    size_t i = 0;
    for (size_t j = 0; j < p.size(); ++j) {
      double y = p[j];
      if (std::fabs(x) < std::fabs(y)) {
        double t = x;
        x = y;
        y = t;
      }
      double hi = x + y;
      double yr = hi - x;
      double lo = y - yr;
      if (lo != 0.0) p[i++] = lo;
      x = hi;
    }
    p.resize(i);
    if (x != 0.0) p.push_back(x);
  }
  double hi = 0.0, lo = 0.0;
  size_t k = p.size();
  if (k > 0) {
    hi = p[--k];
    while (k > 0) {
      double x = hi;
      double y = p[--k];
      hi = x + y;
      double yr = hi - x;
      lo = y - yr;
      if (lo != 0.0) break;
    }
    if (k > 0 && ((lo < 0.0 && p[k - 1] < 0.0) || (lo > 0.0 && p[k - 1] > 0.0))) {
      double y = lo * 2.0;
      double x = hi + y;
      double yr = x - hi;
      if (y == yr) hi = x;
    }
  }
  return hi;
}

// math.sumprod float path (Modules/mathmodule.c, CPython 3.12): triple-length
// accumulation of error-free products (Ogita/Rump/Oishi "SumKVert", K=3).
struct DL {
  double hi, lo;
};
inline DL dl_sum(double a, double b) {
  double x = a + b;
  double z = x - a;
  double y = (a - (x - z)) + (b - z);
  return {x, y};
}
inline DL dl_mul(double x, double y) {
  double z = x * y;
  double zz = std::fma(x, y, -z);
  return {z, zz};
}
struct TL {
  double hi = 0.0, lo = 0.0, tiny = 0.0;
};
inline TL tl_fma(double x, double y, TL t) {
  DL pr = dl_mul(x, y);
  DL sm = dl_sum(t.hi, pr.hi);
  DL r1 = dl_sum(t.lo, pr.lo);
  DL r2 = dl_sum(r1.hi, sm.lo);
  return {sm.hi, r2.hi, t.tiny + r1.lo + r2.lo};
}
inline double tl_to_d(TL t) {
  DL last = dl_sum(t.lo, t.hi);
  return t.tiny + last.lo + last.hi;
}
inline double py_sumprod(const double* a, const double* b, int64_t n) {
  TL t;
  for (int64_t i = 0; i < n; ++i) t = tl_fma(a[i], b[i], t);
  return tl_to_d(t);
}

// Python's two-argument max(a, b): b replaces a only when b > a.
inline double py_max(double a, double b) { return (b > a) ? b : a; }

}  // namespace lsb
