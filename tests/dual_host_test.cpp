// T15: the device dual type compiled for the host.
// Each check prints "name value" lines; tests/test_dual_host.py compares them
// against closed forms and finite differences computed in Python.
#include <cmath>
#include <cstdio>

#include "../paper_2506_00746_b200/csrc/dual.cuh"

using D = feod::dual<double>;

int main() {
  D x(3.0, 1.0);
  D sq = x * x;                                       // x^2 at 3: (9, 6)
  std::printf("square %.17g %.17g\n", sq.v, sq.d);
  D id(5.0, 1.0);                                     // identity: (5, 1)
  std::printf("identity %.17g %.17g\n", id.v, id.d);
  D a(0.7, 0.3), b(-1.9, 2.5);
  D q = a / b;
  std::printf("div %.17g %.17g\n", q.v, q.d);
  D s = feod::sqrt(D(2.0, 1.0));
  std::printf("sqrt %.17g %.17g\n", s.v, s.d);
  D p = feod::pow(D(1.3, 1.0), 0.75);
  std::printf("pow075 %.17g %.17g\n", p.v, p.d);
  D p1 = feod::pow(D(1.3, 1.0), 1.0);
  std::printf("pow1 %.17g %.17g\n", p1.v, p1.d);
  D p0 = feod::pow(D(1.3, 1.0), 0.0);
  std::printf("pow0 %.17g %.17g\n", p0.v, p0.d);
  D ph = feod::pow(D(1.3, 1.0), 0.5);
  std::printf("pow05 %.17g %.17g\n", ph.v, ph.d);
  // seeding linearity: derivative of f(x) = x^3 / (1 + x^2) with seeds 1 and 2.5
  auto f = [](D z) { return z * z * z / (z * z + 1.0); };
  D f1 = f(D(0.8, 1.0)), f2 = f(D(0.8, 2.5));
  std::printf("seed1 %.17g %.17g\n", f1.v, f1.d);
  std::printf("seed25 %.17g %.17g\n", f2.v, f2.d);
  // mixed ops
  D m = 2.0 - (D(0.4, 1.0) * 3.0) + D(0.1, -2.0) / 4.0;
  std::printf("mixed %.17g %.17g\n", m.v, m.d);
  return 0;
}
