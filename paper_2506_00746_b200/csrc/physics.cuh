// Pointwise operator D at one quadrature point, written once as a template over
// the number type T (double for the residual, dual<double> for the JVP and the
// design derivative) — AD confined to D (Eq. 2 at :160).
//
// Metric form: all three fluxes are kappa * grad u, so
// with the symmetric metric M = w detJ J^{-1} J^{-T} and the reference gradient
// gh, the test-side quantity is  Fh = W J^{-1} D = kappa * M gh  and
// |grad u|^2 = gh . M gh / W,  W = w detJ.
//   PLAPLACE: kappa = (eps^2 + |grad u|^2)^((p-2)/2)
//   NLDIFF:   kappa = 1 + u^2                                  (BASELINE configs[2])
//   HEAT:     kappa = rho^3 (1 + u^2)                          (BASELINE configs[4])
#pragma once
#include "common.cuh"
#include "dual.cuh"

namespace feod {

struct Metric { double xx, yy, zz, xy, xz, yz; };

// 1 / x for x > 0 (W = w detJ; feod_create rejects detJ <= 0). Device: the hardware
// approximation (MUFU.RCP64H) and two Newton steps r <- r (2 - x r) -- no IEEE division
// with its special-case paths; the host (tests) divides.
FEOD_HD double recip(double x) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
#else
  return 1.0 / x;
#endif
}

// DIAG: the metric is diagonal (uniform affine grid: M = w_q diag(cx, cy, cz)), so the
// off-diagonal products are skipped (they are exact zeros; IEEE arithmetic would not
// let the compiler drop x * 0.0 on its own).
template <int MODEL, bool DIAG = false, class T, class R>
FEOD_DEV void flux_hat(const T& u, const T gh[3], const Metric& M, double W, const R& rho,
                       const OpParams& P, T Fh[3]) {
  T a[3];
  if constexpr (DIAG && MODEL != PLAPLACE) {
    // a is not needed (see below)
  } else if constexpr (DIAG) {
    a[0] = gh[0] * M.xx;
    a[1] = gh[1] * M.yy;
    a[2] = gh[2] * M.zz;
  } else {
    a[0] = gh[0] * M.xx + gh[1] * M.xy + gh[2] * M.xz;
    a[1] = gh[0] * M.xy + gh[1] * M.yy + gh[2] * M.yz;
    a[2] = gh[0] * M.xz + gh[1] * M.yz + gh[2] * M.zz;
  }
  T kappa;
  if constexpr (MODEL == PLAPLACE && DIAG) {
    // M = s diag(c), W = s vol: |grad u|^2 = gh . M gh / W = sum_d (c_d / vol) gh_d^2 --
    // the same quantity without the per-point reciprocal of W
    T s = gh[0] * (gh[0] * P.cxv) + gh[1] * (gh[1] * P.cyv) + gh[2] * (gh[2] * P.czv) + P.eps2;
    kappa = pow_case(s, P.half_pm2, P.pcase);
  } else if constexpr (MODEL == PLAPLACE) {
    T s = (gh[0] * a[0] + gh[1] * a[1] + gh[2] * a[2]) * recip(W) + P.eps2;
    kappa = pow_case(s, P.half_pm2, P.pcase);
  } else if constexpr (MODEL == NLDIFF) {
    kappa = u * u + 1.0;
  } else {
    auto r3 = rho * rho * rho;
    kappa = r3 * (u * u + 1.0);
  }
  if constexpr (DIAG && MODEL != PLAPLACE) {
    // kappa does not depend on gh: (kappa gh_d) M_dd, the metric applied last (one
    // multiply per component; the same value as kappa (M_dd gh_d) up to rounding order)
    Fh[0] = (kappa * gh[0]) * M.xx;
    Fh[1] = (kappa * gh[1]) * M.yy;
    Fh[2] = (kappa * gh[2]) * M.zz;
  } else {
    Fh[0] = kappa * a[0];
    Fh[1] = kappa * a[1];
    Fh[2] = kappa * a[2];
  }
}

}  // namespace feod
