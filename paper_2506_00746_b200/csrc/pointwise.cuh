// The per-quadrature-point step of every operator mode, shared by both kernel
// families (plane_kernel.cuh for Q3..Q6, col_kernel.cuh for Q1/Q2). This is the
// only place where automatic differentiation happens ("AD ... at the
// level of the integration points", :162 forward mode when D's input and output
// lengths match): the flux D (physics.cuh, written once over the number type) is
// evaluated in double or in dual<double> with the seed each mode needs.
//
// Inputs at the point, per input field f (NIN of them): the value Ul[f] and the
// reference gradient (Uxl, Uyl, Uzl)[f]; the metric M and W = w detJ (perturbed
// meshes; affine meshes pass the constant metric); rho_e (HEAT); sv = the point's
// stored linearisation (MODE_PAJVP).
// Outputs: F0 = (Fx, Fy, Fz, V) of output 0 -- the test-side flux M J^{-1}-mapped
// gradient channel and the value channel that B^T takes back to the nodes --
// F1 likewise for output 1 (MODE_JVPRES), gpart (MODE_DESIGN: -grad lambda . dFh/drho
// accumulated), lv (MODE_LIN: the point's linearisation values).
#pragma once
#include "common.cuh"
#include "dual.cuh"
#include "physics.cuh"

namespace feod {

// Does output o of MODE carry a value channel (test function phi_i itself, not its
// gradient)? Modes without one skip its transposed contraction entirely.
FEOD_HD constexpr bool value_channel(int mode, int o) {
  return mode == MODE_RES || mode == MODE_LIN || mode == MODE_VJP || mode == MODE_RESDES || (mode == MODE_JVPRES && o == 1);
}

template <int MODE, int MODEL, bool DIAG = false>
FEOD_DEV void point_op(const double* Ul, const double* Uxl, const double* Uyl, const double* Uzl, const Metric& M,
                       double W, double rho_e, const OpParams& P, const double* sv, double* F0, double* F1,
                       double& gpart, double* lv) {
  if constexpr (MODE == MODE_RES) {
    const double gh[3] = {Uxl[0], Uyl[0], Uzl[0]};
    double Fh[3];
    flux_hat<MODEL, DIAG>(Ul[0], gh, M, W, rho_e, P, Fh);
    F0[0] = Fh[0]; F0[1] = Fh[1]; F0[2] = Fh[2];
    F0[3] = -P.f * W;   // load term (reading A1)
  } else if constexpr (MODE == MODE_JVP || MODE == MODE_JVPRES) {
    // J(u) v at the point: D along the tangent (v, grad v) -- Eq. 2
    using D = dual<double>;
    const D ud(Ul[0], Ul[1]);
    const D gh[3] = {D(Uxl[0], Uxl[1]), D(Uyl[0], Uyl[1]), D(Uzl[0], Uzl[1])};
    D Fh[3];
    flux_hat<MODEL, DIAG>(ud, gh, M, W, rho_e, P, Fh);
    F0[0] = Fh[0].d; F0[1] = Fh[1].d; F0[2] = Fh[2].d;
    F0[3] = 0.0;
    if constexpr (MODE == MODE_JVPRES) {   // the value part of the same dual pass is F(u)
      F1[0] = Fh[0].v; F1[1] = Fh[1].v; F1[2] = Fh[2].v;
      F1[3] = -P.f * W;
    }
  } else if constexpr (MODE == MODE_VJP) {
    // J^T w at the point (field 1 is w): value channel gw . dFh/du, flux channel
    // (dFh/dgh)^T gw. For the three models dFh/dgh = kappa M + c (M gh)(M gh)^T is
    // symmetric (kappa depends on gh only through gh . M gh), so the transpose is the
    // forward derivative along (0, gw); dFh/du is the one along (1, 0) (A17)
    using D = dual<double>;
    const D uw(Ul[0]);
    const D gw[3] = {D(Uxl[0], Uxl[1]), D(Uyl[0], Uyl[1]), D(Uzl[0], Uzl[1])};
    D Fg[3];
    flux_hat<MODEL, DIAG>(uw, gw, M, W, rho_e, P, Fg);
    F0[0] = Fg[0].d; F0[1] = Fg[1].d; F0[2] = Fg[2].d;
    if constexpr (MODEL == PLAPLACE) {
      // the p-Laplacian flux does not depend on u: dFh/du = 0 exactly, no second dual
      // evaluation (IEEE arithmetic would not let the compiler drop its 0.0 * x terms;
      // it was ~40 % of the point's work: C2 J^T w 258 us against a 181 us JVP)
      F0[3] = 0.0;
    } else {
      const D uu(Ul[0], 1.0);
      const D gu[3] = {D(Uxl[0]), D(Uyl[0]), D(Uzl[0])};
      D Fu[3];
      flux_hat<MODEL, DIAG>(uu, gu, M, W, rho_e, P, Fu);
      F0[3] = Uxl[1] * Fu[0].d + Uyl[1] * Fu[1].d + Uzl[1] * Fu[2].d;
    }
  } else if constexpr (MODE == MODE_LIN) {
    // r = F(u) as MODE_RES, and the linearisation of D at the point for MODE_PAJVP
    // ("store only the innermost, pointwise operator component"):
    // A = dFh/dgh from three dual evaluations along e_x, e_y, e_z (symmetric, reading
    // A17; the upper triangle is stored), b = dFh/du along (1, 0)
    using D = dual<double>;
    const D ud(Ul[0]);
    double A[3][3];
    D Fh[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const D gh[3] = {D(Uxl[0], k == 0 ? 1.0 : 0.0), D(Uyl[0], k == 1 ? 1.0 : 0.0), D(Uzl[0], k == 2 ? 1.0 : 0.0)};
      flux_hat<MODEL, DIAG>(ud, gh, M, W, rho_e, P, Fh);
#pragma unroll
      for (int m = 0; m < 3; ++m) A[m][k] = Fh[m].d;
    }
    F0[0] = Fh[0].v; F0[1] = Fh[1].v; F0[2] = Fh[2].v;
    F0[3] = -P.f * W;
    constexpr int NL = lin_values(MODEL);
    lv[0] = A[0][0]; lv[1] = A[1][1]; lv[2] = A[2][2]; lv[3] = A[0][1]; lv[4] = A[0][2]; lv[5] = A[1][2];
    if constexpr (NL == 9) {
      const D uu(Ul[0], 1.0);
      const D gu[3] = {D(Uxl[0]), D(Uyl[0]), D(Uzl[0])};
      D Fu[3];
      flux_hat<MODEL, DIAG>(uu, gu, M, W, rho_e, P, Fu);
      lv[6] = Fu[0].d; lv[7] = Fu[1].d; lv[8] = Fu[2].d;
    }
  } else if constexpr (MODE == MODE_PAJVP) {
    // J(u0) v from the stored linearisation: F' = A gh_v + b v (field 0 is v)
    const double g0 = Uxl[0], g1 = Uyl[0], g2 = Uzl[0];
    F0[0] = sv[0] * g0 + sv[3] * g1 + sv[4] * g2;
    F0[1] = sv[3] * g0 + sv[1] * g1 + sv[5] * g2;
    F0[2] = sv[4] * g0 + sv[5] * g1 + sv[2] * g2;
    if constexpr (lin_values(MODEL) == 9) {
      F0[0] = fma(sv[6], Ul[0], F0[0]);
      F0[1] = fma(sv[7], Ul[0], F0[1]);
      F0[2] = fma(sv[8], Ul[0], F0[2]);
    }
    F0[3] = 0.0;
  } else if constexpr (MODE == MODE_RESDES) {
    // r and the design derivative from ONE dual evaluation seeded along rho: the value
    // part is the residual's flux, the tangent part dF/drho; field 1 is lambda
    using D = dual<double>;
    const D ud(Ul[0]);
    const D gh[3] = {D(Uxl[0]), D(Uyl[0]), D(Uzl[0])};
    const D rd(rho_e, 1.0);
    D Fh[3];
    flux_hat<MODEL, DIAG>(ud, gh, M, W, rd, P, Fh);
    F0[0] = Fh[0].v; F0[1] = Fh[1].v; F0[2] = Fh[2].v;
    F0[3] = -P.f * W;
    gpart -= Uxl[1] * Fh[0].d + Uyl[1] * Fh[1].d + Uzl[1] * Fh[2].d;
  } else {   // MODE_DESIGN: seed d/drho (PAPER.md:199 adjoint loads); field 1 is lambda
    using D = dual<double>;
    const D ud(Ul[0]);
    const D gh[3] = {D(Uxl[0]), D(Uyl[0]), D(Uzl[0])};
    const D rd(rho_e, 1.0);
    D Fh[3];
    flux_hat<MODEL, DIAG>(ud, gh, M, W, rd, P, Fh);
    gpart -= Uxl[1] * Fh[0].d + Uyl[1] * Fh[1].d + Uzl[1] * Fh[2].d;
  }
}

// Brick tickets (DevState): the CTA that draws the launch's last ticket resets the
// counter (so the next launch starts from 0 whatever happened on the host) and advances
// the epoch: every CTA of the launch read it before its first claim.
FEOD_DEV int claim_brick(DevState* ds, int nbricks, unsigned long long epoch) {
  const unsigned long long t = atomicAdd(&ds->sched, 1ull);
  if (t == (unsigned long long)nbricks + gridDim.x - 1) {
    atomicExch(&ds->sched, 0ull);
    atomicExch(&ds->epoch, epoch + 1);
  }
  return t < (unsigned long long)nbricks ? (int)t : -1;
}

FEOD_DEV unsigned long long read_epoch(const DevState* ds) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(&ds->epoch) : "memory");
  return v;
}

// Start of an operator call, after griddepcontrol.wait (the previous call is complete):
// read this call's epoch E; CTA 0 hands E + 1 (the value the bricks will publish) to the
// scatter fix-up through DevState::cur, then the CTA lets its dependents launch (the
// fence orders the store before the trigger, so the fix-up reads the current value).
FEOD_DEV unsigned long long call_begin(DevState* ds) {
  const unsigned long long e = read_epoch(ds);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(&ds->cur), "l"(e + 1) : "memory");
    __threadfence();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  return e;
}

FEOD_DEV void publish_brick(unsigned long long* bdone, int b, unsigned long long value) {
  __threadfence();
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(bdone + b), "l"(value) : "memory");
}

}  // namespace feod
