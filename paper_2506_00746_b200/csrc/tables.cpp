// Host-side 1D tables of libfeod (product path; written independently of the
// oracle): Gauss-Legendre points/weights on [0,1] (reading A4/A5), GLL nodes of
// Q_k (reading A3), and the Lagrange basis values/derivatives at the points,
// B[i][a] = l_a(x_i), G[i][a] = l_a'(x_i) — the 1D factors of operator B
// (PAPER.md:126-127).
#include <cmath>
#include <vector>

#include "tables.h"

namespace feod {

// P_n(t) and P_n'(t) by the three-term recurrence.
static void legendre(int n, double t, double* P, double* dP) {
  double p0 = 1.0, p1 = t;
  if (n == 0) { *P = 1.0; *dP = 0.0; return; }
  for (int m = 1; m < n; ++m) {
    const double p2 = ((2.0 * m + 1.0) * t * p1 - m * p0) / (m + 1.0);
    p0 = p1;
    p1 = p2;
  }
  *P = p1;
  // (t^2 - 1) P_n' = n (t P_n - P_{n-1})
  *dP = (std::fabs(t * t - 1.0) > 0.0) ? n * (t * p1 - p0) / (t * t - 1.0) : 0.5 * n * (n + 1.0) * (t > 0 ? 1.0 : (n % 2 ? 1.0 : -1.0));
}

void gauss01(int q, double* x, double* w) {
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < q; ++i) {
    double t = -std::cos(pi * (i + 0.75) / (q + 0.5));   // ascending initial guess
    double P = 0, dP = 0;
    for (int it = 0; it < 100; ++it) {
      legendre(q, t, &P, &dP);
      const double dt = P / dP;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    legendre(q, t, &P, &dP);
    x[i] = 0.5 * (1.0 + t);
    w[i] = 1.0 / ((1.0 - t * t) * dP * dP);   // 2/((1-t^2)P'^2), halved for [0,1]
  }
}

void gll01(int k, double* x) {
  const double pi = 3.14159265358979323846;
  x[0] = 0.0;
  x[k] = 1.0;
  for (int i = 1; i < k; ++i) {
    double t = -std::cos(pi * i / k);
    for (int it = 0; it < 100; ++it) {
      double P, dP;
      legendre(k, t, &P, &dP);
      // Legendre ODE: (1-t^2) P'' = 2 t P' - k(k+1) P
      const double d2P = (2.0 * t * dP - k * (k + 1.0) * P) / (1.0 - t * t);
      const double dt = dP / d2P;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    x[i] = 0.5 * (1.0 + t);
  }
}

void lagrange01(int nd, const double* nodes, int nq, const double* pts, double* B, double* G, int ld) {
  for (int i = 0; i < nq; ++i) {
    for (int a = 0; a < nd; ++a) {
      double v = 1.0, d = 0.0;
      for (int m = 0; m < nd; ++m) {
        if (m == a) continue;
        const double inv = 1.0 / (nodes[a] - nodes[m]);
        d = d * (pts[i] - nodes[m]) * inv + v * inv;   // product rule, accumulated
        v *= (pts[i] - nodes[m]) * inv;
      }
      B[i * ld + a] = v;
      G[i * ld + a] = d;
    }
  }
}

}  // namespace feod
