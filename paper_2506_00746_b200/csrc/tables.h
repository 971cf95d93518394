#pragma once
namespace feod {
void gauss01(int q, double* x, double* w);
void gll01(int k, double* x);
// B[i*ld + a] = l_a(pts[i]), G[i*ld + a] = l_a'(pts[i])
void lagrange01(int nd, const double* nodes, int nq, const double* pts, double* B, double* G, int ld);
}  // namespace feod
