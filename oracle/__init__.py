"""CPU oracle for the FEOD hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path
(``paper_2506_00746_b200``, ``libfeod.so``) never imports, links or calls it,
and this package imports nothing from the product path: the two share no code,
tables or constants. Only the seeded input generators in ``workloads/`` serve
both.

What it computes (§2, Eq. 1 line 155 and Eq. 2; reference
"file:line" below is PAPER.md unless marked SPEC.md):

* ``residual``   r = P^T G^T B^T D(B G P u)                         (Eq. 1)
* ``jvp``        J(u) v = P^T G^T B^T J_D(u_q) B G P v              (Eq. 2)
* ``vjp``        J(u)^T w, the transpose of Eq. 2
* ``design_grad`` g_e = -lambda^T dF/drho_e with the derivative taken at the
  integration points ("adjoint loads", line 199)
* ``element_tangent`` K_e = B^T J_D B                              (Eq. 3)
* ``newton_cg`` Jacobian-free Newton with unpreconditioned CG (line 164, 211)

How (deliberately plain): dense, NON-sum-factorised
q^3 x (k+1)^3 tables of basis values and reference gradients, per-point
trilinear Jacobians inverted with ``numpy.linalg.inv``, analytic flux
derivatives (the "HND" hand-coded Jacobian of Table 1) instead of
dual numbers, and a ``numpy.bincount`` scatter. fp64 throughout.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to the
paper or to mathematics, see DESIGN.md §Oracle. The Newton-CG trajectory
beyond roundoff growth is "parity unpinned" (T17).
"""
from .rules import gauss_legendre01, gll_nodes01, lagrange_eval
from .fem import Problem, residual, jvp, vjp, design_grad, element_tangent, dense_jacobian, adjoint_solve
from .fem import residual_rows, jvp_rows, vjp_rows, design_grad_elems, dirichlet_mask, dof_map
from .flux import flux, flux_dg, flux_du, flux_drho
from .newton import newton_cg, bicgstab_fixed, jacobi_diag, cg_fixed

__all__ = [
    "gauss_legendre01", "gll_nodes01", "lagrange_eval", "Problem", "residual", "jvp", "vjp", "adjoint_solve",
    "design_grad", "element_tangent", "dense_jacobian", "residual_rows", "jvp_rows", "vjp_rows",
    "design_grad_elems", "dirichlet_mask", "dof_map", "flux", "flux_dg", "flux_du",
    "flux_drho", "newton_cg", "bicgstab_fixed", "jacobi_diag", "cg_fixed",
]
