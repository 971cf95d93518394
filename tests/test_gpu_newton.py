"""C4 driver (reading A15): Jacobian-free Newton + 20-iteration unpreconditioned
CG using only feod_jvp (libfeod's feod_newton_cg). State-synchronised strict
check (T17): at every oracle Newton iterate the GPU residual and the GPU JVP on
the oracle's CG directions match to 1e-11; loose free-running check of the
||F|| history and final u at 1e-8 (parity beyond roundoff growth is unpinned)."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_util import rel_l2, problem, operator, cuda, host

pytestmark = pytest.mark.gpu


def test_newton_cg_state_synchronised_and_free_running():
    w = W.C4.resized(2)
    d = W.draw(w)
    pr, op = problem(w, d), operator(w, d)
    u0 = np.zeros(w.n_dofs)
    u_ref, norms_ref, iterates, dirs = O.newton_cg(pr, u0, 5, 20, record=True)
    for uk, dk in zip(iterates, dirs):
        assert rel_l2(host(op.residual(cuda(uk))), O.residual(pr, uk)) <= 1e-11
        for p in dk[:3] + dk[-2:]:
            assert rel_l2(host(op.jvp(cuda(uk), cuda(p))), O.jvp(pr, uk, p)) <= 1e-11
    u, norms = op.newton_cg(cuda(u0), 5, 20)
    # Free-running: the 5 x 20 unconverged CG trajectory amplifies roundoff
    # (reading A15/T17: parity unpinned beyond roundoff growth). Measure the
    # amplification on the oracle itself with a roundoff-sized start (1e-15)
    # and allow the GPU 100x that spread.
    pert = 1e-15 * np.random.default_rng(9).uniform(-1, 1, w.n_dofs)
    pert[W.dirichlet_dofs(w.n, w.k, w.faces)] = 0.0
    u_p, norms_p = O.newton_cg(pr, pert, 5, 20)
    spread_n = np.max(np.abs(np.array(norms_p) - norms_ref) / np.array(norms_ref))
    spread_u = rel_l2(u_p, u_ref)
    dev_n = np.max(np.abs(np.array(norms) - norms_ref) / np.array(norms_ref))
    assert dev_n <= 100 * spread_n + 1e-12, (dev_n, spread_n)
    assert rel_l2(host(u), u_ref) <= 100 * spread_u + 1e-12


def test_newton_cg_fullsize_runs():
    w = W.C4
    d = W.draw(w)
    op = operator(w, d)
    u, norms = op.newton_cg(cuda(np.zeros(w.n_dofs)), 5, 20)
    assert len(norms) == 6 and all(np.isfinite(norms))
    assert np.all(np.isfinite(host(u)))
    # A15: at u0 = 0, J = eps^(p-2) K, the first step overshoots (||F|| grows) by design
    assert norms[1] > norms[0]


def test_newton_cg_stored_linearization():
    """Same driver with feod_linearize once per Newton step and feod_jvp_lin in CG
    (NEXT-2): free-running against the oracle with the same roundoff-growth bound."""
    w = W.C4.resized(2)
    d = W.draw(w)
    pr, op = problem(w, d), operator(w, d)
    u0 = np.zeros(w.n_dofs)
    u_ref, norms_ref = O.newton_cg(pr, u0, 5, 20)
    pert = 1e-15 * np.random.default_rng(9).uniform(-1, 1, w.n_dofs)
    pert[W.dirichlet_dofs(w.n, w.k, w.faces)] = 0.0
    u_p, norms_p = O.newton_cg(pr, pert, 5, 20)
    spread_n = np.max(np.abs(np.array(norms_p) - norms_ref) / np.array(norms_ref))
    spread_u = rel_l2(u_p, u_ref)
    op.set_newton_linearization(True)
    u, norms = op.newton_cg(cuda(u0), 5, 20)
    dev_n = np.max(np.abs(np.array(norms) - norms_ref) / np.array(norms_ref))
    assert dev_n <= 100 * spread_n + 1e-12, (dev_n, spread_n)
    assert rel_l2(host(u), u_ref) <= 100 * spread_u + 1e-12


@pytest.mark.parametrize("n", [3, 4])
def test_adjoint_solve_converges_to_dense(n):
    """feod_adjoint_solve (BiCGStab on P^T J^T, NEXT-1) on small C5 heat cases (J
    nonsymmetric). rho = 1 keeps the unpreconditioned iteration well conditioned, so
    120 iterations converge: lambda against the oracle's dense solve. With the
    recipe's rho (cond ~1e4) the first 25 residual norms follow the oracle's
    BiCGStab on the same operator within 100x the oracle's own roundoff spread."""
    w = W.C5.resized(n)
    d = W.draw(w)
    rhs = np.random.default_rng(5).uniform(-1, 1, w.n_dofs)
    mask = W.dirichlet_dofs(w.n, w.k, w.faces)
    d1 = dict(d, rho=np.ones(w.n_elems))
    pr1, op1 = problem(w, d1), operator(w, d1)
    lam_ref = O.adjoint_solve(pr1, d["u"], rhs)
    lam, norms = op1.adjoint_solve(cuda(d["u"]), cuda(rhs), iters=120)
    lam = host(lam)
    assert np.all(lam[mask] == 0.0)
    assert norms[-1] <= 1e-11 * norms[0]
    assert rel_l2(lam, lam_ref) <= 1e-9
    lam2, _ = op1.adjoint_solve(cuda(d["u"]), cuda(rhs), iters=120)   # deterministic
    assert np.array_equal(host(lam2), lam)
    pr, op = problem(w, d), operator(w, d)
    b = rhs.copy()
    b[mask] = 0.0
    def apply(y):
        out = O.vjp(pr, d["u"], y)
        out[mask] = 0.0
        return out
    _, h_ref = O.bicgstab_fixed(apply, b, 25)
    # the oracle's own spread under a roundoff-sized change of the right-hand side
    bp = b * (1.0 + 1e-15 * np.random.default_rng(8).uniform(-1, 1, b.size))
    _, h_p = O.bicgstab_fixed(apply, bp, 25)
    spread = np.abs(np.array(h_p) - h_ref) / np.array(h_ref)
    _, h = op.adjoint_solve(cuda(d["u"]), cuda(rhs), iters=25)
    dev = np.abs(np.array(h) - h_ref) / np.array(h_ref)
    assert np.all(dev <= 100 * np.maximum.accumulate(spread) + 1e-12), (dev, spread)


def test_adjoint_solve_fullsize_runs():
    w = W.C5
    d = W.draw(w)
    op = operator(w, d)
    lam, norms = op.adjoint_solve(cuda(d["u"]), cuda(d["lam"]), iters=30)
    assert np.all(np.isfinite(host(lam))) and norms[-1] < 0.5 * norms[0]


def test_newton_pcg_jacobi():
    """Newton mode 2 (stored linearisation + Jacobi PCG, NEXT-3) free-running against the
    oracle's Jacobi-preconditioned Newton-CG within 100x the oracle's own roundoff spread;
    preconditioning must not be worse than plain CG on the final residual."""
    w = W.C4.resized(2)
    d = W.draw(w)
    pr, op = problem(w, d), operator(w, d)
    u0 = np.zeros(w.n_dofs)
    u_ref, norms_ref = O.newton_cg(pr, u0, 5, 20, jacobi=True)
    pert = 1e-15 * np.random.default_rng(9).uniform(-1, 1, w.n_dofs)
    pert[W.dirichlet_dofs(w.n, w.k, w.faces)] = 0.0
    u_p, norms_p = O.newton_cg(pr, pert, 5, 20, jacobi=True)
    spread_n = np.max(np.abs(np.array(norms_p) - norms_ref) / np.array(norms_ref))
    spread_u = rel_l2(u_p, u_ref)
    op.set_newton_linearization(2)
    u, norms = op.newton_cg(cuda(u0), 5, 20)
    dev_n = np.max(np.abs(np.array(norms) - norms_ref) / np.array(norms_ref))
    assert dev_n <= 100 * spread_n + 1e-12, (dev_n, spread_n)
    assert rel_l2(host(u), u_ref) <= 100 * spread_u + 1e-12


def test_newton_cg_fullsize_state_synchronised_rows():
    """Full-size C4 (A15): after one and two GPU Newton steps from u0 = 0, the GPU
    iterate is checked state-synchronised on sampled rows -- F(u_k) and J(u_{k-1}) delta_k
    against the oracle at the same state -- and the driver's reported ||F|| against the
    norm of the GPU residual (the trajectory itself is parity-unpinned, T17)."""
    from test_gpu_fullsize import sample_rows
    w = W.C4
    d = W.draw(w)
    pr, op = problem(w, d), operator(w, d)
    rows = sample_rows(w, n_random=80, seed=11, op=op)
    u_prev = np.zeros(w.n_dofs)
    for steps in (1, 2):
        u, norms = op.newton_cg(cuda(np.zeros(w.n_dofs)), steps, 20)
        uh = host(u)
        r = host(op.residual(u))
        assert rel_l2(r[rows], O.residual_rows(pr, uh, rows)) <= 1e-11
        delta = uh - u_prev
        Jd = host(op.jvp(cuda(u_prev), cuda(delta)))
        assert rel_l2(Jd[rows], O.jvp_rows(pr, u_prev, delta, rows)) <= 1e-11
        assert abs(norms[steps] - np.linalg.norm(r)) <= 1e-10 * norms[steps]
        u_prev = uh


@pytest.mark.parametrize("stored", [0, 1, 2])
def test_newton_cg_graph_replay_bitwise(stored):
    """NEXT-3: the CG iterations captured as a CUDA graph and replayed per Newton step give
    the same bits as direct launches (deterministic kernels, device-side scheduling state)."""
    import torch
    w = W.C4.resized(3)
    d = W.draw(w)
    op = operator(w, d)
    op.set_newton_linearization(stored)
    u0 = cuda(np.zeros(w.n_dofs))
    op.set_cg_graphs(False)
    u_direct, n_direct = op.newton_cg(u0, 3, 20)
    assert op.cg_graph_launches() == 0
    op.set_cg_graphs(True)
    u_graph, n_graph = op.newton_cg(u0, 3, 20)
    assert op.cg_graph_launches() == 3
    assert torch.equal(u_graph, u_direct) and n_graph == n_direct
    u_again, _ = op.newton_cg(u0, 3, 20)   # replays the cached graph
    assert op.cg_graph_launches() == 6 and torch.equal(u_again, u_direct)


@pytest.mark.parametrize("stored", [0, 1, 2])
def test_newton_cg_fused_update_matches_unfused(stored):
    """NEXT-3: feod_set_cg_fusion (the CG update behind the Q6 operator's assembly, p.Ap formed
    element by element in the operator kernel) against the unfused loop (cg_update on the
    assembled Ap): the same iterates up to the rounding order of the two dot products. A short
    run (2 x 6: the roundoff growth of T17 stays small), then the fused run twice (bitwise
    reproducible)."""
    import torch
    w = W.C4.resized(3)
    d = W.draw(w)
    op = operator(w, d)
    op.set_newton_linearization(stored)
    u0 = cuda(np.zeros(w.n_dofs))
    op.set_cg_fusion(False)
    u_a, n_a = op.newton_cg(u0, 2, 6)
    op.set_cg_fusion(True)
    u_b, n_b = op.newton_cg(u0, 2, 6)
    u_c, n_c = op.newton_cg(u0, 2, 6)
    assert torch.equal(u_b, u_c) and n_b == n_c
    assert rel_l2(host(u_b), host(u_a)) <= 1e-10
    assert np.max(np.abs(np.array(n_b) - np.array(n_a)) / np.array(n_a)) <= 1e-10
