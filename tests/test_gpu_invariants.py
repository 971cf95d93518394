"""GPU-side invariants of the CUDA path itself (no oracle in the loop):
patch test (T9), p=2 Kronecker stiffness (T7), J(0) (T8), symmetry (T10),
Taylor order 2 (T12), host-buffer path, error paths."""
import numpy as np
import pytest

import oracle as O
import workloads as W
from gpu_util import rel_l2, cuda, host

pytestmark = pytest.mark.gpu


def op_for(n, k, model=0, p=2.0, eps=0.0, f=0.0, faces=63, perturbed=False, rho=None):
    import paper_2506_00746_b200 as fe
    verts = W.vertices(n, True) if perturbed else None
    return fe.Operator(n, n, n, k, k + 1, model, p, eps, f, verts, faces,
                       None if rho is None else cuda(rho))


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("perturbed", [False, True])
def test_patch(k, perturbed):
    n = {1: 9, 2: 5, 3: 5, 4: 3, 5: 3, 6: 3}[k]
    op = op_for(n, k, model=0, p=3.0, eps=1e-2, f=0.0, perturbed=perturbed)
    nodes, _ = O.gll_nodes01(k)
    X = W.node_coords(n, k, perturbed, nodes)
    u = X @ np.array([0.3, -0.7, 0.45]) + 0.2
    r = host(op.residual(cuda(u)))
    free = ~W.dirichlet_dofs(n, k, 63)
    # un-cancelled scale: same operator on |grad|-sized random data
    scale = np.linalg.norm(host(op.residual(cuda(np.random.default_rng(0).uniform(-1, 1, u.size)))))
    assert np.linalg.norm(r[free]) <= 1e-12 * max(scale, 1.0)
    c = host(op.residual(cuda(np.full(u.size, 0.37))))
    assert np.max(np.abs(c)) < 1e-13


def kron_K(n, k):
    from test_oracle_fem import kron_stiffness
    return kron_stiffness(n, n, n, k)


@pytest.mark.parametrize("n,k", [(3, 1), (2, 2), (2, 3), (1, 6)])
def test_p2_kronecker_and_J0(n, k):
    K, b = kron_K(n, k)
    N = K.shape[0]
    mask = W.dirichlet_dofs(n, k, 63)
    u = np.random.default_rng(1).uniform(-1, 1, N)
    op = op_for(n, k, model=0, p=2.0, eps=0.0, f=1.0)
    expect = K @ u - b
    expect[mask] = 0.0
    assert rel_l2(host(op.residual(cuda(u))), expect) <= 1e-12
    v = np.random.default_rng(2).uniform(-1, 1, N)
    for model, scale in ((0, 1e-2), (1, 1.0), (2, 0.4 ** 3)):
        opm = op_for(n, k, model=model, p=3.0, eps=1e-2, f=1.0, rho=np.full(n ** 3, 0.4))
        e = scale * (K @ v)
        e[mask] = 0.0
        assert rel_l2(host(opm.jvp(cuda(np.zeros(N)), cuda(v))), e) <= 1e-12


@pytest.mark.parametrize("k,p", [(1, 4.0), (2, 3.0), (3, 3.0), (6, 3.0)])
def test_symmetry_plaplace(k, p):
    n = {1: 9, 2: 5, 3: 5, 6: 2}[k]
    op = op_for(n, k, model=0, p=p, eps=1e-2, f=1.0, perturbed=True)
    mask = W.dirichlet_dofs(n, k, 63)
    rng = np.random.default_rng(k)
    u, x, y = (rng.uniform(-1, 1, mask.size) for _ in range(3))
    x[mask] = 0
    y[mask] = 0
    a = x @ host(op.jvp(cuda(u), cuda(y)))
    b = y @ host(op.jvp(cuda(u), cuda(x)))
    assert abs(a - b) <= 1e-12 * abs(a)


@pytest.mark.parametrize("model,k", [(0, 2), (1, 3), (2, 2)])
def test_taylor(model, k):
    n = 4
    rho = np.random.default_rng(3).uniform(0.1, 1, n ** 3)
    op = op_for(n, k, model=model, p=3.0, eps=1e-2, f=1.0, perturbed=True, rho=rho, faces=63 if model != 2 else 1)
    N = (k * n + 1) ** 3
    rng = np.random.default_rng(4)
    u, v = rng.uniform(-1, 1, N), rng.uniform(-1, 1, N)
    F0, Jv = host(op.residual(cuda(u))), host(op.jvp(cuda(u), cuda(v)))
    errs = [np.linalg.norm(host(op.residual(cuda(u + h * v))) - F0 - h * Jv) for h in (1e-1, 5e-2, 2.5e-2, 1.25e-2)]
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(abs(r - 2) < 0.1 for r in rates), rates
    r, Jv2 = op.jvp_res(cuda(u), cuda(v))
    assert np.array_equal(host(Jv2), Jv)
    assert rel_l2(host(r), F0) <= 1e-14


def test_host_buffer_path_matches_device():
    import torch
    w = W.C3.resized(6)
    d = W.draw(w)
    from gpu_util import operator
    op = operator(w, d)
    uh, vh = torch.as_tensor(d["u"]).pin_memory(), torch.as_tensor(d["v"]).pin_memory()
    assert torch.equal(op.apply_host(0, uh), op.residual(uh.cuda()).cpu())
    assert torch.equal(op.apply_host(1, uh, vh), op.jvp(uh.cuda(), vh.cuda()).cpu())
    rj = op.apply_host(4, uh, vh)   # residual + JVP with overlapped copies
    n = op.n_dofs
    assert torch.equal(rj[:n], op.residual(uh.cuda()).cpu())
    assert torch.equal(rj[n:], op.jvp(uh.cuda(), vh.cuda()).cpu())


@pytest.mark.parametrize("w", [W.C3.resized(6), W.C5.resized(5)], ids=["C3n6", "C5n5"])
def test_host_batch_matches_single_calls(w):
    """feod_apply_host_batch (double-buffered staging, uploads of step b+1 under step b):
    every step bitwise equal to its own feod_apply_host call, for 5 different input pairs
    (odd count: the last step uses set 0 again), for every op; and op 4 against the oracle."""
    import torch
    from gpu_util import operator, problem
    d = W.draw(w)
    op = operator(w, d)
    rng = np.random.default_rng(11)
    us = [torch.as_tensor(d["u"] + 0.1 * rng.standard_normal(w.n_dofs)).pin_memory() for _ in range(5)]
    vs = [torch.as_tensor(rng.standard_normal(w.n_dofs)).pin_memory() for _ in range(5)]
    ops = (0, 1, 3, 4) + ((2,) if w.model == W.HEAT else ())
    for o in ops:
        outs = op.apply_host_batch(o, us, None if o == 0 else vs)
        for b in range(5):
            assert torch.equal(outs[b], op.apply_host(o, us[b], None if o == 0 else vs[b])), (o, b)
    outs = op.apply_host_batch(4, us, vs)
    pr, n = problem(w, d), op.n_dofs
    for b in (0, 4):
        ub, vb = us[b].numpy(), vs[b].numpy()
        assert rel_l2(outs[b][:n].numpy(), O.residual(pr, ub)) <= 1e-11
        assert rel_l2(outs[b][n:].numpy(), O.jvp(pr, ub, vb)) <= 1e-11
    assert op.apply_host_batch(4, [], []) == []


def test_error_paths():
    import torch
    import paper_2506_00746_b200 as fe
    op = op_for(2, 2, model=0, p=3.0, eps=1e-2, f=1.0)
    u = cuda(np.zeros(125))
    with pytest.raises(fe.FeodError) as e:
        op.design_grad(u, u)
    assert e.value.code == fe.FEOD_EINVAL
    with pytest.raises(fe.FeodError):
        op.residual(u, out=u)            # aliasing
    with pytest.raises(fe.FeodError):
        op.residual(cuda(np.zeros(10)))  # wrong length
    with pytest.raises(fe.FeodError):
        op.residual(torch.zeros(125, dtype=torch.float32, device="cuda"))
    bad = W.vertices(2, False).copy()
    bad[[0, 1]] = bad[[1, 0]]            # swap two vertices: inverted element
    with pytest.raises(fe.FeodError) as e:
        fe.Operator(2, 2, 2, 1, 2, 0, 2.0, 0.0, 0.0, bad, 63)
    assert e.value.code == fe.FEOD_EINVAL
    with pytest.raises(fe.FeodError) as e:
        fe.Operator(2, 2, 2, 2, 4)
    assert e.value.code == fe.FEOD_EUNSUPPORTED


def test_nonuniform_box_and_dirichlet_subsets():
    """nx != ny != nz, odd face subsets, stored metric on a uniform grid: full parity."""
    import paper_2506_00746_b200 as fe
    for (nx, ny, nz), k, faces, model in (((5, 3, 9), 2, 1 | 8 | 32, 1), ((10, 3, 2), 1, 2 | 4, 0),
                                          ((3, 5, 4), 3, 16, 2)):
        rng = np.random.default_rng(nx)
        rho = rng.uniform(0.1, 1, nx * ny * nz)
        x = np.arange(nx + 1) / nx
        y = np.arange(ny + 1) / ny
        z = np.arange(nz + 1) / nz
        Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
        verts = np.stack([X, Y, Z], -1).reshape(-1, 3) + 0.01 * rng.uniform(-1, 1, ((nx + 1) * (ny + 1) * (nz + 1), 3)) / max(nx, ny, nz)
        pr = O.Problem(nx, ny, nz, k, k + 1, model, 3.0, 1e-2, 0.5, faces, verts, rho)
        N = pr.n_dofs
        u, v, lam = (rng.uniform(-1, 1, N) for _ in range(3))
        for vv in (None, verts):
            op = fe.Operator(nx, ny, nz, k, k + 1, model, 3.0, 1e-2, 0.5, vv, faces, cuda(rho))
            prv = O.Problem(nx, ny, nz, k, k + 1, model, 3.0, 1e-2, 0.5, faces, vv, rho)
            assert rel_l2(host(op.residual(cuda(u))), O.residual(prv, u)) <= 1e-11
            assert rel_l2(host(op.jvp(cuda(u), cuda(v))), O.jvp(prv, u, v)) <= 1e-11
            if model == 2:
                assert rel_l2(host(op.design_grad(cuda(u), cuda(lam))), O.design_grad(prv, u, lam)) <= 1e-11


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_vjp_adjoint_identity_fullsize(name):
    """<w, J v> = <J^T w, v> through the CUDA path alone at BASELINE size, and J^T w
    ignores w's Dirichlet entries (holds at any size; no oracle in the loop)."""
    import paper_2506_00746_b200 as fe
    import torch
    w = W.CONFIGS[name]
    d = W.draw(w)
    rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
    op = fe.from_workload(w, verts=d["verts"], rho=rho)
    rng = np.random.default_rng(77)
    u, v, a = cuda(d["u"]), cuda(d["v"]), cuda(rng.uniform(-1, 1, op.n_dofs))
    Jv, JTa = op.jvp(u, v), op.vjp(u, a)
    lhs, rhs = float(torch.dot(a, Jv)), float(torch.dot(JTa, v))
    scale = float(torch.dot(a.abs(), Jv.abs()) + torch.dot(JTa.abs(), v.abs()))
    assert abs(lhs - rhs) <= 1e-11 * scale
    mask = cuda(W.dirichlet_dofs(w.n, w.k, w.faces).astype(np.float64))
    a2 = a + 5.0 * mask
    assert torch.equal(op.vjp(u, a2), JTa)


def test_two_handles_on_concurrent_streams_are_bitwise_reproducible():
    """Two operators driven concurrently on two CUDA streams (per-handle ticket counters,
    brick epochs and programmatic dependent launches must not interact) give bitwise
    the results of the same calls run one after the other."""
    import torch
    import paper_2506_00746_b200 as fe
    cases = []
    for w, n in ((W.C3, 18), (W.C5, 17)):
        ww = w.resized(n)
        d = W.draw(ww)
        rho = torch.as_tensor(d["rho"]).cuda() if "rho" in d else None
        op = fe.from_workload(ww, verts=d["verts"], rho=rho)
        cases.append((op, cuda(d["u"]), cuda(d["v"])))
    ref = [(op.residual(u).clone(), op.jvp(u, v).clone(), op.vjp(u, v).clone()) for op, u, v in cases]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[], []]
    for _ in range(6):
        for k, (op, u, v) in enumerate(cases):
            with torch.cuda.stream(streams[k]):
                outs[k].append((op.residual(u), op.jvp(u, v), op.vjp(u, v)))
    torch.cuda.synchronize()
    for k in range(2):
        for r, j, t in outs[k]:
            assert torch.equal(r, ref[k][0]) and torch.equal(j, ref[k][1]) and torch.equal(t, ref[k][2])


def test_q6_long_rows_and_odd_boxes():
    """The Q6 tensor-core path on boxes with nx != ny != nz, odd Dirichlet face subsets and
    rows longer than the default shared-memory row buffers of the assembly (nx = 120:
    7 nx x 8 doubles > 48 KB per CTA, the opt-in path): residual, J v, J^T w, the stored
    linearisation and the Jacobi diagonal against the oracle."""
    import paper_2506_00746_b200 as fe
    for (nx, ny, nz), faces, model in (((120, 1, 1), 1 | 2 | 16, 0), ((3, 2, 4), 4 | 32, 1), ((2, 3, 1), 63, 2)):
        rng = np.random.default_rng(nx + ny)
        rho = rng.uniform(0.1, 1, nx * ny * nz)
        pr = O.Problem(nx, ny, nz, 6, 7, model, 3.0, 1e-2, 0.5, faces, None, rho)
        N = pr.n_dofs
        u, v = (rng.uniform(-1, 1, N) for _ in range(2))
        op = fe.Operator(nx, ny, nz, 6, 7, model, 3.0, 1e-2, 0.5, None, faces, cuda(rho))
        assert rel_l2(host(op.residual(cuda(u))), O.residual(pr, u)) <= 1e-11
        assert rel_l2(host(op.jvp(cuda(u), cuda(v))), O.jvp(pr, u, v)) <= 1e-11
        assert rel_l2(host(op.vjp(cuda(u), cuda(v))), O.vjp(pr, u, v)) <= 1e-11
        op.linearize(cuda(u))
        assert rel_l2(host(op.jvp_lin(cuda(v))), O.jvp(pr, u, v)) <= 1e-11
        assert rel_l2(host(op.jacobi_diag()), O.jacobi_diag(pr, u)) <= 1e-11
