"""feod-b200: Python binding of libfeod (include/feod.h).

Argument marshalling only: every step of the FEOD path (gather, sum-factorised
interpolation, dual-number flux, transposed interpolation, atomic-free scatter,
Dirichlet rows, design reduction, Newton-CG BLAS-1) runs in libfeod's sm_100a
kernels. PyTorch provides device memory and the current CUDA stream. There is
no CPU fallback: if libfeod.so is missing or CUDA is unavailable, constructing
an Operator raises.

    op = Operator(nx, ny, nz, order=3, qorder=4, model=NLDIFF, f=1.0,
                  vertices=verts_numpy_or_None, dirichlet_faces=63)
    r  = op.residual(u)            # PAPER.md Eq. 1 (line 155)
    Jv = op.jvp(u, v)              # PAPER.md Eq. 2 (line 160)
    g  = op.design_grad(u, lam)    # PAPER.md line 199 (HEAT_DESIGN)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FEOD_LIB") or os.path.join(HERE, "libfeod.so")   # FEOD_LIB: experiment builds

PLAPLACE, NLDIFF, HEAT_DESIGN = 0, 1, 2
FEOD_OK, FEOD_EINVAL, FEOD_EUNSUPPORTED, FEOD_ENOMEM, FEOD_ECUDA = 0, -1, -2, -3, -4

# every symbol include/feod.h declares (checked by tests/test_abi.py)
EXPORTS = ("feod_create", "feod_destroy", "feod_set_stream", "feod_set_rho", "feod_num_dofs", "feod_num_elems",
           "feod_residual", "feod_jvp", "feod_jvp_res", "feod_vjp", "feod_linearize", "feod_jvp_lin",
           "feod_set_newton_linearization", "feod_brick_shape", "feod_jacobi_diag", "feod_adjoint_solve", "feod_element_matrices",
           "feod_design_grad", "feod_res_design_grad", "feod_apply_host", "feod_apply_host_batch", "feod_newton_cg",
           "feod_set_cg_graphs", "feod_set_cg_fusion", "feod_cg_graph_launches",
           "feod_dot", "feod_profile_next", "feod_last_error", "feod_version")


class FeodError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libfeod error {code}: {msg}")
        self.code = code


class _Mesh(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("vertices", ctypes.POINTER(ctypes.c_double)), ("dirichlet_faces", ctypes.c_uint32)]


class _Coeffs(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int), ("p", ctypes.c_double), ("eps", ctypes.c_double), ("f", ctypes.c_double),
                ("rho", ctypes.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libfeod.so (raises if absent: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FeodError(FEOD_EUNSUPPORTED, f"{path} not built; run python -m paper_2506_00746_b200.build")
    lib = ctypes.CDLL(path)
    vp, dp, i64 = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64
    lib.feod_create.argtypes = [ctypes.POINTER(_Mesh), ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Coeffs), vp,
                                ctypes.POINTER(vp)]
    lib.feod_destroy.argtypes = [vp]
    lib.feod_set_stream.argtypes = [vp, vp]
    lib.feod_set_rho.argtypes = [vp, dp]
    lib.feod_num_dofs.argtypes = [vp]
    lib.feod_num_dofs.restype = i64
    lib.feod_num_elems.argtypes = [vp]
    lib.feod_num_elems.restype = i64
    lib.feod_brick_shape.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int)]
    lib.feod_residual.argtypes = [vp, dp, dp]
    lib.feod_jvp.argtypes = [vp, dp, dp, dp]
    lib.feod_jvp_res.argtypes = [vp, dp, dp, dp, dp]
    lib.feod_design_grad.argtypes = [vp, dp, dp, dp]
    lib.feod_res_design_grad.argtypes = [vp, dp, dp, dp, dp]
    lib.feod_vjp.argtypes = [vp, dp, dp, dp]
    lib.feod_linearize.argtypes = [vp, dp, dp]
    lib.feod_jvp_lin.argtypes = [vp, dp, dp]
    lib.feod_set_newton_linearization.argtypes = [vp, ctypes.c_int]
    lib.feod_jacobi_diag.argtypes = [vp, dp]
    lib.feod_element_matrices.argtypes = [vp, dp, i64, i64, ctypes.c_int, dp]
    lib.feod_adjoint_solve.argtypes = [vp, dp, dp, dp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.feod_apply_host.argtypes = [vp, ctypes.c_int, dp, dp, dp]
    lib.feod_apply_host_batch.argtypes = [vp, ctypes.c_int, i64, vp, vp, vp]
    lib.feod_newton_cg.argtypes = [vp, dp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    lib.feod_set_cg_graphs.argtypes = [vp, ctypes.c_int]
    lib.feod_set_cg_fusion.argtypes = [vp, ctypes.c_int]
    lib.feod_cg_graph_launches.argtypes = [vp]
    lib.feod_cg_graph_launches.restype = i64
    lib.feod_dot.argtypes = [vp, dp, dp, i64, dp]
    lib.feod_profile_next.argtypes = [vp, vp, vp]
    lib.feod_last_error.restype = ctypes.c_char_p
    lib.feod_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(rc):
    if rc != FEOD_OK:
        raise FeodError(rc, _lib.feod_last_error().decode())


class Operator:
    """Handle on one FEOD operator (feod_create ... feod_destroy)."""

    def __init__(self, nx, ny, nz, order, qorder=None, model=PLAPLACE, p=2.0, eps=0.0, f=0.0,
                 vertices=None, dirichlet_faces=63, rho=None, device=None):
        import torch
        if not torch.cuda.is_available():
            raise FeodError(FEOD_ECUDA, "CUDA device required (no CPU fallback)")
        self._torch = torch
        self.lib = load_library()
        self.device = torch.device(device or "cuda")
        self.nx, self.ny, self.nz, self.order = int(nx), int(ny), int(nz), int(order)
        self.qorder = int(qorder if qorder is not None else order + 1)
        self.model = int(model)
        self._rho = None
        if rho is not None:
            self._rho = self._dev(rho, self.nx * self.ny * self.nz, "rho")
        mesh = _Mesh(self.nx, self.ny, self.nz, None, int(dirichlet_faces))
        if vertices is not None:
            self._verts = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64))
            if self._verts.size != (self.nx + 1) * (self.ny + 1) * (self.nz + 1) * 3:
                raise FeodError(FEOD_EINVAL, "vertices must have (nx+1)(ny+1)(nz+1) x 3 entries")
            mesh.vertices = self._verts.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        coeffs = _Coeffs(self.model, float(p), float(eps), float(f),
                         self._rho.data_ptr() if self._rho is not None else None)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(self.lib.feod_create(ctypes.byref(mesh), self.order, self.qorder, ctypes.byref(coeffs),
                                        self._stream(), ctypes.byref(h)))
        self.h = h
        self.n_dofs = int(self.lib.feod_num_dofs(h))
        self.n_elems = int(self.lib.feod_num_elems(h))

    # ------------------------------------------------------------------ helpers
    def _stream(self):
        return ctypes.c_void_p(self._torch.cuda.current_stream(self.device).cuda_stream)

    def _dev(self, x, n, name):
        t = self._torch
        if not isinstance(x, t.Tensor):
            x = t.as_tensor(np.asarray(x, dtype=np.float64))
        if x.dtype != t.float64:
            raise FeodError(FEOD_EINVAL, f"{name} must be float64")
        if x.numel() != n:
            raise FeodError(FEOD_EINVAL, f"{name} must have {n} entries, got {x.numel()}")
        if x.device.type != "cuda":
            x = x.to(self.device)
        elif x.device != self._cuda_device():
            raise FeodError(FEOD_EINVAL, f"{name} lives on {x.device}, the operator on {self._cuda_device()}")
        return x.contiguous().view(-1)

    def _cuda_device(self):
        t = self._torch
        d = self.device
        return d if d.index is not None else t.device("cuda", t.cuda.current_device())

    def _out(self, out, n, name="out", shape=None):
        """Validate a caller-supplied output: float64, exactly n entries, this device, contiguous."""
        t = self._torch
        if out is None:
            return t.empty(shape if shape is not None else (n,), dtype=t.float64, device=self._cuda_device())
        if not isinstance(out, t.Tensor) or out.dtype != t.float64 or out.numel() != n:
            raise FeodError(FEOD_EINVAL, f"{name} must be a float64 tensor with {n} entries")
        if out.device != self._cuda_device() or not out.is_contiguous():
            raise FeodError(FEOD_EINVAL, f"{name} must be contiguous on {self._cuda_device()}")
        return out

    def _sync_stream(self):
        _check(self.lib.feod_set_stream(self.h, self._stream()))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.feod_destroy(h)
            self.h = None

    # ------------------------------------------------------------------ operations
    def residual(self, u, out=None):
        u = self._dev(u, self.n_dofs, "u")
        r = self._out(out, self.n_dofs)
        self._sync_stream()
        _check(self.lib.feod_residual(self.h, u.data_ptr(), r.data_ptr()))
        return r

    def jvp(self, u, v, out=None):
        u, v = self._dev(u, self.n_dofs, "u"), self._dev(v, self.n_dofs, "v")
        Jv = self._out(out, self.n_dofs)
        self._sync_stream()
        _check(self.lib.feod_jvp(self.h, u.data_ptr(), v.data_ptr(), Jv.data_ptr()))
        return Jv

    def jvp_res(self, u, v, out=None):
        """(F(u), J(u) v) from one dual pass (feod_jvp_res); out = (r, Jv) optional."""
        u, v = self._dev(u, self.n_dofs, "u"), self._dev(v, self.n_dofs, "v")
        r, Jv = (None, None) if out is None else out
        r, Jv = self._out(r, self.n_dofs, "out[0]"), self._out(Jv, self.n_dofs, "out[1]")
        self._sync_stream()
        _check(self.lib.feod_jvp_res(self.h, u.data_ptr(), v.data_ptr(), r.data_ptr(), Jv.data_ptr()))
        return r, Jv

    def vjp(self, u, w, out=None):
        """J(u)^T w (feod_vjp): w's Dirichlet entries ignored, every row kept."""
        u, w = self._dev(u, self.n_dofs, "u"), self._dev(w, self.n_dofs, "w")
        JTw = self._out(out, self.n_dofs)
        self._sync_stream()
        _check(self.lib.feod_vjp(self.h, u.data_ptr(), w.data_ptr(), JTw.data_ptr()))
        return JTw

    def linearize(self, u, out=None):
        """r = F(u), and store the pointwise linearisation at u (feod_linearize)."""
        u = self._dev(u, self.n_dofs, "u")
        r = self._out(out, self.n_dofs)
        self._sync_stream()
        _check(self.lib.feod_linearize(self.h, u.data_ptr(), r.data_ptr()))
        return r

    def jvp_lin(self, v, out=None):
        """J(u) v at the u of the last linearize() (feod_jvp_lin)."""
        v = self._dev(v, self.n_dofs, "v")
        Jv = self._out(out, self.n_dofs)
        self._sync_stream()
        _check(self.lib.feod_jvp_lin(self.h, v.data_ptr(), Jv.data_ptr()))
        return Jv

    def adjoint_solve(self, u, rhs, iters=50):
        """lambda from `iters` BiCGStab iterations on P^T J(u)^T lambda = P^T rhs
        (feod_adjoint_solve); returns (lambda, residual-norm history)."""
        u, rhs = self._dev(u, self.n_dofs, "u"), self._dev(rhs, self.n_dofs, "rhs")
        lam = self._torch.empty_like(u)
        norms = (ctypes.c_double * (iters + 1))()
        self._sync_stream()
        _check(self.lib.feod_adjoint_solve(self.h, u.data_ptr(), rhs.data_ptr(), lam.data_ptr(), int(iters), norms))
        return lam, list(norms)

    def set_newton_linearization(self, stored):
        """0/False matrix-free, 1/True stored linearisation, 2 stored + Jacobi PCG."""
        _check(self.lib.feod_set_newton_linearization(self.h, int(stored)))

    def element_matrices(self, u, e0=0, ne=None, elm=False, out=None):
        """K_e = B^T J_D B for elements e0 .. e0+ne-1 (feod_element_matrices), shape (ne, nd^3, nd^3)."""
        u = self._dev(u, self.n_dofs, "u")
        ne = self.n_elems - e0 if ne is None else ne
        nn = (self.order + 1) ** 3
        if ne < 0 or e0 < 0 or e0 + ne > self.n_elems:
            raise FeodError(FEOD_EINVAL, "element range out of bounds")
        Ke = self._out(out, ne * nn * nn, shape=(ne, nn, nn))
        self._sync_stream()
        _check(self.lib.feod_element_matrices(self.h, u.data_ptr(), int(e0), int(ne), 1 if elm else 0, Ke.data_ptr()))
        return Ke

    def jacobi_diag(self, out=None):
        """Diagonal of J at the last linearize() (feod_jacobi_diag)."""
        d = self._out(out, self.n_dofs)
        self._sync_stream()
        _check(self.lib.feod_jacobi_diag(self.h, d.data_ptr()))
        return d

    def design_grad(self, u, lam, out=None):
        u, lam = self._dev(u, self.n_dofs, "u"), self._dev(lam, self.n_dofs, "lam")
        g = self._out(out, self.n_elems)
        self._sync_stream()
        _check(self.lib.feod_design_grad(self.h, u.data_ptr(), lam.data_ptr(), g.data_ptr()))
        return g

    def brick_shape(self):
        """(bx, by, bz): elements per brick of the operator kernels (feod_brick_shape)."""
        b = [ctypes.c_int() for _ in range(3)]
        _check(self.lib.feod_brick_shape(self.h, *[ctypes.byref(x) for x in b]))
        return tuple(x.value for x in b)

    def res_design_grad(self, u, lam, out=None):
        """(r, g): F(u) and the design gradient from one dual pass (feod_res_design_grad)."""
        u, lam = self._dev(u, self.n_dofs, "u"), self._dev(lam, self.n_dofs, "lam")
        r, g = (None, None) if out is None else out
        r, g = self._out(r, self.n_dofs, "out[0]"), self._out(g, self.n_elems, "out[1]")
        self._sync_stream()
        _check(self.lib.feod_res_design_grad(self.h, u.data_ptr(), lam.data_ptr(), r.data_ptr(), g.data_ptr()))
        return r, g

    def set_rho(self, rho):
        self._rho = self._dev(rho, self.n_elems, "rho")
        _check(self.lib.feod_set_rho(self.h, self._rho.data_ptr()))

    def apply_host(self, op, in0, in1=None, out=None):
        """Host-buffer path (feod_apply_host): H2D, compute, D2H, synchronise."""
        t = self._torch
        n_out = self.n_elems if op == 2 else (2 * self.n_dofs if op == 4 else self.n_dofs)
        a = in0 if isinstance(in0, t.Tensor) else t.as_tensor(np.asarray(in0, np.float64))
        b = None if in1 is None else (in1 if isinstance(in1, t.Tensor) else t.as_tensor(np.asarray(in1, np.float64)))
        for x, name in ((a, "in0"), (b, "in1")):
            if x is not None and (x.device.type != "cpu" or x.dtype != t.float64 or x.numel() != self.n_dofs):
                raise FeodError(FEOD_EINVAL, f"{name}: host float64 vector of length N expected")
        if out is None:
            res = t.empty(n_out, dtype=t.float64, pin_memory=True)
        else:
            res = out
            if (not isinstance(res, t.Tensor) or res.device.type != "cpu" or res.dtype != t.float64
                    or res.numel() != n_out or not res.is_contiguous()):
                raise FeodError(FEOD_EINVAL, f"out: contiguous host float64 tensor of {n_out} entries expected")
        self._sync_stream()
        _check(self.lib.feod_apply_host(self.h, int(op), a.data_ptr(), 0 if b is None else b.data_ptr(),
                                        res.data_ptr()))
        return res

    def apply_host_batch(self, op, ins0, ins1=None, outs=None):
        """A stream of host-buffer problems (feod_apply_host_batch): step b maps ins0[b]
        (and ins1[b]) to outs[b]; uploads of step b+1 overlap step b's operator and
        downloads. Returns the list of output tensors."""
        t = self._torch
        nb = len(ins0)
        n_out = self.n_elems if op == 2 else (2 * self.n_dofs if op == 4 else self.n_dofs)
        if op != 0 and (ins1 is None or len(ins1) != nb):
            raise FeodError(FEOD_EINVAL, "ins1: one host vector per step expected")
        for lst, name in ((ins0, "ins0"), (ins1 if op != 0 else (), "ins1")):
            for x in lst:
                if (not isinstance(x, t.Tensor) or x.device.type != "cpu" or x.dtype != t.float64
                        or x.numel() != self.n_dofs or not x.is_contiguous()):
                    raise FeodError(FEOD_EINVAL, f"{name}: contiguous host float64 tensors of length N expected")
        if outs is None:
            outs = [t.empty(n_out, dtype=t.float64, pin_memory=True) for _ in range(nb)]
        if len(outs) != nb:
            raise FeodError(FEOD_EINVAL, "outs: one host buffer per step expected")
        for o in outs:
            if (not isinstance(o, t.Tensor) or o.device.type != "cpu" or o.dtype != t.float64
                    or o.numel() != n_out or not o.is_contiguous()):
                raise FeodError(FEOD_EINVAL, f"outs: contiguous host float64 tensors of {n_out} entries expected")
        P = ctypes.c_void_p * max(nb, 1)
        a = P(*[x.data_ptr() for x in ins0])
        b = P(*[x.data_ptr() for x in ins1]) if op != 0 else None
        o = P(*[x.data_ptr() for x in outs])
        self._sync_stream()
        _check(self.lib.feod_apply_host_batch(self.h, int(op), nb, a, b, o))
        return outs

    def newton_cg(self, u0, newton_steps=5, cg_iters=20):
        u = self._dev(u0, self.n_dofs, "u0").clone()
        norms = (ctypes.c_double * (newton_steps + 1))()
        self._sync_stream()
        _check(self.lib.feod_newton_cg(self.h, u.data_ptr(), int(newton_steps), int(cg_iters), norms))
        return u, list(norms)

    def set_cg_graphs(self, enable):
        """Capture the CG iterations of feod_newton_cg as a CUDA graph (default on)."""
        _check(self.lib.feod_set_cg_graphs(self.h, 1 if enable else 0))

    def set_cg_fusion(self, enable):
        """Fuse the CG update into the Q6 tensor-core operator call of feod_newton_cg (default on)."""
        _check(self.lib.feod_set_cg_fusion(self.h, 1 if enable else 0))

    def cg_graph_launches(self):
        return int(self.lib.feod_cg_graph_launches(self.h))

    def profile_next(self, ev_begin, ev_end):
        """Time the fused kernel of the next call with two torch.cuda.Event(enable_timing=True)."""
        _check(self.lib.feod_profile_next(self.h, ctypes.c_void_p(ev_begin.cuda_event),
                                          ctypes.c_void_p(ev_end.cuda_event)))

    def dot(self, x, y):
        if x.numel() != y.numel():
            raise FeodError(FEOD_EINVAL, f"dot: x has {x.numel()} entries, y {y.numel()}")
        x, y = self._dev(x, x.numel(), "x"), self._dev(y, x.numel(), "y")
        out = self._torch.empty(1, dtype=self._torch.float64, device=self.device)
        self._sync_stream()
        _check(self.lib.feod_dot(self.h, x.data_ptr(), y.data_ptr(), x.numel(), out.data_ptr()))
        return out


def from_workload(w, verts=None, rho=None, device=None) -> Operator:
    """Operator for a workloads.Workload (n^3 unit cube)."""
    return Operator(w.n, w.n, w.n, w.k, w.q, w.model, w.p, w.eps, w.f, verts, w.faces, rho, device)
