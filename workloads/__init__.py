"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NO arithmetic of the method (no basis, no quadrature, no
flux): only the input recipe of SURVEY.md §8(d) / DESIGN.md "Input recipe":

* the five workloads of BASELINE.json ``configs`` (C1..C5) as plain data;
* the mesh vertex array, uniform or with the sinusoidal node perturbation
  (BASELINE.json configs[1..2]; reading A6 in DESIGN.md);
* the seeded draws u, v, lambda, rho (reading A9: ``numpy.random.default_rng``
  with the config index as seed, full-length draws in a fixed order, then the
  Dirichlet entries set to zero).

The paper (§2) meshes "a cube ... using 200K elements" and
names no public dataset; these generators stand in for that workload.

Both sides consume the arrays produced here; neither side's results feed back.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# Face bits for the Dirichlet boundary (include/feod.h FEOD_FACE_*).
FACE_X0, FACE_X1, FACE_Y0, FACE_Y1, FACE_Z0, FACE_Z1 = 1, 2, 4, 8, 16, 32
ALL_FACES = 63

PLAPLACE, NLDIFF, HEAT = 0, 1, 2
MODEL_NAMES = {PLAPLACE: "p-Laplacian", NLDIFF: "nonlinear diffusion", HEAT: "heat design"}


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    n: int              # hex elements per axis (unit cube)
    k: int              # polynomial order Q_k
    q: int              # Gauss points per axis
    model: int
    p: float = 2.0
    eps: float = 0.0
    f: float = 1.0
    faces: int = ALL_FACES
    perturbed: bool = False
    seed: int = 0
    u_scale: float = 1.0   # u ~ u_scale * U[-1,1]

    @property
    def n_dofs(self) -> int:
        return (self.k * self.n + 1) ** 3

    @property
    def n_elems(self) -> int:
        return self.n ** 3

    def resized(self, n: int) -> "Workload":
        """Same recipe on an n^3 mesh (reduced-size parity cases)."""
        return dataclasses.replace(self, n=n, name=f"{self.name}@n{n}")


# BASELINE.json configs[0..4]; readings A8 (C2/C4 BCs and f) and A9 (seeds) in DESIGN.md.
C1 = Workload("C1", n=4, k=2, q=3, model=PLAPLACE, p=3.0, eps=1e-2, f=1.0, seed=1)
C2 = Workload("C2", n=128, k=1, q=2, model=PLAPLACE, p=4.0, eps=1e-3, f=1.0, perturbed=True, seed=2)
C3 = Workload("C3", n=64, k=3, q=4, model=NLDIFF, f=1.0, perturbed=True, seed=3, u_scale=0.5)
C4 = Workload("C4", n=32, k=6, q=7, model=PLAPLACE, p=3.0, eps=1e-2, f=1.0, seed=4)
C5 = Workload("C5", n=96, k=2, q=3, model=HEAT, f=1.0, faces=FACE_X0, seed=5)
CONFIGS = {w.name: w for w in (C1, C2, C3, C4, C5)}


def vertices(n: int, perturbed: bool) -> np.ndarray:
    """(n+1)^3 x 3 vertex coordinates of the unit cube, x-fastest.

    Perturbed (reading A6): every vertex moves by
    delta = 0.1 h sin(2 pi x) sin(2 pi y) sin(2 pi z) in each coordinate, with
    delta forced to exactly 0 on boundary vertices.
    """
    h = 1.0 / n
    t = np.arange(n + 1, dtype=np.float64) / n
    z, y, x = np.meshgrid(t, t, t, indexing="ij")     # x fastest in C order
    X = np.stack([x, y, z], axis=-1).reshape(-1, 3).copy()
    if perturbed:
        s = np.sin(2 * np.pi * t)
        s[0] = 0.0
        s[-1] = 0.0
        d = 0.1 * h * (s[None, None, :] * s[None, :, None] * s[:, None, None])
        X += d.reshape(-1, 1)
    return X


def dirichlet_dofs(n: int, k: int, faces: int) -> np.ndarray:
    """Boolean mask over the (k n + 1)^3 lexicographic DOFs lying on flagged faces."""
    m = k * n + 1
    i = np.arange(m)
    K, J, I = np.meshgrid(i, i, i, indexing="ij")
    mask = np.zeros((m, m, m), dtype=bool)
    if faces & FACE_X0: mask |= I == 0
    if faces & FACE_X1: mask |= I == m - 1
    if faces & FACE_Y0: mask |= J == 0
    if faces & FACE_Y1: mask |= J == m - 1
    if faces & FACE_Z0: mask |= K == 0
    if faces & FACE_Z1: mask |= K == m - 1
    return mask.reshape(-1)


def draw(w: Workload) -> dict:
    """Seeded inputs in the fixed order of SURVEY.md §8(d).

    C1-C4: u, v ~ U[-1,1] (u scaled by u_scale); C5: rho ~ U[0.1,1] (E), then u,
    lambda, then a 4th draw v for the Q2 JVP datapoint. Dirichlet entries of
    u, v, lambda are zeroed after drawing.
    """
    rng = np.random.default_rng(w.seed)
    N, E = w.n_dofs, w.n_elems
    out = {}
    if w.model == HEAT:
        out["rho"] = rng.uniform(0.1, 1.0, E)
        out["u"] = rng.uniform(-1.0, 1.0, N)
        out["lam"] = rng.uniform(-1.0, 1.0, N)
        out["v"] = rng.uniform(-1.0, 1.0, N)
    else:
        out["u"] = w.u_scale * rng.uniform(-1.0, 1.0, N)
        out["v"] = rng.uniform(-1.0, 1.0, N)
    mask = dirichlet_dofs(w.n, w.k, w.faces)
    for key in ("u", "v", "lam"):
        if key in out:
            out[key][mask] = 0.0
    out["verts"] = vertices(w.n, w.perturbed) if w.perturbed else None
    return out


def node_coords(n: int, k: int, perturbed: bool, gll01) -> np.ndarray:
    """Physical coordinates of all DOF nodes (needed only by the patch test, A7).

    ``gll01`` are the k+1 reference node positions on [0,1], supplied by the
    caller (each side brings its own); the trilinear vertex interpolation here
    is input construction (the exact linear field u = a.x + c at the nodes).
    """
    X = vertices(n, perturbed).reshape(n + 1, n + 1, n + 1, 3)
    m = k * n + 1
    out = np.empty((m, m, m, 3))
    gll01 = np.asarray(gll01, dtype=np.float64)
    for ez in range(n):
        for ey in range(n):
            for ex in range(n):
                for c in range(k + 1):
                    for b in range(k + 1):
                        for a in range(k + 1):
                            xi, eta, zeta = gll01[a], gll01[b], gll01[c]
                            acc = np.zeros(3)
                            for dz in (0, 1):
                                for dy in (0, 1):
                                    for dx in (0, 1):
                                        wgt = ((xi if dx else 1 - xi) * (eta if dy else 1 - eta)
                                               * (zeta if dz else 1 - zeta))
                                        acc += wgt * X[ez + dz, ey + dy, ex + dx]
                            out[k * ez + c, k * ey + b, k * ex + a] = acc
    return out.reshape(-1, 3)
