"""CPU checks of the C-ABI boundary: libfeod.so loads, exports every symbol
include/feod.h declares, and rejects bad arguments before touching a GPU."""
import ctypes
import os
import re

import pytest

import paper_2506_00746_b200 as fe
from paper_2506_00746_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return fe.load_library()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "feod.h")).read()
    return sorted(set(re.findall(r"FEOD_API\s+[\w\s\*]+?\b(feod_\w+)\s*\(", text)))


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for s in ("feod_create", "feod_residual", "feod_jvp", "feod_design_grad", "feod_destroy"):
        assert s in syms
    assert set(syms) == set(fe.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for s in header_symbols():
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.feod_version()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True)
    arches = set(re.findall(r"sm_\d+a?", out.stdout))
    assert arches == {"sm_100a"}, arches


def _mesh(nx=2, ny=2, nz=2, faces=63):
    return fe._Mesh(nx, ny, nz, None, faces)


def _create(lib, mesh, order, q, coeffs):
    h = ctypes.c_void_p()
    return lib.feod_create(ctypes.byref(mesh) if mesh is not None else None, order, q,
                           ctypes.byref(coeffs) if coeffs is not None else None, None, ctypes.byref(h))


def test_argument_validation_without_gpu(lib):
    ok = fe._Coeffs(fe.PLAPLACE, 3.0, 1e-2, 1.0, None)
    assert _create(lib, None, 2, 3, ok) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 3, None) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(0, 2, 2), 2, 3, ok) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 0, 1, ok) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 9, 10, ok) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 0, ok) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 5, ok) == fe.FEOD_EUNSUPPORTED
    assert _create(lib, _mesh(), 7, 8, ok) == fe.FEOD_EUNSUPPORTED
    assert _create(lib, _mesh(faces=64), 2, 3, ok) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 3, fe._Coeffs(fe.PLAPLACE, 1.5, 0.0, 1.0, None)) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 3, fe._Coeffs(fe.PLAPLACE, 3.0, -1.0, 1.0, None)) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 3, fe._Coeffs(fe.HEAT_DESIGN, 2.0, 0.0, 1.0, None)) == fe.FEOD_EINVAL
    assert _create(lib, _mesh(), 2, 3, fe._Coeffs(7, 2.0, 0.0, 1.0, None)) == fe.FEOD_EINVAL
    assert b"rho" in lib.feod_last_error() or len(lib.feod_last_error()) > 0
    for fn, nargs in (("feod_residual", 3), ("feod_jvp", 4), ("feod_design_grad", 4), ("feod_destroy", 1)):
        assert getattr(lib, fn)(*([None] * nargs)) == fe.FEOD_EINVAL
    assert lib.feod_element_matrices(None, None, 0, 1, 0, None) == fe.FEOD_EINVAL
    assert lib.feod_apply_host(None, 4, None, None, None) == fe.FEOD_EINVAL
    assert lib.feod_apply_host_batch(None, 4, 2, None, None, None) == fe.FEOD_EINVAL
    assert lib.feod_num_dofs(None) == -1
    assert lib.feod_set_cg_fusion(None, 1) == fe.FEOD_EINVAL
    assert lib.feod_set_cg_graphs(None, 1) == fe.FEOD_EINVAL


def test_operator_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fe.FeodError):
        fe.Operator(2, 2, 2, 2)
