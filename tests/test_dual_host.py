"""T15: dual<double> (paper_2506_00746_b200/csrc/dual.cuh) compiled for the host
with g++; values against closed forms and central finite differences."""
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def out(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("dual") / "dual_host_test")
    subprocess.run(["g++", "-O1", "-std=c++17", os.path.join(HERE, "dual_host_test.cpp"), "-o", exe], check=True)
    res = subprocess.run([exe], capture_output=True, text=True, check=True)
    return {ln.split()[0]: (float(ln.split()[1]), float(ln.split()[2])) for ln in res.stdout.splitlines()}


def fd(f, x, h=1e-6):
    return (f(x + h) - f(x - h)) / (2 * h)


def test_closed_forms(out):
    assert out["square"] == (9.0, 6.0)
    assert out["identity"] == (5.0, 1.0)
    assert out["pow1"] == (1.3, 1.0)
    assert out["pow0"] == (1.0, 0.0)


def test_rules_vs_fd(out):
    # a/b with a = 0.7 + 0.3 t, b = -1.9 + 2.5 t
    g = lambda t: (0.7 + 0.3 * t) / (-1.9 + 2.5 * t)
    assert abs(out["div"][0] - g(0)) < 1e-15
    assert abs(out["div"][1] - fd(g, 0.0)) < 1e-8
    assert abs(out["sqrt"][0] - np.sqrt(2)) < 1e-15
    assert abs(out["sqrt"][1] - 0.5 / np.sqrt(2)) < 1e-15
    assert abs(out["pow075"][0] - 1.3 ** 0.75) < 1e-15
    assert abs(out["pow075"][1] - fd(lambda x: x ** 0.75, 1.3)) < 1e-8
    assert abs(out["pow05"][0] - np.sqrt(1.3)) < 1e-15
    assert abs(out["pow05"][1] - fd(np.sqrt, 1.3)) < 1e-8
    f = lambda x: x ** 3 / (x * x + 1)
    assert abs(out["seed1"][1] - fd(f, 0.8)) < 1e-8
    assert abs(out["mixed"][0] - (2 - 1.2 + 0.025)) < 1e-15
    assert abs(out["mixed"][1] - (-3.0 - 0.5)) < 1e-15


def test_seeding_linearity(out):
    assert abs(out["seed25"][1] - 2.5 * out["seed1"][1]) < 1e-15
    assert out["seed25"][0] == out["seed1"][0]
