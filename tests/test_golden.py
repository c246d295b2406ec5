"""The oracle against the golden fixtures of tests/golden/ (closed forms and hand-worked
values, each cited in its file header)."""

import os

import numpy as np
import pytest

import scinputs
from oracle import ari, chebyshev, laplacian

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.loadtxt(os.path.join(GOLDEN, name), comments="#", ndmin=2)


@pytest.mark.parametrize("name,maker", [
    ("ring8_spectrum.txt", lambda: scinputs.ring(8)),
    ("ring13_spectrum.txt", lambda: scinputs.ring(13)),
    ("path3_spectrum.txt", lambda: scinputs.path(3)),
    ("path10_spectrum.txt", lambda: scinputs.path(10)),
])
def test_laplacian_spectrum_golden(name, maker):
    want = load(name)[:, 0]
    got = np.linalg.eigvalsh(laplacian.laplacian_dense(maker()))
    assert np.allclose(got, want, atol=1e-12)


def test_cheb_coefficients_golden():
    tab = load("cheb_step_half.txt")
    c = chebyshev.lowpass_coeffs(0.5 * 7.3, 7.3, int(tab[-1, 0]))
    assert np.allclose(c, tab[:, 1], atol=1e-15)


def test_ari_golden():
    for line in open(os.path.join(GOLDEN, "ari_hand.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v, a, b = line.split(";")
        a = np.array(a.split(), dtype=np.int64)
        b = np.array(b.split(), dtype=np.int64)
        assert ari.ari(a, b) == pytest.approx(float(v), abs=1e-15)
