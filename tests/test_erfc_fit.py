"""The fp64 erfc used by the flux kernels (csrc/common.cuh erfc_exp, coefficients in
csrc/erfc_fit.h from scripts/fit_erfc.py): the same Horner evaluation in the monomial
basis, done here in numpy (one Horner chain, and the device's four interleaved chains in t^4),
against the C library's erfc (math.erfc) over z in [-40, 40]."""
import json
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def erfc_fit(z, K, c, split=False):
    a = np.abs(z)
    r = 1.0 / (a + K)
    t = (a - K) * r
    if split:  # common.cuh HGKS_POLY_SPLIT: P = P0(s) + t P1(s) + t^2 P2(s) + t^3 P3(s), s = t^4
        s4 = (t * t) * (t * t)
        Pi = []
        for i in range(4):
            top = len(c) - 1 - ((len(c) - 1 - i) % 4)
            p = np.full_like(t, c[top])
            for k in range(top - 4, -1, -4):
                p = p * s4 + c[k]
            Pi.append(p)
        P = ((Pi[3] * t + Pi[2]) * t + Pi[1]) * t + Pi[0]
    else:
        P = np.zeros_like(t)
        for ck in c[::-1]:
            P = P * t + ck
    v = P * r * np.exp(-z * z)
    return np.where(z >= 0, v, 2.0 - v)


def test_header_matches_fit_record():
    fit = json.load(open(os.path.join(ROOT, "tests", "golden", "erfc_fit.json")))
    h = open(os.path.join(ROOT, "paper_2407_00656_b200", "csrc", "erfc_fit.h")).read()
    assert float(re.search(r"#define HGKS_ERFC_K (\S+)", h).group(1)) == fit["K"]
    coef = [float(v) for v in re.findall(r"^\s+(-?[0-9.e+-]+),? \\$", h, re.M)]
    assert coef == fit["coef"]


@pytest.mark.parametrize("split", [False, True])
def test_erfc_fit_accuracy(split):
    fit = json.load(open(os.path.join(ROOT, "tests", "golden", "erfc_fit.json")))
    z = np.concatenate([np.linspace(-8, 8, 160001), np.linspace(-40, -8, 3201), np.linspace(8, 40, 3201),
                        [0.0, -0.0, 1e-300, -1e-300]])
    got = erfc_fit(z, fit["K"], np.array(fit["coef"]), split)
    ref = np.array([math.erfc(v) for v in z])
    assert np.max(np.abs(got - ref)) < 4e-15
    # relative accuracy where the half-range moment is small (z >= 0): erfc * e^{z^2} = erfcx
    pos = (z >= 0) & (z < 26)
    assert np.max(np.abs(got[pos] - ref[pos]) / ref[pos]) < 1e-13
