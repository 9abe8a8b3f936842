"""The fp64 erfc used by the flux kernels (csrc/common.cuh erfc_exp, coefficients in
csrc/erfc_fit.h from scripts/fit_erfc.py): the same Horner evaluation in the monomial
basis, done here in numpy, against the C library's erfc (math.erfc) over z in [-40, 40]."""
import json
import math
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def erfc_fit(z, K, c):
    a = np.abs(z)
    r = 1.0 / (a + K)
    t = (a - K) * r
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


def test_erfc_fit_accuracy():
    fit = json.load(open(os.path.join(ROOT, "tests", "golden", "erfc_fit.json")))
    z = np.concatenate([np.linspace(-8, 8, 160001), np.linspace(-40, -8, 3201), np.linspace(8, 40, 3201),
                        [0.0, -0.0, 1e-300, -1e-300]])
    got = erfc_fit(z, fit["K"], np.array(fit["coef"]))
    ref = np.array([math.erfc(v) for v in z])
    assert np.max(np.abs(got - ref)) < 4e-15
    # relative accuracy where the half-range moment is small (z >= 0): erfc * e^{z^2} = erfcx
    pos = (z >= 0) & (z < 26)
    assert np.max(np.abs(got[pos] - ref[pos]) / ref[pos]) < 1e-13
