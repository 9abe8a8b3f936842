"""exp_neg (csrc/common.cuh), the fp64 exp of non-positive arguments in the flux
kernels: the same reduction and series evaluated here in numpy (without fused
multiply-adds, so slightly less exact than the device) against numpy's exp."""
import math
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def device_constants():
    """ln2 split and the even / odd Horner coefficients (kExpEven / kExpOdd) of the split branch."""
    src = open(os.path.join(ROOT, "paper_2407_00656_b200", "csrc", "common.cuh")).read()
    body = src[src.index("double exp_neg(double x)"):src.index("float exp_neg(float x)")]
    lo, hi = [float(v) for v in re.findall(r"fma\(-k, ([0-9.e+-]+)", body)]
    arr = lambda name: [float(v) for v in re.search(name + r"\[\d+\] = \{([^}]*)\}", src).group(1).replace("\n", " ").split(",")]
    ce, co = arr("kExpEven"), arr("kExpOdd")
    return lo, hi, ce, co


def test_series_coefficients_are_inverse_factorials():
    _, _, ce, co = device_constants()
    assert len(ce) == 7 and len(co) == 6
    for j, c in enumerate(ce):
        assert c == 1.0 / math.factorial(12 - 2 * j)
    for j, c in enumerate(co):
        assert c == 1.0 / math.factorial(11 - 2 * j)


def test_exp_neg_accuracy():
    ln2_lo, ln2_hi, ce, co = device_constants()
    assert ln2_hi + ln2_lo == math.log(2.0) or abs(ln2_hi + ln2_lo - math.log(2.0)) < 1e-17
    x = np.concatenate([-np.logspace(-20, np.log10(700), 100001), np.linspace(-700, 0, 100001), [0.0, -0.0]])
    k = np.rint(np.maximum(x, -708.0) * 1.4426950408889634)
    r = (x - k * ln2_hi) - k * ln2_lo
    r2 = r * r
    pe = np.full_like(r, ce[0])
    for c in ce[1:]:
        pe = pe * r2 + c
    po = np.full_like(r, co[0])
    for c in co[1:]:
        po = po * r2 + c
    p = po * r + pe
    got = np.ldexp(p, k.astype(int))
    assert np.max(np.abs(got - np.exp(x)) / np.exp(x)) < 5e-16
