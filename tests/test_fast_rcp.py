"""rcp_pos / rsqrt_pos (csrc/common.cuh): the MUFU estimates (relative error below 2^-22 for
the fp64 rcp / rsqrt approximations) refined by two Newton steps reach double precision.
Evaluated here in numpy from a worst-case perturbed start, with the device's update formulas."""
import numpy as np


def test_two_newton_steps_reach_double_precision():
    rng = np.random.default_rng(3)
    x = np.exp(rng.uniform(np.log(1e-300), np.log(1e300), 200001))
    for d in (2.0 ** -22, -(2.0 ** -22)):
        y = (1.0 / x) * (1.0 + d)  # reciprocal estimate
        for _ in range(2):
            e = 1.0 - x * y
            y = y + y * e
        assert np.max(np.abs(y * x - 1.0)) < 4e-16
        z = (1.0 / np.sqrt(x)) * (1.0 + d)  # rsqrt estimate
        hx = 0.5 * x
        for _ in range(2):
            z = z * (1.5 - hx * z * z)
        assert np.max(np.abs(z * np.sqrt(x) - 1.0)) < 6e-16
