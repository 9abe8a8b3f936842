"""Post-processing of the sphere workload (scripts/sphere_wake.py):
the wake length and separation angle readers recover values planted in
synthetic axisymmetric fields on the real cubed-sphere mesh."""
import os, sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import sphere_wake as SW  # noqa: E402
from paper_2407_00656_b200 import workloads as W  # noqa: E402


def planted_field(mi, L_true, theta_true):
    """rho = 1; axial velocity reversed inside the bubble 0.5 < x < 0.5 + L (near the
    axis); near the wall u_alpha = cos-like profile changing sign at theta_true."""
    c = SW.cell_centroids(mi)
    r = np.linalg.norm(c, axis=1)
    Q = np.zeros((mi.n_cells, 5))
    Q[:, 0] = 1.0
    x_end = 0.5 + L_true
    # axial: linear in x, zero at x_end, negative before
    u = np.where(c[:, 0] > 0.5, (c[:, 0] - x_end), 1.0)
    alpha = np.arccos(np.clip(-c[:, 0] / r, -1, 1))
    ua = np.sin(alpha) * np.sign(np.radians(theta_true) - alpha) * np.abs(alpha - np.radians(theta_true))
    perp = np.stack([np.zeros_like(r), c[:, 1], c[:, 2]], 1)
    perp /= np.maximum(np.linalg.norm(perp, axis=1), 1e-300)[:, None]
    ea = np.stack([np.sin(alpha), np.cos(alpha) * perp[:, 1], np.cos(alpha) * perp[:, 2]], 1)
    vel = ua[:, None] * ea
    near_axis = (c[:, 0] > 0) & (np.hypot(c[:, 1], c[:, 2]) < 0.3 * r)
    vel[near_axis] = 0.0
    vel[near_axis, 0] = u[near_axis]
    Q[:, 1:4] = vel
    Q[:, 4] = 2.5
    return Q


def test_planted_wake_and_separation():
    N = 9
    mi = W.sphere_shell(N)
    nr = 2 * N
    Q = planted_field(mi, L_true=0.9, theta_true=128.0)
    L = SW.wake_length(mi, Q, nr)
    # samples are cell centroids along the axis; linear interpolation of a linear profile is exact
    assert abs(L - 0.9 / 1.0) < 1e-6, L
    th = SW.separation_angle(mi, Q, np.arange(0, mi.n_cells, nr))
    assert th is not None and abs(th - 128.0) < 1.5, th


def test_attached_flow_has_no_wake():
    mi = W.sphere_shell(7)
    c = SW.cell_centroids(mi)
    Q = np.zeros((mi.n_cells, 5)); Q[:, 0] = 1.0; Q[:, 1] = 0.3; Q[:, 4] = 2.5
    assert SW.wake_length(mi, Q, 14) == 0.0
    assert SW.separation_angle(mi, Q, np.arange(0, mi.n_cells, 14)) is None
