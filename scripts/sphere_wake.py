"""Flow past a sphere to steady state (Tables 8-9).

    python scripts/sphere_wake.py --N 35 --ma 0.2535 --re 118 --t-end 150
    python scripts/sphere_wake.py --N 35 --ma 1.5 --re 300 --t-end 60

Runs the CUDA path from the free-stream state and reports, every
chunk of steps, the residual and the two quantities of Tables 8-9:

* L, the closed wake length: distance (in D) from the rear of the sphere to the
  point on the downstream axis where the axial velocity changes from reversed
  to forward (reading R28);
* theta, the separation angle: the polar angle, measured from the front
  stagnation point, at which the wall-tangential velocity of the first cell
  layer changes sign (azimuthally averaged, reading R28).

The paper does not define either procedure; these readings are the usual ones
for this benchmark.  Only post-processing lives here (numpy on the solver's
state); every step runs in libhgks.
"""
import argparse, json, os, sys, time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def cell_centroids(mi):
    """Mean of the cell's nodes (adequate for locating cells in the analysis)."""
    nodes = mi.cell_nodes[:, :8]
    return mi.xyz[nodes].mean(axis=1)


def wake_length(mi, Q, nr, r_in=0.5):
    """Closed wake length L/D behind a sphere of radius r_in centred at the origin,
    free stream along +x.  In each radial layer (workloads.sphere_shell orders
    cells radius-fastest, nr layers) the downstream cell whose centroid is closest
    to the +x axis gives one sample of the axial velocity; L is where it turns from
    reversed to forward (linear interpolation).  0 when there is no reversed flow."""
    c = cell_centroids(mi)
    u = Q[:, 1] / Q[:, 0]
    off = np.hypot(c[:, 1], c[:, 2])
    layer = np.arange(mi.n_cells) % nr
    cand = np.where(c[:, 0] > 0)[0]
    xs, us = np.empty(nr), np.empty(nr)
    for k in range(nr):
        ck = cand[layer[cand] == k]
        i = ck[np.argmin(off[ck])]
        xs[k], us[k] = c[i, 0], u[i]
    if us[0] >= 0:
        return 0.0
    for i in range(1, nr):
        if us[i - 1] < 0 <= us[i]:
            x0 = xs[i - 1] - us[i - 1] * (xs[i] - xs[i - 1]) / (us[i] - us[i - 1])
            return float(x0 - r_in) / (2 * r_in)
    return float(xs[-1] - r_in) / (2 * r_in)


def separation_angle(mi, Q, first_layer, bin_deg=1.0):
    """Separation angle (degrees from the front stagnation point) from the first
    cell layer: azimuthally averaged wall-tangential velocity u_alpha (positive
    when moving from front to rear) binned in alpha; the first bin past 90 deg
    where it turns negative, interpolated.  None when the flow stays attached."""
    c = cell_centroids(mi)[first_layer]
    q = Q[first_layer]
    vel = q[:, 1:4] / q[:, :1]
    r = np.linalg.norm(c, axis=1)
    alpha = np.arccos(np.clip(-c[:, 0] / r, -1, 1))  # 0 at the front stagnation point (-x)
    perp = np.stack([np.zeros_like(r), c[:, 1], c[:, 2]], 1)
    pn = np.linalg.norm(perp, axis=1)
    perp = perp / np.maximum(pn, 1e-300)[:, None]
    # e_alpha = d/d alpha of (-cos a, sin a * perp) = (sin a, cos a * perp)
    ua = vel[:, 0] * np.sin(alpha) + np.cos(alpha) * np.einsum("ij,ij->i", vel, perp)
    deg = np.degrees(alpha)
    nb = int(round(180 / bin_deg))
    idx = np.minimum((deg / bin_deg).astype(int), nb - 1)
    cnt = np.bincount(idx, minlength=nb)
    mean = np.bincount(idx, weights=ua, minlength=nb) / np.maximum(cnt, 1)
    centers = (np.arange(nb) + 0.5) * bin_deg
    ok = cnt > 0
    centers, mean = centers[ok], mean[ok]
    for i in range(1, len(mean)):
        if centers[i] > 90 and mean[i - 1] > 0 >= mean[i]:
            return float(centers[i - 1] + mean[i - 1] * (centers[i] - centers[i - 1]) / (mean[i - 1] - mean[i]))
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=35)
    ap.add_argument("--ma", type=float, default=0.2535)
    ap.add_argument("--re", type=float, default=118.0)
    ap.add_argument("--t-end", type=float, default=150.0)
    ap.add_argument("--chunk", type=int, default=2000)
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--prandtl", type=float, default=1.0, help="Pr of the heat-flux correction (R29); 1 = none")
    ap.add_argument("--tol", type=float, default=1e-6, help="stop when the density residual falls below")
    ap.add_argument("--out", default=None, help="save the final state (.npy)")
    args = ap.parse_args()
    from paper_2407_00656_b200 import hgks, workloads as W
    gam = 1.4
    mi = W.sphere_shell(args.N)
    nr = 2 * args.N
    first_layer = np.arange(0, mi.n_cells, nr)  # workloads.sphere_shell: radial index fastest
    fs = (1.0, args.ma, 0.0, 0.0, 1.0 / gam)
    Q0 = W.uniform_state(mi.n_cells, 1.0, (args.ma, 0.0, 0.0), 1.0 / gam, gamma=gam)
    cfg = hgks.SolverConfig(gamma=gam, cfl=0.5, tau_mode=1, mu_inf=args.ma / args.re, c1=1.0, t_inf=1.0 / gam,
                            prandtl=args.prandtl,
                            freestream=fs, precision=args.precision)
    s = hgks.Solver(hgks.Mesh(mi), Q0, cfg)
    Qp, _, tp = s.get_state()
    t0 = time.time()
    steps = 0
    while True:
        info = s.step(args.chunk)
        steps += info["steps_done"]
        Q, _, t = s.get_state()
        res = float(np.abs(Q[:, 0] - Qp[:, 0]).mean() / max(t - tp, 1e-300))
        L = wake_length(mi, Q, nr)
        th = separation_angle(mi, Q, first_layer)
        print(json.dumps(dict(N=args.N, ma=args.ma, re=args.re, steps=steps, t=t, dt=info["last_dt"], residual=res,
                              L=L, theta=th, fallbacks=info["fallbacks"], secs=time.time() - t0)), flush=True)
        Qp, tp = Q, t
        if t >= args.t_end or res < args.tol:
            break
    if args.out:
        np.save(args.out, Q)
    s.close()


if __name__ == "__main__":
    main()
