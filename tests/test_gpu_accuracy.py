"""Table 3 on the CUDA path: the accuracy test to t = 2 at N = 20, 40, 80 under
the adopted readings (R6a: CFL 0.7; R9 dQ0), against the paper's printed L1 errors.

The bar is the reading's own justification (R6a, profiles/r02/t3_readings.md):
the sweep over the dQ0 readings and CFL 0.3/0.5/0.7 reproduced T3 within 2 % at N >= 20 only
at CFL 0.7; the test allows 5 % and asks for the paper's asymptotic order (2.99, 3.00) to
within 0.1.  N = 10 is pinned on the oracle side (tests/test_oracle_scheme.py)."""
import numpy as np
import pytest

from paper_2407_00656_b200 import hgks, workloads as W

pytestmark = pytest.mark.gpu

T3 = {20: 8.7117e-3, 40: 1.0994e-3, 80: 1.3768e-4}


def l1_at_t2(N, cfl=0.7):
    mi = W.kuhn_box(N)
    s = hgks.Solver(hgks.Mesh(mi), W.advection_ic(mi), hgks.SolverConfig(cfl=cfl))
    while s.step(500, t_stop=2.0)["t"] < 2.0:
        pass
    Q, _, t = s.get_state()
    assert t == 2.0
    e = Q[:, 0] - W.advection_ic(mi, t=t)[:, 0]
    return float(np.abs(e).mean())  # equal tet volumes: L1 = sum |e| V / V_D = mean |e| (R22)


def test_table3_on_gpu(cuda_ok):
    L1 = {N: l1_at_t2(N) for N in (20, 40, 80)}
    for N, v in L1.items():
        assert abs(v / T3[N] - 1) <= 0.05, (N, v, T3[N])
    for a, b in ((20, 40), (40, 80)):
        order = np.log2(L1[a] / L1[b])
        assert abs(order - np.log2(T3[a] / T3[b])) <= 0.1, (a, b, order)
