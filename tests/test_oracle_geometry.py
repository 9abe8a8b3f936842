"""Oracle pins: geometry (O1), connectivity and stencils (O2/O3) against closed
forms, invariants and brute force independent of the oracle's own code."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import workloads as W


def single_cell(kind):
    if kind == "tet":
        xyz = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
        cn = np.full((1, 8), -1, np.int64)
        cn[0, :4] = [0, 1, 2, 3]
        faces = [[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]]
        t = W.TET
    else:
        xyz = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]], float)
        cn = np.arange(8, dtype=np.int64)[None, :]
        faces = [[0, 1, 2, 3], [0, 1, 5, 4], [1, 2, 6, 5], [2, 3, 7, 6], [3, 0, 4, 7], [4, 5, 6, 7]]
        t = W.HEX
    bf = np.full((len(faces), 4), -1, np.int64)
    for k, f in enumerate(faces):
        bf[k, :len(f)] = f
    return W.MeshInput(xyz=xyz, cell_type=np.array([t], np.int8), cell_nodes=cn, bface_nodes=bf,
                       bface_tag=np.full(len(faces), W.BC_WALL, np.int32))


def test_regular_tet_volume_centroid():
    """SPEC S:61-63 'regular tet -> volume 1/6, centroid (1/4,1/4,1/4)'."""
    m = O.OracleMesh(single_cell("tet"))
    V, c, M2 = m.geometry()
    assert abs(V[0] - 1 / 6) < 1e-15
    assert np.allclose(c[0], 0.25, atol=1e-15)
    # second central moments of the unit simplex: var = 3/80, cov = -1/80
    assert np.allclose(M2[0], (np.eye(3) * 4 - 1) / 80.0, atol=1e-15)
    assert m.n_ghosts == 4  # one mirror ghost per wall face (Alg. 1 ghosts, R25)
    # ghost centroid = mirror of the centroid across the face plane x=0
    Vg, cg, _ = m.geometry()
    f = m.faces()
    k = [i for i in range(4) if np.allclose(f["gp_n"][i, 0], [-1, 0, 0])][0]
    assert np.allclose(cg[1 + k], [-0.25, 0.25, 0.25])


def test_unit_hex_gauss_points():
    """unit-square face -> 4 GPs at 1/2 +- 1/(2 sqrt 3), weights 1/4."""
    m = O.OracleMesh(single_cell("hex"))
    V, c, M2 = m.geometry()
    assert abs(V[0] - 1.0) < 1e-14 and np.allclose(c[0], 0.5)
    assert np.allclose(M2[0], np.eye(3) / 12.0, atol=1e-15)
    f = m.faces()
    q = {0.5 - 0.5 / np.sqrt(3), 0.5 + 0.5 / np.sqrt(3)}
    for i in range(6):
        assert f["ngp"][i] == 4
        assert np.allclose(f["gp_wS"][i], 0.25)
        x = f["gp_x"][i]
        n = f["gp_n"][i][0]
        ax = int(np.argmax(np.abs(n)))
        other = [a for a in range(3) if a != ax]
        got = {round(v, 12) for v in x[:, other].ravel()}
        assert got == {round(v, 12) for v in q}
        # outward normal
        assert np.sign(n[ax]) == (1 if x[0, ax] > 0.5 else -1)


@pytest.mark.parametrize("mk", [lambda: W.kuhn_box(4), lambda: W.kuhn_box(5, jitter=0.1),
                                lambda: W.cartesian_hex_box(5, jitter=0.15)])
def test_closure_volume_and_quadrature(mk):
    mi = mk()
    m = O.OracleMesh(mi)
    V, c, M2 = m.geometry()
    assert abs(V[: m.n_cells].sum() - 8.0) < 1e-12  # sum V = V_D
    f = m.faces()
    cf = m.cell_faces()
    # closed cells: sum over faces and Gauss points of omega S n = 0 (A.8)
    for i in range(0, m.n_cells, 7):
        s = np.zeros(3)
        for p in range(6):
            fi = cf[i, p]
            if fi < 0:
                continue
            sg = 1.0 if f["owner"][fi] == i else -1.0
            ng = f["ngp"][fi]
            s += sg * (f["gp_wS"][fi, :ng, None] * f["gp_n"][fi, :ng]).sum(0)
        assert np.abs(s).max() < 1e-14
    # face quadrature exact for degree 2: int_face (x.a)^2 on triangles vs vertex formula
    if mi.cell_type[0] == W.TET:
        a = np.array([0.3, -0.7, 0.5])
        for fi in range(0, m.n_faces, 11):
            x = f["gp_x"][fi, :3]
            area = f["gp_wS"][fi, :3].sum()
            quad = (f["gp_wS"][fi, :3] * (x @ a) ** 2).sum()
            # exact: area/6 * (s1^2+s2^2+s3^2 + s1 s2 + s1 s3 + s2 s3) for the vertex values s_k;
            # vertices recovered from the GPs: v = 2*(sum x)/3... use barycentric inversion
            M = np.array([[2 / 3, 1 / 6, 1 / 6], [1 / 6, 2 / 3, 1 / 6], [1 / 6, 1 / 6, 2 / 3]])
            v = np.linalg.solve(M, x)
            s = v @ a
            exact = area / 6 * (s @ s + s[0] * s[1] + s[0] * s[2] + s[1] * s[2])
            assert abs(quad - exact) < 1e-14 * max(1, abs(exact))


def kuhn_adjacency(N):
    """Independent face adjacency of the periodic Kuhn box from node keys (wrapped indices)."""
    mi = W.kuhn_box(N)
    ijk = np.rint(mi.xyz / (2.0 / N)).astype(int) % N
    wrapped = ijk[:, 0] * N * N + ijk[:, 1] * N + ijk[:, 2]
    faces = {}
    for c in range(mi.n_cells):
        nodes = wrapped[mi.cell_nodes[c, :4]]
        for p in range(4):
            key = tuple(sorted(np.delete(nodes, p)))
            # faces with identical wrapped keys are the same periodic face
            faces.setdefault(key, []).append(c)
    adj = [set() for _ in range(mi.n_cells)]
    for key, cs in faces.items():
        assert len(cs) == 2
        adj[cs[0]].add(cs[1])
        adj[cs[1]].add(cs[0])
    return mi, adj


def test_kuhn_stencils_equal_depth2_bfs():
    """Alg. 1 big stencil == depth-2 BFS; 14 cells for every Kuhn tet;
    sub-stencils of 6 distinct cells."""
    mi, adj = kuhn_adjacency(5)
    m = O.OracleMesh(mi)
    assert m.n_faces == 2 * m.n_cells
    assert m.min_stencil == m.max_stencil == 14
    for i in range(m.n_cells):
        ids, _ = m.big_stencil(i)
        bfs = set(adj[i]) | set().union(*[adj[j] for j in adj[i]])
        bfs.discard(i)
        assert set(ids.tolist()) == bfs
        # first layer comes first, in face order
        assert set(ids[:4].tolist()) == adj[i]
        for mm in range(4):
            sub = m.sub_stencil(i, mm)
            assert len(sub) == 6 and len(set(sub.tolist())) == 6
            assert set(sub.tolist()) <= bfs


def test_hex_box_stencil_24_and_substencils():
    """Cartesian hex interior: 6 + 18 = 24 neighbours; 8 sub-stencils
    {i_1 or i_6, two adjacent ring faces}."""
    mi = W.cartesian_hex_box(5)
    m = O.OracleMesh(mi)
    assert m.min_stencil == m.max_stencil == 24
    V, c, _ = m.geometry()
    i = 62
    ids, sh = m.big_stencil(i)
    first = ids[:6]
    # local faces 0 and 5 are the -z / +z neighbours for the VTK-ordered unit hexes
    d = (c[first] + sh[:6]) - c[i]
    assert np.allclose(d[0], [0, 0, -0.4]) and np.allclose(d[5], [0, 0, 0.4])
    ring = [1, 2, 3, 4]
    for mm in range(8):
        sub = m.sub_stencil(i, mm)
        assert len(sub) == 3
        assert sub[0] == first[0 if mm < 4 else 5]
        r1, r2 = ring[mm % 4], ring[(mm + 1) % 4]
        assert list(sub[1:]) == [first[r1], first[r2]]


def test_tiny_periodic_box_rejected():
    with pytest.raises(O.OracleError):
        O.OracleMesh(W.kuhn_box(2))


# --------------------------------------------------------------------------- #
# triangular prisms (reading R30)
# --------------------------------------------------------------------------- #
def single_prism(v):
    xyz = np.asarray(v, float)
    cn = np.full((1, 8), -1, np.int64)
    cn[0, :6] = np.arange(6)
    faces = [[0, 1, 2], [3, 4, 5], [0, 1, 4, 3], [1, 2, 5, 4], [2, 0, 3, 5]]
    bf = np.full((5, 4), -1, np.int64)
    for k, f in enumerate(faces):
        bf[k, :len(f)] = f
    return W.MeshInput(xyz=xyz, cell_type=np.array([W.PRISM], np.int8), cell_nodes=cn, bface_nodes=bf,
                       bface_tag=np.full(5, W.BC_WALL, np.int32))


def tet_moments(v):
    """V, centroid, M2 of a tet from its vertices (closed forms, independent of the oracle)."""
    v = np.asarray(v, float)
    V = abs(np.linalg.det(v[1:] - v[0])) / 6.0
    c = v.mean(0)
    d = v - c
    return V, c, (d.T @ d) / 20.0


def test_right_prism_closed_forms():
    """Unit right prism (triangle (0,0),(1,0),(0,1) x [0,1]): V = 1/2, centroid (1/3, 1/3, 1/2),
    var x = var y = 1/18, cov xy = -1/36, var z = 1/12; five faces, two triangles + three quads."""
    m = O.OracleMesh(single_prism([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]]))
    V, c, M2 = m.geometry()
    assert abs(V[0] - 0.5) < 1e-15 and np.allclose(c[0], [1 / 3, 1 / 3, 0.5], atol=1e-15)
    exp = np.array([[1 / 18, -1 / 36, 0], [-1 / 36, 1 / 18, 0], [0, 0, 1 / 12]])
    assert np.allclose(M2[0], exp, atol=1e-15)
    f = m.faces()
    assert m.n_faces == 5 and sorted(f["ngp"].tolist()) == [3, 3, 4, 4, 4]


def test_oblique_prism_vs_three_tets():
    """A skewed straight prism (top = bottom + a shift, planar faces) is exactly the union of
    the tets (A,B,C,D), (B,C,D,E), (C,D,E,F): V, centroid and M2 from their closed forms."""
    A, B, C = np.array([0.1, 0.0, 0.2]), np.array([1.3, 0.2, 0.0]), np.array([0.4, 1.1, 0.3])
    t = np.array([0.3, -0.2, 0.9])
    v = [A, B, C, A + t, B + t, C + t]
    m = O.OracleMesh(single_prism(v))
    V, c, M2 = m.geometry()
    parts = [tet_moments([v[0], v[1], v[2], v[3]]), tet_moments([v[1], v[2], v[3], v[4]]),
             tet_moments([v[2], v[3], v[4], v[5]])]
    Vt = sum(p[0] for p in parts)
    ct = sum(p[0] * p[1] for p in parts) / Vt
    St = sum(p[0] * (p[2] + np.outer(p[1] - ct, p[1] - ct)) for p in parts) / Vt
    assert abs(V[0] - Vt) < 1e-14 and np.allclose(c[0], ct, atol=1e-14)
    assert np.allclose(M2[0], St, atol=1e-14)


def hybrid_adjacency(mi, N):
    """Face neighbours of the periodic hybrid box from wrapped node keys (independent of the
    oracle); faces of a prism in R30's order (0/1 triangles, 2..4 sides)."""
    ijk = np.rint(mi.xyz / (2.0 / N)).astype(int) % N
    wrapped = ijk[:, 0] * N * N + ijk[:, 1] * N + ijk[:, 2]
    tet_f = [[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]]
    pri_f = [[0, 1, 2], [3, 4, 5], [0, 1, 4, 3], [1, 2, 5, 4], [2, 0, 3, 5]]
    owners = {}
    for c in range(mi.n_cells):
        fl = tet_f if mi.cell_type[c] == W.TET else pri_f
        for p, f in enumerate(fl):
            owners.setdefault(tuple(sorted(wrapped[mi.cell_nodes[c, f]])), []).append((c, p))
    nb = [[-1] * (4 if mi.cell_type[c] == W.TET else 5) for c in range(mi.n_cells)]
    for key, cp in owners.items():
        assert len(cp) == 2, key
        (a, pa), (b, pb) = cp
        nb[a][pa] = b
        nb[b][pb] = a
    return nb


def test_hybrid_box_connectivity_and_closure():
    """Hybrid tet/prism box: every face matched (conforming layers, periodic), sum V = V_D,
    closed cells, big stencil = depth-2 BFS, prism sub-stencils = R30 (one triangle neighbour +
    two ring-adjacent sides), tet sub-stencils = R16 with all the other face neighbours of a
    prism neighbour (7 members)."""
    N = 6
    mi = W.hybrid_box(N)
    nb = hybrid_adjacency(mi, N)
    m = O.OracleMesh(mi)
    V, c, _ = m.geometry()
    assert abs(V[: m.n_cells].sum() - 8.0) < 1e-12
    f = m.faces()
    cf = m.cell_faces()
    for i in range(0, m.n_cells, 5):
        s = np.zeros(3)
        for p in range(6):
            fi = cf[i, p]
            if fi < 0:
                continue
            sg = 1.0 if f["owner"][fi] == i else -1.0
            ng = f["ngp"][fi]
            s += sg * (f["gp_wS"][fi, :ng, None] * f["gp_n"][fi, :ng]).sum(0)
        assert np.abs(s).max() < 1e-14
    ps = [(0, 2, 3), (0, 3, 4), (0, 4, 2), (1, 2, 3), (1, 3, 4), (1, 4, 2)]
    tri = [(0, 1, 2), (0, 1, 3), (1, 2, 3), (2, 0, 3)]
    saw7 = False
    for i in range(m.n_cells):
        ids, _ = m.big_stencil(i)
        bfs = set(nb[i]) | set().union(*[set(nb[j]) for j in nb[i]])
        bfs.discard(i)
        assert set(ids.tolist()) == bfs and list(ids[:len(nb[i])]) == nb[i]
        if mi.cell_type[i] == W.PRISM:
            for mm, t in enumerate(ps):
                assert list(m.sub_stencil(i, mm)) == [nb[i][q] for q in t]
        else:
            for mm in range(4):
                exp = [nb[i][q] for q in tri[mm]]
                for x in nb[nb[i][mm]]:
                    if x != i and x not in exp:
                        exp.append(x)
                sub = list(m.sub_stencil(i, mm))
                assert sub == exp, (i, mm)
                saw7 |= len(sub) == 7
    assert saw7  # tets next to prism layers
