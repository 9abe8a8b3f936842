"""Seeded, synthetic workload generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the HGKS method (no reconstruction, no flux,
no time stepping).  It only produces the *inputs* of a run -- node/cell arrays,
periodic box, boundary-face tags and initial cell averages -- and the exact
solution of the accuracy test, so that both sides of every parity test consume
byte-identical inputs.

Workloads:
  * Kuhn box (C1, C2, C5): the periodic box [0, Lx]x[0, Ly]x[0, Lz] split into
    cubes of edge h, each cube cut into 6 tetrahedra ("every
    cubic is divided into six tetrahedron cells"; Kuhn/Freudenthal split,
    DESIGN.md reading R3).
  * Accuracy-test initial condition: rho = 1 + 0.2 sin(pi(x+y+z)),
    p = 1, U = V = W = 1, as EXACT cell averages (reading R5).
  * Cubed-sphere hexahedral shell (C3/C4): six blocks of
    N x N x 2N hexahedra (the grading and outer radius are readings R24).
  * Hybrid tet/prism box (BASELINE configs[2] "mixed tet/prism cells"): the
    Kuhn box with its lowest z-layers of cubes cut into two triangular prisms each instead of
    six tets (conforming: both cut the cube's horizontal faces along the same diagonal).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

TET = 4
PRISM = 6  # triangular prism (VTK wedge node order: 0-1-2 one triangle, 3-4-5 the other, i+3 above i)
HEX = 8
BC_WALL = 1
BC_FARFIELD = 2


@dataclass
class MeshInput:
    """Plain arrays describing an unstructured mesh (the C-ABI's hgks_mesh_desc)."""

    xyz: np.ndarray                 # [n_nodes, 3] float64
    cell_type: np.ndarray           # [n_cells] int8 (TET=4 / HEX=8)
    cell_nodes: np.ndarray          # [n_cells, 8] int64, -1 padded
    periodic_length: np.ndarray = field(default_factory=lambda: np.zeros(3))  # 0 = not periodic
    periodic_origin: np.ndarray = field(default_factory=lambda: np.zeros(3))
    bface_nodes: np.ndarray = field(default_factory=lambda: np.zeros((0, 4), np.int64))
    bface_tag: np.ndarray = field(default_factory=lambda: np.zeros((0,), np.int32))
    name: str = ""

    @property
    def n_cells(self) -> int:
        return int(self.cell_type.shape[0])

    @property
    def n_nodes(self) -> int:
        return int(self.xyz.shape[0])


# --------------------------------------------------------------------------- #
# Kuhn (Freudenthal) periodic tetrahedral box
# --------------------------------------------------------------------------- #
# Tet sigma of the cube with min corner v0 has vertices
#   v0, v0+e_s0, v0+e_s0+e_s1, v0+e_s0+e_s1+e_s2     (s = permutation of 0,1,2)
KUHN_PERMS = list(itertools.permutations(range(3)))


def kuhn_box(nx: int, ny: int | None = None, nz: int | None = None, h: float | None = None,
             jitter: float = 0.0, seed: int = 656) -> MeshInput:
    """Periodic Kuhn box of nx*ny*nz cubes (6 tets each).

    Default cube edge h = 2/nx so that nx=ny=nz=N gives the paper's [0,2]^3 box
    with 6N^3 tets.  ``jitter`` > 0 moves every node that is
    strictly inside the box by U[-jitter*h, jitter*h] per axis (seed 656,
    SURVEY.md 8(d) "Unit tests"), keeping boundary faces planar and periodic.
    """
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    h = 2.0 / nx if h is None else h
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    xyz = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3).astype(np.float64) * h

    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    n_cubes = ci.size
    cells = np.full((n_cubes, 6, 8), -1, dtype=np.int64)
    for t, perm in enumerate(KUHN_PERMS):
        pos = np.stack([ci, cj, ck], axis=-1).copy()
        cells[:, t, 0] = nid(pos[:, 0], pos[:, 1], pos[:, 2])
        for v, axis in enumerate(perm):
            pos[:, axis] += 1
            cells[:, t, v + 1] = nid(pos[:, 0], pos[:, 1], pos[:, 2])
    cells = cells.reshape(-1, 8)
    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        d = rng.uniform(-jitter * h, jitter * h, size=xyz.shape)
        L = np.array([nx, ny, nz]) * h
        interior = np.all((xyz > 0.5 * h * 1e-6) & (xyz < L - 0.5 * h * 1e-6), axis=1)
        xyz = xyz + d * interior[:, None]
    return MeshInput(
        xyz=xyz,
        cell_type=np.full(cells.shape[0], TET, dtype=np.int8),
        cell_nodes=cells,
        periodic_length=np.array([nx * h, ny * h, nz * h], dtype=np.float64),
        periodic_origin=np.zeros(3),
        name=f"kuhn_{nx}x{ny}x{nz}" + ("_jit" if jitter > 0 else ""),
    )


def hybrid_box(n: int, prism_layers: int | None = None, h: float | None = None, jitter: float = 0.0,
               seed: int = 656) -> MeshInput:
    """Periodic n^3 box of cubes (edge h = 2/n): the cubes of the lowest ``prism_layers``
    z-layers (default n // 2) are cut along the x-y diagonal (0,0)-(1,1) into two triangular
    prisms, the others into the six Kuhn tets of ``kuhn_box``.  The Kuhn split cuts a cube's
    bottom and top faces along the same diagonal, so prism and tet layers meet conformingly
    (also across the periodic z wrap).  ``jitter`` moves interior nodes as in ``kuhn_box``."""
    prism_layers = n // 2 if prism_layers is None else prism_layers
    h = 2.0 / n if h is None else h
    ii, jj, kk = np.meshgrid(np.arange(n + 1), np.arange(n + 1), np.arange(n + 1), indexing="ij")
    xyz = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3).astype(np.float64) * h

    def nid(i, j, k):
        return (i * (n + 1) + j) * (n + 1) + k

    ci, cj, ck = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    cells, types = [], []
    for c in range(ci.size):
        i, j, k = int(ci[c]), int(cj[c]), int(ck[c])
        v = lambda a, b, d: nid(i + a, j + b, k + d)  # noqa: E731
        if k < prism_layers:
            for tri in (((0, 0), (1, 0), (1, 1)), ((0, 0), (1, 1), (0, 1))):
                cells.append([v(a, b, 0) for a, b in tri] + [v(a, b, 1) for a, b in tri] + [-1, -1])
                types.append(PRISM)
        else:
            for perm in KUHN_PERMS:
                pos = [i, j, k]
                row = [nid(*pos)]
                for axis in perm:
                    pos[axis] += 1
                    row.append(nid(*pos))
                cells.append(row + [-1, -1, -1, -1])
                types.append(TET)
    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        d = rng.uniform(-jitter * h, jitter * h, size=xyz.shape)
        L = np.array([n, n, n]) * h
        interior = np.all((xyz > 0.5 * h * 1e-6) & (xyz < L - 0.5 * h * 1e-6), axis=1)
        xyz = xyz + d * interior[:, None]
    return MeshInput(
        xyz=xyz,
        cell_type=np.array(types, dtype=np.int8),
        cell_nodes=np.array(cells, dtype=np.int64),
        periodic_length=np.array([n * h, n * h, n * h]),
        periodic_origin=np.zeros(3),
        name=f"hybrid_{n}_{prism_layers}" + ("_jit" if jitter > 0 else ""),
    )


def cartesian_hex_box(nx: int, ny: int | None = None, nz: int | None = None,
                      h: float | None = None, jitter: float = 0.0, seed: int = 656) -> MeshInput:
    """Periodic box of hexahedra in VTK/Gmsh node order (bottom 0-3, top 4-7)."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    h = 2.0 / nx if h is None else h
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    xyz = np.stack([ii, jj, kk], axis=-1).reshape(-1, 3).astype(np.float64) * h

    def nid(i, j, k):
        return (i * (ny + 1) + j) * (nz + 1) + k

    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    corners = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    cells = np.stack([nid(ci + a, cj + b, ck + c) for (a, b, c) in corners], axis=-1).astype(np.int64)
    if jitter > 0.0:
        rng = np.random.default_rng(seed)
        d = rng.uniform(-jitter * h, jitter * h, size=xyz.shape)
        L = np.array([nx, ny, nz]) * h
        interior = np.all((xyz > 1e-9 * h) & (xyz < L - 1e-9 * h), axis=1)
        xyz = xyz + d * interior[:, None]
    return MeshInput(
        xyz=xyz,
        cell_type=np.full(cells.shape[0], HEX, dtype=np.int8),
        cell_nodes=cells,
        periodic_length=np.array([nx * h, ny * h, nz * h]),
        name=f"hexbox_{nx}x{ny}x{nz}" + ("_jit" if jitter > 0 else ""),
    )


def walled_hex_box(n: int, h: float | None = None, jitter: float = 0.0, seed: int = 656) -> MeshInput:
    """Closed n^3 hex box whose six sides are all WALL boundary faces (no periodicity):
    the wall-pin workload (every wall corner case: cells with 1, 2 and 3 wall faces)."""
    mi = cartesian_hex_box(n, h=h, jitter=jitter, seed=seed)
    mi.periodic_length = np.zeros(3)

    def nid(i, j, k):
        return (i * (n + 1) + j) * (n + 1) + k

    quads = []
    for a in range(n):
        for b in range(n):
            for c0 in (0, n):
                quads.append([nid(c0, a, b), nid(c0, a + 1, b), nid(c0, a + 1, b + 1), nid(c0, a, b + 1)])
                quads.append([nid(a, c0, b), nid(a + 1, c0, b), nid(a + 1, c0, b + 1), nid(a, c0, b + 1)])
                quads.append([nid(a, b, c0), nid(a + 1, b, c0), nid(a + 1, b + 1, c0), nid(a, b + 1, c0)])
    mi.bface_nodes = np.array(quads, np.int64)
    mi.bface_tag = np.full(len(quads), BC_WALL, np.int32)
    mi.name = f"walled_hexbox_{n}" + ("_jit" if jitter > 0 else "")
    return mi


_CELL_FACES = {
    TET: [[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]],
    PRISM: [[0, 1, 2], [3, 4, 5], [0, 1, 4, 3], [1, 2, 5, 4], [2, 0, 3, 5]],
    8: [[0, 1, 2, 3], [0, 1, 5, 4], [1, 2, 6, 5], [2, 3, 7, 6], [3, 0, 4, 7], [4, 5, 6, 7]],
}


def close_with_walls(mi: MeshInput) -> MeshInput:
    """Drop the periodicity of ``mi`` and tag every face without a partner (matched by node
    ids) as a WALL boundary face."""
    owners = {}
    for c in range(mi.n_cells):
        for f in _CELL_FACES[int(mi.cell_type[c])]:
            nodes = mi.cell_nodes[c, f]
            key = tuple(sorted(nodes.tolist()))
            owners[key] = None if key in owners else nodes
    faces = [nodes for nodes in owners.values() if nodes is not None]
    bf = np.full((len(faces), 4), -1, np.int64)
    for k, nodes in enumerate(faces):
        bf[k, :len(nodes)] = nodes
    mi.periodic_length = np.zeros(3)
    mi.bface_nodes = bf
    mi.bface_tag = np.full(len(faces), BC_WALL, np.int32)
    mi.name += "_walled"
    return mi


def walled_hybrid_box(n: int, jitter: float = 0.0, seed: int = 656) -> MeshInput:
    """``hybrid_box`` closed by walls on all six sides: wall faces of both kinds (prism
    sides and tet faces on the x / y sides, prism bottoms at z = 0, tet faces at the top)."""
    return close_with_walls(hybrid_box(n, jitter=jitter, seed=seed))


# --------------------------------------------------------------------------- #
# Cubed-sphere hexahedral shell (C3/C4)
# --------------------------------------------------------------------------- #
def sphere_shell(n: int, r_in: float = 0.5, r_out: float = 10.0, first_cell: float = 0.01,
                 radial_cells: int | None = None) -> MeshInput:
    """Six-block cubed-sphere shell of 6*n*n*(2n) hexahedra.

    Blocks use the equiangular gnomonic map; radial spacing is geometric with
    first cell ``first_cell`` (D=1 sphere: r_in=0.5; outer radius 20D = 10,
    reading R24).  Hex nodes 0-3 lie on the inner radial surface and 4-7 on the
    outer one, so local faces 0 and 5 are the radial pair (reading R17).
    Boundary faces: the sphere surface is WALL, the outer surface FARFIELD.
    Nodes are shared between blocks (conforming mesh).
    """
    nr = 2 * n if radial_cells is None else radial_cells
    # geometric grading: r_k = r_in + first_cell * (q^k - 1)/(q - 1), r_nr = r_out
    span = r_out - r_in

    def total(q):
        return first_cell * (q ** nr - 1.0) / (q - 1.0) if abs(q - 1.0) > 1e-14 else first_cell * nr

    lo, hi = 1.0 + 1e-12, 2.0
    while total(hi) < span:
        hi *= 1.5
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if total(mid) < span:
            lo = mid
        else:
            hi = mid
    q = 0.5 * (lo + hi)
    radii = r_in + first_cell * (q ** np.arange(nr + 1) - 1.0) / (q - 1.0)
    radii[-1] = r_out

    # unit-sphere points of the 6 faces, equiangular: a, b in [-pi/4, pi/4]
    ang = np.linspace(-np.pi / 4, np.pi / 4, n + 1)
    ta = np.tan(ang)

    def face_dirs(f):
        A, B = np.meshgrid(ta, ta, indexing="ij")
        one = np.ones_like(A)
        if f == 0:
            v = np.stack([one, A, B], -1)
        elif f == 1:
            v = np.stack([-one, B, A], -1)
        elif f == 2:
            v = np.stack([B, one, A], -1)
        elif f == 3:
            v = np.stack([A, -one, B], -1)
        elif f == 4:
            v = np.stack([A, B, one], -1)
        else:
            v = np.stack([B, A, -one], -1)
        return v / np.linalg.norm(v, axis=-1, keepdims=True)

    # dedupe surface directions across blocks (shared block edges)
    dirs = []
    for f in range(6):
        dirs.append(face_dirs(f).reshape(-1, 3))
    alld = np.concatenate(dirs, 0)
    key = np.round(alld * 1e9).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    inv = inv.ravel()
    ndir = first.size
    udirs = alld[first]
    dir_id = [inv[f * (n + 1) ** 2:(f + 1) * (n + 1) ** 2].reshape(n + 1, n + 1) for f in range(6)]
    xyz = (radii[:, None, None] * udirs[None, :, :]).reshape(-1, 3)

    def nid(r, d):
        return r * ndir + d

    blocks = []
    rr = np.arange(nr)[None, None, :]
    for f in range(6):
        D = dir_id[f].astype(np.int64)
        d00, d10 = D[:-1, :-1, None], D[1:, :-1, None]
        d11, d01 = D[1:, 1:, None], D[:-1, 1:, None]
        c = np.stack([nid(rr, d00), nid(rr, d10), nid(rr, d11), nid(rr, d01),
                      nid(rr + 1, d00), nid(rr + 1, d10), nid(rr + 1, d11), nid(rr + 1, d01)], axis=-1)
        blocks.append(c.reshape(-1, 8))   # order: i, j, r (r fastest)
    cells = np.concatenate(blocks, 0).astype(np.int64)
    # orient every hex so that bottom face (0,1,2,3) has its right-hand normal
    # pointing into the cell (i.e. outwards radially), as for the unit cube.
    p = xyz[cells]
    nrm = np.cross(p[:, 1] - p[:, 0], p[:, 3] - p[:, 0])
    up = p[:, 4] - p[:, 0]
    flip = np.einsum("ij,ij->i", nrm, up) < 0
    cells[flip] = cells[flip][:, [0, 3, 2, 1, 4, 7, 6, 5]]
    # boundary faces: inner (wall) = bottom faces of r=0 cells, outer = top faces of r=nr-1
    nrad = nr
    bottom = cells[0::nrad][:, [0, 1, 2, 3]]
    top = cells[nrad - 1::nrad][:, [4, 5, 6, 7]]
    bface = np.concatenate([bottom, top], 0)
    tags = np.concatenate([np.full(bottom.shape[0], BC_WALL), np.full(top.shape[0], BC_FARFIELD)]).astype(np.int32)
    return MeshInput(
        xyz=xyz,
        cell_type=np.full(cells.shape[0], HEX, dtype=np.int8),
        cell_nodes=cells,
        bface_nodes=bface.astype(np.int64),
        bface_tag=tags,
        name=f"sphere_{n}",
    )


def _prisms_to_tets(pr: np.ndarray) -> np.ndarray:
    """Split prisms [n][6] (bottom 012, top 345, 3 over 0) into 3 tets each so that every quad
    face is cut along the diagonal through its smallest node id (the neighbour's split of a
    shared quad agrees, so the tet mesh stays conforming): rotate / flip the prism to put its
    smallest node at slot 0, then the quad (1,2,5,4) decides between the two 3-tet splits."""
    pr = pr.copy()
    m = np.argmin(pr, axis=1)
    flip = m >= 3
    pr[flip] = pr[flip][:, [3, 4, 5, 0, 1, 2]]
    m = np.where(flip, m - 3, m)
    for r in (1, 2):  # rotate the triangles so slot m goes to slot 0
        sel = m == r
        rot = [r, (r + 1) % 3, (r + 2) % 3]
        pr[sel] = pr[sel][:, rot + [x + 3 for x in rot]]
    d15 = np.minimum(pr[:, 1], pr[:, 5]) < np.minimum(pr[:, 2], pr[:, 4])
    a = np.where(d15[:, None], pr[:, [0, 1, 2, 5]], pr[:, [0, 1, 2, 4]])
    b = np.where(d15[:, None], pr[:, [0, 1, 5, 4]], pr[:, [0, 4, 2, 5]])
    c = pr[:, [0, 4, 5, 3]]
    return np.stack([a, b, c], 1).reshape(-1, 4)


def sphere_hybrid(n: int, prism_layers: int | None = None, **shell_kw) -> MeshInput:
    """Hybrid tet/prism sphere mesh (BASELINE.json config 3: "mixed tet/prism cells"): the
    cubed-sphere shell of ``sphere_shell`` with every hex cut into two prisms along the
    (0,2)/(4,6) diagonal of its spherical faces; the first ``prism_layers`` radial layers
    (default half) stay prisms (the boundary layer), the outer ones are split into tets
    (``_prisms_to_tets``).  Wall faces on the sphere and farfield faces outside are triangles.
    Cells: 6 n^2 per radial layer x (2 per prism layer + 6 per tet layer)."""
    sh = sphere_shell(n, **shell_kw)
    hx = sh.cell_nodes
    nr = hx.shape[0] // (6 * n * n)
    prism_layers = nr // 2 if prism_layers is None else prism_layers
    r = np.arange(hx.shape[0]) % nr
    pa = hx[:, [0, 1, 2, 4, 5, 6]]
    pb = hx[:, [0, 2, 3, 4, 6, 7]]
    prisms = np.stack([pa, pb], 1).reshape(-1, 6)
    pr_r = np.repeat(r, 2)
    keep = prisms[pr_r < prism_layers]
    tets = _prisms_to_tets(prisms[pr_r >= prism_layers])
    cells = np.full((keep.shape[0] + tets.shape[0], 8), -1, np.int64)
    cells[:keep.shape[0], :6] = keep
    cells[keep.shape[0]:, :4] = tets
    types = np.concatenate([np.full(keep.shape[0], PRISM), np.full(tets.shape[0], TET)]).astype(np.int8)
    inner, outer = hx[r == 0], hx[r == nr - 1]
    wall = np.concatenate([inner[:, [0, 1, 2]], inner[:, [0, 2, 3]]], 0)
    far = np.concatenate([outer[:, [4, 5, 6]], outer[:, [4, 6, 7]]], 0)
    bf = np.full((wall.shape[0] + far.shape[0], 4), -1, np.int64)
    bf[:wall.shape[0], :3] = wall
    bf[wall.shape[0]:, :3] = far
    tags = np.concatenate([np.full(wall.shape[0], BC_WALL), np.full(far.shape[0], BC_FARFIELD)]).astype(np.int32)
    return MeshInput(xyz=sh.xyz, cell_type=types, cell_nodes=cells, bface_nodes=bf, bface_tag=tags,
                     name=f"sphere_hybrid_{n}_{prism_layers}")


# --------------------------------------------------------------------------- #
# Initial conditions (inputs, not method arithmetic)
# --------------------------------------------------------------------------- #
def _tet_quadrature(order: int = 6):
    """Collapsed (Duffy) Gauss-Legendre product rule on the unit tetrahedron.

    Returns barycentric-free reference points (xi, eta, zeta) and weights that
    sum to 1 (i.e. it computes the MEAN over the tet). Exact for polynomials of
    total degree <= 2*order-3.
    """
    g, w = np.polynomial.legendre.leggauss(order)
    g = 0.5 * (g + 1.0)
    w = 0.5 * w
    pts, wts = [], []
    for a, wa in zip(g, w):
        for b, wb in zip(g, w):
            for c, wc in zip(g, w):
                x = a * (1 - b) * (1 - c)
                y = b * (1 - c)
                z = c
                jac = (1 - b) * (1 - c) ** 2
                pts.append((x, y, z))
                wts.append(wa * wb * wc * jac)
    pts = np.array(pts)
    wts = np.array(wts) * 6.0  # volume of unit tet is 1/6 -> mean weights sum to 1
    return pts, wts


def tet_cell_means(mesh: MeshInput, func, order: int = 6) -> np.ndarray:
    """Mean of ``func(x, y, z)`` over each tet of ``mesh`` by Duffy quadrature."""
    pts, wts = _tet_quadrature(order)
    v = mesh.xyz[mesh.cell_nodes[:, :4]]                # [n, 4, 3]
    e = v[:, 1:, :] - v[:, :1, :]                        # [n, 3, 3]
    X = v[:, None, 0, :] + np.einsum("qk,nkd->nqd", pts, e)
    vals = func(X[..., 0], X[..., 1], X[..., 2])
    return vals @ wts


def kuhn_density_mean(mesh: MeshInput, t: float = 0.0, amp: float = 0.2) -> np.ndarray:
    """Exact mean of rho = 1 + amp*sin(pi(x+y+z-3t)) over each tet.

    For any tet whose vertex values of s = x+y+z are s0, s0+h, s0+2h, s0+3h
    (every Kuhn tet), Hermite-Genocchi gives
        mean sin(pi s) = [G(s0+3h) - 3G(s0+2h) + 3G(s0+h) - G(s0)] / h^3,
    G(s) = cos(pi s)/pi^3.  Falls back to quadrature for other tets.
    """
    v = mesh.xyz[mesh.cell_nodes[:, :4]]
    s = v.sum(axis=-1) - 3.0 * t
    s_sorted = np.sort(s, axis=1)
    d = np.diff(s_sorted, axis=1)
    h = d[:, 0]
    kuhn = np.all(np.abs(d - h[:, None]) < 1e-12 * np.maximum(1.0, np.abs(s_sorted[:, :1])), axis=1) & (h > 0)
    G = lambda x: np.cos(np.pi * x) / np.pi ** 3
    s0 = s_sorted[:, 0]
    out = np.empty(mesh.n_cells)
    hk = h[kuhn]
    s0k = s0[kuhn]
    out[kuhn] = 1.0 + amp * (G(s0k + 3 * hk) - 3 * G(s0k + 2 * hk) + 3 * G(s0k + hk) - G(s0k)) / hk ** 3
    # general tets with well-separated vertex values: the same identity with unequal
    # spacing, mean f(s) = 3! G[s0, s1, s2, s3] (third divided difference, G^(3) = f)
    gap = d.min(axis=1)
    span = s_sorted[:, 3] - s_sorted[:, 0]
    gen = ~kuhn & (gap > 0.05 * np.maximum(span, 1e-300))
    if gen.any():
        x = s_sorted[gen]
        dd = G(x)
        for k in range(1, 4):
            dd = (dd[:, 1:] - dd[:, :-1]) / (x[:, k:] - x[:, :-k])
        out[gen] = 1.0 + amp * 6.0 * dd[:, 0]
        kuhn = kuhn | gen
    if (~kuhn).any():
        sub = MeshInput(xyz=mesh.xyz, cell_type=mesh.cell_type[~kuhn], cell_nodes=mesh.cell_nodes[~kuhn])
        out[~kuhn] = tet_cell_means(sub, lambda x, y, z: 1.0 + amp * np.sin(np.pi * (x + y + z - 3.0 * t)), order=8)
    return out


def advection_ic(mesh: MeshInput, gamma: float = 1.4, t: float = 0.0) -> np.ndarray:
    """Accuracy-test cell averages Q = (rho, rhoU, rhoV, rhoW, rhoE), [n, 5].

    PAPER.md:944-953: rho = 1+0.2 sin(pi(x+y+z)), p = 1, U=V=W=1.  Because U and p
    are constant, mean(rhoU) = mean(rho), mean(rhoE) = 1/(gamma-1) + 1.5 mean(rho).
    ``t`` gives the exact solution's averages at time t (reading R2: x+y+z-3t).
    """
    rho = kuhn_density_mean(mesh, t=t)
    Q = np.empty((mesh.n_cells, 5))
    Q[:, 0] = rho
    Q[:, 1] = rho
    Q[:, 2] = rho
    Q[:, 3] = rho
    Q[:, 4] = 1.0 / (gamma - 1.0) + 1.5 * rho
    return Q


def uniform_state(n_cells: int, rho: float, vel, p: float, gamma: float = 1.4) -> np.ndarray:
    vel = np.asarray(vel, dtype=np.float64)
    Q = np.empty((n_cells, 5))
    Q[:, 0] = rho
    Q[:, 1:4] = rho * vel[None, :]
    Q[:, 4] = p / (gamma - 1.0) + 0.5 * rho * float(vel @ vel)
    return Q


def cell_centroids_simple(mesh: MeshInput) -> np.ndarray:
    """Vertex average (used only to place input patterns, never by the method)."""
    k = mesh.cell_type.astype(np.int64)  # node count = type code (TET 4, PRISM 6, HEX 8)
    out = np.zeros((mesh.n_cells, 3))
    for nv in (4, 6, 8):
        m = k == nv
        if m.any():
            out[m] = mesh.xyz[mesh.cell_nodes[m, :nv]].mean(axis=1)
    return out


def density_step_ic(mesh: MeshInput, gamma: float = 1.4) -> np.ndarray:
    """C1s stress input: rho = 1 where floor(x+y+z) even else 0.5; U=V=W=1, p=1."""
    c = cell_centroids_simple(mesh)
    par = np.floor(c.sum(axis=1)).astype(np.int64) % 2
    rho = np.where(par == 0, 1.0, 0.5)
    Q = np.empty((mesh.n_cells, 5))
    Q[:, 0] = rho
    Q[:, 1:4] = rho[:, None]
    Q[:, 4] = 1.0 / (gamma - 1.0) + 1.5 * rho
    return Q


def spike_state(mesh: MeshInput, amp: float = 30.0, cell: int = 100, gamma: float = 1.4) -> np.ndarray:
    """Positivity-fallback stress input (R21): uniform flow (rho = p = 1, U = (0.5, 0.3, 0.2))
    with one cell of density and pressure x amp; its neighbours' reconstructions overshoot
    below zero at some Gauss points within a step."""
    u = np.array([0.5, 0.3, 0.2])
    Q = uniform_state(mesh.n_cells, 1.0, tuple(u), 1.0, gamma=gamma)
    Q[cell] = [amp, *(amp * u), amp / (gamma - 1.0) + 0.5 * amp * float(u @ u)]
    return Q


def random_smooth_ic(mesh: MeshInput, seed: int = 118, gamma: float = 1.4,
                     base=(1.0, 0.3, 0.1, -0.2, 1.0 / 1.4), amp: float = 0.05) -> np.ndarray:
    """Smooth seeded perturbation of a uniform state (parity IC for C3/C4 and hex boxes).

    rho and p are multiplied by 1 + amp * sum_k sin(k_k . x + phi_k) with four
    random wave vectors k_k in 2*pi*{1..3}^3/Lref and phases from default_rng(seed)
    (SURVEY.md 8(d) "Parity IC for C3/C4").
    """
    rng = np.random.default_rng(seed)
    c = cell_centroids_simple(mesh)
    L = mesh.periodic_length.copy()
    lref = np.where(L > 0, L, 20.0)
    kk = rng.integers(1, 4, size=(4, 3)) * 2 * np.pi / lref[None, :]
    ph = rng.uniform(0, 2 * np.pi, size=4)
    pert = 1.0 + amp * np.sin(c @ kk.T + ph[None, :]).sum(axis=1)
    rho0, u, v, w, p0 = base
    rho = rho0 * pert
    p = p0 * pert
    Q = np.empty((mesh.n_cells, 5))
    Q[:, 0] = rho
    Q[:, 1] = rho * u
    Q[:, 2] = rho * v
    Q[:, 3] = rho * w
    Q[:, 4] = p / (gamma - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
    return Q


def random_states(n: int, seed: int = 20240700, gamma: float = 1.4):
    """Random primitive states for unit tests (SURVEY.md 8(d) 'Unit tests').

    rho, p ~ U[0.1, 10]; Mach ~ U[0, 3] in a random direction.
    Returns (rho, vel[n,3], p).
    """
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.1, 10.0, n)
    p = rng.uniform(0.1, 10.0, n)
    c = np.sqrt(gamma * p / rho)
    ma = rng.uniform(0.0, 3.0, n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    vel = d * (ma * c)[:, None]
    return rho, vel, p
