"""CPU checks of the C-ABI library: it loads, exports every symbol include/hgks.h
declares, and its host-side setup (geometry, faces, stencils, partition) agrees
with the oracle's independently built tables.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_00656_b200 import hgks, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hgks.h")).read()
    return sorted(set(re.findall(r"\b(hgks_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = hgks.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(hgks.EXPORTS)
    assert b"sm_100a" in lib.hgks_version()


def test_library_contains_sm100a_cubin():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", hgks.lib()._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("mk", [lambda: W.kuhn_box(6), lambda: W.kuhn_box(5, jitter=0.1),
                                lambda: W.cartesian_hex_box(5, jitter=0.1), lambda: W.hybrid_box(6, jitter=0.1),
                                lambda: W.hybrid_box(5, prism_layers=5), lambda: W.walled_hybrid_box(5)])
def test_host_setup_matches_oracle_counts(mk):
    mi = mk()
    m = hgks.Mesh(mi)
    info = m.info()
    om = O.OracleMesh(mi)
    assert info["n_cells_global"] == om.n_cells == info["n_owned"]
    assert info["n_faces"] == om.n_faces
    assert info["stencil_min"] == om.min_stencil and info["stencil_max"] == om.max_stencil
    assert info["n_sub"] == om.n_subs
    assert info["n_ghost"] == 0 and info["n_peers"] == 0 and info["n_bghost"] == om.n_ghosts
    assert info["n_early_cells"] == info["n_owned"] and info["n_early_faces"] == info["n_faces"] - info["n_faces_bc"]


def test_sphere_shell_boundary_faces():
    mi = W.sphere_shell(4)
    m = hgks.Mesh(mi)
    info = m.info()
    om = O.OracleMesh(mi)
    assert info["n_cells_global"] == 6 * 4 * 4 * 8
    assert info["n_faces"] == om.n_faces
    assert info["n_faces_bc"] == 2 * 6 * 16 == om.n_ghosts == info["n_bghost"]


def test_errors_are_reported_not_thrown():
    mi = W.kuhn_box(4)
    bad = W.MeshInput(xyz=mi.xyz, cell_type=mi.cell_type.copy(), cell_nodes=mi.cell_nodes.copy(),
                      periodic_length=mi.periodic_length)
    bad.cell_nodes[3, 1] = 10 ** 9
    with pytest.raises(hgks.HgksError) as e:
        hgks.Mesh(bad)
    assert e.value.code == 2 and "cell 3" in str(e.value)
    mixed = W.MeshInput(xyz=mi.xyz, cell_type=mi.cell_type.copy(), cell_nodes=mi.cell_nodes,
                        periodic_length=mi.periodic_length)
    mixed.cell_type[5] = 8
    with pytest.raises(hgks.HgksError) as e:
        hgks.Mesh(mixed)
    assert e.value.code == 2
    openm = W.MeshInput(xyz=mi.xyz, cell_type=mi.cell_type, cell_nodes=mi.cell_nodes)  # not periodic
    with pytest.raises(hgks.HgksError) as e:
        hgks.Mesh(openm)
    assert e.value.code == 2 and "boundary face" in str(e.value)
    with pytest.raises(hgks.HgksError):
        hgks.Mesh(W.kuhn_box(2))  # periodic box too small for the 2-layer stencil


def test_workspace_size_scales_with_cells():
    cfg = hgks.SolverConfig()
    a = hgks.Mesh(W.kuhn_box(6)).workspace_size(cfg)
    b = hgks.Mesh(W.kuhn_box(12)).workspace_size(cfg)
    per_cell = (b - a) / (6 * 12 ** 3 - 6 * 6 ** 3)
    # operators 198 doubles + record 50 + state/face/update data: ~2.5-3.5 KB per tet
    assert 2000 < per_cell < 4000, per_cell


def test_solver_without_cuda_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has CUDA")
    mi = W.kuhn_box(4)
    with pytest.raises(RuntimeError, match="CUDA"):
        hgks.Solver(hgks.Mesh(mi), W.advection_ic(mi))


def test_ctypes_structs_match_header_layout(tmp_path):
    """The binding's ctypes structures have the header's field offsets and sizes
    (compiled with gcc against include/hgks.h): no silent drift of the ABI."""
    import subprocess
    pairs = [("hgks_mesh_desc", hgks.MeshDesc), ("hgks_config", hgks.Config), ("hgks_dist", hgks.Dist),
             ("hgks_mesh_stats", hgks.MeshStats), ("hgks_step_info", hgks.StepInfo)]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hgks.h"', "int main(void) {"]
    for cname, cls in pairs:
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, cls in pairs:
        assert got[(cname, "size")] == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert got[(cname, fname)] == getattr(cls, fname).offset, (cname, fname)


def test_p2p_and_put_map_argument_errors():
    """HGKS_TRANSPORT_P2P setup calls and the put map report bad arguments as status
    codes (no GPU needed): NULL handles -> HGKS_E_ARG; rank out of range -> HGKS_E_ARG."""
    L = hgks.lib()
    buf = (ctypes.c_uint8 * hgks.P2P_HANDLE_BYTES)()
    assert L.hgks_p2p_export(None, ctypes.cast(buf, ctypes.c_void_p)) == 1
    assert L.hgks_p2p_connect(None, ctypes.cast(buf, ctypes.c_void_p)) == 1
    mesh = hgks.Mesh(W.kuhn_box(8, 8, 6, h=0.25), n_ranks=2)
    with pytest.raises(hgks.HgksError) as e:
        mesh.put_map(2)
    assert e.value.code == 1
    rr, row = mesh.put_map(1)
    assert rr.size == mesh.info(1)["send_cells"] and set(rr.tolist()) == {0}


def test_hybrid_sphere_counts_and_volume():
    """Hybrid sphere (f4): the prism/tet split of the cubed-sphere shell keeps its volume
    (oracle geometry of both meshes), every wall / farfield face is a triangle, and the host
    setup's counts equal the oracle's."""
    mi = W.sphere_hybrid(4)
    assert set(np.unique(mi.cell_type).tolist()) == {W.TET, W.PRISM}
    assert np.all(mi.bface_nodes[:, 3] == -1)
    info = hgks.Mesh(mi).info()
    om = O.OracleMesh(mi)
    assert info["n_faces"] == om.n_faces and info["n_bghost"] == om.n_ghosts == 2 * 2 * 6 * 16
    assert info["stencil_min"] == om.min_stencil and info["stencil_max"] == om.max_stencil
    hs = W.sphere_shell(4)
    V = om.geometry()[0][: mi.n_cells].sum()
    Vh = O.OracleMesh(hs).geometry()[0][: hs.n_cells].sum()
    assert abs(V - Vh) <= 1e-12 * Vh
