"""General-mesh path, CPU side: the C ABI of
include/tpgpu_mesh.h is exported, its structs match the ctypes mirror, and the
host mesher restated in libtpgpu (build_rectilinear_mesh + refine_uniform +
transformer_regions, mesh.hpp:105-246) reproduces the reference mesher bit
for bit; the reference's own mesh tests (tests/test_mesh.cpp) restated on it.
No device call is made here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2502_21013_b200 import api, mesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tpgpu_mesh.h")


def test_library_exports_every_mesh_symbol():
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    names = sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", text)))
    lib = api.lib()
    assert [n for n in names if not hasattr(lib, n)] == []
    assert set(names) == set(mesh.MESH_EXPORTS)


def test_mesh_struct_layout_matches_c(tmp_path):
    structs = {"tp_exp_material": mesh.TpExpMaterial, "tp_mesh_desc": mesh.TpMeshDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, val = line.split()
        py = structs[cname]
        got = C.sizeof(py) if field == "size" else getattr(py, field).offset
        assert got == int(val), (cname, field, got, val)


def areas(V, T):
    a, b, c = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    return 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))


def test_transformer_mesh_40x40_has_2142_dofs():
    # proj/test_output.txt:40 (acceptance: transformer 40x40 = 2142 DoF)
    V, T, R, n = mesh.transformer_mesh(40, 40, 0)
    assert n == 2142


@pytest.mark.parametrize("refinements", [0, 1, 2])
def test_transformer_geometry(refinements):
    # Mesh.TriangleAreasArePositiveAndSumToDomain / UniformRefinementPreservesGeometry
    V, T, R, n = mesh.transformer_mesh(40, 40, refinements)
    A = areas(V, T)
    assert (A > 0).all()
    assert abs(A.sum() - 0.355 * 0.466) < 1e-12
    # every region of the painter's list is present, winding areas as drawn
    for reg, area in ((3, 2 * 0.013 * 0.22), (4, 2 * 0.013 * 0.22)):
        assert abs(A[R == reg].sum() - area) < 1e-12


def test_refinement_quadruples_triangles_and_keeps_parents():
    V0, T0, R0, n0 = mesh.transformer_mesh(20, 16, 0)
    V1, T1, R1, n1 = mesh.transformer_mesh(20, 16, 1)
    assert len(T1) == 4 * len(T0)
    assert np.array_equal(V1[:len(V0)], V0)       # parents keep their numbers
    assert np.array_equal(R1, np.repeat(R0, 4))   # children inherit the label
    assert n1 > n0                                # Mesh.RefinementGrowsDofCount


def test_invalid_mesh_arguments_raise():
    with pytest.raises(ValueError):
        mesh.transformer_mesh(0, 40, 0)
    with pytest.raises(ValueError):
        mesh.transformer_mesh(40, 40, -1)


@pytest.mark.parametrize("nx,ny,refinements", [(40, 40, 0), (40, 40, 1), (13, 7, 0), (80, 60, 1), (40, 40, 2)])
def test_mesher_matches_reference_bitwise(ref, nx, ny, refinements):
    V, T, R, n = mesh.transformer_mesh(nx, ny, refinements)
    Vr, Tr, Rr, nr = ref.tr_mesh(nx, ny, refinements)
    assert n == nr
    assert V.shape == Vr.shape and np.array_equal(V.view(np.uint64), Vr.view(np.uint64))
    assert np.array_equal(T, Tr) and np.array_equal(R, Rr)


def test_transformer_material_table_matches_reference(ref):
    m = mesh.transformer_materials()
    mr = (mesh.TpExpMaterial * 5)()
    assert ref._trlib().tpref_tr_material(mr) == 0
    for r in range(5):
        for f, _ in mesh.TpExpMaterial._fields_:
            assert getattr(m[r], f) == getattr(mr[r], f), (r, f)


def test_mesh_problem_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    with pytest.raises(RuntimeError):
        mesh.MeshProblem.transformer()


def test_oracle_transformer_matches_golden(ref):
    """The checker (the reference's own transformer pipeline in oracle/_ref)
    reproduces the committed fixture bit for bit (same host arithmetic)."""
    from paper_2502_21013_b200.abi import default_cfg
    g = np.load(os.path.join(ROOT, "tests", "golden", "transformer_reference.npz"))
    c = ref.tr_cfg(nx=12, ny=10, steps=8, j_amp=9.5e5)
    cfg = default_cfg(tol=1e-8)
    U0, counts = ref.tr_static_init(c, cfg)
    nu, q = ref.tr_choose_nu_hat(c, U0, cfg)
    r = ref.tr_solve_m1(c, nu, q, U0, cfg)
    assert np.array_equal(counts, g["small_newton_counts"]) and r.iterations == int(g["small_iterations"])
    assert np.array_equal(U0, g["small_U0"]) and np.array_equal(r.U, g["small_U"])
