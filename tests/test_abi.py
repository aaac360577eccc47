"""C ABI boundary (CPU-only): libtpgpu.so loads, exports every function that
include/tpgpu.h declares, and the ctypes mirror matches the C struct layout.
No compute call is made here (no GPU in the CPU suite)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2502_21013_b200 import abi, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tpgpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", text)) - {"tp_iterate_cb"})


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(api.EXPORTS)


def test_version_and_defaults_without_gpu():
    lib = api.lib()
    assert lib.tp_version() == 1
    cfg = abi.TpSolverCfg()
    lib.tp_solver_cfg_default(C.byref(cfg))
    ref = abi.default_cfg()
    for f, _ in abi.TpSolverCfg._fields_:
        if f == "threads":
            continue
        assert getattr(cfg, f) == getattr(ref, f), f


@pytest.mark.parametrize("config", [0, 1, 2, 3, 4, 5])
def test_baseline_descriptors(config):
    d = api.baseline_desc(config)
    assert d.cells in (32, 256, 512, 1024, 2048)
    assert d.steps in (64, 256, 512, 1024, 2048)
    assert 1 <= d.n_materials <= abi.TP_MAX_MATERIALS


def test_unknown_config_is_invalid_argument():
    with pytest.raises(ValueError):
        api.baseline_desc(42)


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    structs = {"tp_rect": abi.TpRect, "tp_material": abi.TpMaterial,
               "tp_problem_desc": abi.TpProblemDesc, "tp_solver_cfg": abi.TpSolverCfg,
               "tp_report": abi.TpReport}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, val = line.split()
        py = structs[cname]
        got = C.sizeof(py) if field == "size" else getattr(py, field).offset
        assert got == int(val), (cname, field, got, val)


def test_problem_create_without_gpu_fails_loudly():
    """No silent CPU fallback: without a usable device creation is an error."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    with pytest.raises(RuntimeError):
        api.Problem(api.baseline_desc(0))


def test_tpfem_adapter_compiles_against_reference_headers(tmp_path):
    """include/tpgpu_tpfem.hpp (the reference-side binding) type-checks
    against the reference's own headers (shim SparseSolver for Eigen)."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers not present")
    src = tmp_path / "use.cpp"
    src.write_text('#include "tpgpu_tpfem.hpp"\n'
                   "int f(){ tp_problem_desc d; tp_problem_desc_baseline(0,&d);"
                   " tpgpu::GpuProblem p(d); tpfem::SolverConfig c; c.tol=1e-8;"
                   " auto U0 = tpgpu::static_init(p, c); tpgpu::choose_nu_hat(p, c);"
                   " auto r = tpgpu::solve_m1_fixed_point(p, U0, c); return r.second.iterations; }\n"
                   "int g(){ auto m = tpfem::build_rectilinear_mesh(tpfem::transformer_regions(), 40, 40);"
                   " tpgpu::GpuMeshProblem p(m, tpfem::MaterialTable::transformer(), 64, 0.02);"
                   " tpfem::SolverConfig c; auto U0 = tpgpu::static_init(p, c); tpgpu::choose_nu_hat(p, c);"
                   " return tpgpu::solve_m1_fixed_point(p, U0, c).second.iterations; }\n")
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "oracle", "shim"),
                    "-I", ref_inc, "-I", os.path.join(ROOT, "include"), str(src)], check=True)
