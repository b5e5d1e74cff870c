"""The C++ drop-in shim (include/bsfv_sip.hpp) compiles against the C-ABI
library and maps statuses to the reference's exception classes."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1303_4538_b200")


def build(tmp_path):
    exe = str(tmp_path / "shim_example")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_example.cpp"), "-L", LIBDIR,
                    "-lsip_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_reports_missing_device(tmp_path):
    exe = build(tmp_path)
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present (covered by the gpu test)")
    except Exception:
        pass
    r = subprocess.run([exe, "8"], capture_output=True, text=True)
    assert r.returncode == 3 and "CUDA error" in r.stdout


@pytest.mark.gpu
def test_shim_solve_matches_oracle(gpu, tmp_path):
    from oracle import oracle as O
    exe = build(tmp_path)
    for prec, flag in (("f64", "d"), ("f32", "s")):
        r = subprocess.run([exe, "12", flag], capture_output=True, text=True, check=True)
        out = r.stdout.splitlines()
        assert out[-1] == "misuse ok" and out[-3] == "stale ok", out[-3:]
        norms = np.array([float(x) for x in out[:-3]])
        A = O.generate(0, 1303, (12, 12, 12))
        ref = O.solve(A, O.field(12, 12, 12), 0.92, 5, prec)
        np.testing.assert_allclose(norms, ref, rtol=1e-12)
        # residual_general (fp64) of phi0 = 0 is su: its L1 is sum |Q|
        l1 = float(out[-2].split()[-1])
        np.testing.assert_allclose(l1, np.abs(A["Q"][1:-1, 1:-1, 1:-1]).sum(), rtol=1e-12)


def build_flow(tmp_path):
    exe = str(tmp_path / "flow_example")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "flow_example.cpp"), "-L", LIBDIR,
                    "-lsip_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_flow_shim_compiles_and_reports_missing_device(tmp_path):
    exe = build_flow(tmp_path)
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present (covered by the gpu test)")
    except Exception:
        pass
    r = subprocess.run([exe, "8"], capture_output=True, text=True)
    assert r.returncode == 3 and "CUDA error" in r.stdout


@pytest.mark.gpu
def test_flow_shim_reuses_one_factorization(gpu, tmp_path):
    """PressureSolver (C++ shim): 100 pressure_correct steps on one
    factorisation, NonConvergenceError carries the defect."""
    exe = build_flow(tmp_path)
    r = subprocess.run([exe, "16"], capture_output=True, text=True, check=True)
    out = r.stdout.splitlines()
    assert out[-1] == "factorizations 1" and out[-2] == "noconv ok", out[-2:]
    steps = [ln.split() for ln in out if ln.startswith("step")]
    assert len(steps) == 4
    for s in steps:
        d0, d1 = float(s[5]), float(s[7])
        assert int(s[3]) >= 1 and d1 <= 0.1 * d0


REF_INCLUDE = "/root/reference/proj/include"


def build_ref(tmp_path):
    exe = str(tmp_path / "shim_ref_example")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "shim_ref_example.cpp"), "-L", LIBDIR,
                    "-lsip_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers only in the build container")
def test_shim_with_reference_field_and_errors(tmp_path):
    """The shim compiled against the reference's own headers: bsfv::FieldD as
    the field type and BSFV_SIP_USE_REFERENCE_ERRORS=1, so a library failure
    surfaces as the reference's bsfv::Error (here: no CUDA device)."""
    exe = build_ref(tmp_path)
    try:
        import torch
        gpu = torch.cuda.is_available()
    except Exception:
        gpu = False
    r = subprocess.run([exe, "8"], capture_output=True, text=True)
    if gpu:
        out = r.stdout.splitlines()
        assert r.returncode == 0 and out[-2] == "factorizations 1" and out[-1] == "stale ok", out
    else:
        assert r.returncode == 3 and r.stdout.startswith("bsfv::Error: sip_create: CUDA error"), r.stdout
