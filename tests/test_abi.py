"""The C-ABI library (include/truncmul_b200.h) loads, exports every declared
symbol, and the host-side mirror behaves like the reference's API on the
parts that need no GPU."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import paper_1703_00640_b200 as tm
from paper_1703_00640_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    L = _native.load()
    names = _native.header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    for name in names:
        assert f" T {name}" in out, name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_last_error():
    L = _native.load()
    assert b"sm_100a" in L.tmg_version()
    with pytest.raises(tm.InputOutOfRange):
        tm.required_precision(tm.Mode.LOW, 0, 10)
    assert "chunk width" in _native.last_error()


def test_no_cpu_fallback_without_device():
    """On a machine without a usable GPU the product path must fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(tm.CudaError):
        tm.Context(0)


def test_limbs_round_trip_and_range():
    rng = np.random.default_rng(0)
    for n in (1, 63, 64, 65, 1000):
        x = int.from_bytes(rng.bytes((n + 7) // 8), "little") & ((1 << n) - 1)
        a = tm.to_limbs(x, n)
        assert len(a) == (n + 63) // 64
        assert tm.from_limbs(a) == x
        with pytest.raises(tm.InputOutOfRange):
            tm.to_limbs(1 << n, n)
    with pytest.raises(tm.InputOutOfRange):
        tm.to_limbs(-1, 10)
    with pytest.raises(tm.InputOutOfRange):
        tm.to_limbs(np.array([0, 1], dtype=np.uint64), 64)
    assert len(tm.to_limbs(np.array([5], dtype=np.uint64), 200)) == 4


def test_params_c_round_trip():
    p = tm.select_params(1 << 20, tm.Mode.HIGH)
    assert tm.Params.from_c(p.to_c()) == p


def _build_c_demo(tmp_path):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_1703_00640_b200")
    exe = str(tmp_path / "c_abi_demo")
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "c_abi_demo.c"), "-L", lib, "-ltruncmul_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    """The header is plain C: a C program that uses the ABI builds and links."""
    assert os.path.exists(_build_c_demo(tmp_path))


@pytest.mark.gpu
def test_c_demo_runs(tmp_path):
    """Full/low/high products from C against a schoolbook product, the
    precision refusal and its escalation."""
    import subprocess
    r = subprocess.run([_build_c_demo(tmp_path)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout


def _build_cpp_demo(tmp_path):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_1703_00640_b200")
    exe = str(tmp_path / "cpp_api_demo")
    subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "cpp_api_demo.cpp"), "-L", lib, "-ltruncmul_b200",
                    "-Wl,-rpath," + lib, "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_cpp_api_parameters(tmp_path):
    """The C++ host API (truncmul_b200.hpp: products.hpp names and errors.hpp
    exceptions over the C-ABI) builds, and its parameter functions run
    without a GPU: select/validate/required_precision, the fallback mode and
    the InputOutOfRange / UnsupportedLength exceptions."""
    import subprocess
    env = dict(os.environ, TMG_DEMO_PARAMS_ONLY="1")
    r = subprocess.run([_build_cpp_demo(tmp_path)], capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "params OK" in r.stdout


@pytest.mark.gpu
def test_cpp_api_products(tmp_path):
    """Full/low/high products through the C++ host API against a schoolbook
    product, and the reference's exceptions (InputOutOfRange,
    ConvolutionPrecisionFailure) raised from C-ABI error codes."""
    import subprocess
    r = subprocess.run([_build_cpp_demo(tmp_path)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout.splitlines()[-1]


@pytest.mark.gpu
def test_every_context_option_is_accepted():
    """Every TMG_OPT_* the header declares is handled by
    tmg_context_set_option (and an unknown one is refused)."""
    import re
    import paper_1703_00640_b200 as tm
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hdr = open(os.path.join(root, "include", "truncmul_b200.h")).read()
    opts = {m.group(1): int(m.group(2)) for m in re.finditer(r"(TMG_OPT_\w+)\s*=\s*(\d+)", hdr)}
    assert len(opts) >= 14
    c = tm.Context(0)
    for name, val in opts.items():
        assert getattr(tm._native, name) == val, name
        c.set_option(val, 0)
    with pytest.raises(tm.InputOutOfRange):
        c.set_option(999, 1)
    c.close()
