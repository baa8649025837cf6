"""Host-side checks of the C-ABI library that need no GPU: it builds for sm_100a, loads,
exports every symbol include/lshbloom.h declares, and rejects bad arguments before touching
CUDA.  No compute calls are made here."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2411_04257_b200 as pkg
from paper_2411_04257_b200 import build as libbuild
from paper_2411_04257_b200._native import LSHBloom, LSHBloomError, _Config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lshbloom.h")


@pytest.fixture(scope="module")
def lib():
    libbuild.build()
    return pkg.load_library()


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LSHBLOOM_API\s+[\w\s\*]+?\b(lshbloom_\w+)\s*\(", text)))


def test_header_declares_every_export():
    assert _declared() == sorted(pkg.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libbuild.LIB]).decode()
    exported = set(re.findall(r"\bT (lshbloom_\w+)", out))
    assert set(_declared()) <= exported
    for name in _declared():
        assert hasattr(lib, name)


def test_library_is_sm100a(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libbuild.LIB]).decode()
    assert "sm_100a" in out


def test_header_compiles_as_c():
    src = '#include "lshbloom.h"\nint main(void){ lshbloom_batch b; lshbloom_config c; (void)b; (void)c; return 0; }\n'
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-I",
                           os.path.join(ROOT, "include"), "-x", "c", "-"], input=src.encode(), check=True)


@pytest.mark.parametrize("kw", [
    dict(num_perm=0, b=1, r=1), dict(num_perm=128, b=0, r=8), dict(num_perm=128, b=16, r=9),
    dict(num_perm=2048, b=16, r=8), dict(num_perm=128, b=65, r=1), dict(num_perm=128, b=16, r=0),
])
def test_create_rejects_bad_lsh_params(lib, kw):
    with pytest.raises(LSHBloomError) as e:
        LSHBloom(kw["num_perm"], kw["b"], kw["r"], 1000, 1e-5, 0, device=0)
    assert e.value.code == 1


@pytest.mark.parametrize("fp", [0.0, 1.0, -1.0, 2.0, float("nan")])
def test_create_rejects_bad_fp_rate(lib, fp):
    with pytest.raises(LSHBloomError) as e:
        LSHBloom(128, 16, 8, 1000, fp, 0, device=0)
    assert e.value.code == 1 and "fp_rate" in str(e.value)


def test_create_rejects_bad_sharding_and_size(lib):
    with pytest.raises(LSHBloomError) as e:
        LSHBloom(128, 4, 8, 1000, 1e-5, 0, device=0, rank=2, world=2)
    assert e.value.code == 1
    with pytest.raises(LSHBloomError) as e:
        LSHBloom(128, 4, 8, 1000, 1e-5, 0, device=0, world=5)
    assert e.value.code == 1
    with pytest.raises(LSHBloomError) as e:   # m > 2^36 bits
        LSHBloom(128, 4, 8, 10**10, 1e-9, 0, device=0)
    assert e.value.code == 1
    with pytest.raises(LSHBloomError) as e:   # n_expected = 0
        LSHBloom(128, 4, 8, 0, 1e-5, 0, device=0)
    assert e.value.code == 1


def test_null_pointer_usage_errors(lib):
    vp = ctypes.c_void_p
    lib.lshbloom_destroy(None)                                 # NULL-safe
    assert lib.lshbloom_create_ex(None, ctypes.byref(vp())) == 1
    assert lib.lshbloom_signatures(None, None, None) == 1
    assert lib.lshbloom_query_insert(None, None, None) == 1
    assert lib.lshbloom_reset(None) == 1
    assert lib.lshbloom_launch_count(None) == 0


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(LSHBloomError) as e:
        LSHBloom(128, 16, 8, 1000, 1e-5, 0, device=0)
    assert e.value.code in (3, 4)


def test_product_path_never_imports_oracle():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2411_04257_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "lshbloom_oracle" not in text, f


# --------------------------------------------------------------------------- host planner
# lshbloom_optimal_params / lshbloom_plan are host-only (no CUDA); compared with the oracle's
# independently written planner (pinned in tests/test_oracle_classic.py) and the paper.

@pytest.mark.parametrize("T,num_perm", [(0.8, 128), (0.5, 48), (0.3, 64), (0.9, 32), (0.7, 256), (1.0, 16)])
def test_library_optimal_params_matches_oracle(lib, T, num_perm):
    import oracle
    assert pkg.optimal_params(T, num_perm) == oracle.optimal_params(T, num_perm)


def test_library_plan_matches_oracle_and_paper(lib):
    import oracle
    for n, pe, T, npm in [(5e9, 1e-5, 0.8, 128), (1e10, 1e-10, 0.8, 128), (1e11, 1e-5, 0.8, 128),
                          (39e6, 1e-4, 0.5, 256)]:
        got, want = pkg.plan(int(n), pe, T, npm), oracle.plan(int(n), pe, T, npm)
        for key in ("b", "r", "m", "k", "total_bytes"):
            assert got[key] == want[key], (n, key)
    assert round(pkg.plan(int(5e9), 1e-5)["total_bytes"] / 1e9, 2) == 160.51     # Table 1


def test_library_planner_rejects_bad_arguments(lib):
    for T in (0.0, 1.5, float("nan")):
        with pytest.raises(LSHBloomError):
            pkg.optimal_params(T, 128)
    with pytest.raises(LSHBloomError):
        pkg.optimal_params(0.8, 1)
    with pytest.raises(LSHBloomError):
        pkg.plan(0, 1e-5)
    with pytest.raises(LSHBloomError):
        pkg.plan(100, 1.0)
