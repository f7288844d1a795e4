"""The C-ABI library (libaz.so) loads without a GPU and exports every entry point that
include/az.h declares; the Python binding registers argument types for each of them.  No compute
call is made (CPU-only check)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "az.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(az_[A-Za-z0-9_]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def libpath():
    from paper_2308_14490_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    return B.LIB


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for n in ["az_plan_create", "az_plan_destroy", "az_apply_A", "az_apply_At", "az_apply_Zstar", "az_solve"]:
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    missing = [n for n in _declared() if not hasattr(L, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol(libpath):
    from paper_2308_14490_b200 import _lib
    declared = set(_declared())
    assert set(_lib.EXPORTED) <= declared
    missing = declared - set(_lib.EXPORTED)
    assert not missing, missing


def test_status_strings_without_gpu(libpath):
    L = ctypes.CDLL(libpath)
    L.az_status_string.restype = ctypes.c_char_p
    L.az_status_string.argtypes = [ctypes.c_int]
    assert L.az_status_string(0)
    assert L.az_status_string(100)


def test_library_exports_nothing_undeclared(libpath):
    """Every exported az_* symbol of libaz.so is declared in include/az.h (no hidden entry points)."""
    import shutil
    import subprocess
    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("az_")}
    extra = exported - set(_declared())
    assert not extra, sorted(extra)


def test_only_tests_bench_and_smoke_import_the_oracle():
    """The oracle is test infrastructure: outside tests/ and oracle/ itself, only bench.py (its CPU
    baseline legs) and __graft_entry__.py (smoke) may import it; the product package never does."""
    import ast
    allowed = {"bench.py", "__graft_entry__.py"}
    offenders = []
    for dirpath, _, files in os.walk(ROOT):
        rel = os.path.relpath(dirpath, ROOT)
        if rel.split(os.sep)[0] in ("tests", "oracle", ".git", "build", "baseline", "gpurun_out"):
            continue
        for f in files:
            if not f.endswith(".py"):
                continue
            path = os.path.join(dirpath, f)
            if os.path.relpath(path, ROOT) in allowed:
                continue
            tree = ast.parse(open(path).read())
            for node in ast.walk(tree):
                mods = []
                if isinstance(node, ast.Import):
                    mods = [a.name for a in node.names]
                elif isinstance(node, ast.ImportFrom) and node.module:
                    mods = [node.module]
                if any(m == "oracle" or m.startswith("oracle.") for m in mods):
                    offenders.append(os.path.relpath(path, ROOT))
    assert not offenders, offenders
