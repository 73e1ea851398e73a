"""CPU-only checks of the C-ABI boundary (no compute calls without a GPU):
the library builds for sm_100a, loads, exports every symbol include/crius.h
declares, and validates its inputs before touching the device."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2403_16125_b200 as pkg
from paper_2403_16125_b200 import build as B
from paper_2403_16125_b200 import workload as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    return pkg.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "crius.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(crius_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("crius_load_profiles", "crius_enumerate_cells", "crius_estimate_cells",
              "crius_schedule_round"):
        assert s in syms
    assert sorted(pkg.EXPORTS) == syms


def test_library_exports_every_declared_symbol(L):
    out = subprocess.check_output(["nm", "-D", "--defined-only", pkg.LIB_PATH]).decode()
    exported = set(re.findall(r" T (crius_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(L, s)


def test_library_is_sm100a(L):
    out = subprocess.check_output(["cuobjdump", "--list-elf", pkg.LIB_PATH]).decode()
    assert "sm_100a" in out


def _load(pr, **over):
    """Call crius_load_profiles with the binding's marshalling; returns (code, msg)."""
    cr = pkg.Crius.__new__(pkg.Crius)
    cr._keep = []
    cl, jb, cf = pkg.Crius._structs(cr, pr)
    for k, v in over.items():
        setattr(cf, k, v)
    ctx = C.c_void_p()
    code = pkg.lib().crius_load_profiles(C.byref(ctx), C.byref(cl), C.byref(jb), C.byref(cf), 0,
                                         None)
    return code, pkg.lib().crius_last_error().decode()


@pytest.mark.parametrize("mutate,needle", [
    (lambda pr: pr.ng.__setitem__(0, 3), "N_G must be a power of two"),
    (lambda pr: pr.gb.__setitem__(0, 6), "global batch"),
    (lambda pr: pr.cap.__setitem__(0, 5), "capacity"),
    (lambda pr: pr.gpn.__setitem__(1, 3), "gpus_per_node"),
    (lambda pr: pr.kst.__setitem__(0, 0), "k_state"),
    (lambda pr: setattr(pr, "g_max", 128), "g_max"),
    (lambda pr: setattr(pr, "depth", 17), "search_depth"),
    (lambda pr: setattr(pr, "s_max", 0), "s_max"),
])
def test_loader_rejects_bad_inputs(L, mutate, needle):
    pr = W.make_config(2)
    mutate(pr)
    code, msg = _load(pr)
    assert code == 2 and needle in msg, msg


def test_loader_rejects_bad_b_values(L):
    pr = W.make_config(3)
    pr.b_values = np.array([1, 4, 2], np.int32)
    code, msg = _load(pr)
    assert code == 2 and "ascending" in msg


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU error path")
def test_no_gpu_fails_loudly(L):
    code, msg = _load(W.make_config(1))
    assert code == 4 and "no CUDA device" in msg
    with pytest.raises(pkg.CriusError):
        pkg.Crius(W.make_config(1))


def test_product_path_does_not_import_oracle():
    """The product package never references the oracle (test infrastructure)."""
    pkg_dir = os.path.join(ROOT, "paper_2403_16125_b200")
    for root, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                assert "import oracle" not in src and "crius_oracle" not in src, f
