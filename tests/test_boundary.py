"""CPU-side checks of the drop-in boundary: libacrgpu.so loads, exports every
symbol include/acrgpu.h declares, and its structure compiler reproduces the
reference's cluster / block cluster trees exactly (checked against the oracle,
which restates proj/core/src/cluster.cpp:39-126)."""
import os
import re

import numpy as np
import pytest

from paper_1701_00182_b200 import acr, problems as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "acrgpu.h")).read()
    return sorted(set(re.findall(r"\b(acrgpu_[a-z_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    L = acr.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(acr.SYMBOLS)
    assert b"sm_100a" in L.acrgpu_version()


@pytest.mark.parametrize("side,leaf,eta,weak", [(16, 8, 2.0, False), (32, 32, 2.0, False), (64, 32, 2.0, False),
                                                (32, 16, 2.0, True), (12, 8, 2.0, False), (10, 4, 1.0, False),
                                                (128, 64, 2.0, False)])
def test_structure_matches_oracle(oracle, side, leaf, eta, weak):
    coords = P.plane_coords(side)
    perm, leaves = acr.structure(coords, leaf, eta, weak)
    s = oracle.Structure(coords, leaf, eta, weak)
    assert np.array_equal(perm, s.perm())
    assert np.array_equal(leaves, s.leaves())


def test_structure_counts_survey():
    # C1 210 dense / 274 Rk; C2-C4 1004 / 1634; C5 2116 / 3954
    for side, leaf, nd, nk in ((32, 32, 210, 274), (64, 32, 1004, 1634), (128, 64, 2116, 3954)):
        _, leaves = acr.structure(P.plane_coords(side), leaf)
        assert (leaves[:, 4] == 0).sum() == nd
        assert (leaves[:, 4] == 1).sum() == nk


def test_structure_errors():
    with pytest.raises(acr.UsageError):
        acr.structure(np.zeros((0, 2)), 32)
    with pytest.raises(acr.UsageError):
        acr.structure(P.plane_coords(4), 0)
    with pytest.raises(acr.UsageError):
        acr.structure(P.plane_coords(4), 4, eta=0.0)


def test_dense_mode_rejected():
    with pytest.raises(acr.UsageError):
        acr._cfg(acr.AcrConfig(mode=acr.ArithmeticMode.Dense))


SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "shim", "acr_shim_check.cpp")


def build_shim(out):
    """INTEGRATION.md §2's reference-side C++ shim, compiled against include/acrgpu.h and
    linked with libacrgpu.so (stand-ins for the Eigen-based reference types)."""
    import subprocess
    from paper_1701_00182_b200 import build as B
    lib = B.build()
    libdir = os.path.dirname(lib)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["g++", "-std=c++17", "-O1", "-Wall", "-Wno-misleading-indentation", "-Werror",
                    "-I", os.path.join(root, "include"), SHIM, "-L", libdir, "-lacrgpu",
                    f"-Wl,-rpath,{libdir}", "-o", out], check=True)
    return out


def test_cpp_shim_compiles_and_links(tmp_path):
    exe = build_shim(str(tmp_path / "acr_shim_check"))
    assert os.path.exists(exe)
