"""Matrix Market I/O for block-tridiagonal systems (reference mmio.hpp / mmio.cpp).

    write_matrix_market / read_matrix_market   mmio.cpp:30-65  (coordinate real general, 1-based)
    write_plane_vector / read_plane_vector     mmio.cpp:67-84  (one value per line)
    write_system / read_system                 mmio.cpp:86-113 (D_j.mtx, E_j.mtx (j>=1),
                                                                F_j.mtx (j<=n-2), f_j.txt)

Numbers are written like the reference's ``setprecision(17)`` stream (``%.17g``), so a
system written here and one written by the reference's ``acr generate`` are the same
files.  Read blocks go through the PlaneBlock sort/merge (block.cpp:7-29); coordinates
are reconstructed for an nx x nx plane grid when dim is a square, else (i, 0)
(mmio.cpp:13-26).
"""
from __future__ import annotations

import math
import os

import numpy as np

from . import problems as P
from .acr import Error


def _g17(v: float) -> str:
    from .report import fmt_double
    return fmt_double(v)


def grid_coords(dim: int) -> np.ndarray:
    nx = int(round(math.sqrt(dim)))
    if nx * nx == dim:
        return P.plane_coords(nx)
    return np.stack([np.arange(dim, dtype=np.float64), np.zeros(dim)], axis=1)


def write_matrix_market(block, dim: int, path: str) -> None:
    """block = (rows, cols, vals), already merged (a System block)."""
    r, c, v = block
    try:
        with open(path, "w") as out:
            out.write("%%MatrixMarket matrix coordinate real general\n")
            out.write(f"{dim} {dim} {len(r)}\n")
            out.write("".join(f"{int(a) + 1} {int(b) + 1} {_g17(x)}\n" for a, b, x in zip(r, c, v)))
    except OSError:
        raise Error(f"cannot open for writing: {path}") from None


def read_matrix_market(path: str):
    """Returns (dim, (rows, cols, vals)) after the PlaneBlock sort/merge."""
    try:
        fh = open(path)
    except OSError:
        raise Error(f"cannot open for reading: {path}") from None
    with fh:
        first = fh.readline()
        if not first.startswith("%%MatrixMarket"):
            raise Error(f"not a Matrix Market file: {path}")
        line = fh.readline()
        while line and line.startswith("%"):
            line = fh.readline()
        if not line:
            raise Error(f"truncated Matrix Market file: {path}")
        hdr = line.split()
        rows, cols, nnz = int(hdr[0]), int(hdr[1]), int(hdr[2])
        if rows != cols or rows <= 0:
            raise Error(f"plane blocks must be square: {path}")
        toks = fh.read().split()
    if len(toks) < 3 * nnz:
        raise Error(f"truncated entries in: {path}")
    t = np.array(toks[:3 * nnz], dtype=object).reshape(nnz, 3) if nnz else np.zeros((0, 3), object)
    r = t[:, 0].astype(np.int64) - 1
    c = t[:, 1].astype(np.int64) - 1
    v = t[:, 2].astype(np.float64)
    if nnz and (r.min() < 0 or r.max() >= rows or c.min() < 0 or c.max() >= rows):
        raise Error("PlaneBlock: entry index out of range")
    return rows, P._plane_block([r], [c], [v])


def write_plane_vector(v, path: str) -> None:
    try:
        with open(path, "w") as out:
            out.write("".join(_g17(x) + "\n" for x in np.asarray(v, np.float64)))
    except OSError:
        raise Error(f"cannot open for writing: {path}") from None


def read_plane_vector(path: str) -> np.ndarray:
    try:
        with open(path) as fh:
            return np.array([float(t) for t in fh.read().split()], dtype=np.float64)
    except OSError:
        raise Error(f"cannot open for reading: {path}") from None


def write_system(system, directory: str, rhs_index: int = 0) -> None:
    os.makedirs(directory, exist_ok=True)
    n, d = system.n, system.dim
    for j in range(n):
        write_matrix_market(system.D(j), d, os.path.join(directory, f"D_{j}.mtx"))
        write_plane_vector(system.rhs[rhs_index, j], os.path.join(directory, f"f_{j}.txt"))
    for j in range(1, n):
        write_matrix_market(system.E(j), d, os.path.join(directory, f"E_{j}.mtx"))
    for j in range(n - 1):
        write_matrix_market(system.F(j), d, os.path.join(directory, f"F_{j}.mtx"))


def read_system(directory: str, plane_count: int):
    from .acr import DimensionError
    if plane_count < 1:
        raise DimensionError("BlockTridiagonalSystem: need at least one plane")
    blocks, rhs, dims = [], [], []
    for j in range(plane_count):
        dim, b = read_matrix_market(os.path.join(directory, f"D_{j}.mtx"))
        dims.append(dim)
        blocks.append(b)
        rhs.append(read_plane_vector(os.path.join(directory, f"f_{j}.txt")))
    for j in range(1, plane_count):
        dim, b = read_matrix_market(os.path.join(directory, f"E_{j}.mtx"))
        dims.append(dim)
        blocks.append(b)
    for j in range(plane_count - 1):
        dim, b = read_matrix_market(os.path.join(directory, f"F_{j}.mtx"))
        dims.append(dim)
        blocks.append(b)
    d = dims[0]
    if any(x != d for x in dims) or any(len(f) != d for f in rhs):
        raise DimensionError("BlockTridiagonalSystem: plane dimensions disagree")
    return P._assemble(plane_count, d, grid_coords(d), blocks, np.stack(rhs)[None], os.path.basename(directory))
