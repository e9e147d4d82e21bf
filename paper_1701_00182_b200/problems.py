"""Seeded block-tridiagonal systems: the reference's generators and the
BASELINE.json configurations C1-C5.

Layout (shared by the product C-ABI ``include/acrgpu.h`` and the CPU oracle):
a system of ``n`` planes of ``dim`` unknowns is stored as 3n-2 sparse plane
blocks in COO form -- blocks ``0..n-1`` are D(j), ``n..2n-2`` are E(j) for
j = 1..n-1 (E(j) couples plane j to plane j-1), ``2n-1..3n-3`` are F(j) for
j = 0..n-2 (couples j to j+1); block b owns entries ``blk_off[b]:blk_off[b+1]``.
This is ``BlockTridiagonalSystem`` (reference proj/core/include/acr/block.hpp:67-92)
flattened.  Right-hand sides are ``rhs[r, j, i]`` (RHS r, plane j, point i).

Generators:
  poisson(n)            reference assemble_poisson   (proj/core/src/discretize.cpp:46-71)
  poisson2d_block(n)    reference poisson2d_block    (discretize.cpp:227-242)
  convdiff_vortex(n, alpha, a)  reference assemble_convdiff (discretize.cpp:73-174)
  helmholtz_fem(n, kappa)       reference assemble_helmholtz (discretize.cpp:176-214)
  assemble(kind, n, ...)        reference assemble(ProblemSpec) (discretize.hpp:55)
  config_system(k)      BASELINE.json configs[k-1] with the builder decisions of
                        SURVEY.md §8(d) (documented in DESIGN.md §2).
The portable RNG is splitmix64 -> 53-bit doubles; Box-Muller for
N(0,1).  It replaces the reference's implementation-defined std::uniform_real.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(seed: int, stream: int, count: int) -> np.ndarray:
    """``count`` splitmix64 outputs of the counter sequence keyed by (seed, stream)."""
    base = np.uint64((seed * 0x632BE59BD9B4E019 + stream * 0x9E3779B97F4A7C15 + 0x1234567) & 0xFFFFFFFFFFFFFFFF)
    i = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = base + i * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, stream: int, count: int) -> np.ndarray:
    z = splitmix64(seed, stream, count)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform_pm1(seed: int, stream: int, count: int) -> np.ndarray:
    return 2.0 * uniform01(seed, stream, count) - 1.0


def normal(seed: int, stream: int, count: int) -> np.ndarray:
    m = (count + 1) // 2
    u = uniform01(seed, stream, 2 * m)
    u1 = np.maximum(u[:m], 1e-300)
    u2 = u[m:]
    r = np.sqrt(-2.0 * np.log(u1))
    out = np.concatenate([r * np.cos(2 * math.pi * u2), r * np.sin(2 * math.pi * u2)])
    return out[:count]


@dataclasses.dataclass
class System:
    """A block-tridiagonal system in the shared COO layout (see module doc)."""

    n: int
    dim: int
    coords: np.ndarray      # (dim, 2) float64, plane point coordinates
    blk_off: np.ndarray     # (3n-1,) int64
    rows: np.ndarray        # int32
    cols: np.ndarray        # int32
    vals: np.ndarray        # float64
    rhs: np.ndarray         # (nrhs, n, dim) float64
    name: str = ""

    @property
    def nblocks(self) -> int:
        return 3 * self.n - 2

    @property
    def total_dim(self) -> int:
        return self.n * self.dim

    def block(self, b: int):
        s, e = int(self.blk_off[b]), int(self.blk_off[b + 1])
        return self.rows[s:e], self.cols[s:e], self.vals[s:e]

    def D(self, j):
        return self.block(j)

    def E(self, j):  # couples j -> j-1, j in [1, n)
        return self.block(self.n + j - 1)

    def F(self, j):  # couples j -> j+1, j in [0, n-1)
        return self.block(2 * self.n - 1 + j)

    def apply(self, u: np.ndarray) -> np.ndarray:
        """y_j = E_j u_{j-1} + D_j u_j + F_j u_{j+1} (reference block.cpp:89-107).
        u: (nrhs, n, dim) or (n, dim)."""
        squeeze = u.ndim == 2
        if squeeze:
            u = u[None]
        y = np.zeros_like(u)
        n = self.n
        for j in range(n):
            r, c, v = self.D(j)
            np.add.at(y[:, j], (slice(None), r), (v[None, :] * u[:, j][:, c]))
            if j > 0:
                r, c, v = self.E(j)
                np.add.at(y[:, j], (slice(None), r), (v[None, :] * u[:, j - 1][:, c]))
            if j < n - 1:
                r, c, v = self.F(j)
                np.add.at(y[:, j], (slice(None), r), (v[None, :] * u[:, j + 1][:, c]))
        return y[0] if squeeze else y

    def relative_residual(self, u: np.ndarray, rhs: np.ndarray | None = None) -> float:
        """||A u - f||_2 / ||f||_2 over all planes and RHS (reference block.cpp:109-123)."""
        f = self.rhs if rhs is None else rhs
        if u.ndim == 2:
            u = u[None]
        if f.ndim == 2:
            f = f[None]
        fn = float(np.sum(f * f))
        if fn == 0.0:
            raise ZeroDivisionError("relative residual undefined: right-hand side has zero norm")
        r = self.apply(u) - f
        return math.sqrt(float(np.sum(r * r)) / fn)

    def to_dense(self) -> np.ndarray:
        """Full operator (small n only; reference block.cpp:74-86)."""
        N = self.total_dim
        A = np.zeros((N, N))
        d = self.dim
        for j in range(self.n):
            r, c, v = self.D(j)
            np.add.at(A, (j * d + r, j * d + c), v)
            if j > 0:
                r, c, v = self.E(j)
                np.add.at(A, (j * d + r, (j - 1) * d + c), v)
            if j < self.n - 1:
                r, c, v = self.F(j)
                np.add.at(A, (j * d + r, (j + 1) * d + c), v)
        return A


def plane_coords(n: int) -> np.ndarray:
    """Grid node coordinates ((i+1)h, (j+1)h), index j*n+i (discretize.cpp:12-19)."""
    h = 1.0 / (n + 1)
    j, i = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    return np.stack([(i.ravel() + 1) * h, (j.ravel() + 1) * h], axis=1).astype(np.float64)


def _assemble(n, dim, coords, blocks, rhs, name=""):
    """blocks: list of (rows, cols, vals) in block order D.., E(1..), F(..n-2)."""
    counts = [len(b[0]) for b in blocks]
    off = np.zeros(len(blocks) + 1, dtype=np.int64)
    off[1:] = np.cumsum(counts)
    rows = np.concatenate([np.asarray(b[0], np.int32) for b in blocks]) if blocks else np.zeros(0, np.int32)
    cols = np.concatenate([np.asarray(b[1], np.int32) for b in blocks]) if blocks else np.zeros(0, np.int32)
    vals = np.concatenate([np.asarray(b[2], np.float64) for b in blocks]) if blocks else np.zeros(0)
    return System(n, dim, np.ascontiguousarray(coords, np.float64), off, rows, cols, vals,
                  np.ascontiguousarray(rhs, np.float64), name)


def _stencil_block(n, center, west, east, south, north):
    j, i = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i = i.ravel()
    j = j.ravel()
    r = j * n + i
    m = n * n
    rs, cs, vs = [r], [r], [np.broadcast_to(np.asarray(center, np.float64), (m,))]
    for mask, off, coef in ((i > 0, -1, west), (i < n - 1, 1, east), (j > 0, -n, south), (j < n - 1, n, north)):
        c = np.broadcast_to(np.asarray(coef, np.float64), (m,))
        rs.append(r[mask])
        cs.append(r[mask] + off)
        vs.append(c[mask])
    rows = np.concatenate(rs)
    cols = np.concatenate(cs)
    vals = np.concatenate(vs)
    order = np.lexsort((cols, rows))
    return rows[order].astype(np.int32), cols[order].astype(np.int32), vals[order].astype(np.float64)


def _diag_block(m, diag):
    r = np.arange(m, dtype=np.int32)
    return r, r.copy(), np.broadcast_to(np.asarray(diag, np.float64), (m,)).copy()


def _constant_coeff(n, center, west, east, south, north, elow, fhigh, rhs, name):
    m = n * n
    coords = plane_coords(n)
    D = _stencil_block(n, center, west, east, south, north)
    E = _diag_block(m, elow)
    F = _diag_block(m, fhigh)
    blocks = [D] * n + [E] * (n - 1) + [F] * (n - 1)
    return _assemble(n, m, coords, blocks, rhs, name)


def poisson(n: int, rhs: np.ndarray | None = None) -> System:
    """Reference assemble_poisson: 7-point star, h^2-scaled, centre 6, E=F=-I,
    f = h^2 (proj/core/src/discretize.cpp:46-71)."""
    if n < 2:
        raise ValueError("GridSpec: n must be >= 2")
    h = 1.0 / (n + 1)
    if rhs is None:
        rhs = np.full((1, n, n * n), h * h)
    return _constant_coeff(n, 6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, rhs, f"poisson{n}")


def poisson2d_block(n: int):
    """Reference poisson2d_block: 5-point 2D Laplacian plane block (centre 4)
    (discretize.cpp:227-242).  Returns (rows, cols, vals, coords)."""
    r, c, v = _stencil_block(n, 4.0, -1.0, -1.0, -1.0, -1.0)
    return r, c, v, plane_coords(n)


def identity_system(n: int, dim: int, rhs: np.ndarray) -> System:
    """n identity planes, no coupling (proj/tests/test_helpers.hpp:50-62)."""
    side = int(round(math.sqrt(dim)))
    coords = np.stack([np.arange(dim) % side, np.arange(dim) // side], axis=1).astype(np.float64)
    I = _diag_block(dim, 1.0)
    Z = (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    blocks = [I] * n + [Z] * (2 * (n - 1))
    return _assemble(n, dim, coords, blocks, rhs.reshape(1, n, dim), "identity")


# ----------------------------------------------------------------------------
# BASELINE.json configurations (SURVEY.md §8(d) builder decisions)
# ----------------------------------------------------------------------------

def seeded_rhs(seed: int, nrhs: int, n: int, dim: int) -> np.ndarray:
    return uniform_pm1(seed, 1, nrhs * n * dim).reshape(nrhs, n, dim)


def kappa_field(n: int, seed: int) -> np.ndarray:
    """kappa = exp(g) on the (n+2)^3 node lattice (boundary nodes included):
    g i.i.d. N(0,1), three 3x3x3 box-filter passes with clamp padding, then
    standardised and scaled so max(g)-min(g) = ln(100) (contrast exactly 100)."""
    g = normal(seed, 2, (n + 2) ** 3).reshape(n + 2, n + 2, n + 2)
    for _ in range(3):
        p = np.pad(g, 1, mode="edge")
        acc = np.zeros_like(g)
        for dz in range(3):
            for dy in range(3):
                for dx in range(3):
                    acc += p[dz:dz + n + 2, dy:dy + n + 2, dx:dx + n + 2]
        g = acc / 27.0
    g = (g - g.mean()) / g.std()
    g = g * (math.log(100.0) / (g.max() - g.min()))
    return np.exp(g)  # indexed [z, y, x]


def vardiff(n: int, seed: int, nrhs: int = 1, name: str = "") -> System:
    """-div(kappa grad u) = f, 7-point FD, harmonic-mean face coefficients,
    h^2-scaled, symmetric (BASELINE configs 2 and 5)."""
    kap = kappa_field(n, seed)
    m = n * n

    def face(a, b):
        return 2.0 * a * b / (a + b)

    inner = kap[1:n + 1, 1:n + 1, 1:n + 1]  # [z, y, x] of the unknowns
    kw = face(inner, kap[1:n + 1, 1:n + 1, 0:n])
    ke = face(inner, kap[1:n + 1, 1:n + 1, 2:n + 2])
    ks = face(inner, kap[1:n + 1, 0:n, 1:n + 1])
    kn = face(inner, kap[1:n + 1, 2:n + 2, 1:n + 1])
    kd = face(inner, kap[0:n, 1:n + 1, 1:n + 1])
    ku = face(inner, kap[2:n + 2, 1:n + 1, 1:n + 1])
    center = kw + ke + ks + kn + kd + ku
    Ds, Es, Fs = [], [], []
    for z in range(n):
        Ds.append(_stencil_block(n, center[z].ravel(), -kw[z].ravel(), -ke[z].ravel(), -ks[z].ravel(), -kn[z].ravel()))
    for z in range(1, n):
        Es.append(_diag_block(m, -kd[z].ravel()))
    for z in range(n - 1):
        Fs.append(_diag_block(m, -ku[z].ravel()))
    rhs = seeded_rhs(seed, nrhs, n, m)
    return _assemble(n, m, plane_coords(n), Ds + Es + Fs, rhs, name or f"vardiff{n}")


def convdiff_upwind(n: int, seed: int, beta: float = 50.0, nrhs: int = 1) -> System:
    """-lap u + beta.grad u, beta = (b,b,b), first-order upwind (backward
    differences for b > 0), h^2-scaled, nonsymmetric (BASELINE config 3)."""
    h = 1.0 / (n + 1)
    bh = beta * h
    rhs = seeded_rhs(seed, nrhs, n, n * n)
    return _constant_coeff(n, 6.0 + 3.0 * bh, -1.0 - bh, -1.0, -1.0 - bh, -1.0, -1.0 - bh, -1.0, rhs,
                           f"convdiff{n}")


def helmholtz7(n: int, seed: int, omega: float = 2 * math.pi * 6.4, nrhs: int = 1) -> System:
    """-lap u - omega^2 u, 7-point FD, h^2-scaled; RHS = unit point source at
    node (n/2, n/2, n/2) plus 1e-3 * U[-1,1] (BASELINE config 4)."""
    h = 1.0 / (n + 1)
    rhs = 1e-3 * seeded_rhs(seed, nrhs, n, n * n)
    c = n // 2
    rhs[:, c, c * n + c] += 1.0
    return _constant_coeff(n, 6.0 - omega * omega * h * h, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0, rhs,
                           f"helmholtz{n}")


# ----------------------------------------------------------------------------
# The reference's own generators behind acr::assemble (discretize.hpp:10-55)
# ----------------------------------------------------------------------------

PROBLEM_KINDS = ("poisson", "convdiff", "helmholtz")


def parse_problem_kind(name: str) -> str:
    """discretize.cpp:25-30 (UsageError on unknown names is raised by the caller's layer)."""
    if name not in PROBLEM_KINDS:
        raise ValueError(f"unknown problem kind: {name}")
    return name


def helmholtz_kappa_for(n: int) -> float:
    """~12 points per wavelength (discretize.cpp:41-44)."""
    return n / 2.0


def _plane_block(entries_r, entries_c, entries_v):
    """PlaneBlock construction (block.cpp:7-29): sort by (row, col) -- stable, so
    duplicates keep their insertion order -- then sum duplicates left to right."""
    r = np.concatenate(entries_r).astype(np.int64)
    c = np.concatenate(entries_c).astype(np.int64)
    v = np.concatenate(entries_v).astype(np.float64)
    order = np.lexsort((c, r))  # lexsort is stable
    r, c, v = r[order], c[order], v[order]
    if len(r) == 0:
        return r.astype(np.int32), c.astype(np.int32), v
    new = np.ones(len(r), bool)
    new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    starts = np.flatnonzero(new)
    out_v = np.add.reduceat(v, starts)  # runs of <= 8 duplicates sum left to right
    return r[starts].astype(np.int32), c[starts].astype(np.int32), out_v


def convdiff_vortex(n: int, alpha: float, a: float = 1.0) -> System:
    """Reference assemble_convdiff (discretize.cpp:73-174): 7-point diffusion plus
    alpha * b(x).grad u with the three-component vortex field b and first-order upwind
    differences, h^2-scaled; the right-hand side is A applied to the sampled reference
    solution sum_d sin(pi x_d) + sin(3 pi x_d), which is returned as ``exact``."""
    if alpha < 0:
        raise ValueError("assemble_convdiff: alpha must be nonnegative")
    if n < 2:
        raise ValueError("GridSpec: n must be >= 2")
    h = 1.0 / (n + 1)
    m = n * n
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i = ii.ravel()
    j = jj.ravel()
    r = j * n + i
    x = (i + 1) * h
    y = (j + 1) * h
    t = 2.0 * math.pi * a
    Dblocks, Eblocks, Fblocks = [], [], []
    for z in range(n):
        zc = (z + 1) * h
        # per-row insertion order of the reference: centre, W, E, S, N, then E/F -1,
        # then the three upwind terms.  Stable sorting keeps that order within a row,
        # so build columns of (row, insertion slot) and sort once.
        dr, dc, dv, ds = [], [], [], []
        er, ec, ev = [], [], []
        fr, fc, fv = [], [], []

        def add(lst, rows, cols, vals, slot):
            lst[0].append(rows)
            lst[1].append(cols)
            lst[2].append(np.broadcast_to(np.asarray(vals, np.float64), rows.shape).copy())
            if len(lst) > 3:
                lst[3].append(np.full(rows.shape, slot))

        D = (dr, dc, dv, ds)
        add(D, r, r, 6.0, 0)
        msk = i > 0
        add(D, r[msk], r[msk] - 1, -1.0, 1)
        msk = i < n - 1
        add(D, r[msk], r[msk] + 1, -1.0, 2)
        msk = j > 0
        add(D, r[msk], r[msk] - n, -1.0, 3)
        msk = j < n - 1
        add(D, r[msk], r[msk] + n, -1.0, 4)
        er.append(r)
        ec.append(r)
        ev.append(np.full(m, -1.0))
        fr.append(r)
        fc.append(r)
        fv.append(np.full(m, -1.0))
        if alpha != 0.0:
            b1 = np.sin(t * x) * np.sin(t * (0.125 + y)) + np.sin(t * (0.125 + zc)) * np.sin(t * x)
            b2 = np.cos(t * x) * np.cos(t * (0.125 + y)) + np.cos(t * (0.125 + y)) * np.cos(t * zc)
            b3 = np.cos(t * x) * np.cos(t * (0.125 + zc)) + np.sin(t * (0.125 + y)) * np.sin(t * zc)
            slot = 5
            for bd, lo_in, hi_in, off, axis in ((b1, i > 0, i < n - 1, 1, 0), (b2, j > 0, j < n - 1, n, 1),
                                                (b3, None, None, 0, 2)):
                c = alpha * h * bd
                nz = c != 0.0
                pos = nz & (bd > 0)
                neg = nz & ~(bd > 0)
                # diagonal: +c when bd > 0, -c otherwise (both inserted into D)
                add(D, r[pos], r[pos], c[pos], slot)
                add(D, r[neg], r[neg], -c[neg], slot)
                if axis < 2:
                    lo = pos & lo_in
                    add(D, r[lo], r[lo] - off, -c[lo], slot + 1)
                    hi = neg & hi_in
                    add(D, r[hi], r[hi] + off, c[hi], slot + 1)
                else:
                    if z > 0:
                        er.append(r[pos])
                        ec.append(r[pos])
                        ev.append(-c[pos])
                    if z < n - 1:
                        fr.append(r[neg])
                        fc.append(r[neg])
                        fv.append(c[neg])
                slot += 2
        # reference order within a row: insertion order; rows interleave, so sort by
        # (row, slot) first to reproduce it, then the PlaneBlock sort/merge
        R = np.concatenate(dr)
        S = np.concatenate(ds)
        o = np.lexsort((S, R))
        Dblocks.append(_plane_block([R[o]], [np.concatenate(dc)[o]], [np.concatenate(dv)[o]]))
        Eblocks.append(_plane_block(er, ec, ev))
        Fblocks.append(_plane_block(fr, fc, fv))
    u = np.empty((n, m))
    for z in range(n):
        zc = (z + 1) * h
        u[z] = (np.sin(math.pi * x) + np.sin(math.pi * y) + math.sin(math.pi * zc) +
                np.sin(3 * math.pi * x) + np.sin(3 * math.pi * y) + math.sin(3 * math.pi * zc))
    blocks = Dblocks + Eblocks[1:] + Fblocks[:-1]
    sysm = _assemble(n, m, plane_coords(n), blocks, np.zeros((1, n, m)), f"convdiff_vortex{n}")
    sysm.rhs = sysm.apply(u[None])
    sysm.exact = u
    return sysm


def helmholtz_fem(n: int, kappa: float) -> System:
    """Reference assemble_helmholtz (discretize.cpp:176-214): 27-point trilinear FEM
    K - kappa^2 M from 1D stiffness/mass stencils; D/E/F are 9-point plane blocks;
    f = h^3."""
    if n < 2:
        raise ValueError("GridSpec: n must be >= 2")
    h = 1.0 / (n + 1)
    m = n * n
    k1 = (-1.0 / h, 2.0 / h, -1.0 / h)
    m1 = (h / 6.0, 4.0 * h / 6.0, h / 6.0)
    w = np.zeros((3, 3, 3))
    for dz in range(3):
        for dy in range(3):
            for dx in range(3):
                w[dx, dy, dz] = (k1[dx] * m1[dy] * m1[dz] + m1[dx] * k1[dy] * m1[dz] + m1[dx] * m1[dy] * k1[dz]
                                 - kappa * kappa * m1[dx] * m1[dy] * m1[dz])
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    i = ii.ravel()
    j = jj.ravel()
    r = j * n + i
    out = {0: ([], [], []), 1: ([], [], []), 2: ([], [], [])}
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            ok = (i + dx >= 0) & (i + dx < n) & (j + dy >= 0) & (j + dy < n)
            c = (j + dy) * n + (i + dx)
            for dz in range(3):
                out[dz][0].append(r[ok])
                out[dz][1].append(c[ok])
                out[dz][2].append(np.full(int(ok.sum()), w[dx + 1, dy + 1, dz]))
    D = _plane_block(*out[1])
    E = _plane_block(*out[0])
    F = _plane_block(*out[2])
    blocks = [D] * n + [E] * (n - 1) + [F] * (n - 1)
    return _assemble(n, m, plane_coords(n), blocks, np.full((1, n, m), h ** 3), f"helmholtz_fem{n}")


def assemble(kind: str, n: int, alpha: float = 0.0, a: float = 1.0, kappa: float = 0.0) -> System:
    """acr::assemble(ProblemSpec) (discretize.hpp:55; report.cpp:333-339 passes kappa
    through, 0 meaning helmholtz_kappa_for(n) at the CLI)."""
    kind = parse_problem_kind(kind)
    if kind == "poisson":
        return poisson(n)
    if kind == "convdiff":
        return convdiff_vortex(n, alpha, a)
    return helmholtz_fem(n, kappa if kappa > 0 else helmholtz_kappa_for(n))


def first_planes(sysm: System, k: int) -> System:
    """The first k planes of a system (its leading k x k block sub-system: D_0..D_{k-1},
    E_1..E_{k-1}, F_0..F_{k-2}, rhs planes 0..k-1).  Used to exercise a configuration's
    full plane size (e.g. C5's 16384-point planes, leaf 64) with fewer planes."""
    if not 1 <= k <= sysm.n:
        raise ValueError("first_planes: need 1 <= k <= n")
    n = sysm.n
    blocks = [sysm.block(j) for j in range(k)]
    blocks += [sysm.block(n + j - 1) for j in range(1, k)]
    blocks += [sysm.block(2 * n - 1 + j) for j in range(k - 1)]
    return _assemble(k, sysm.dim, sysm.coords, blocks, sysm.rhs[:, :k], f"{sysm.name}[:{k}]")


#: BASELINE.json configs (1-based).  ``n`` may be overridden for parity-size runs.
CONFIGS = {
    1: dict(kind="poisson", n=32, leaf=32, eps=1e-6, nrhs=1),
    2: dict(kind="vardiff", n=64, leaf=32, eps=1e-6, nrhs=1),
    3: dict(kind="convdiff", n=64, leaf=32, eps=1e-6, nrhs=1),
    4: dict(kind="helmholtz", n=64, leaf=32, eps=1e-4, nrhs=1),
    5: dict(kind="vardiff", n=128, leaf=64, eps=1e-6, nrhs=16),
}


def config_system(k: int, n: int | None = None, seed: int = 2024, nrhs: int | None = None) -> System:
    c = CONFIGS[k]
    n = c["n"] if n is None else n
    nrhs = c["nrhs"] if nrhs is None else nrhs
    if c["kind"] == "poisson":
        sysm = poisson(n, rhs=seeded_rhs(seed, nrhs, n, n * n))
    elif c["kind"] == "vardiff":
        sysm = vardiff(n, seed, nrhs)
    elif c["kind"] == "convdiff":
        sysm = convdiff_upwind(n, seed, nrhs=nrhs)
    else:
        sysm = helmholtz7(n, seed, nrhs=nrhs)
    sysm.name = f"C{k}:{c['kind']}{n}"
    return sysm
