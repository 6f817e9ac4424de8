"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the aFSAI method's arithmetic (SURVEY.md §8(c),
task rule ③): it only builds SPD matrices shaped like the paper's test
problems (Table 1, P:1183-1205 weak-scaling Poisson) and
right-hand sides.  Every matrix it returns is a full (both triangles) CSR with
strictly increasing columns per row, the diagonal present and positive, and
BITWISE symmetric values (each off-diagonal value is computed once and
mirrored).

Layout of a returned ``CSR``: ``rowptr`` int64[n+1], ``col`` int32[nnz],
``val`` float64[nnz] (the C-ABI layout of include/afsai.h).

Seeds: numpy PCG64 with the root seed 20101417, one ``spawn`` child per purpose
(SURVEY.md §8(d) "Concrete synthetic inputs").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ROOT_SEED = 20101417

# purpose -> spawn index (stable; never reorder)
_PURPOSES = {
    "hetero_K": 0,
    "fe_E": 1,
    "rhs": 2,
    "random_spd": 3,
    "random_sparse": 4,
    "sample_rows": 5,
    "vectors": 6,
}


def rng(purpose: str, sub: int = 0) -> np.random.Generator:
    """Deterministic generator for one purpose (and an optional sub-stream)."""
    ss = np.random.SeedSequence(ROOT_SEED)
    child = ss.spawn(len(_PURPOSES))[_PURPOSES[purpose]]
    if sub:
        child = child.spawn(sub + 1)[sub]
    return np.random.Generator(np.random.PCG64(child))


@dataclass
class CSR:
    n: int
    rowptr: np.ndarray  # int64[n+1]
    col: np.ndarray     # int32[nnz]
    val: np.ndarray     # float64[nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col.astype(np.int64), self.rowptr), shape=(self.n, self.n))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.rowptr))
        d[rows, self.col] = self.val
        return d

    def bandwidth(self) -> int:
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.rowptr))
        return int(np.max(np.abs(rows - self.col.astype(np.int64)))) if self.nnz else 0


def _from_row_blocks(n: int, cols: np.ndarray, vals: np.ndarray, valid: np.ndarray, name: str) -> CSR:
    """cols/vals/valid: shape (n, k) with each row's candidate columns already ascending."""
    cnt = valid.sum(axis=1).astype(np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    return CSR(n, rowptr, cols[valid].astype(np.int32), vals[valid].astype(np.float64), name)


def from_dense(a: np.ndarray, name: str = "dense") -> CSR:
    """Full CSR of a dense symmetric matrix, storing only nonzeros (diagonal always kept)."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    mask = (a != 0.0) | np.eye(n, dtype=bool)
    cols = np.broadcast_to(np.arange(n), (n, n))
    return _from_row_blocks(n, cols, a, mask, name)


def from_dense_full(a: np.ndarray, name: str = "dense_full") -> CSR:
    """Full CSR storing every entry (explicit zeros included)."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    cols = np.broadcast_to(np.arange(n), (n, n))
    return _from_row_blocks(n, cols, a, np.ones((n, n), dtype=bool), name)


# ---------------------------------------------------------------- stencils
def tridiag(n: int, diag: float = 2.0, off: float = -1.0) -> CSR:
    """1D Laplacian tri(off, diag, off) (SURVEY.md §8(c) pin P2)."""
    offs = np.array([-1, 0, 1])
    i = np.arange(n)[:, None]
    cols = i + offs[None, :]
    valid = (cols >= 0) & (cols < n)
    vals = np.where(offs[None, :] == 0, diag, off) * np.ones((n, 1))
    return _from_row_blocks(n, np.where(valid, cols, 0), vals, valid, f"tri{n}")


def poisson2d(nx: int, ny: int) -> CSR:
    """2D 5-point Laplacian, x fastest, Dirichlet truncation: diag 4, off-diagonals -1
    (BASELINE.json configs[0])."""
    n = nx * ny
    idx = np.arange(n, dtype=np.int64)
    x, y = idx % nx, idx // nx
    offs = [(0, -1), (-1, 0), (0, 0), (1, 0), (0, 1)]  # (dx, dy) in ascending column order
    cols = np.empty((n, 5), dtype=np.int64)
    valid = np.empty((n, 5), dtype=bool)
    vals = np.empty((n, 5))
    for k, (dx, dy) in enumerate(offs):
        xx, yy = x + dx, y + dy
        valid[:, k] = (xx >= 0) & (xx < nx) & (yy >= 0) & (yy < ny)
        cols[:, k] = np.where(valid[:, k], xx + nx * yy, 0)
        vals[:, k] = 4.0 if (dx, dy) == (0, 0) else -1.0
    return _from_row_blocks(n, cols, vals, valid, f"poisson2d_{nx}x{ny}")


def poisson3d(nx: int, ny: int | None = None, nz: int | None = None) -> CSR:
    """3D 7-point Poisson, natural order (x fastest), Dirichlet truncation: diag 6,
    off-diagonals -1 (SPEC.md S:522-530 generate_poisson7; PAPER.md P:1195-1196;
    BASELINE.json configs[1])."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    cols = np.empty((n, 7), dtype=np.int64)
    valid = np.empty((n, 7), dtype=bool)
    vals = np.empty((n, 7))
    for k, (dx, dy, dz) in enumerate(offs):
        xx, yy, zz = x + dx, y + dy, z + dz
        valid[:, k] = (xx >= 0) & (xx < nx) & (yy >= 0) & (yy < ny) & (zz >= 0) & (zz < nz)
        cols[:, k] = np.where(valid[:, k], xx + nx * (yy + ny * zz), 0)
        vals[:, k] = 6.0 if (dx, dy, dz) == (0, 0, 0) else -1.0
    return _from_row_blocks(n, cols, vals, valid, f"poisson3d_{nx}x{ny}x{nz}")


def hetero_poisson3d(nx: int, ny: int | None = None, nz: int | None = None,
                     aniso=(1.0, 1.0, 0.01), sigma: float = 1.0) -> CSR:
    """Cell-centred FV 7-point discretisation of -div(K grad u):
    K_cell = exp(2*sigma*xi), xi iid N(0,1); face transmissibility
    T = aniso_axis * 2*Ka*Kb/(Ka+Kb) (commutative -> exactly symmetric); Dirichlet walls
    add aniso_axis*2*K_cell to the diagonal; diag = fixed-order sum of the 6 face terms
    (-z, -y, -x, +x, +y, +z).  Off-diagonal = -T."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n = nx * ny * nz
    K = np.exp(2.0 * sigma * rng("hetero_K").standard_normal(n))
    idx = np.arange(n, dtype=np.int64)
    x, y, z = idx % nx, (idx // nx) % ny, idx // (nx * ny)
    face_order = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    terms = {}
    nbr = {}
    for (dx, dy, dz) in face_order:
        a = aniso[0] if dx else (aniso[1] if dy else aniso[2])
        xx, yy, zz = x + dx, y + dy, z + dz
        inside = (xx >= 0) & (xx < nx) & (yy >= 0) & (yy < ny) & (zz >= 0) & (zz < nz)
        j = np.where(inside, xx + nx * (yy + ny * zz), 0)
        Kb = K[j]
        T_in = a * ((2.0 * (K * Kb)) / (K + Kb))   # K*Kb and K+Kb are commutative in fp
        T_wall = a * (2.0 * K)
        terms[(dx, dy, dz)] = np.where(inside, T_in, T_wall)
        nbr[(dx, dy, dz)] = (inside, j, T_in)
    diag = np.zeros(n)
    for f in face_order:
        diag = diag + terms[f]
    col_order = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), None, (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    cols = np.empty((n, 7), dtype=np.int64)
    valid = np.empty((n, 7), dtype=bool)
    vals = np.empty((n, 7))
    for k, f in enumerate(col_order):
        if f is None:
            cols[:, k], valid[:, k], vals[:, k] = idx, True, diag
        else:
            inside, j, T_in = nbr[f]
            cols[:, k], valid[:, k], vals[:, k] = j, inside, -T_in
    return _from_row_blocks(n, cols, vals, valid, f"hetero3d_{nx}x{ny}x{nz}")


# ---------------------------------------------------------------- FE elasticity
def _q1_hex_stiffness(nu: float = 0.3) -> np.ndarray:
    """24x24 stiffness of a unit-cube trilinear hex, E = 1, 2x2x2 Gauss; local node
    l = lx + 2*ly + 4*lz, dof-minor (3*l + d).  Made bitwise symmetric."""
    c = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu))
    D = np.zeros((6, 6))
    D[:3, :3] = nu
    np.fill_diagonal(D[:3, :3], 1.0 - nu)
    D[3:, 3:] = np.eye(3) * (1.0 - 2.0 * nu) / 2.0
    D *= c
    g = 1.0 / np.sqrt(3.0)
    pts = [(-g + 1) / 2, (g + 1) / 2]   # Gauss points mapped to [0,1]
    Ke = np.zeros((24, 24))
    for px in pts:
        for py in pts:
            for pz in pts:
                dN = np.zeros((8, 3))
                for l in range(8):
                    lx, ly, lz = l & 1, (l >> 1) & 1, (l >> 2) & 1
                    fx = px if lx else 1 - px
                    fy = py if ly else 1 - py
                    fz = pz if lz else 1 - pz
                    sx = 1.0 if lx else -1.0
                    sy = 1.0 if ly else -1.0
                    sz = 1.0 if lz else -1.0
                    dN[l] = (sx * fy * fz, fx * sy * fz, fx * fy * sz)
                B = np.zeros((6, 24))
                for l in range(8):
                    B[0, 3 * l + 0] = dN[l, 0]
                    B[1, 3 * l + 1] = dN[l, 1]
                    B[2, 3 * l + 2] = dN[l, 2]
                    B[3, 3 * l + 0] = dN[l, 1]; B[3, 3 * l + 1] = dN[l, 0]
                    B[4, 3 * l + 1] = dN[l, 2]; B[4, 3 * l + 2] = dN[l, 1]
                    B[5, 3 * l + 0] = dN[l, 2]; B[5, 3 * l + 2] = dN[l, 0]
                Ke += B.T @ D @ B * 0.125   # weight 1 per point on [-1,1]^3 -> det J = 1/8
    return (Ke + Ke.T) / 2.0


def fe_elasticity(N: int, nu: float = 0.3, hetero: bool = True) -> CSR:
    """Synthetic 3D hexahedral FE elasticity, shaped like the
    paper's geomechanics matrices: Q1 hexes, h = 1, 2x2x2 Gauss,
    N x N x N free nodes (the z = 0 plane is clamped and eliminated), 3 dof/node,
    node-major, x fastest; per-element log10 E ~ U(-1, 1).  Couplings summed in
    ascending element order, then the strictly-upper part is mirrored from the lower."""
    n = 3 * N * N * N
    step = 3 * N * N * max(1, 2_000_000 // (3 * N * N))   # whole node planes, ~2M rows per slab
    if n <= step:
        return fe_elasticity_rows(N, 0, n, nu, hetero)
    # large N (M5): slabs of rows (bitwise the full matrix's rows), concatenated;
    # bounded peak memory instead of the (n/3) x 27 x 3 x 3 block array at once
    parts = [fe_elasticity_rows(N, a, min(n, a + step), nu, hetero) for a in range(0, n, step)]
    nnz = sum(p.nnz for p in parts)
    rowptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    r = e = 0
    rowptr[0] = 0
    for p in parts:
        rowptr[r + 1: r + p.n + 1] = p.rowptr[1:] + e
        col[e: e + p.nnz] = p.col
        val[e: e + p.nnz] = p.val
        r += p.n
        e += p.nnz
    return CSR(n, rowptr, col, val, f"fe_{N}")


def fe_elasticity_rows(N: int, row_lo: int, row_hi: int, nu: float = 0.3, hetero: bool = True) -> CSR:
    """Rows [row_lo, row_hi) of fe_elasticity(N), bitwise identical to the full
    matrix's rows (every node's couplings depend only on its own coordinates and the
    global element moduli; the mirror needs the blocks of nodes one plane away).
    Returned as a CSR with n = row_hi - row_lo rows, GLOBAL column indices, and
    attribute n_cols = 3 N^3 (multi-GPU slabs without building the whole matrix)."""
    Ke = _q1_hex_stiffness(nu)
    ne_x = N - 1
    ne_z = N
    n_el = ne_x * ne_x * ne_z
    if hetero:
        E = 10.0 ** rng("fe_E").uniform(-1.0, 1.0, n_el)
    else:
        E = np.ones(n_el)
    nn_all = N * N * N
    node_lo, node_hi = row_lo // 3, -(-row_hi // 3)
    halo = N * N + N + 1
    g_lo, g_hi = max(0, node_lo - halo), min(nn_all, node_hi + halo)
    a = np.arange(g_lo, g_hi, dtype=np.int64)   # computed nodes (slab + mirror halo)
    nn = len(a)
    ax, ay, az = a % N, (a // N) % N, a // (N * N) + 1   # az: physical plane index 1..N
    offsets = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    dindex = {d: k for k, d in enumerate(offsets)}
    blocks = np.zeros((nn, 27, 3, 3))
    # la descending == element id ascending for a fixed node pair
    for la in range(7, -1, -1):
        lx, ly, lz = la & 1, (la >> 1) & 1, (la >> 2) & 1
        ex, ey, ez = ax - lx, ay - ly, az - lz   # element origin (physical)
        ok = (ex >= 0) & (ex < ne_x) & (ey >= 0) & (ey < ne_x) & (ez >= 0) & (ez < ne_z)
        eid = np.where(ok, ex + ne_x * (ey + ne_x * ez), 0)
        Ee = np.where(ok, E[eid], 0.0)
        for lb in range(8):
            mx, my, mz = lb & 1, (lb >> 1) & 1, (lb >> 2) & 1
            d = (mx - lx, my - ly, mz - lz)
            bz = ez + mz   # physical plane of node b; must be free (>= 1)
            okb = ok & (bz >= 1)
            blk = Ke[3 * la:3 * la + 3, 3 * lb:3 * lb + 3]
            contrib = np.where(okb[:, None, None], Ee[:, None, None] * blk[None], 0.0)
            k = dindex[d]
            blocks[:, k] = blocks[:, k] + contrib
    # neighbour validity (node b exists and is free), for the slab nodes only
    s0, s1 = node_lo - g_lo, node_hi - g_lo
    asl = a[s0:s1]
    sx, sy, sz = ax[s0:s1], ay[s0:s1], az[s0:s1]
    ns = len(asl)
    valid = np.zeros((ns, 27), dtype=bool)
    bidx = np.zeros((ns, 27), dtype=np.int64)
    for k, (dx, dy, dz) in enumerate(offsets):
        bx, by, bz = sx + dx, sy + dy, sz + dz
        v = (bx >= 0) & (bx < N) & (by >= 0) & (by < N) & (bz >= 1) & (bz <= N)
        valid[:, k] = v
        bidx[:, k] = np.where(v, bx + N * (by + N * (bz - 1)), g_lo)
    # mirror: upper entries (3b+j > 3a+i) := lower entries of the transposed block
    rows_g = 3 * asl[:, None, None, None] + np.arange(3)[None, None, :, None]
    cols_g = 3 * bidx[:, :, None, None] + np.arange(3)[None, None, None, :]
    upper = (cols_g > rows_g) & valid[:, :, None, None]
    opp = np.array([dindex[(-dx, -dy, -dz)] for (dx, dy, dz) in offsets])
    mirrored = blocks[bidx - g_lo, opp[None, :]]     # (ns, 27, 3, 3) block of (b, -d)
    mirrored = np.swapaxes(mirrored, 2, 3)
    blocks = np.where(upper, mirrored, blocks[s0:s1])
    del mirrored, upper
    # rows 3a+i: columns over d ascending (== b ascending), then j
    vals = np.transpose(blocks, (0, 2, 1, 3)).reshape(ns * 3, 81)
    cols = np.transpose(np.broadcast_to(cols_g, (ns, 27, 3, 3)), (0, 2, 1, 3)).reshape(ns * 3, 81)
    vmask = np.broadcast_to(valid[:, None, :, None], (ns, 3, 27, 3)).reshape(ns * 3, 81)
    r0, r1 = row_lo - 3 * node_lo, row_hi - 3 * node_lo
    out = _from_row_blocks(r1 - r0, cols[r0:r1], vals[r0:r1], vmask[r0:r1], f"fe_{N}")
    out.n_cols = 3 * nn_all
    return out


# ---------------------------------------------------------------- random SPD (tests)
def random_spd_dense(n: int, sub: int = 0, shift: float = 1.0) -> np.ndarray:
    """Dense random SPD, bitwise symmetric (lower triangle mirrored)."""
    g = rng("random_spd", sub)
    B = g.standard_normal((n, n))
    A = B @ B.T / n + shift * np.eye(n)
    L = np.tril(A)
    return L + np.tril(L, -1).T


def random_sparse_spd(n: int, nnz_per_row: int = 6, sub: int = 0, bandwidth: int | None = None) -> CSR:
    """Random sparse SPD: random symmetric pattern (optionally banded), random values,
    diagonal = sum |offdiag| + U(0.5, 1.5) (strictly diagonally dominant).
    Bitwise symmetric by mirroring the lower triangle."""
    g = rng("random_sparse", sub)
    k = max(1, nnz_per_row // 2)
    rows = np.repeat(np.arange(n), k)
    if bandwidth is None:
        cols = g.integers(0, n, size=n * k)
    else:
        cols = rows - g.integers(1, bandwidth + 1, size=n * k)
    keep = (cols < rows) & (cols >= 0)
    rows, cols = rows[keep], cols[keep]
    key = np.unique(rows.astype(np.int64) * n + cols)
    r, c = key // n, key % n
    v = g.uniform(-1.0, 1.0, size=len(key))
    import scipy.sparse as sp
    Lo = sp.coo_matrix((v, (r, c)), shape=(n, n)).tocsr()
    Lo.sum_duplicates()
    absrow = np.abs(Lo).sum(axis=1).A1 + np.abs(Lo).sum(axis=0).A1
    d = absrow + g.uniform(0.5, 1.5, size=n)
    A = (Lo + Lo.T + sp.diags(d)).tocsr()
    A.sort_indices()
    return CSR(n, A.indptr.astype(np.int64), A.indices.astype(np.int32), A.data.astype(np.float64),
               f"rsparse{n}_{sub}")


def arrow_spd(n: int) -> CSR:
    """Tridiagonal 1D Laplacian plus a hub: row/column 0 coupled to every row
    (a_0j = a_j0 = -0.5 / n^0.5).  Every row's pattern can select column 0, so
    G^T's row 0 is about n long (exercises the long-row transpose path).
    Strictly diagonally dominant, hence SPD; bitwise symmetric by construction."""
    c = -0.5 / np.sqrt(n)
    d = np.full(n, 3.0)
    d[0] = 2.0 + (n - 1) * abs(c)
    rows, cols, vals = [], [], []
    for i in range(n):
        cs = {i: d[i]}
        if i > 0:
            cs[0] = c if i > 1 else c - 1.0
            cs[i - 1] = cs.get(i - 1, 0.0) + (-1.0 if i > 1 else 0.0)
        if i < n - 1:
            cs[i + 1] = cs.get(i + 1, 0.0) + (-1.0 if i + 1 > 1 else 0.0)
        if i == 0:
            for j in range(1, n):
                cs[j] = c if j > 1 else c - 1.0
        for j in sorted(cs):
            rows.append(i)
            cols.append(j)
            vals.append(cs[j])
    rows = np.asarray(rows)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    np.cumsum(rowptr, out=rowptr)
    return CSR(n, rowptr, np.asarray(cols, dtype=np.int32), np.asarray(vals, dtype=np.float64), f"arrow{n}")


def diagonal(d) -> CSR:
    d = np.asarray(d, dtype=np.float64)
    n = len(d)
    return CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), d.copy(), f"diag{n}")


def rhs_for(A: CSR, sub: int = 0):
    """x* ~ U(-1, 1) from the seeded generator and b = A x* (scipy SpMV; input prep only,
    SURVEY.md §8(c) Q12)."""
    x = rng("rhs", sub).uniform(-1.0, 1.0, A.n)
    b = A.to_scipy() @ x
    return b, x


# ---------------------------------------------------------------- named configs
# BASELINE.json configs -> (generator, aFSAI params).  SURVEY.md §8(d) table.
CONFIGS = {
    "M1": dict(desc="2D 5-point Laplacian 32x32 (n=1024), aFSAI 10x1, fp64, 1 GPU",
               make=lambda: poisson2d(32, 32), nsteps=10, s=1, eps=0.0, max_row_nnz=1000),
    "M2": dict(desc="3D 7-point Poisson 100^3 (1M rows), aFSAI 20x2, PCG to 1e-8",
               make=lambda: poisson3d(100), nsteps=20, s=2, eps=0.0, max_row_nnz=1000),
    "M3": dict(desc="3D heterogeneous/anisotropic Poisson 200^3 (8M rows), aFSAI 20x2",
               make=lambda: hetero_poisson3d(200), nsteps=20, s=2, eps=0.0, max_row_nnz=1000),
    "M4": dict(desc="synthetic hex FE elasticity 79^3 nodes x 3 dof (1.48M rows), aFSAI 30x3, cap 100",
               make=lambda: fe_elasticity(79), nsteps=30, s=3, eps=0.0, max_row_nnz=100),
    "M5": dict(desc="synthetic hex FE elasticity 159^3 nodes x 3 dof (12.06M rows), aFSAI 30x3, cap 100",
               make=lambda: fe_elasticity(159), nsteps=30, s=3, eps=0.0, max_row_nnz=100),
}


def sample_rows(n: int, k: int, sub: int = 0) -> np.ndarray:
    """Seeded sorted sample of k distinct rows (plus row 0 and row n-1)."""
    g = rng("sample_rows", sub)
    s = g.choice(n, size=min(k, n), replace=False)
    return np.unique(np.concatenate([s, [0, n - 1]])).astype(np.int64)
