"""CPU oracle for the FlashMP hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This module restates, in plain numpy, the algorithm of the reference package
(`/root/reference/pkg/src/flashmp`, cited below as `ref:<file>:<line>`).  It is
the checker the CUDA path is compared against.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it; the product package never does (it fails loudly when its
CUDA library is missing instead of falling back to anything here).

Parity pinning: `tests/golden/make_golden.py` imports the reference itself (in
the build container, where /root/reference exists) and stores its outputs as
fixtures under `tests/golden/`; `tests/test_oracle.py` checks every function
here against those fixtures and against the reference's own known-answer
values (closed-form singular values, flop totals, correction sizes).

Conventions (ref:grid.py:1-14): a field on a box (nx, ny, nz) is a float64
array of shape (3, nz, ny, nx) -- component-major, x fastest.  Flat index of
(c, i, j, k) is c*V + k*nx*ny + j*nx + i.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

CONDITION_LIMIT = 1e14          # ref:subdomain.py:48
DIVERGENCE_LIMIT = 1e8          # ref:krylov.py:41
REORTH_THRESHOLD = 1e-8         # ref:krylov.py:42


# --------------------------------------------------------------------------- stencils
# axis name -> numpy axis of a (nz, ny, nx) component array (ref:operators.py:34)
AX = {"x": 2, "y": 1, "z": 0}


def dfwd(u: np.ndarray, axis: int) -> np.ndarray:
    """Forward difference with a zero ghost after the last cell (ref:operators.py:94-96)."""
    padded = np.concatenate([u, np.zeros_like(np.take(u, [0], axis=axis))], axis=axis)
    return np.diff(padded, axis=axis)


def dbwd(u: np.ndarray, axis: int) -> np.ndarray:
    """Backward difference with a zero ghost before the first cell (ref:operators.py:97-99)."""
    padded = np.concatenate([np.zeros_like(np.take(u, [0], axis=axis)), u], axis=axis)
    return np.diff(padded, axis=axis)


def curl(kind: str, F: np.ndarray) -> np.ndarray:
    """Curl of a (3, nz, ny, nx) field with all-forward / all-backward differences
    (ref:operators.py:104-125): x = D_y F_z - D_z F_y, y = D_z F_x - D_x F_z,
    z = D_x F_y - D_y F_x."""
    d = dfwd if kind == "forward" else dbwd
    fx, fy, fz = F
    return np.stack([
        d(fz, AX["y"]) - d(fy, AX["z"]),
        d(fx, AX["z"]) - d(fz, AX["x"]),
        d(fy, AX["x"]) - d(fx, AX["y"]),
    ])


def double_curl(F: np.ndarray) -> np.ndarray:
    """M F = curl_b(curl_f F) (ref:operators.py:128-131)."""
    return curl("backward", curl("forward", F))


@lru_cache(maxsize=None)
def deltas(dims: tuple[int, int, int]) -> np.ndarray:
    """Boundary weights Lambda as (3, nz, ny, nx) (ref:operators.py:137-164):
    component x counts (j==0)+(k==0), y counts (i==0)+(k==0), z counts (i==0)+(j==0)."""
    nx, ny, nz = dims
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    out = np.stack([(j == 0) * 1.0 + (k == 0), (i == 0) * 1.0 + (k == 0),
                    (i == 0) * 1.0 + (j == 0)])
    out.setflags(write=False)
    return out


def apply_A(alpha: float, F: np.ndarray, boundary: bool = True) -> np.ndarray:
    """A F = F + alpha (M F [+ Lambda F])  (ref:operators.py:167-175)."""
    dims = (F.shape[3], F.shape[2], F.shape[1])
    t = double_curl(F)
    if boundary:
        t = t + deltas(dims) * F
    return F + alpha * t


# --------------------------------------------------------------------------- transform
@dataclass(frozen=True)
class Svd1D:
    n: int
    U: np.ndarray
    S: np.ndarray
    Vt: np.ndarray


@lru_cache(maxsize=None)
def axis_svd(n: int) -> Svd1D:
    """SVD of the n x n forward difference (-1 diagonal, +1 superdiagonal) with the
    reference's sign gauge: first entry of each V^T row above 1e-14 in magnitude is
    made positive, flipping the matching U column (ref:transform.py:46-63)."""
    D = np.diag(-np.ones(n)) + np.diag(np.ones(n - 1), 1)
    U, S, Vt = np.linalg.svd(D)
    for r in range(n):
        nz = np.nonzero(np.abs(Vt[r]) > 1e-14)[0][0]
        if Vt[r, nz] < 0:
            Vt[r] *= -1.0
            U[:, r] *= -1.0
    return Svd1D(n, U, S, Vt)


def sigma_closed_form(n: int) -> np.ndarray:
    """Known answer: sigma_k = 2 sin((2k-1) pi / (4n+2)), k = 1..n, descending."""
    k = np.arange(n, 0, -1)
    return 2.0 * np.sin((2 * k - 1) * np.pi / (4 * n + 2))


def factors(dims, inverse: bool):
    """Per-component (Tx, Ty, Tz) of the transform (ref:transform.py:120-132):
    inverse uses U for the component's own axis and V on the other two; forward
    uses the transposes."""
    sx, sy, sz = (axis_svd(n) for n in dims)
    U = (sx.U, sy.U, sz.U)
    V = (sx.Vt.T, sy.Vt.T, sz.Vt.T)
    table = [tuple(U[a] if a == c else V[a] for a in range(3)) for c in range(3)]
    if inverse:
        return table
    return [tuple(T.T for T in row) for row in table]


def mode_product(T: np.ndarray, F: np.ndarray, axis: str) -> np.ndarray:
    """out = T applied along one axis of a (nz, ny, nx, ...) array (ref:transform.py:79-101)."""
    a = AX[axis]
    return np.moveaxis(np.tensordot(T, F, axes=([1], [a])), 0, a)


def transform(F: np.ndarray, dims, inverse: bool) -> np.ndarray:
    """Forward / inverse orthogonal transform of a (3, nz, ny, nx, ...) stack, axes in
    the order x, y, z (ref:transform.py:135-160)."""
    out = np.empty_like(F)
    for c, (tx, ty, tz) in enumerate(factors(dims, inverse)):
        out[c] = mode_product(tz, mode_product(ty, mode_product(tx, F[c], "x"), "y"), "z")
    return out


# --------------------------------------------------------------------------- subdomain
def point_block_inverses(dims, alpha: float) -> np.ndarray:
    """B^-1 per transformed point, (nz, ny, nx, 3, 3) (ref:subdomain.py:137-153):
    B = I + alpha (|s|^2 I - s s^T), B^-1 = (I - uu^T)/(1 + alpha|s|^2) + uu^T."""
    nx, ny, nz = dims
    s = np.stack(np.broadcast_arrays(axis_svd(nx).S[None, None, :], axis_svd(ny).S[None, :, None],
                                     axis_svd(nz).S[:, None, None]), axis=-1)
    s2 = (s * s).sum(-1)
    uu = s[..., :, None] * s[..., None, :] / s2[..., None, None]
    return (np.eye(3) - uu) / (1.0 + alpha * s2)[..., None, None] + uu


def correction_rows(dims):
    """Boundary slots with nonzero delta, component-major ascending, and their
    weights (ref:subdomain.py:183-194)."""
    nx, ny, nz = dims
    V = nx * ny * nz
    d = deltas(tuple(dims)).reshape(3, V)
    rows = np.concatenate([np.nonzero(d[c])[0] + c * V for c in range(3)])
    return rows, d.reshape(-1)[rows]


def correction_size(dims) -> int:
    """m = sum_l n_l (n_p + n_q - 1) (ref:subdomain.py:235-238)."""
    nx, ny, nz = dims
    return nx * (ny + nz - 1) + ny * (nx + nz - 1) + nz * (nx + ny - 1)


class DegenerateConfigurationError(RuntimeError):
    pass


@dataclass
class SubdomainData:
    dims: tuple
    alpha: float
    binv: np.ndarray
    rows: np.ndarray | None = None
    values: np.ndarray | None = None
    Cinv: np.ndarray | None = None


def exact_solve(dims, binv: np.ndarray, x: np.ndarray) -> np.ndarray:
    """(I + alpha M)^-1 x for x of shape (3V,) or (3V, b) (ref:subdomain.py:156-179)."""
    nx, ny, nz = dims
    batch = x.shape[1:]
    F = x.reshape((3, nz, ny, nx) + batch)
    hat = transform(F, dims, inverse=False)
    solved = np.einsum("kjiab,bkji...->akji...", binv, hat)
    return transform(solved, dims, inverse=True).reshape(x.shape)


def precompute(dims, alpha: float) -> SubdomainData:
    """Block inverses plus the Woodbury data C^-1 (ref:subdomain.py:182-252)."""
    dims = tuple(dims)
    binv = point_block_inverses(dims, alpha)
    data = SubdomainData(dims, alpha, binv)
    if alpha == 0.0:
        return data
    rows, values = correction_rows(dims)
    m, dof = rows.size, 3 * int(np.prod(dims))
    C = np.empty((m, m))
    step = max(1, min(m, (1 << 23) // dof))
    for lo in range(0, m, step):
        cols = np.arange(lo, min(lo + step, m))
        X = np.zeros((dof, cols.size))
        X[rows[cols], np.arange(cols.size)] = 1.0
        C[:, cols] = exact_solve(dims, binv, X)[rows]
    C[np.diag_indices(m)] += 1.0 / (alpha * values)
    try:
        Cinv = np.linalg.inv(C)
    except np.linalg.LinAlgError as exc:
        raise DegenerateConfigurationError(str(exc)) from exc
    if np.abs(C).sum(0).max() * np.abs(Cinv).sum(0).max() > CONDITION_LIMIT:
        raise DegenerateConfigurationError(f"correction matrix ill-conditioned for {dims}")
    data.rows, data.values, data.Cinv = rows, values, Cinv
    return data


def precompute_faces(dims, alpha: float) -> SubdomainData:
    """The same Woodbury data as `precompute` (ref:subdomain.py:196-215), with C assembled in
    closed form instead of m exact solves on unit vectors -- setup acceleration for the timed
    CPU baseline, checked equal to `precompute` in tests/test_oracle.py.

    A unit vector at correction point p = (c, k, j, i) transforms to a rank-one tensor
    Fz_c[:, k] x Fy_c[:, j] x Fx_c[:, i] in component c; B^-1 couples it into component c'; the
    inverse transform and the row selection read it back at q = (c', k', j', i').  Correction
    points lie on the low faces (fixed coordinate 0), so every (component, face) pair of rows
    and columns is one einsum whose fixed axes contract against one factor row/column:
        C0[q, p] = sum_{kk,jj,ii} Iz_c'[k', kk] Iy_c'[j', jj] Ix_c'[i', ii] binv[kk,jj,ii,c',c]
                                  Fz_c[kk, k] Fy_c[jj, j] Fx_c[ii, i]."""
    dims = tuple(dims)
    nx, ny, nz = dims
    binv = point_block_inverses(dims, alpha)
    data = SubdomainData(dims, alpha, binv)
    if alpha == 0.0:
        return data
    rows, values = correction_rows(dims)
    m, V = rows.size, nx * ny * nz
    pos = np.full(3 * V, -1, dtype=np.int64)
    pos[rows] = np.arange(m)
    fwd, inv = factors(dims, inverse=False), factors(dims, inverse=True)
    faces = {0: ("y", "z"), 1: ("x", "z"), 2: ("x", "y")}   # low faces carrying each component's deltas
    ext = {"x": nx, "y": ny, "z": nz}

    def side(c, fixed, mats, row):
        """einsum operands / subscripts / point positions of one (component, face) side."""
        T = dict(zip("xyz", mats[c]))
        letters = {"z": "KJI"[0], "y": "KJI"[1], "x": "KJI"[2]} if row else {"z": "k", "y": "j", "x": "i"}
        inner = {"z": "a", "y": "b", "x": "d"}
        ops, subs, free = [], [], []
        for ax in "zyx":
            if ax == fixed:
                ops.append(T[ax][0, :] if row else T[ax][:, 0])
                subs.append(inner[ax])
            else:
                ops.append(T[ax])
                subs.append(letters[ax] + inner[ax] if row else inner[ax] + letters[ax])
                free.append(ax)
        grids = np.meshgrid(*[np.arange(ext[a]) for a in free], indexing="ij")
        coord = {a: g.ravel() for a, g in zip(free, grids)}
        coord[fixed] = np.zeros_like(grids[0].ravel())
        lin = c * V + coord["z"] * nx * ny + coord["y"] * nx + coord["x"]
        return ops, subs, "".join(letters[a] for a in free), pos[lin]

    C = np.empty((m, m))
    for cq in range(3):
        for fq in faces[cq]:
            rops, rsubs, rout, rpos = side(cq, fq, inv, True)
            for cp in range(3):
                for fp in faces[cp]:
                    cops, csubs, cout, cpos = side(cp, fp, fwd, False)
                    spec = ",".join(rsubs + ["abd"] + csubs) + "->" + rout + cout
                    blk = np.einsum(spec, *rops, binv[:, :, :, cq, cp], *cops, optimize="greedy")
                    C[np.ix_(rpos, cpos)] = blk.reshape(rpos.size, cpos.size)
    C[np.diag_indices(m)] += 1.0 / (alpha * values)
    try:
        Cinv = np.linalg.inv(C)
    except np.linalg.LinAlgError as exc:
        raise DegenerateConfigurationError(str(exc)) from exc
    if np.abs(C).sum(0).max() * np.abs(Cinv).sum(0).max() > CONDITION_LIMIT:
        raise DegenerateConfigurationError(f"correction matrix ill-conditioned for {dims}")
    data.rows, data.values, data.Cinv = rows, values, Cinv
    return data


def solve(data: SubdomainData, r: np.ndarray) -> np.ndarray:
    """Woodbury solve of I + alpha (M + Lambda) (ref:subdomain.py:265-287)."""
    if data.alpha == 0.0:
        return r.copy()
    e0 = exact_solve(data.dims, data.binv, r)
    rhs = np.zeros_like(e0)
    rhs[data.rows] = data.Cinv @ e0[data.rows]
    return e0 - exact_solve(data.dims, data.binv, rhs)


def analytic_flops(dims, m: int) -> dict:
    """Cost model (ref:subdomain.py:221-232)."""
    nx, ny, nz = dims
    V = nx * ny * nz
    exact = 12 * V * (nx + ny + nz) + 18 * V
    return {"exact": exact, "correction": 2 * m * m, "solve": 2 * exact + 2 * m * m,
            "bytes_resident": 8 * m * m + 48 * V + 72 * V + sum(8 * (2 * n * n + n) for n in dims)}


# --------------------------------------------------------------------------- partition
@dataclass(frozen=True)
class Rank:
    rank: int
    coords: tuple
    owned_lo: tuple
    owned: tuple
    ext_lo: tuple
    ext: tuple
    neighbors: tuple


def partition(gdims, grid, overlap: int) -> list[Rank]:
    """Owned tiles, clamped extended boxes and the 26-neighbour lists, rank x-fastest
    (ref:schwarz.py:78-123)."""
    if min(grid) < 1 or overlap < 0:
        raise ValueError("bad partition")
    if any(n % p for n, p in zip(gdims, grid)):
        raise ValueError("extent not divisible by grid")
    tile = tuple(n // p for n, p in zip(gdims, grid))
    if overlap > min(tile):
        raise ValueError("overlap exceeds tile")
    px, py, pz = grid
    out = []
    for cz in range(pz):
        for cy in range(py):
            for cx in range(px):
                c = (cx, cy, cz)
                lo = tuple(ci * t for ci, t in zip(c, tile))
                elo = tuple(max(0, l - overlap) for l in lo)
                ehi = tuple(min(n, l + t + overlap) for n, l, t in zip(gdims, lo, tile))
                nb = []
                if overlap > 0:
                    for dz in (-1, 0, 1):
                        for dy in (-1, 0, 1):
                            for dx in (-1, 0, 1):
                                q = (cx + dx, cy + dy, cz + dz)
                                if (dx, dy, dz) != (0, 0, 0) and all(0 <= a < b for a, b in zip(q, grid)):
                                    nb.append(((dx, dy, dz), q[0] + px * (q[1] + py * q[2])))
                out.append(Rank(cx + px * (cy + py * cz), c, lo, tile, elo,
                                tuple(h - l for l, h in zip(elo, ehi)), tuple(nb)))
    return out


def region(F: np.ndarray, lo, dims) -> np.ndarray:
    """View of a (3, NZ, NY, NX) field over the box at lo with extents dims."""
    return F[:, lo[2]:lo[2] + dims[2], lo[1]:lo[1] + dims[1], lo[0]:lo[0] + dims[0]]


def scatter(gdims, ranks, g: np.ndarray) -> list[np.ndarray]:
    """Global component-major vector -> per-rank owned vectors (ref:schwarz.py:273-281)."""
    G = g.reshape(3, gdims[2], gdims[1], gdims[0])
    return [np.ascontiguousarray(region(G, r.owned_lo, r.owned)).ravel() for r in ranks]


def gather(gdims, ranks, parts) -> np.ndarray:
    """Inverse of scatter (ref:schwarz.py:284-292)."""
    G = np.empty((3, gdims[2], gdims[1], gdims[0]))
    for r, p in zip(ranks, parts):
        region(G, r.owned_lo, r.owned)[...] = p.reshape(3, r.owned[2], r.owned[1], r.owned[0])
    return G.ravel()


_CACHE: dict = {}


def solver_data(dims, alpha, closed_form: bool = False) -> SubdomainData:
    """Per-(extents, alpha) cache (ref:schwarz.py:295-305); closed_form=True builds a missing
    entry with precompute_faces (same data, faster setup)."""
    key = (tuple(dims), float(alpha))
    if key not in _CACHE:
        _CACHE[key] = (precompute_faces if closed_form else precompute)(dims, alpha)
    return _CACHE[key]


def ras_apply(gdims, ranks, alpha: float, r: np.ndarray) -> np.ndarray:
    """Restricted additive Schwarz on a global vector (ref:schwarz.py:320-339): restrict
    to each extended box (the halo exchange mirrors global values,
    ref:tests/test_schwarz.py:76-89), Woodbury solve, keep the owned part."""
    R = r.reshape(3, gdims[2], gdims[1], gdims[0])
    Z = np.empty_like(R)
    for rk in ranks:
        d = solver_data(rk.ext, alpha)
        e = solve(d, np.ascontiguousarray(region(R, rk.ext_lo, rk.ext)).ravel())
        e = e.reshape(3, rk.ext[2], rk.ext[1], rk.ext[0])
        off = tuple(o - l for o, l in zip(rk.owned_lo, rk.ext_lo))
        region(Z, rk.owned_lo, rk.owned)[...] = region(e, off, rk.owned)
    return Z.ravel()


def op_apply(gdims, alpha: float, x: np.ndarray, boundary: bool = True) -> np.ndarray:
    """Global SpMV; the reference's DistributedOperator equals the global CSR to 1e-14
    (ref:schwarz.py:347-388, ref:tests/test_schwarz.py:216-238)."""
    F = x.reshape(3, gdims[2], gdims[1], gdims[0])
    return apply_A(alpha, F, boundary).ravel()


# --------------------------------------------------------------------------- krylov
@dataclass
class Trace:
    method: str
    iterations: int = 0
    converged: bool = False
    final_relres: float = math.inf
    relres: list = field(default_factory=list)
    failure: str | None = None


def bicgstab(op, prec, b: np.ndarray, tol=1e-12, max_iter=1000):
    """Right-preconditioned BiCGSTAB with the reference's exact update order and exits
    (ref:krylov.py:146-239). op/prec map global vectors to global vectors."""
    rep = Trace("bicgstab")
    bnorm = math.sqrt(float(b @ b))
    x = np.zeros_like(b)
    if bnorm == 0.0:
        rep.converged, rep.final_relres, rep.relres = True, 0.0, [0.0]
        return x, rep
    r, rs = b.copy(), b.copy()
    p, v = np.zeros_like(b), np.zeros_like(b)
    rho_old = alpha = omega = 1.0
    rep.relres.append(1.0)
    for it in range(1, max_iter + 1):
        rho = float(rs @ r)
        if rho == 0.0:
            rep.failure = "rho"
            break
        beta = (rho / rho_old) * (alpha / omega)
        p = r + beta * (p - omega * v)
        ph = prec(p) if prec else p
        v = op(ph)
        den = float(rs @ v)
        if den == 0.0:
            rep.failure = "denominator"
            break
        alpha = rho / den
        s = r - alpha * v
        sh = prec(s) if prec else s
        t = op(sh)
        ts, tt = float(t @ s), float(t @ t)
        omega = ts / tt if tt != 0.0 else 0.0
        x += alpha * ph
        x += omega * sh
        r = s - omega * t
        rho_old = rho
        rep.iterations = it
        res = b - op(x)
        relres = math.sqrt(float(res @ res)) / bnorm
        rep.relres.append(relres)
        rep.final_relres = relres
        if relres <= tol:
            rep.converged = True
            break
        if not math.isfinite(relres) or relres > DIVERGENCE_LIMIT:
            rep.failure = "divergence"
            break
        if omega == 0.0:
            rep.failure = "omega"
            break
    return x, rep


def gmres(op, prec, b: np.ndarray, restart=30, tol=1e-12, max_iter=1000):
    """Left-preconditioned restarted GMRES with MGS, one-shot re-orthogonalisation and
    Givens rotations; true residual traced every iteration (ref:krylov.py:242-383)."""
    rep = Trace("gmres")
    P = prec if prec else (lambda u: u.copy())
    nrm = lambda u: math.sqrt(float(u @ u))
    bnorm = nrm(b)
    x = np.zeros_like(b)
    if bnorm == 0.0:
        rep.converged, rep.final_relres, rep.relres = True, 0.0, [0.0]
        return x, rep
    rep.relres.append(1.0)
    k, total, pr0, r, relres = restart, 0, None, b.copy(), 1.0
    while total < max_iter:
        z = P(r)
        beta = nrm(z)
        pr0 = beta if pr0 is None else pr0
        if beta == 0.0:
            rep.converged = relres <= tol
            break
        Q = [z / beta]
        H = np.zeros((k + 1, k))
        g = np.zeros(k + 1)
        g[0] = beta
        cs, sn = np.zeros(k), np.zeros(k)
        inner, stop, xc = 0, False, x
        for j in range(k):
            if total >= max_iter:
                break
            w = P(op(Q[j]))
            for i in range(j + 1):
                H[i, j] = float(Q[i] @ w)
                w -= H[i, j] * Q[i]
            hn = nrm(w)
            cn = math.sqrt(float(H[:j + 1, j] @ H[:j + 1, j]) + hn * hn)
            if cn > 0.0 and hn <= REORTH_THRESHOLD * cn:
                for i in range(j + 1):
                    c = float(Q[i] @ w)
                    H[i, j] += c
                    w -= c * Q[i]
                hn = nrm(w)
            H[j + 1, j] = hn
            happy = hn == 0.0 or (cn > 0.0 and hn < 1e-14 * cn)
            if not happy:
                Q.append(w / hn)
            for i in range(j):
                H[i, j], H[i + 1, j] = (cs[i] * H[i, j] + sn[i] * H[i + 1, j],
                                        -sn[i] * H[i, j] + cs[i] * H[i + 1, j])
            den = math.hypot(H[j, j], H[j + 1, j])
            if den == 0.0:
                rep.failure = "zero column"
                stop = True
                break
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j], H[j + 1, j] = den, 0.0
            g[j + 1], g[j] = -sn[j] * g[j], cs[j] * g[j]
            est = abs(g[j + 1]) / pr0 if pr0 > 0 else 0.0
            inner, total = j + 1, total + 1
            rep.iterations = total
            y = np.linalg.solve(np.triu(H[:inner, :inner]), g[:inner])
            xc = x.copy()
            for i in range(inner):
                xc += float(y[i]) * Q[i]
            relres = nrm(b - op(xc)) / bnorm
            rep.relres.append(relres)
            rep.final_relres = relres
            if not math.isfinite(relres) or relres > DIVERGENCE_LIMIT:
                rep.failure = "divergence"
                stop = True
                break
            if happy or est <= tol or relres <= tol:
                stop = True
                break
        if inner:
            x = xc
        if relres <= tol:
            rep.converged = True
            break
        if rep.failure is not None or (not stop and total >= max_iter):
            break
        r = b - op(x)
    return x, rep


# --------------------------------------------------------------------------- CN step
def build_rhs(E: np.ndarray, H: np.ndarray, dt: float) -> np.ndarray:
    """R = E + dt curl_b(H) - alpha M E, alpha = dt^2/4 (ref:cn_driver.py:54-59)."""
    return E + dt * curl("backward", H) - (dt * dt / 4.0) * double_curl(E)


def cn_step(E, H, dt, solve_fn):
    """One implicit step: solve A E_new = R, then H -= dt/2 (C_f E_new + C_f E)
    (ref:cn_driver.py:82-94). solve_fn maps the global RHS to (E_new, Trace)."""
    R = build_rhs(E, H, dt)
    e_new, rep = solve_fn(R)
    if not rep.converged:
        raise RuntimeError("step failed to converge")
    e_new = e_new.reshape(E.shape)
    h_new = H - 0.5 * dt * (curl("forward", e_new) + curl("forward", E))
    return e_new, h_new, rep


def proc_grid_for(n: int) -> tuple:
    """Most cubic factorisation, ties to the larger px (ref:cli.py:214-231)."""
    best = None
    for px in range(1, n + 1):
        if n % px:
            continue
        for py in range(1, n // px + 1):
            if (n // px) % py:
                continue
            pz = n // px // py
            key = (max(px, py, pz) - min(px, py, pz), -px)
            if best is None or key < best[0]:
                best = (key, (px, py, pz))
    return best[1]
