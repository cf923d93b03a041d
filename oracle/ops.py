"""Sum-factorised elemental operators, element-major restatement.

Restates reference ``speckern/operators.py`` for hex/prism/pyr/tet with the
lane axis of the reference (``(g, n, w)``) replaced by one group holding every
element: arrays are ``(n_data, E)``.  Contraction order, triangular bounds and
the collapsed-vertex rank-one corrections follow the reference line by line.
TEST INFRASTRUCTURE (see ``oracle/__init__.py``).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from oracle.elements import RefElement, mode_count, qcounts
from oracle.geom import Geometry, payload_dxi, payload_lam, payload_w


def _sel(pair, deriv: bool) -> np.ndarray:
    """``_pick`` (operators.py:118-119)."""
    return pair[1] if deriv else pair[0]


@lru_cache(maxsize=None)
def _offsets(shape: str, P: int):
    """Mode-run offsets (operators.py:82-115): prism per p -> (off, nq, nr);
    tet/pyr per p -> tuple per q of (off, nr)."""
    p1 = P + 1
    off = 0
    out = []
    for p in range(p1):
        if shape == "prism":
            out.append((off, p1, p1 - p))
            off += p1 * (p1 - p)
            continue
        row = []
        for q in range(p1 - p if shape == "tet" else p1):
            nr = p1 - p - q if shape == "tet" else p1 - max(p, q)
            row.append((off, nr))
            off += nr
        out.append(tuple(row))
    return tuple(out)


# ---------------------------------------------------------------------------
# forward sweeps B (and D_k B when ``dmode`` = k): (nm, E) -> (nq, E)


def _bwd_hex(el, x, dmode):
    """operators.py:149-159."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = x.shape[1]
    b1, b2, b3 = (_sel(el.a[d], dmode == d) for d in range(3))
    t = b1 @ x.reshape(p1, p1 * p1 * E)
    t = np.matmul(b2, t.reshape(q1, p1, p1 * E))
    u = np.matmul(b3, t.reshape(q1, q2, p1, E))
    return u.reshape(q1 * q2 * q3, E)


def _bwd_prism(el, x, dmode):
    """operators.py:275-295."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = x.shape[1]
    a1 = _sel(el.a[0], dmode == 0)
    a2 = _sel(el.a[1], dmode == 1)
    t2 = np.empty((p1, q2, q3, E))
    segs = _offsets("prism", el.P)
    for p, (off, nq, nr) in enumerate(segs):
        slab = x[off : off + nq * nr].reshape(nq, nr, E)
        t1 = np.matmul(_sel(el.c3[p], dmode == 2), slab)  # (nq, q3, E)
        t2[p] = (a2 @ t1.reshape(nq, q3 * E)).reshape(q2, q3, E)
    off0, nq0, nr0 = segs[0]
    edge = x[off0 : off0 + nq0 * nr0].reshape(nq0, nr0, E)[:, 1, :]  # modes (0,q,1)
    tmp = a2 @ edge  # (q2, E)
    ccol = _sel(el.c3[0], dmode == 2)[:, 1]
    t2[1] += tmp[:, None, :] * ccol[None, :, None]
    return (a1 @ t2.reshape(p1, q2 * q3 * E)).reshape(q1 * q2 * q3, E)


def _bwd_pyr(el, x, dmode):
    """operators.py:321-351."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = x.shape[1]
    a1 = _sel(el.a[0], dmode == 0)
    a2 = _sel(el.a[1], dmode == 1)
    t2 = np.empty((p1, q2, q3, E))
    for p, row in enumerate(_offsets("pyr", el.P)):
        t1 = np.empty((p1, q3, E))
        for q, (off, nr) in enumerate(row):
            t1[q] = _sel(el.c3[max(p, q)], dmode == 2) @ x[off : off + nr]
        t2[p] = (a2 @ t1.reshape(p1, q3 * E)).reshape(q2, q3, E)
    u001 = x[1]
    ccol = _sel(el.c3[0], dmode == 2)[:, 1]
    ones2 = np.zeros(q2) if dmode == 1 else np.ones(q2)
    t2[1] += ones2[:, None, None] * ccol[None, :, None] * u001[None, None, :]
    t2[0] += a2[:, 1][:, None, None] * ccol[None, :, None] * u001[None, None, :]
    return (a1 @ t2.reshape(p1, q2 * q3 * E)).reshape(q1 * q2 * q3, E)


def _bwd_tet(el, x, dmode):
    """operators.py:209-245."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = x.shape[1]
    a1 = _sel(el.a[0], dmode == 0)
    segs = _offsets("tet", el.P)
    t2 = np.zeros((p1, q2, q3, E))
    for p, row in enumerate(segs):
        t1 = np.empty((len(row), q3, E))
        for q, (off, nr) in enumerate(row):
            t1[q] = _sel(el.c3[p + q], dmode == 2) @ x[off : off + nr]
        t2[p] = (_sel(el.b2[p], dmode == 1) @ t1.reshape(len(row), q3 * E)).reshape(q2, q3, E)
    off01, nr01 = segs[0][1]
    tmp = _sel(el.c3[1], dmode == 2) @ x[off01 : off01 + nr01]  # (q3, E)
    bcol = _sel(el.b2[0], dmode == 1)[:, 1]
    t2[1] += bcol[:, None, None] * tmp[None, :, :]
    u001 = x[1]
    ccol = _sel(el.c3[0], dmode == 2)[:, 1]
    ones2 = np.zeros(q2) if dmode == 1 else np.ones(q2)
    t2[1] += ones2[:, None, None] * ccol[None, :, None] * u001[None, None, :]
    t2[0] += bcol[:, None, None] * ccol[None, :, None] * u001[None, None, :]
    return (a1 @ t2.reshape(p1, q2 * q3 * E)).reshape(q1 * q2 * q3, E)


# ---------------------------------------------------------------------------
# transposed sweeps B^T (and (D_k B)^T): (nq, E) -> (nm, E)


def _bwdt_hex(el, y, dmode):
    """operators.py:162-172."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = y.shape[1]
    b1, b2, b3 = (_sel(el.a[d], dmode == d) for d in range(3))
    t = np.matmul(b3.T, y.reshape(q1, q2, q3, E))
    t = np.matmul(b2.T, t.reshape(q1, q2, p1 * E))
    return (b1.T @ t.reshape(q1, p1 * p1 * E)).reshape(p1**3, E)


def _bwdt_prism(el, y, dmode):
    """operators.py:298-318."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = y.shape[1]
    a1 = _sel(el.a[0], dmode == 0)
    a2 = _sel(el.a[1], dmode == 1)
    segs = _offsets("prism", el.P)
    t2 = (a1.T @ y.reshape(q1, q2 * q3 * E)).reshape(p1, q2, q3, E)
    out = np.empty((el.nm, E))
    for p, (off, nq, nr) in enumerate(segs):
        t1 = (a2.T @ t2[p].reshape(q2, q3 * E)).reshape(nq, q3, E)
        out[off : off + nq * nr] = np.matmul(_sel(el.c3[p], dmode == 2).T, t1).reshape(nq * nr, E)
    ccol = _sel(el.c3[0], dmode == 2)[:, 1]
    tmp = np.einsum("k,jke->je", ccol, t2[1])
    off0, nq0, nr0 = segs[0]
    out[off0 + 1 + nr0 * np.arange(nq0)] += a2.T @ tmp
    return out


def _bwdt_pyr(el, y, dmode):
    """operators.py:354-373."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = y.shape[1]
    a1 = _sel(el.a[0], dmode == 0)
    a2 = _sel(el.a[1], dmode == 1)
    t2 = (a1.T @ y.reshape(q1, q2 * q3 * E)).reshape(p1, q2, q3, E)
    out = np.empty((el.nm, E))
    for p, row in enumerate(_offsets("pyr", el.P)):
        t1 = (a2.T @ t2[p].reshape(q2, q3 * E)).reshape(p1, q3, E)
        for q, (off, nr) in enumerate(row):
            out[off : off + nr] = _sel(el.c3[max(p, q)], dmode == 2).T @ t1[q]
    ccol = _sel(el.c3[0], dmode == 2)[:, 1]
    ones2 = np.zeros(q2) if dmode == 1 else np.ones(q2)
    out[1] += np.einsum("j,k,jke->e", ones2, ccol, t2[1])
    out[1] += np.einsum("j,k,jke->e", a2[:, 1], ccol, t2[0])
    return out


def _bwdt_tet(el, y, dmode):
    """operators.py:248-272."""
    q1, q2, q3 = el.q
    p1 = el.P + 1
    E = y.shape[1]
    a1 = _sel(el.a[0], dmode == 0)
    segs = _offsets("tet", el.P)
    t2 = (a1.T @ y.reshape(q1, q2 * q3 * E)).reshape(p1, q2, q3, E)
    out = np.empty((el.nm, E))
    for p, row in enumerate(segs):
        bm = _sel(el.b2[p], dmode == 1)
        t1 = (bm.T @ t2[p].reshape(q2, q3 * E)).reshape(len(row), q3, E)
        for q, (off, nr) in enumerate(row):
            out[off : off + nr] = _sel(el.c3[p + q], dmode == 2).T @ t1[q]
    off01, nr01 = segs[0][1]
    bcol = _sel(el.b2[0], dmode == 1)[:, 1]
    tmp = np.einsum("j,jke->ke", bcol, t2[1])
    out[off01 : off01 + nr01] += _sel(el.c3[1], dmode == 2).T @ tmp
    ccol = _sel(el.c3[0], dmode == 2)[:, 1]
    ones2 = np.zeros(q2) if dmode == 1 else np.ones(q2)
    out[1] += np.einsum("j,k,jke->e", ones2, ccol, t2[1])
    out[1] += np.einsum("j,k,jke->e", bcol, ccol, t2[0])
    return out


_BWD = {"hex": _bwd_hex, "prism": _bwd_prism, "pyr": _bwd_pyr, "tet": _bwd_tet}
_BWDT = {"hex": _bwdt_hex, "prism": _bwdt_prism, "pyr": _bwdt_pyr, "tet": _bwdt_tet}


def bwd(el: RefElement, x: np.ndarray, dmode=None) -> np.ndarray:
    """Sum-factorised B (or D_k B) (operators.py:376-383, 429-431)."""
    return _BWD[el.shape](el, np.ascontiguousarray(x, dtype=float), dmode)


def bwdt(el: RefElement, y: np.ndarray, dmode=None) -> np.ndarray:
    """Sum-factorised B^T (or (D_k B)^T) (operators.py:384-391)."""
    return _BWDT[el.shape](el, np.ascontiguousarray(y, dtype=float), dmode)


def colloc(el: RefElement, u: np.ndarray, d: int, transpose: bool = False) -> np.ndarray:
    """Collocation sweep D_d (or D_d^T) along tensor axis d (operators.py:449-464)."""
    E = u.shape[1]
    full = u.reshape(*el.q, E)
    mat = el.D[d].T if transpose else el.D[d]
    out = np.moveaxis(np.tensordot(mat, full, axes=([1], [d])), 0, d)
    return np.ascontiguousarray(out).reshape(el.nq, E)


# ---------------------------------------------------------------------------
# pointwise metric


def _g_apply(el: RefElement, v: list, transpose: bool) -> list:
    """Chain rule t = G v or G^T v over structural nonzeros (operators.py:471-490)."""
    if el.shape == "hex":
        return v
    out = []
    for i in range(3):
        acc = None
        for j in range(3):
            g = el.G[:, j, i] if transpose else el.G[:, i, j]
            if not np.any(g):
                continue
            term = v[j] if np.all(g == 1.0) else v[j] * g[:, None]
            acc = term if acc is None else acc + term
        out.append(acc)
    return out


def _metric(el: RefElement, geo: Geometry, v: list, lam_payload=None) -> list:
    """v' = G^T (Lam (G v)) with W folded (operators.py:502-523)."""
    t = _g_apply(el, v, False)
    lam = payload_lam(el, geo) if lam_payload is None else lam_payload
    w = []
    for j in range(3):
        acc = lam[0][j] * t[0]
        for i in range(1, 3):
            acc = acc + lam[i][j] * t[i]
        w.append(acc)
    if not geo.deformed:
        w = [wj * el.refw[:, None] for wj in w]
    return _g_apply(el, w, True)


def _apply_w(el: RefElement, geo: Geometry, u: np.ndarray) -> np.ndarray:
    """operators.py:493-499."""
    if geo.deformed:
        return u * geo.jac.T
    return (u * el.refw[:, None]) * geo.jac[None, :]


# ---------------------------------------------------------------------------
# block-level operators, (n_data, E) in and out


def bwd_trans(el, geo, x):
    """operators.py:551-561."""
    return bwd(el, x)


def iproduct_wrt_base(el, geo, u):
    """operators.py:564-574."""
    return bwdt(el, _apply_w(el, geo, u))


def phys_deriv(el, geo, u):
    """operators.py:577-596: returns (3, nq, E)."""
    v = [colloc(el, u, k) for k in range(3)]
    t = _g_apply(el, v, False)
    dxi = payload_dxi(el, geo)
    out = []
    for j in range(3):
        acc = dxi[0][j] * t[0]
        for i in range(1, 3):
            acc = acc + dxi[i][j] * t[i]
        out.append(acc)
    return np.stack(out)


def iproduct_wrt_deriv_base(el, geo, v):
    """operators.py:599-619: v is (3, nq, E)."""
    acc = None
    for k in range(3):
        term = bwdt(el, _apply_w(el, geo, v[k]), dmode=k)
        acc = term if acc is None else acc + term
    return acc


def mass(el, geo, x):
    """operators.py:622-633."""
    return bwdt(el, _apply_w(el, geo, bwd(el, x)))


def helmholtz_noncoll(el, geo, x, lam):
    """operators.py:636-667 (Alg. 5)."""
    if lam < 0.0:
        raise ValueError("lam must be nonnegative")
    u = bwd(el, x)
    v = [bwd(el, x, dmode=k) for k in range(3)]
    vp = _metric(el, geo, v)
    acc = bwdt(el, vp[0], dmode=0)
    for k in range(1, 3):
        acc = acc + bwdt(el, vp[k], dmode=k)
    return acc + lam * bwdt(el, _apply_w(el, geo, u))


def helmholtz_coll(el, geo, x, lam, lam_payload=None):
    """operators.py:670-699 (Alg. 6)."""
    if lam < 0.0:
        raise ValueError("lam must be nonnegative")
    u = bwd(el, x)
    v = [colloc(el, u, k) for k in range(3)]
    vp = _metric(el, geo, v, lam_payload)
    up = colloc(el, vp[0], 0, True)
    for k in range(1, 3):
        up = up + colloc(el, vp[k], k, True)
    up = up + lam * _apply_w(el, geo, u)
    return bwdt(el, up)


# ---------------------------------------------------------------------------
# counters and harness helpers


def _bwd_flops(shape: str, P: int) -> int:
    """operators.py:783-818 (3D shapes)."""
    q1, q2, q3 = qcounts(shape, P)
    p1 = P + 1
    ntri = p1 * (p1 + 1) // 2
    if shape == "hex":
        return 2 * (q1 * p1**3 + q1 * q2 * p1**2 + q1 * q2 * q3 * p1)
    step3 = 2 * q1 * q2 * q3 * p1
    if shape == "prism":
        return 2 * q3 * p1 * ntri + 2 * p1 * q2 * p1 * q3 + step3 + 2 * q2 * p1 + 2 * q2 * q3
    if shape == "pyr":
        npyr = p1 * (p1 + 1) * (2 * p1 + 1) // 6
        return 2 * q3 * npyr + 2 * p1 * q2 * p1 * q3 + step3 + 4 * q2 * q3
    ntet = p1 * (p1 + 1) * (p1 + 2) // 6
    return 2 * q3 * ntet + 2 * q2 * q3 * ntri + step3 + 2 * q3 * P + 2 * q2 * q3 + 8 * q2 * q3


def flops(kind: str, shape: str, P: int) -> int:
    """operator_flops for SUM_FAC (operators.py:835-876)."""
    q = qcounts(shape, P)
    nq = q[0] * q[1] * q[2]
    nm = mode_count(shape, P)
    b = _bwd_flops(shape, P)
    sweep = sum(2 * nq * x for x in q)
    nnz = {"hex": 0, "prism": 4, "pyr": 5, "tet": 6}[shape]
    metric = 2 * nq * (2 * nnz + 9) + 3 * nq
    return {
        "bwdtrans": b,
        "iproduct": b + nq,
        "physderiv": sweep + metric,
        "iproduct_deriv": 3 * (b + nq) + 2 * nm,
        "mass": 2 * b + nq,
        "helmholtz_noncoll": 8 * b + metric + nq + 4 * nm,
        "helmholtz_coll": 2 * b + 2 * sweep + metric + nq + 5 * nq,
    }[kind]


def bytes_per_element(kind: str, shape: str, P: int, deformed: bool) -> int:
    """_bytes_estimate per element (bench.py:175-189), extended to stiffness
    (lam = 0: the W stream is not read)."""
    q = qcounts(shape, P)
    nq = q[0] * q[1] * q[2]
    nm = mode_count(shape, P)
    per = nq if deformed else 1
    if kind == "bwdtrans":
        return 8 * (nm + nq)
    if kind == "mass":
        return 8 * (2 * nm + per)
    if kind == "stiffness":
        return 8 * (2 * nm + 6 * per)
    return 8 * (2 * nm + 7 * per)


def rel_diff(a: np.ndarray, b: np.ndarray) -> float:
    """Max-normalised error (bench.py:192-194)."""
    scale = max(float(np.max(np.abs(a))), float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / scale)


def bench_coeffs(shape_index: int, P: int, nm: int, n: int, seed: int = 0) -> np.ndarray:
    """Seeded U[-1,1] coefficients drawn element-major (bench.py:167-172,
    seed key bench.py:260-262); returns (nm, n)."""
    rng = np.random.default_rng([seed, shape_index, P, 1])
    return np.ascontiguousarray(rng.uniform(-1.0, 1.0, size=(n, nm)).T)
