"""CPU checks of the pyramid C0 assembly restatement (oracle/assembly.py):
six pyramids per cube (apex = cube centre), base axes along the global axes;
neighbouring pyramids agree on every shared triangular face (siblings) and
base quad (adjacent cubes), and the assembled operator has the C0
invariants."""

import numpy as np
import pytest

import oracle.assembly as A
from oracle.elements import mode_set


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5])
def test_pyr_map_is_conforming(P):
    nx, ny, nz = 2, 2, 2
    pyrs, _, _ = A._pyr_topology(nx, ny, nz)
    l2g, ls, _ = A._pyr_numbering(nx, ny, nz, P)
    x = np.random.default_rng(P).standard_normal(ls[2 * nz + 1])
    owners: dict = {}
    for e, t in enumerate(pyrs):
        for loc in ((0, 1, 4), (3, 2, 4), (0, 3, 4), (1, 2, 4)):
            owners.setdefault(("t", tuple(sorted(t[i] for i in loc))), []).append((e, loc))
        owners.setdefault(("q", tuple(sorted(t[:4]))), []).append((e, (0, 1, 2, 3)))
    rng = np.random.default_rng(3)
    nshared = {"t": 0, "q": 0}
    for (kind, face), own in owners.items():
        if len(own) < 2:
            continue
        assert len(own) == 2
        nshared[kind] += 1
        vals = []
        if kind == "t":
            w = np.array([[0.2, 0.3, 0.5], [0.6, 0.25, 0.15], [0.1, 0.1, 0.8], [1 / 3, 1 / 3, 1 / 3]])
            gv = sorted(pyrs[own[0][0]][i] for i in own[0][1])
            for e, loc in own:
                idx = [loc[[pyrs[e][i] for i in loc].index(v)] for v in gv]  # local vertex of each global one
                xi = w @ A.PYR_REF[idx]
                vals.append(A.pyr_eval(P, x[l2g[e]], A.pyr_collapse(xi)))
        else:
            s = rng.uniform(0.05, 0.95, (5, 2))
            # bilinear point of the physical square: both bases run along the same global axes
            for e, _ in own:
                xi = np.stack([2 * s[:, 0] - 1, 2 * s[:, 1] - 1, -np.ones(5)], axis=1)
                vals.append(A.pyr_eval(P, x[l2g[e]], A.pyr_collapse(xi)))
        assert np.allclose(vals[0], vals[1], rtol=0, atol=1e-12 * max(1.0, np.abs(vals[0]).max())), (kind, face, P)
    assert nshared["t"] == 12 * nx * ny * nz and nshared["q"] > 0


@pytest.mark.parametrize("P", [1, 2, 3])
def test_pyr_assembled_invariants(P):
    nx, ny, nz = 2, 2, 2
    n = A.pyr_n_global(nx, ny, nz, P)
    l2g, ls, plane = A._pyr_numbering(nx, ny, nz, P)
    assert len(np.unique(l2g)) == n and plane == (nx * P + 1) * (ny * P + 1)
    vert = [m for m, md in enumerate(mode_set("pyr", P)) if md in ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1))]
    one = np.zeros(n)
    one[l2g[:, vert].ravel()] = 1.0
    assert np.max(np.abs(A.assembled_helmholtz_pyr(nx, ny, nz, P, one, 0.0))) <= 1e-11
    rng = np.random.default_rng(2)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    a = u @ A.assembled_helmholtz_pyr(nx, ny, nz, P, v, 0.9)
    b = v @ A.assembled_helmholtz_pyr(nx, ny, nz, P, u, 0.9)
    assert abs(a - b) <= 1e-11 * abs(a)


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_product_pyr_numbering_matches_oracle(P, world):
    from paper_2604_04644_b200.assembly import _pyr_maps
    from paper_2604_04644_b200.sharding import partition

    nx, ny, nz = 2, 3, 4
    l2g_o, ls, plane = A._pyr_numbering(nx, ny, nz, P)
    per = nx * ny * 6
    for r in range(world):
        z0, nzl = partition(nz, world, r)
        _, l2g, n, layer = _pyr_maps(nx, ny, nz, z0, nzl, P)
        assert layer == plane
        assert np.array_equal(l2g, l2g_o[z0 * per:(z0 + nzl) * per] - ls[2 * z0])
        assert n == ls[2 * (z0 + nzl) + 1] - ls[2 * z0]
