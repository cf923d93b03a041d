"""CPU checks of the prism C0 assembly restatement (oracle/assembly.py): the
signed local-to-global map is conforming -- every element's expansion of a
random global vector agrees with its neighbours' on every shared quad face
(triangle edge x extrusion) and triangular face (between layers) -- and the
assembled operator has the C0 invariants (stiffness kills constants, mass
of the constant = volume, symmetry)."""

import numpy as np
import pytest

import oracle.assembly as A
from oracle.elements import mode_set

EDGE_ETA = {  # local edge -> (eta1, eta3) as functions of the edge parameter s (start -> end vertex)
    (0, 1): lambda s: (s, -np.ones_like(s)),
    (1, 2): lambda s: (np.ones_like(s), s),
    (0, 2): lambda s: (-np.ones_like(s), s),
}


def _local(x, l2g, sgn, e):
    return sgn[e] * x[l2g[e]]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5])
def test_prism_map_is_conforming(P):
    nx, nw, nz = 2, 3, 2
    tris, _ = A._tri_topology(nx, nw)
    l2g, sgn = A.prism_local_to_global(nx, nw, nz, P)
    x = np.random.default_rng(P).standard_normal(A.prism_n_global(nx, nw, nz, P))
    nt = len(tris)
    s = np.array([-0.8, -0.3, 0.15, 0.6, 0.95])
    eta2 = np.array([-0.9, -0.1, 0.4, 0.8, 0.2])
    # quad faces: elements of one layer sharing a triangle edge
    owners: dict = {}
    for t, v in enumerate(tris):
        for a, b in ((0, 1), (1, 2), (0, 2)):
            owners.setdefault((min(v[a], v[b]), max(v[a], v[b])), []).append((t, a, b))
    shared = 0
    for (lo, hi), own in owners.items():
        if len(own) < 2:
            continue
        shared += 1
        vals = []
        for t, a, b in own:
            sl = s if tris[t][a] == lo else -s  # local parameter of the same physical points
            e1, e3 = EDGE_ETA[(a, b)](sl)
            eta = np.stack([e1, eta2, e3], axis=1)
            for ez in range(nz):
                pass
            vals.append(A.prism_eval(P, _local(x, l2g, sgn, t + nt), eta))  # layer 1
        assert np.allclose(vals[0], vals[1], rtol=0, atol=1e-12 * np.abs(vals[0]).max()), ((lo, hi), P)
    assert shared == 3 * nx * nw - nx - nw
    # triangular faces between layers: top of layer 0 = bottom of layer 1
    rng = np.random.default_rng(7)
    e1 = rng.uniform(-1, 1, 6)
    e3 = rng.uniform(-1, 0.9, 6)
    for t in range(nt):
        top = A.prism_eval(P, _local(x, l2g, sgn, t), np.stack([e1, np.ones(6), e3], axis=1))
        bot = A.prism_eval(P, _local(x, l2g, sgn, t + nt), np.stack([e1, -np.ones(6), e3], axis=1))
        assert np.allclose(top, bot, rtol=0, atol=1e-12 * max(1.0, np.abs(top).max()))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_prism_map_covers_every_dof(P):
    nx, nw, nz = 2, 2, 3
    l2g, _ = A.prism_local_to_global(nx, nw, nz, P)
    n = A.prism_n_global(nx, nw, nz, P)
    assert l2g.min() == 0 and l2g.max() == n - 1
    assert len(np.unique(l2g)) == n
    assert l2g.shape[1] == len(mode_set("prism", P))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_prism_assembled_invariants(P):
    nx, nw, nz = 2, 2, 2
    n = A.prism_n_global(nx, nw, nz, P)
    l2g, sgn = A.prism_local_to_global(nx, nw, nz, P)
    # the constant 1: every vertex mode 1 (vertex dofs are those of local modes (0,q,0),(1,q,0),(0,q,1), q < 2)
    one = np.zeros(n)
    modes = mode_set("prism", P)
    for m, (p, q, r) in enumerate(modes):
        if q < 2 and (p, r) in ((0, 0), (1, 0), (0, 1)):
            one[l2g[:, m]] = 1.0
    assert np.max(np.abs(A.assembled_helmholtz_prism(nx, nw, nz, P, one, 0.0))) <= 1e-12
    vol = one @ A.assembled_helmholtz_prism(nx, nw, nz, P, one, 1.0)
    assert abs(vol - nx * nw * nz) <= 1e-3 * nx * nw * nz  # deformed box volume, amp 0.05
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    a = u @ A.assembled_helmholtz_prism(nx, nw, nz, P, v, 1.3)
    b = v @ A.assembled_helmholtz_prism(nx, nw, nz, P, u, 1.3)
    assert abs(a - b) <= 1e-11 * abs(a)
