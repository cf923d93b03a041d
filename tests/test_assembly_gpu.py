"""Assembled C0 Helmholtz on a conforming hex mesh (device gather ->
elemental kernel -> deterministic scatter) against the CPU restatement
oracle/assembly.py, plus the C0 invariants."""

import numpy as np
import pytest

import oracle as O
import oracle.assembly as A

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("P", [1, 2, 4, 6])
def test_assembled_matches_oracle(torch, P):
    from paper_2604_04644_b200.assembly import C0HexMesh

    nx, ny, nz = 4, 3, 5
    mesh = C0HexMesh(nx, ny, nz, P)
    N = A.n_global(nx, ny, nz, P)
    assert mesh.n_dofs == N
    x = np.random.default_rng(P).standard_normal(N)
    for lam in (0.0, 1.0):
        y = mesh.helmholtz(torch.from_numpy(x).cuda(), lam).cpu().numpy()
        assert O.rel_diff(y, A.assembled_helmholtz(nx, ny, nz, P, x, lam)) <= 1e-12


def test_assembled_stiffness_annihilates_constants(torch):
    from paper_2604_04644_b200.assembly import C0HexMesh

    nx, ny, nz, P = 3, 3, 4, 3
    mesh = C0HexMesh(nx, ny, nz, P)
    Nx, Ny = nx * P + 1, ny * P + 1
    g = np.arange(mesh.n_dofs)
    c = ((g % Nx % P == 0) & ((g // Nx) % Ny % P == 0) & ((g // (Nx * Ny)) % P == 0)).astype(float)
    y = mesh.helmholtz(torch.from_numpy(c).cuda(), 0.0).cpu().numpy()
    assert np.max(np.abs(y)) <= 1e-12
    # and the mass of the constant is the (deformed) volume
    vol = c @ mesh.helmholtz(torch.from_numpy(c).cuda(), 1.0).cpu().numpy()
    assert abs(vol - nx * ny * nz) <= 1e-6 * nx * ny * nz


@pytest.mark.parametrize("P,dims", [(4, (13, 7, 11)), (3, (9, 5, 6)), (8, (5, 4, 3))])
def test_fused_gather_many_tiles(torch, P, dims):
    """The gather fused into the Helmholtz tile load (sk_helmholtz_apply_c0):
    tiles straddle mesh rows (nx not a multiple of the tile width) and
    element layers; identical to the stand-alone gather route and to the
    oracle."""
    from paper_2604_04644_b200.assembly import C0HexMesh

    nx, ny, nz = dims
    mesh = C0HexMesh(nx, ny, nz, P)
    x = np.random.default_rng(P + 100).standard_normal(mesh.n_dofs)
    y = mesh.helmholtz(torch.from_numpy(x).cuda(), 0.8).cpu().numpy()
    assert O.rel_diff(y, A.assembled_helmholtz(nx, ny, nz, P, x, 0.8)) <= 1e-12


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6])
def test_assembled_prism_matches_oracle(torch, P):
    """Assembled C0 prism Helmholtz (signed gather -> prism kernels ->
    CSR scatter) against the oracle's signed assembly on the same deformed
    extruded-triangle mesh; the oracle's map is conformity-checked on CPU
    (tests/test_c0_prism_oracle.py)."""
    from paper_2604_04644_b200.assembly import C0PrismMesh

    nx, nw, nz = 3, 2, 3
    mesh = C0PrismMesh(nx, nw, nz, P)
    N = A.prism_n_global(nx, nw, nz, P)
    assert mesh.n_dofs == N
    x = np.random.default_rng(P).standard_normal(N)
    for lam in (0.0, 1.0):
        y = mesh.helmholtz(torch.from_numpy(x).cuda(), lam).cpu().numpy()
        assert O.rel_diff(y, A.assembled_helmholtz_prism(nx, nw, nz, P, x, lam)) <= 1e-12, lam


def test_assembled_prism_stiffness_annihilates_constants(torch):
    from paper_2604_04644_b200.assembly import C0PrismMesh

    nx, nw, nz, P = 4, 3, 2, 3
    mesh = C0PrismMesh(nx, nw, nz, P)
    nv = (nx + 1) * (nw + 1)
    c = np.zeros(mesh.n_dofs)
    for layer in range(0, nz * P + 1, P):  # vertex nodes of the extrusion
        c[layer * mesh.layer: layer * mesh.layer + nv] = 1.0
    y = mesh.helmholtz(torch.from_numpy(c).cuda(), 0.0).cpu().numpy()
    assert np.max(np.abs(y)) <= 1e-12
    vol = c @ mesh.helmholtz(torch.from_numpy(c).cuda(), 1.0).cpu().numpy()
    assert abs(vol - nx * nw * nz) <= 1e-3 * nx * nw * nz


def test_assembled_prism_many_tiles(torch):
    """A larger mesh (many CTA tiles, ragged last tile) at P=4."""
    from paper_2604_04644_b200.assembly import C0PrismMesh

    nx, nw, nz, P = 7, 5, 4, 4
    mesh = C0PrismMesh(nx, nw, nz, P)
    x = np.random.default_rng(11).standard_normal(mesh.n_dofs)
    y = mesh.helmholtz(torch.from_numpy(x).cuda(), 0.8).cpu().numpy()
    assert O.rel_diff(y, A.assembled_helmholtz_prism(nx, nw, nz, P, x, 0.8)) <= 1e-12


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6])
def test_assembled_tet_matches_oracle(torch, P):
    """Assembled C0 tet Helmholtz (Kuhn tets in global vertex order, reflected
    half with w|det J|) against the oracle on the same mesh."""
    from paper_2604_04644_b200.assembly import C0TetMesh

    nx, ny, nz = 2, 3, 2
    mesh = C0TetMesh(nx, ny, nz, P)
    N = A.tet_n_global(nx, ny, nz, P)
    assert mesh.n_dofs == N
    x = np.random.default_rng(P).standard_normal(N)
    for lam in (0.0, 1.0):
        y = mesh.helmholtz(torch.from_numpy(x).cuda(), lam).cpu().numpy()
        assert O.rel_diff(y, A.assembled_helmholtz_tet(nx, ny, nz, P, x, lam)) <= 1e-12, lam


def test_assembled_tet_stiffness_annihilates_constants(torch):
    from paper_2604_04644_b200.assembly import C0TetMesh

    mesh = C0TetMesh(3, 2, 3, 3)
    x = np.zeros(mesh.n_dofs)
    l2g = mesh._l2g.cpu().numpy().reshape(mesh.E, -1)
    modes = mesh.basis.modes
    vert = [m for m, md in enumerate(modes) if md in ((0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1))]
    x[l2g[:, vert].ravel()] = 1.0
    y = mesh.helmholtz(torch.from_numpy(x).cuda(), 0.0).cpu().numpy()
    assert np.max(np.abs(y)) <= 1e-11


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6])
def test_assembled_pyr_matches_oracle(torch, P):
    """Assembled C0 pyramid Helmholtz (six pyramids per cube, bases along the
    global axes) against the oracle on the same mesh."""
    from paper_2604_04644_b200.assembly import C0PyrMesh

    nx, ny, nz = 2, 2, 3
    mesh = C0PyrMesh(nx, ny, nz, P)
    N = A.pyr_n_global(nx, ny, nz, P)
    assert mesh.n_dofs == N
    x = np.random.default_rng(P).standard_normal(N)
    for lam in (0.0, 1.0):
        y = mesh.helmholtz(torch.from_numpy(x).cuda(), lam).cpu().numpy()
        assert O.rel_diff(y, A.assembled_helmholtz_pyr(nx, ny, nz, P, x, lam)) <= 1e-12, lam


@pytest.mark.parametrize("kind", ["prism", "tet", "pyr"])
def test_compact_maps_bitwise(torch, monkeypatch, kind):
    """The compact int32 maps (sk_c0_gather_map32 / sk_c0_scatter_map32,
    sign folded into the index) and the gather fused into the elemental
    kernel (sk_helmholtz_apply_c0_mapped) give bitwise the results of the
    int64 index + double sign maps, on meshes with signed (prism) and
    unsigned maps, Helmholtz and stiffness."""
    from paper_2604_04644_b200 import assembly as M

    cls, dims = {"prism": (M.C0PrismMesh, (5, 4, 3)), "tet": (M.C0TetMesh, (3, 2, 3)),
                 "pyr": (M.C0PyrMesh, (3, 2, 3))}[kind]
    ys = []
    for map32, fused in (("0", "0"), ("1", "0"), ("1", "1")):
        monkeypatch.setenv("SK_C0_MAP32", map32)
        monkeypatch.setenv("SK_C0_FUSED", fused)
        mesh = cls(*dims, 4)
        assert (mesh._map32 is None) == (map32 == "0")
        x = np.random.default_rng(3).standard_normal(mesh.n_dofs)
        for lam in (0.9, 0.0):
            ys.append(mesh.helmholtz(torch.from_numpy(x).cuda(), lam).cpu().numpy())
    # wide maps, compact maps, compact maps with the gather fused into the kernel
    assert np.array_equal(ys[0], ys[2]) and np.array_equal(ys[0], ys[4])
    assert np.array_equal(ys[1], ys[3]) and np.array_equal(ys[1], ys[5])
