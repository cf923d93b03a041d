"""Host-side multi-GPU logic on CPU: contiguous partitioning, per-element
seeding (a rank's slice equals the same elements of the unsharded mesh), and
the gather / max-over-ranks collectives over a world_size-2 gloo group."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
from paper_2604_04644_b200.sharding import partition


@pytest.mark.parametrize("n", [0, 1, 7, 64, 1000, 1 << 20])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_partition_covers_exactly_once(n, world):
    seen = 0
    for r in range(world):
        first, count = partition(n, world, r)
        assert first == seen
        seen += count
        assert abs(count - n / world) < 1
    assert seen == n


def test_partition_rejects_bad_rank():
    with pytest.raises(ValueError):
        partition(10, 2, 2)
    with pytest.raises(ValueError):
        partition(-1, 2, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2604_04644_b200.sharding import gather_blocks, max_over_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape, P, n = "tet", 3, 37
    el = O.element(shape, P)
    first, count = partition(n, world, rank)
    # this rank's slice of the seeded mesh and of the bench coefficients
    params = O.deformation_params(count, seed=4, first=first)
    from oracle.geom import deformed_coords

    geo = O.deformed_geometry_from_coords(el, deformed_coords(el, params))
    x_all = O.bench_coeffs(O.SHAPE_INDEX[shape], P, el.nm, n, seed=4)
    local = O.helmholtz_coll(el, geo, x_all[:, first : first + count], 1.0)
    full = gather_blocks(local[None])
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), full)
        np.save(os.path.join(out_dir, "tmax.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shards_match_unsharded(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    full = np.load(tmp_path / "gathered.npy")[0]
    el = O.element("tet", 3)
    geo = O.synthetic_geometry(el, True, 37, seed=4)
    x = O.bench_coeffs(O.SHAPE_INDEX["tet"], 3, el.nm, 37, seed=4)
    ref = O.helmholtz_coll(el, geo, x, 1.0)
    # per-element seeding: identical inputs; only BLAS blocking differs
    assert O.rel_diff(full, ref) <= 1e-15
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0


def _c0_worker(rank, world, port, out_dir):
    """Each rank assembles its z-slab with the oracle, exchanges the shared
    DOF layers over gloo with the product's exchange routine."""
    import torch
    import torch.distributed as dist

    import oracle.assembly as A
    from oracle.elements import element
    from oracle.geom import deformed_geometry_from_coords
    from oracle.ops import helmholtz_coll
    from paper_2604_04644_b200.assembly import exchange_interfaces

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz, P = 3, 2, 5, 2
    z0, nzl = partition(nz, world, rank)
    layer = (nx * P + 1) * (ny * P + 1)
    N = A.n_global(nx, ny, nz, P)
    x = np.random.default_rng(7).standard_normal(N)
    first, E = z0 * nx * ny, nzl * nx * ny
    el = element("hex", P)
    geo = deformed_geometry_from_coords(el, A.mesh_coords(nx, ny, nz, P, first=first, count=E))
    l2g = A.local_to_global(nx, ny, nz, P, first=first, count=E)
    ye = helmholtz_coll(el, geo, x[l2g].T, 1.0)
    lo = z0 * P * layer
    y = np.zeros((nzl * P + 1) * layer)
    np.add.at(y, l2g.T.ravel() - lo, ye.ravel())
    t = torch.from_numpy(y)
    exchange_interfaces(t, layer)
    np.save(os.path.join(out_dir, f"slab{rank}.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_c0_interface_exchange(tmp_path):
    import oracle.assembly as A

    world = 2
    mp.start_processes(_c0_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    nx, ny, nz, P = 3, 2, 5, 2
    layer = (nx * P + 1) * (ny * P + 1)
    N = A.n_global(nx, ny, nz, P)
    x = np.random.default_rng(7).standard_normal(N)
    ref = A.assembled_helmholtz(nx, ny, nz, P, x, 1.0)
    for r in range(world):
        z0, nzl = partition(nz, world, r)
        got = np.load(tmp_path / f"slab{r}.npy")
        lo = z0 * P * layer
        assert O.rel_diff(got, ref[lo : lo + got.size]) <= 1e-13
