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
