"""Multi-rank execution of the device path on one GPU: two processes share
cuda:0 and a world_size-2 gloo group (the same code path bench.py runs under
torchrun with NCCL, one rank per GPU).

* every rank runs the CUDA Helmholtz / mass kernels on its contiguous shard
  of each block of a mixed mesh (sharding.make_sharded_field); the gathered
  result equals the unsharded oracle on the same seeded mesh;
* every rank runs the assembled C0 hex apply on its z-slab (fused gather ->
  elemental kernel -> scatter on the device) and sums the shared DOF layers
  with its neighbour (assembly.exchange_interfaces over gloo); each slab
  equals the assembled oracle."""

import os
import socket

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


SHAPES = ["hex", "prism", "pyr", "tet"]
N_EL, P_MIX = 45, 4


def _shard_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import paper_2604_04644_b200 as sk
    from paper_2604_04644_b200 import _lib
    from paper_2604_04644_b200.sharding import gather_blocks, make_sharded_field

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fld, ranges = make_sharded_field([sk.Shape(s) for s in SHAPES], P_MIX, sk.GeometryClass.DEFORMED, N_EL,
                                     rank, world, interleave_width=1, seed=6)
    n0 = _lib.launch_count()
    for k, (blk, (first, count)) in enumerate(zip(fld.blocks, ranges)):
        x = O.bench_coeffs(O.SHAPE_INDEX[SHAPES[k]], P_MIX, blk.basis.n_modes, N_EL, seed=6 + k)
        blk.set_elements(x[None, :, first:first + count])
    helm = sk.apply_to_field(sk.OperatorKind.HELMHOLTZ_COLL, fld, lam=1.3)
    mass = sk.apply_to_field(sk.OperatorKind.MASS, fld)
    torch.cuda.synchronize()
    launched = _lib.launch_count() - n0
    for k in range(len(SHAPES)):
        h = gather_blocks(helm.blocks[k].get_elements())
        m = gather_blocks(mass.blocks[k].get_elements())
        if rank == 0:
            np.save(os.path.join(out_dir, f"helm{k}.npy"), h)
            np.save(os.path.join(out_dir, f"mass{k}.npy"), m)
    np.save(os.path.join(out_dir, f"launched{rank}.npy"), np.array([launched]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_cuda_shards_match_unsharded(cuda, tmp_path):
    import torch.multiprocessing as mp

    world = 2
    mp.start_processes(_shard_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    for r in range(world):
        assert int(np.load(tmp_path / f"launched{r}.npy")[0]) >= 2 * len(SHAPES)  # CUDA kernels on every rank
    for k, s in enumerate(SHAPES):
        el = O.element(s, P_MIX)
        geo = O.synthetic_geometry(el, True, N_EL, seed=6 + k)
        x = O.bench_coeffs(O.SHAPE_INDEX[s], P_MIX, el.nm, N_EL, seed=6 + k)
        h = np.load(tmp_path / f"helm{k}.npy")[0]
        m = np.load(tmp_path / f"mass{k}.npy")[0]
        assert h.shape == (el.nm, N_EL)
        assert O.rel_diff(h, O.helmholtz_coll(el, geo, x, 1.3)) <= 1e-12, s
        assert O.rel_diff(m, O.mass(el, geo, x)) <= 1e-12, s


C0 = (5, 3, 6, 3)  # nx, ny, nz, P


def _c0_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle.assembly as A
    from paper_2604_04644_b200.assembly import C0HexMesh

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz, P = C0
    mesh = C0HexMesh(nx, ny, nz, P, rank=rank, world=world)
    x = np.random.default_rng(3).standard_normal(A.n_global(nx, ny, nz, P))
    xs = torch.from_numpy(x[mesh.slab_slice()].copy()).cuda()
    y = mesh.helmholtz(xs, 1.0)  # device gather/apply/scatter, then the layer exchange
    assert y.is_cuda
    np.save(os.path.join(out_dir, f"slab{rank}_dev.npy"), y.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_c0_slabs_with_exchange(cuda, tmp_path):
    import torch.multiprocessing as mp

    import oracle.assembly as A
    from paper_2604_04644_b200.sharding import partition

    world = 2
    mp.start_processes(_c0_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    nx, ny, nz, P = C0
    layer = (nx * P + 1) * (ny * P + 1)
    x = np.random.default_rng(3).standard_normal(A.n_global(nx, ny, nz, P))
    ref = A.assembled_helmholtz(nx, ny, nz, P, x, 1.0)
    for r in range(world):
        z0, _ = partition(nz, world, r)
        got = np.load(tmp_path / f"slab{r}_dev.npy")
        lo = z0 * P * layer
        assert O.rel_diff(got, ref[lo:lo + got.size]) <= 1e-12, r


C0P = (3, 2, 5, 3)  # nx, nw, nz, P


def _c0_prism_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle.assembly as A
    from paper_2604_04644_b200.assembly import C0PrismMesh

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, nw, nz, P = C0P
    mesh = C0PrismMesh(nx, nw, nz, P, rank=rank, world=world)
    x = np.random.default_rng(4).standard_normal(A.prism_n_global(nx, nw, nz, P))
    y = mesh.helmholtz(torch.from_numpy(x[mesh.slab_slice()].copy()).cuda(), 1.0)
    np.save(os.path.join(out_dir, f"pslab{rank}.npy"), y.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_c0_prism_slabs_with_exchange(cuda, tmp_path):
    import torch.multiprocessing as mp

    import oracle.assembly as A
    from paper_2604_04644_b200.sharding import partition

    world = 2
    mp.start_processes(_c0_prism_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    nx, nw, nz, P = C0P
    n2d = A.prism_n_global(nx, nw, nz, P) // (nz * P + 1)
    x = np.random.default_rng(4).standard_normal(A.prism_n_global(nx, nw, nz, P))
    ref = A.assembled_helmholtz_prism(nx, nw, nz, P, x, 1.0)
    for r in range(world):
        z0, _ = partition(nz, world, r)
        got = np.load(tmp_path / f"pslab{r}.npy")
        lo = z0 * P * n2d
        assert O.rel_diff(got, ref[lo:lo + got.size]) <= 1e-12, r


C0T = (2, 2, 4, 3)  # nx, ny, nz, P


def _c0_tet_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle.assembly as A
    from paper_2604_04644_b200.assembly import C0TetMesh

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz, P = C0T
    mesh = C0TetMesh(nx, ny, nz, P, rank=rank, world=world)
    x = np.random.default_rng(5).standard_normal(A.tet_n_global(nx, ny, nz, P))
    y = mesh.helmholtz(torch.from_numpy(x[mesh.slab_slice()].copy()).cuda(), 1.0)
    np.save(os.path.join(out_dir, f"tslab{rank}.npy"), y.cpu().numpy())
    np.save(os.path.join(out_dir, f"tslice{rank}.npy"), np.array([mesh.slab_slice().start, mesh.slab_slice().stop]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_c0_tet_slabs_with_exchange(cuda, tmp_path):
    import torch.multiprocessing as mp

    import oracle.assembly as A

    world = 2
    mp.start_processes(_c0_tet_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    nx, ny, nz, P = C0T
    x = np.random.default_rng(5).standard_normal(A.tet_n_global(nx, ny, nz, P))
    ref = A.assembled_helmholtz_tet(nx, ny, nz, P, x, 1.0)
    for r in range(world):
        got = np.load(tmp_path / f"tslab{r}.npy")
        lo, hi = np.load(tmp_path / f"tslice{r}.npy")
        assert O.rel_diff(got, ref[lo:hi]) <= 1e-12, r


C0Y = (2, 2, 3, 2)  # nx, ny, nz, P


def _c0_pyr_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle.assembly as A
    from paper_2604_04644_b200.assembly import C0PyrMesh

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz, P = C0Y
    mesh = C0PyrMesh(nx, ny, nz, P, rank=rank, world=world)
    x = np.random.default_rng(6).standard_normal(A.pyr_n_global(nx, ny, nz, P))
    sl = mesh.slab_slice()
    y = mesh.helmholtz(torch.from_numpy(x[sl].copy()).cuda(), 1.0)
    np.save(os.path.join(out_dir, f"yslab{rank}.npy"), y.cpu().numpy())
    np.save(os.path.join(out_dir, f"yslice{rank}.npy"), np.array([sl.start, sl.stop]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_c0_pyr_slabs_with_exchange(cuda, tmp_path):
    import torch.multiprocessing as mp

    import oracle.assembly as A

    world = 2
    mp.start_processes(_c0_pyr_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    nx, ny, nz, P = C0Y
    x = np.random.default_rng(6).standard_normal(A.pyr_n_global(nx, ny, nz, P))
    ref = A.assembled_helmholtz_pyr(nx, ny, nz, P, x, 1.0)
    for r in range(world):
        got = np.load(tmp_path / f"yslab{r}.npy")
        lo, hi = np.load(tmp_path / f"yslice{r}.npy")
        assert O.rel_diff(got, ref[lo:hi]) <= 1e-12, r
