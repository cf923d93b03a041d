"""Contiguous element sharding across GPUs.

Every in-scope operator is elemental (no element couples to another,
operators.py:17-19), so a block shards as contiguous element
ranges with no data-path collective: each rank builds and applies only its
slice.  The synthetic meshes are seeded per element index
(geometry.py:265, 288), so a slice [first, first + count) of a seed-s mesh is
bit-identical to the same elements of the unsharded mesh.  Collectives appear
only outside the timed region: max-over-ranks timing and gathering outputs
for parity checks.
"""

from __future__ import annotations

from paper_2604_04644_b200.field_block import Block, Field, FieldState, default_interleave_width
from paper_2604_04644_b200.geometry import GeometryClass, make_synthetic_factors
from paper_2604_04644_b200.shapes import Shape, build_shape_basis

__all__ = ["partition", "make_sharded_field", "gather_blocks", "max_over_ranks"]


def partition(n_elements: int, world: int, rank: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous slice: near-equal, the first
    ``n % world`` ranks take one extra element."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_elements < 0:
        raise ValueError("element count must be nonnegative")
    base, extra = divmod(n_elements, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def make_sharded_field(
    shapes,
    order: int,
    geometry_class: GeometryClass,
    n_elements,
    rank: int,
    world: int,
    state: FieldState = FieldState.COEFF,
    n_components: int = 1,
    interleave_width: int | None = None,
    seed: int = 0,
) -> tuple[Field, list[tuple[int, int]]]:
    """This rank's slice of ``make_field(shapes, ...)``: block k holds
    elements [first_k, first_k + count_k) of the seed + k mesh.  Returns the
    field and the (first, count) of every block."""
    if isinstance(shapes, Shape):
        shapes = [shapes]
    if isinstance(n_elements, int):
        n_elements = [n_elements] * len(shapes)
    width = default_interleave_width() if interleave_width is None else interleave_width
    blocks, ranges = [], []
    for k, (shp, ne) in enumerate(zip(shapes, n_elements)):
        first, count = partition(ne, world, rank)
        basis = build_shape_basis(shp, order)
        fac = make_synthetic_factors(basis, geometry_class, count, seed=seed + k, first=first)
        blocks.append(Block(basis, fac, state, n_components, width))
        ranges.append((first, count))
    return Field(blocks), ranges


def gather_blocks(local, group=None):
    """All-gather per-rank canonical element arrays (n_comp, n_data, count)
    along the element axis (outside the timed region; gloo or NCCL)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.as_tensor(np.ascontiguousarray(local), dtype=torch.float64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([t.shape[-1]], dtype=torch.int64, device=dev), group=group)
    n_max = int(max(c.item() for c in counts))
    pad = torch.zeros(t.shape[:-1] + (n_max,), dtype=t.dtype, device=dev)
    pad[..., : t.shape[-1]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return np.concatenate([p[..., : int(c.item())].cpu().numpy() for p, c in zip(parts, counts)], axis=-1)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank scalar (time-like metrics: the slowest rank)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
