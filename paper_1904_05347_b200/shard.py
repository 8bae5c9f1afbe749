"""Multi-GPU decomposition of the tilekit hot path.

The reference has no distributed code: every output element is owned by one
logical thread and computed from its own ordered sum, so ANY disjoint
partition of the outputs is exact.  The B200 build therefore shards with no
data-path collective (one process per GPU, launched by torchrun):

* convolution: by batch -- NHWC is batch-outermost, so rank r owns images
  [lo, hi) as one contiguous slice of input and output.  Filters are
  replicated once, outside any timed region.
* GEMM (column-major C = A B): by column panels of C -- a panel needs only
  the matching column block of B; A is replicated.  Panels are rounded to a
  multiple of the tile width so no tile straddles two ranks.

Collectives appear only in the plumbing: a barrier + MAX all-reduce of the
device time (every multi-GPU number is the slowest rank), and an optional
gather of the shards to rank 0 for verification.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) slice of `total` units owned by `rank` (the first
    total % world ranks get one extra unit)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def panel_range(n: int, world: int, rank: int, align: int = 256) -> Tuple[int, int]:
    """Column-panel slice of an n-column output, panel edges on multiples of
    `align` (the tensor-core N tile) except at the end."""
    blocks = (n + align - 1) // align
    lo_b, hi_b = shard_range(blocks, world, rank)
    return min(n, lo_b * align), min(n, hi_b * align)


def all_shards(total: int, world: int) -> List[Tuple[int, int]]:
    return [shard_range(total, world, r) for r in range(world)]


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (device time) over the process group; the
    identity without an initialised group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_batch_shards(local, total_batch: int, dst: int = 0):
    """Verification-only gather of per-rank batch shards (tensors of shape
    [hi-lo, ...]) into a full batch on rank `dst` (None elsewhere)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    shapes = all_shards(total_batch, world)
    if rank == dst:
        parts = [torch.empty((hi - lo,) + tuple(local.shape[1:]), dtype=local.dtype,
                             device=local.device) for lo, hi in shapes]
        parts[rank].copy_(local)
        for r, buf in enumerate(parts):
            if r != rank and buf.shape[0] > 0:
                dist.recv(buf, src=r)
        return torch.cat(parts, dim=0)
    if local.shape[0] > 0:
        dist.send(local.contiguous(), dst=dst)
    return None


# ---------------------------------------------------------------------------
# Logical full-batch tensors, sharded without communication
# ---------------------------------------------------------------------------
def image_seed(base: int, layer: int, image: int) -> int:
    """Seed of image `image` (global index) of layer `layer`'s input: the
    logical batch-256 tensor is defined image by image, so a rank
    materialises exactly its slice [lo, hi) and any other rank can rebuild
    it bit for bit for verification."""
    return base + layer * 1_000_003 + image


def seeded_images(hwc, lo: int, hi: int, base: int, layer: int, device):
    """Images [lo, hi) of the logical NHWC tensor (uniform [-1, 1))."""
    import torch
    out = torch.empty((hi - lo,) + tuple(hwc), device=device)
    gen = torch.Generator(device=device)
    for i in range(lo, hi):
        gen.manual_seed(image_seed(base, layer, i))
        out[i - lo].uniform_(-1.0, 1.0, generator=gen)
    return out


def seeded_columns(rows: int, lo: int, hi: int, base: int, block: int, device):
    """Columns [lo, hi) of a logical column-major rows x n matrix, generated
    in blocks of `block` columns (lo, hi multiples of `block` except the
    end): a rank builds its own column panel of B without communication."""
    import torch
    out = torch.empty((hi - lo) * rows, device=device)
    gen = torch.Generator(device=device)
    for b0 in range(lo, hi, block):
        b1 = min(hi, b0 + block)
        gen.manual_seed(base + b0 // block)
        out[(b0 - lo) * rows:(b1 - lo) * rows].uniform_(-1.0, 1.0, generator=gen)
    return out


def broadcast_(t, src: int = 0):
    """One-time replication of a shared operand (filters, GEMM A) over NCCL
    (NVLink); identity without a process group.  Never on the timed path."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(t, src=src)
    return t


def all_gather_scalar(value: float, device=None) -> List[float]:
    """Per-rank scalars (device times) on every rank, in rank order."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(value)]
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [float(p.item()) for p in parts]


def gather_to(local, dst: int = 0):
    """Verification-only gather of equally shaped per-rank tensors to `dst`
    (a list in rank order there, None elsewhere)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [local]
    world, rank = dist.get_world_size(), dist.get_rank()
    if rank == dst:
        parts = [local if r == rank else torch.empty_like(local) for r in range(world)]
        for r in range(world):
            if r != rank:
                dist.recv(parts[r], src=r)
        return parts
    dist.send(local.contiguous(), dst=dst)
    return None
