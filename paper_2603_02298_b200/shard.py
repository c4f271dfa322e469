"""Multi-GPU sharding of the hot path: every shard is an independent range of tile
coordinates, there is no collective on the data path. torch.distributed (NCCL on GPUs, gloo in the CPU
tests) is used only afterwards, to gather per-shard checksums for verification.

    copy / index maps   contiguous ranges of the integral coordinate, cut at whole slices of the outermost
                        mode so that every rank keeps the planned (vec / tiled) kernels
    gemm                contiguous ranges of 128 x 256 output tiles (tlb_gemm_tile_count), cut at groups of 4 tiles
                        (512 x 256 pair tiles) so that every rank keeps the wide cta_group::2 plan; batched problems
                        by whole batches
"""
from __future__ import annotations

from .host import L, Layout


def even_split(n_units: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """[begin, end) of `rank` when n_units are dealt out in contiguous, `align`-aligned, balanced ranges."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world")
    blocks = (n_units + align - 1) // align
    lo = (blocks * rank) // world
    hi = (blocks * (rank + 1)) // world
    return min(lo * align, n_units), min(hi * align, n_units)


def copy_range(layout: Layout | str, world: int, rank: int) -> tuple[int, int]:
    """Range of integral coordinates of `layout`'s domain owned by `rank`: whole slices of the outermost
    non-trivial flat mode (its colex prefix product is the alignment)."""
    lay = L(layout) if isinstance(layout, str) else layout
    size = lay.size
    outer = 1
    for e, *_ in reversed(lay.modes):
        if e > 1:
            outer = e
            break
    prefix = size // outer
    return even_split(size, world, rank, align=prefix)


def gemm_tile_range(tile_count: int, world: int, rank: int) -> tuple[int, int]:
    """Tile ids [begin, end) of `rank`. Cuts fall on groups of 4 tiles (one 512 x 256 pair tile of the wide tcgen05
    plan, which is two 256 x 256 blocks of the cta_group::2 plan) whenever that still deals every rank the same
    number of tiles, else on tile pairs."""
    return even_split(tile_count, world, rank, align=4 if tile_count % (4 * world) == 0 else 2)


def batch_range(batches: int, world: int, rank: int) -> tuple[int, int]:
    return even_split(batches, world, rank)


def checksum64(t) -> int:
    """Order-independent 64-bit checksum of a tensor's bit pattern (sum of 32-bit words mod 2^64)."""
    import torch
    flat = t.contiguous().view(torch.uint8).view(-1)
    pad = (-flat.numel()) % 4
    if pad:
        flat = torch.cat([flat, torch.zeros(pad, dtype=torch.uint8, device=flat.device)])
    words = flat.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    return int(words.sum().item()) & 0xFFFFFFFFFFFFFFFF


def gather_checksums(local: int, device=None) -> list[int]:
    """all_gather of one 64-bit checksum per rank (the only collective this package issues)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [local]
    # int64 carrier: reinterpret the unsigned value
    v = local - (1 << 64) if local >= (1 << 63) else local
    mine = torch.tensor([v], dtype=torch.int64, device=device)
    out = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(out, mine)
    return [int(x.item()) & 0xFFFFFFFFFFFFFFFF for x in out]
