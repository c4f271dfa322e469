"""CPU, world_size 2 over gloo: the multi-GPU path of SURVEY.md 8(e). Each rank derives its own shard from
the host logic (paper_2603_02298_b200.shard), runs it (here on the CPU checker, on the box through libtlb), and
the ranks exchange only checksums; rank 0 compares the assembled result with the single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_02298_b200 import L, shard


def test_even_split_partitions_exactly():
    for n, world, align in [(512, 8, 2), (2048, 3, 2), (10, 4, 1), (7, 8, 1), (4096 * 262144, 8, 262144), (6, 4, 2)]:
        cuts = [shard.even_split(n, world, r, align) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n
        for (a, b), (c, d) in zip(cuts, cuts[1:]):
            assert b == c and a <= b
        assert all(a % align == 0 for a, _ in cuts)


def test_copy_ranges_follow_the_outermost_mode():
    c3 = "((8,128),(4,64),4096):((1,2048),(8,32),262144)"
    for world in (1, 2, 4, 8):
        cuts = [shard.copy_range(c3, world, r) for r in range(world)]
        assert cuts[-1][1] == L(c3).size
        assert all(a % 262144 == 0 and b % 262144 == 0 for a, b in cuts)       # whole tiles
        assert len({b - a for a, b in cuts}) == 1                               # equal work per GPU
    c1 = "(8192,8192):(8192,1)"
    assert shard.copy_range(c1, 8, 3) == (3 * 8192 * 1024, 4 * 8192 * 1024)
    # the planner keeps the tiled kernel on every shard (host-only dry run)
    from paper_2603_02298_b200 import host
    for r in range(4):
        b, e = shard.copy_range(c1, 4, r)
        assert host.copy_plan(c1, "(8192,8192):(1,8192)", 4, b, e) == "tiled"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
    import oracle_util as ou
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # --- copy shard: C3 in small (8 tiles), each rank permutes its own tiles into a shared-shape buffer
        s = "((8,128),(4,64),8):((1,2048),(8,32),262144)"
        d = "((8,128),(4,64),8):((128,1),(65536,1024),262144)"
        n = L(s).size
        src = (np.arange(n, dtype=np.int64) * 2654435761 % (1 << 31)).astype(np.int32)
        dst = np.full(n, -1, dtype=np.int32)
        b, e = shard.copy_range(s, world, rank)
        assert ou.orc_copy(s, src, d, dst, i_begin=b, i_end=e) == 0
        touched = dst != -1
        assert touched.sum() == e - b
        mine = shard.checksum64(torch.from_numpy(dst[touched].copy()))
        sums = shard.gather_checksums(mine)
        # --- gemm shard: rows of C by tile range (M = 512 -> 2 blocks of 256 rows; one per rank)
        M, N, K = 512, 256, 64
        la, lb, lc = f"({M},{K}):({K},1)", f"({N},{K}):({K},1)", f"({M},{N}):(1,{M})"
        i, p = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
        a = ((i * 7 + p * 3 + 1) % 11).astype(np.int64).ravel()
        j, p = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
        bb = ((j * 5 + p * 2 + 2) % 13).astype(np.int64).ravel()
        tiles = 2 * 2                       # transposed plan: rows = N (1 block), cols = M (2 blocks) -> 4 tiles
        t0, t1 = shard.gemm_tile_range(tiles, world, rank)
        assert (t1 - t0) * world == tiles and t0 % 2 == 0
        # rank r owns C columns block r of the transposed problem == rows [256 r, 256 (r + 1)) of C
        rows = slice(256 * rank, 256 * (rank + 1))
        c_full = np.zeros(M * N, dtype=np.int64)
        assert ou.orc_gemm_i64(la, a, lb, bb, lc, c_full) == 0
        part = c_full.reshape(N, M)[:, rows]
        gsum = shard.gather_checksums(shard.checksum64(torch.from_numpy(np.ascontiguousarray(part))))
        if rank == 0:
            whole = np.full(n, -1, dtype=np.int32)
            assert ou.orc_copy(s, src, d, whole) == 0
            want = []
            for r in range(world):
                rb, re_ = shard.copy_range(s, world, r)
                ref = np.full(n, -1, dtype=np.int32)
                ou.orc_copy(s, src, d, ref, i_begin=rb, i_end=re_)
                want.append(shard.checksum64(torch.from_numpy(ref[ref != -1].copy())))
            results["copy_ok"] = sums == want
            results["gemm_ok"] = gsum == [shard.checksum64(torch.from_numpy(np.ascontiguousarray(
                c_full.reshape(N, M)[:, 256 * r:256 * (r + 1)]))) for r in range(world)]
            results["world"] = dist.get_world_size()
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_run_over_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    assert results.get("world") == 2
    assert results.get("copy_ok") is True
    assert results.get("gemm_ok") is True


def test_bench_gpus_flag_is_never_silently_ignored():
    """bench.py --gpus N: outside torchrun it must start N ranks or fail loudly (here: no GPU at all), and under
    torchrun WORLD_SIZE must agree with --gpus."""
    import subprocess
    import sys
    from pathlib import Path
    bench = str(Path(__file__).resolve().parent.parent / "bench.py")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    if not torch.cuda.is_available():
        r = subprocess.run([sys.executable, bench, "--gpus", "2", "--steps", "3"], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode != 0 and "CUDA device(s)" in r.stderr and r.stdout.strip() == ""
    r = subprocess.run([sys.executable, bench, "--gpus", "2"], capture_output=True, text=True, env=dict(env, WORLD_SIZE="4"), timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=4" in r.stderr
