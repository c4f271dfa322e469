"""GPU, two ranks: the multi-GPU path of SURVEY.md 8(e) through libtlb. Each of two processes derives its shard from
paper_2603_02298_b200.shard (copy_range / gemm_tile_range / batch_range), runs it with tlb_copy / tlb_gemm_bf16 /
tlb_gemm_bf16_batched / tlb_eval_range on the GPU, and the shards are assembled on rank 0 and compared, cell by cell,
with the oracle's single-process result. The box has one GPU, so both ranks use cuda:0 (one process per rank, as under
torchrun) and the ranks talk over gloo; on a multi-GPU box bench.py does the same per device over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, results):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import oracle_util as ou
    from paper_2603_02298_b200 import L, abi, host, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        lib = abi.load()
        n0 = lib.tlb_launch_count()
        ok = {}
        # ---- copy: C3 in small (8 tiles) and C1 in small, every rank copies its own coordinate range
        for name, s, d in [("c3", "((8,128),(4,64),8):((1,2048),(8,32),262144)", "((8,128),(4,64),8):((128,1),(65536,1024),262144)"),
                           ("c1", "(512,1024):(1024,1)", "(512,1024):(1,512)")]:
            n = L(s).size
            src = (np.arange(n, dtype=np.int64) * 2654435761 % (1 << 31)).astype(np.int32)
            tsrc = torch.from_numpy(src).cuda()
            tdst = torch.full((n,), -1, dtype=torch.int32, device="cuda")
            b, e = shard.copy_range(s, world, rank)
            plan = host.copy(host.tensor_of(s, tsrc), host.tensor_of(d, tdst), b, e)
            torch.cuda.synchronize()
            part = tdst.cpu()
            assert int((part != -1).sum()) == e - b and plan == "tiled", (name, plan)
            parts = [torch.empty_like(part) for _ in range(world)] if rank == 0 else None
            dist.gather(part, parts, dst=0)
            if rank == 0:
                whole = np.full(n, -1, dtype=np.int32)
                for p in parts:
                    pn = p.numpy()
                    assert ((whole == -1) | (pn == -1)).all()          # shards are disjoint
                    whole = np.where(pn != -1, pn, whole)
                want = np.full(n, -1, dtype=np.int32)
                assert ou.orc_copy(s, src, d, want) == 0
                ok[name] = bool((whole == want).all())
        # ---- GEMM by tile-id ranges: C starts at zero on every rank, the shards sum to the full product (exact KAT)
        M, N, K = 1024, 2048, 256
        la, lb, lc = f"({M},{K}):({K},1)", f"({N},{K}):({K},1)", f"({M},{N}):(1,{M})"
        i, p = np.meshgrid(np.arange(M), np.arange(K), indexing="ij")
        a = ou.f32_to_bf16_bits(((i * 7 + p * 3 + 1) % 11).astype(np.float32))
        j, p = np.meshgrid(np.arange(N), np.arange(K), indexing="ij")
        bb = ou.f32_to_bf16_bits(((j * 5 + p * 2 + 2) % 13).astype(np.float32))
        ta_ = torch.from_numpy(a.view(np.int16).ravel().copy()).cuda()
        tb_ = torch.from_numpy(bb.view(np.int16).ravel().copy()).cuda()
        tc_ = torch.zeros(M * N, dtype=torch.float32, device="cuda")
        ta, tb, tc = (host.tensor_of(t, buf, ranked=True) for t, buf in ((la, ta_), (lb, tb_), (lc, tc_)))
        tiles = host.gemm_tile_count(ta, tb, tc)
        t0, t1 = shard.gemm_tile_range(tiles, world, rank)
        plan = host.gemm_bf16(ta, tb, tc, t0, t1)
        torch.cuda.synchronize()
        part = tc_.cpu()
        dist.reduce(part, dst=0, op=dist.ReduceOp.SUM)                 # disjoint tiles: the sum assembles C
        if rank == 0:
            want = np.zeros(M * N, dtype=np.float32)
            st, _ = ou.orc_gemm_bf16(la, a.ravel(), lb, bb.ravel(), lc, want)
            ok["gemm"] = st == 0 and bool((part.numpy() == want).all()) and plan.startswith("umma")
            ok["gemm_plan"] = plan
        # ---- batched GEMM by whole batches (C4's sharding)
        B_, Mb, Kb = 4, 256, 128
        rng = np.random.default_rng(5)
        ab = ou.f32_to_bf16_bits(rng.integers(-3, 4, (B_, Mb, Kb)).astype(np.float32))
        bbt = ou.f32_to_bf16_bits(rng.integers(-3, 4, (B_, Mb, Kb)).astype(np.float32))
        ta_ = torch.from_numpy(ab.view(np.int16).ravel().copy()).cuda()
        tb_ = torch.from_numpy(bbt.view(np.int16).ravel().copy()).cuda()
        tc_ = torch.zeros(B_ * Mb * Mb, dtype=torch.float32, device="cuda")
        lab, lcb = f"({Mb},{Kb}):({Kb},1)", f"({Mb},{Mb}):(1,{Mb})"
        t3 = [(host.make_tensor(L(t).lower(ranked=True), buf.data_ptr(), buf.numel(), eb), None)
              for t, buf, eb in ((lab, ta_, 2), (lab, tb_, 2), (lcb, tc_, 4))]
        b0, b1 = shard.batch_range(B_, world, rank)
        host.gemm_bf16_batched(*t3, Mb * Kb, Mb * Kb, Mb * Mb, b0, b1)
        torch.cuda.synchronize()
        part = tc_.cpu()
        dist.reduce(part, dst=0, op=dist.ReduceOp.SUM)
        if rank == 0:
            good = True
            for bi in range(B_):
                want = np.zeros(Mb * Mb, dtype=np.float32)
                st, _ = ou.orc_gemm_bf16(lab, ab[bi].ravel(), lab, bbt[bi].ravel(), lcb, want)
                good = good and st == 0 and bool((part.numpy()[bi * Mb * Mb:(bi + 1) * Mb * Mb] == want).all())
            ok["batched"] = good
        # ---- index maps: each rank evaluates its slice of one chunk
        Lt = "((128,64),(512,1024)):((65536,1),(8388608,64))"
        chunk, base = 1 << 20, 9 * 2**28
        c0, c1 = shard.even_split(chunk, world, rank, align=4096)
        out = torch.empty(c1 - c0, dtype=torch.int64, device="cuda")
        host.eval_range(Lt, base + c0, c1 - c0, out)
        torch.cuda.synchronize()
        sums = shard.gather_checksums(shard.checksum64(out.cpu()))
        if rank == 0:
            want = ou.orc_eval_range(Lt, base, chunk)
            ok["eval"] = sums == [shard.checksum64(torch.from_numpy(want[slice(*shard.even_split(chunk, world, r, align=4096))].copy()))
                                  for r in range(world)]
            ok["launches_rank0"] = int(lib.tlb_launch_count() - n0)
            ok["world"] = dist.get_world_size()
            results.update(ok)
    finally:
        dist.destroy_process_group()


def test_two_ranks_shard_the_problems_through_libtlb():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    r = dict(results)
    assert r.get("world") == 2, r
    assert r.get("c3") is True and r.get("c1") is True, r
    assert r.get("gemm") is True, r
    assert r.get("batched") is True, r
    assert r.get("eval") is True, r
    assert r.get("launches_rank0", 0) >= 5, r


def test_bench_refuses_more_gpus_than_the_box_has():
    """`python bench.py --gpus N` spawns one rank per GPU; asking for more GPUs than exist must fail loudly, not
    quietly run one rank."""
    import subprocess
    import sys
    from pathlib import Path
    n = torch.cuda.device_count()
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(Path(__file__).resolve().parent.parent / "bench.py"), "--gpus", str(n + 1),
                        "--steps", "3", "--warmup", "3", "--gemm-only", "--no-cpu"], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode != 0
    assert "CUDA device(s)" in r.stderr and not r.stdout.strip().startswith("{")
