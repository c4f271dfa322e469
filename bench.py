#!/usr/bin/env python
"""Benchmark of the layout-driven hot path (BASELINE.json: "copy GB/s & GEMM TFLOP/s (% of B200 roofline)
vs CPU ref, 1/2/4/8 GPUs").

    python bench.py --gpus N --steps K --warmup W            # our arm (libtlb.so, sm_100a)
    python bench.py --impl reference --gpus N ...            # the reference's own CPU implementation

One JSON line on stdout (rank 0). The headline workload is BASELINE.json configs[1] (C2: bf16 4096^3 TN GEMM,
fp32 accumulate); a "step" is one such GEMM per GPU (weak scaling: every rank owns one independent problem,
no collective on the data path). The copy / index-map configs (C1, C3, C5) and the batched GEMM (C4) are timed in
the same run and reported under "other_configs", each with its own roofline, CPU baseline and end-to-end figure;
at N > 1 they are the NAMED problem sharded by tile-coordinate ranges (strong scaling, paper_2603_02298_b200.shard).

Launch: under torchrun (the driver's N > 1 command) RANK / LOCAL_RANK / WORLD_SIZE come from the environment. A plain
`python bench.py --gpus N` with N > 1 re-launches itself under torch.distributed.run with N ranks (and fails loudly when
the box has fewer than N GPUs), so both spellings measure the same thing.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

L2_BYTES = 126 * 1024 * 1024
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["_source"] = "measured"
        return d
    d = dict(FALLBACK_PEAKS)
    d["_source"] = "fallback"
    return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md recipe)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self, period_ms: int = 100):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", str(period_ms), "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self, t0: float, t1: float):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        rows = [r for (t, r) in self.rows if t0 - 0.05 <= t <= t1 + 0.15] or [r for (_, r) in self.rows]
        sm, mx, reasons, pw = [], None, set(), []
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                pw.append(float(r[3]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), r[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> None:
    """`python bench.py --gpus N` (N > 1) outside torchrun: start N ranks, one per GPU, and exit with their status."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}: launch one rank per GPU "
                     f"(torchrun --nproc-per-node {args.gpus})")
        return
    if args.gpus <= 1 or args.impl == "reference":   # the CPU arm runs on rank 0 alone: nothing to spawn
        return
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not (args.share_gpu and have >= 1):
        sys.exit(f"bench.py: --gpus {args.gpus} requested but this box has {have} CUDA device(s); the multi-GPU path is "
                 f"one process per GPU and is never emulated")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# --------------------------------------------------------------------------------------------
# CPU legs: the reference's own implementation (oracle/_ref when it was built, else the C port)
# --------------------------------------------------------------------------------------------
def cpu_gemm_sample(m_rows: int, n_cols: int, K: int, threads: int):
    """tla::gemm (tensor.hpp:214) on an (m_rows*threads) x n_cols x K sub-problem of the TN workload, one row
    block per host thread. Returns (seconds, macs, kind)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    import oracle_util as ou
    kind = "reference" if ou.have_ref() else "port"
    la, lb, lc = f"({m_rows},{K}):({K},1)", f"({n_cols},{K}):({K},1)", f"({m_rows},{n_cols}):(1,{m_rows})"
    i, p = np.meshgrid(np.arange(m_rows), np.arange(K), indexing="ij")
    j, p2 = np.meshgrid(np.arange(n_cols), np.arange(K), indexing="ij")
    b = ((j * 5 + p2 * 2 + 2) % 13).astype(np.int64).ravel()
    blocks = []
    for t in range(threads):
        a = (((i + t * m_rows) * 7 + p * 3 + 1) % 11).astype(np.int64).ravel()
        blocks.append((a, np.zeros(m_rows * n_cols, dtype=np.int64)))

    def work(t):
        a, c = blocks[t]
        if kind == "reference":
            st = ou.ref_gemm(la, a, lb, b, lc, c)
        else:
            st = ou.orc_gemm_i64(la, a, lb, b, lc, c)
        assert st == 0

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, range(threads)))
    dt = time.perf_counter() - t0
    return dt, m_rows * threads * n_cols * K, kind


def cpu_copy_baseline(src: str, dst: str, elem_bytes: int, what: str):
    """tla::copy (tensor.hpp:195-199) on a bounded slice of the workload: verbatim on 1 core and its loop body on all
    host threads. GB/s counts 2 x elem_bytes per element, the GPU workload's bytes (the reference
    itself moves 8-byte Int cells)."""
    import numpy as np
    import oracle_util as ou
    from paper_2603_02298_b200 import L
    n = L(src).size
    threads = os.cpu_count() or 1
    if ou.have_ref():
        s1, c1 = ou.ref_copy_bench(src, dst, 1)
        sn, cn = ou.ref_copy_bench(src, dst, threads)
        assert c1 == cn, "1-core and N-thread reference copies disagree"
        kind = "reference"
    else:   # GPU box without the prebuilt reference: the C port, one core
        a = np.arange(ou.cosize_of(src), dtype=np.int64) * 3 + 1
        b = np.full(ou.cosize_of(dst), -1, dtype=np.int64)
        t0 = time.perf_counter()
        assert ou.orc_copy(src, a, dst, b) == 0
        s1 = sn = time.perf_counter() - t0
        threads_used = 1
        kind = "port"
    gb = 2.0 * elem_bytes * n / 1e9
    return {"value": gb / sn, "unit": "GB/s", "cores": threads if kind == "reference" else 1, "kind": kind,
            "one_core_value": gb / s1, "ns_per_element_one_core": s1 / n * 1e9,
            "sample": f"tla::copy {'verbatim (unmodified reference headers)' if kind == 'reference' else '(C port)'} on {what}: "
                      f"{n} elements, {s1:.2f} s on 1 core, {sn:.2f} s with the loop body on {threads if kind == 'reference' else 1} threads; "
                      f"bytes counted as 2 x {elem_bytes} B per element"}


def cpu_eval_baseline(layout: str, n: int):
    import oracle_util as ou
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    if ou.have_ref():
        ou.ref_eval_range_mt(layout, 2**31, n, threads)
        kind = "reference"
    else:
        ou.orc_eval_range(layout, 2**31, n)
        threads, kind = 1, "port"
    dt = time.perf_counter() - t0
    return {"value": n * 8 / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": kind, "evals_per_s": n / dt,
            "sample": f"tla::eval_int ({'unmodified reference' if kind == 'reference' else 'C port'}) on {n} consecutive indices "
                      f"of the 2^32-element layout, {threads} host threads, {dt:.2f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    K = 4096
    # calibrate ns/MAC on a tiny block, then size one step so the whole run ends within ~2 minutes
    dt, macs, kind = cpu_gemm_sample(2, 16, K, threads)
    per_mac = dt * threads / macs
    budget = 110.0 / max(args.steps + args.warmup, 1)
    n_cols = 64
    m_rows = max(1, min(64, int(budget / (per_mac * n_cols * K))))
    for _ in range(args.warmup):
        cpu_gemm_sample(m_rows, n_cols, K, threads)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        _, m, kind = cpu_gemm_sample(m_rows, n_cols, K, threads)
        total += m
    dt = time.perf_counter() - t0
    tflops = 2.0 * total / dt / 1e12
    sample = (f"tla::gemm verbatim ({'unmodified reference headers' if kind == 'reference' else 'C port of tensor.hpp:214'}, "
              f"checked int64) on a {m_rows * threads}x{n_cols}x{K} sub-problem of the 4096^3 TN workload per step, "
              f"{threads} host threads")
    line = {
        "impl": "reference", "metric": "gemm_tflops", "value": tflops, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / max(args.steps, 1) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "C2: 4096^3 TN GEMM (configs[1]); CPU arm runs a bounded sub-problem per step"},
        "cpu_baseline": {"value": tflops, "unit": "TFLOP/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": tflops, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------------
RED_DEV = "cuda"   # where the max-over-ranks reduction lives ("cpu" under --share-gpu: gloo)


def timed(torch, dist, world, fn, steps, warmup):
    """W warm-up calls, then exactly K calls between barrier+synchronize, CUDA events on the launching stream,
    max over ranks. Returns seconds."""
    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        fn(warmup + i)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=RED_DEV)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms / 1e3


def wall_timed(torch, dist, world, fn, steps, warmup=2):
    """Synchronous host-buffer calls (the e2e legs): wall clock around K calls, max over ranks. Returns seconds."""
    for _ in range(warmup):
        fn()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    sec = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([sec], dtype=torch.float64, device=RED_DEV)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    return sec


def traffic_for(config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full capture of the
    same workload (profiles/traffic.json, written by tools/ncu_summary.py: not measured in this run, the capture it
    came from is named in traffic_source); None when no capture exists."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        e = json.loads(p.read_text()).get(config)
        return (e["dram_bytes_per_launch"], e.get("source")) if e else (None, None)
    return None, None


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_02298_b200 import abi, host, shard

    rank, world, local = dist_env()
    assert torch.cuda.is_available(), "bench.py needs a CUDA device: libtlb has no CPU fallback"
    global RED_DEV
    if args.share_gpu and world > 1:
        # functional test of the N-rank code path on a box with fewer GPUs: every rank uses cuda:0, ranks talk over gloo
        local = 0
        RED_DEV = "cpu"
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    assert local < torch.cuda.device_count(), f"rank {rank}: LOCAL_RANK {local} has no GPU (one process per GPU)"
    torch.cuda.set_device(local)
    if world > 1 and not args.share_gpu:
        # communicator set-up is logged (NCCL INFO, INIT subsystem) so that the number of ranks is visible to whoever
        # launched this; the data path below never uses the communicator
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = abi.load()
    host.config("GEMM_CLOCK", "1")  # the GEMM kernels stamp {clock64, globaltimer}: SM clock under load
    pk = peaks()
    K, W = args.steps, args.warmup
    only = set(args.only.split(",")) if args.only else None

    # ---- C2: bf16 4096^3 TN GEMM, fp32 accumulate (C += A B^T), one problem per rank -----------------
    M = N = Kd = 4096
    nsets = 3  # 3 x (32 + 32 + 64 MiB) = 384 MiB of operands rotate through a 126 MB L2
    g = torch.Generator(device="cuda").manual_seed(rank)
    sets = []
    for s in range(nsets):
        a = (torch.rand(M * Kd, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        b = (torch.rand(N * Kd, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        c = torch.zeros(M * N, dtype=torch.float32, device="cuda")
        ta = host.tensor_of(f"({M},{Kd}):({Kd},1)", a.view(torch.int16), ranked=True)
        tb = host.tensor_of(f"({N},{Kd}):({Kd},1)", b.view(torch.int16), ranked=True)
        tc = host.tensor_of(f"({M},{N}):(1,{M})", c, ranked=True)
        sets.append((ta, tb, tc))
    lib.tlb_gemm_set_path({"auto": 0, "1sm": 2, "2sm": 3}[args.gemm_path])

    def gemm_step(i):
        ta, tb, tc = sets[i % nsets]
        host.gemm_bf16(ta, tb, tc)

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
        time.sleep(0.3)
    n0 = lib.tlb_launch_count()
    w0 = time.time()
    sec = timed(torch, dist, world, gemm_step, K, W)
    w1 = time.time()
    plan = lib.tlb_last_plan().decode()
    launches = int(lib.tlb_launch_count() - n0) - W  # warm-up launches are outside the timed region
    clocks = sampler.stop(w0, w1) if rank == 0 else None
    if rank == 0:
        # nvidia-smi samples every 100 ms and a 50-step region lasts ~5 ms, so the SM clock the kernel actually ran
        # at is measured inside the kernel (CTA 0: clock64 delta / globaltimer delta, median over the launches)
        import ctypes as C
        mhz, us, nl = C.c_double(0), C.c_double(0), C.c_uint32(0)
        lib.tlb_gemm_clock_stats(C.byref(mhz), C.byref(us), C.byref(nl))
        if nl.value:
            clocks["sm_mhz_in_kernel"] = round(mhz.value, 1)
            clocks["kernel_us_in_kernel"] = round(us.value, 2)
            clocks["launches_sampled"] = nl.value
            if clocks.get("sm_max_mhz") and mhz.value < 0.97 * clocks["sm_max_mhz"] and not clocks["reasons"]:
                clocks["note"] = "SM clock below max inside the kernel: power management under tensor load (sw_power_cap regime)"
    flops = 2.0 * M * N * Kd
    value = flops * K * world / sec / 1e12
    kernel_s = sec / K
    burst = sec < 1.0
    peak = pk["bf16_tflops"] if burst else pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    achieved = flops / kernel_s / 1e12
    tr, tr_src = traffic_for("C2")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": tr, "traffic_source": tr_src,
                "kernel": f"{'umma_wide_kernel' if plan.endswith('wide') else 'umma_gemm_kernel'} ({plan})",
                "peak_source": f"{pk['_source']} {'burst' if burst else 'sustained'} cuBLAS bf16",
                "frac_of_nominal_2250": achieved / 2250.0, "algorithmic_flop_per_launch": flops}

    # ---- e2e: the reference-facing call with HOST buffers (pinned), H2D + D2H inside the timed region ----
    ha = (torch.rand(M * Kd) * 2 - 1).to(torch.bfloat16).view(torch.int16).pin_memory()
    hb = (torch.rand(N * Kd) * 2 - 1).to(torch.bfloat16).view(torch.int16).pin_memory()
    hc = torch.zeros(M * N, dtype=torch.float32).pin_memory()
    eta = host.tensor_of(f"({M},{Kd}):({Kd},1)", ha, ranked=True)
    etb = host.tensor_of(f"({N},{Kd}):({Kd},1)", hb, ranked=True)
    etc = host.tensor_of(f"({M},{N}):(1,{M})", hc, ranked=True)
    ke = max(3, min(K, 10))
    e2e_s = wall_timed(torch, dist, world, lambda: host.gemm_bf16_host(eta, etb, etc), ke, 3)  # synchronous: returns after the D2H of C
    # verification gather (outside every timed region): one 64-bit checksum of C per rank over NCCL
    sums = shard.gather_checksums(shard.checksum64(sets[0][2][1][1]), device=RED_DEV)
    verify = {"collective": f"all_gather of per-rank C checksums ({'gloo, shared GPU' if args.share_gpu else 'nccl'})" if world > 1 else "none (1 GPU)",
              "ranks_reporting": len(sums), "all_nonzero": all(x != 0 for x in sums)}
    e2e = {"value": flops * ke * world / e2e_s / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": (M * Kd + N * Kd) * 2 + M * N * 4, "d2h_bytes_per_step": M * N * 4,
           "steps": ke, "ms_per_step": e2e_s / ke * 1e3, "api": "tlb_gemm_bf16_host (pinned host buffers)"}
    # context, not a target: the vendor library on the same box, same shape and timing recipe (cuBLAS writes bf16 C and
    # does not read it; this path reads and writes fp32 C), and torch's copy_ on the C1 footprint
    library = None
    if rank == 0 and world == 1 and not only:
        lsets = [[(torch.rand(M, Kd, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2)] for _ in range(nsets)]
        lsec = timed(torch, dist, 1, lambda i: torch.matmul(lsets[i % nsets][0], lsets[i % nsets][1].t()), K, W)
        x_ = torch.empty(8192 * 8192, dtype=torch.float32, device="cuda")
        y_ = torch.empty_like(x_)
        csec = timed(torch, dist, 1, lambda i: y_.copy_(x_), K, W)
        library = {"cublas_bf16_4096_tflops": flops * K / lsec / 1e12, "torch_copy_512MiB_gbs": 2 * x_.numel() * 4 * K / csec / 1e9,
                   "note": "torch.matmul bf16->bf16 / torch copy_ timed in this process with the same recipe"}
        # the like-for-like of the headline: the library's bf16 x bf16 GEMM with an fp32 output (beta = 0: C written, not
        # read) and with fp32 C accumulated in place (beta = 1: C += A B^T, the reference's contract, tensor.hpp:226)
        try:
            c32 = [torch.zeros(M, N, dtype=torch.float32, device="cuda") for _ in range(nsets)]
            fsec = timed(torch, dist, 1, lambda i: torch.mm(lsets[i % nsets][0], lsets[i % nsets][1].t(), out_dtype=torch.float32,
                                                             out=c32[i % nsets]), K, W)
            library["cublas_bf16_fp32_out_4096_tflops"] = flops * K / fsec / 1e12
            asec = timed(torch, dist, 1, lambda i: torch.addmm(c32[i % nsets], lsets[i % nsets][0], lsets[i % nsets][1].t(),
                                                                out_dtype=torch.float32, out=c32[i % nsets]), K, W)
            library["cublas_bf16_fp32_c_accumulate_4096_tflops"] = flops * K / asec / 1e12
            del c32
        except Exception as ex:  # an older torch without out_dtype: the bf16 -> bf16 figure stands alone
            library["fp32_out_note"] = f"torch.mm(out_dtype=float32) unavailable: {type(ex).__name__}"
        del lsets, x_, y_
    del ha, hb, hc, sets
    torch.cuda.empty_cache()

    other = []
    if not args.gemm_only:
        other = other_configs(torch, dist, world, rank, lib, host, shard, pk, K, W, args, only)

    if rank == 0 and world == 1 and not only:
        # LAST, so that it does not pre-heat the other configs: an untimed half-second loop of the C2 step with nvidia-smi
        # sampling every 20 ms. Long enough for the samples to see the load (the timed region is not); it records the
        # power-capped operating point as context.
        psets = []
        for s_ in range(nsets):
            a_ = (torch.rand(M * Kd, device="cuda") * 2 - 1).to(torch.bfloat16)
            b_ = (torch.rand(N * Kd, device="cuda") * 2 - 1).to(torch.bfloat16)
            c_ = torch.zeros(M * N, dtype=torch.float32, device="cuda")
            psets.append((host.tensor_of(f"({M},{Kd}):({Kd},1)", a_.view(torch.int16), ranked=True),
                          host.tensor_of(f"({N},{Kd}):({Kd},1)", b_.view(torch.int16), ranked=True),
                          host.tensor_of(f"({M},{N}):(1,{M})", c_, ranked=True)))
        for i in range(3):
            host.gemm_bf16(*psets[i % nsets])
        torch.cuda.synchronize()
        probe = ClockSampler(local)
        probe.start(20)
        time.sleep(0.1)
        n_probe = max(50, int(0.5 / max(sec / K, 1e-6)))
        p0 = time.time()
        psec = timed(torch, dist, 1, lambda i: host.gemm_bf16(*psets[i % nsets]), n_probe, 0)
        p1 = time.time()
        pc = probe.stop(p0 + 0.1, p1)
        clocks["sustained_probe"] = {"steps": n_probe, "seconds": round(psec, 3), "tflops": flops * n_probe / psec / 1e12,
                                     "sm_mhz": pc["sm_mhz"], "power_w": pc.get("power_w"), "reasons": pc["reasons"],
                                     "samples": pc.get("samples"),
                                     "frac_of_sustained_peak": flops * n_probe / psec / 1e12 / pk.get("bf16_tflops_sustained", pk["bf16_tflops"])}
        del psets

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:   # N = 1 only: at N > 1 the other ranks would idle at the next barrier
        threads = os.cpu_count() or 1
        dt, macs, kind = cpu_gemm_sample(2, 16, 4096, threads)
        per_mac = dt * threads / macs
        m_rows = max(1, min(64, int(15.0 / (per_mac * 64 * 4096))))
        dt, macs, kind = cpu_gemm_sample(m_rows, 64, 4096, threads)
        cpu = {"value": 2.0 * macs / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
               "sample": f"tla::gemm verbatim (checked int64) on a {m_rows * threads}x64x4096 sub-problem of the "
                         f"4096^3 TN workload, {threads} host threads, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": "gemm_tflops", "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": sec / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "C2: bf16 4096^3 TN GEMM, fp32 accumulate, C += A*B^T (configs[1]), one problem per GPU",
                       "M": M, "N": N, "K": Kd, "plan": plan,
                       "l2": f"{nsets} rotating operand sets ({nsets * 128} MiB) > 126 MB L2",
                       "sharding": "independent problems per rank, no data-path collective"},
            "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
            "verify": verify, "library_same_box": library, "other_configs": other,
        }
        if args.share_gpu and world > 1:
            line["shared_gpu"] = "all ranks on cuda:0 (functional test of the N-rank path; NOT a scaling measurement)"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def other_configs(torch, dist, world, rank, lib, host, shard, pk, K, W, args, only):
    """C1 (8192^2 fp32 transpose), C3 (4 GiB hierarchical permute), C5 (2^32 index maps, 2^28-element chunks), two
    fallback-plan copies, C2 with bf16 C and C4: same timing rules, own roofline. Inputs exceed L2 (512 MiB / 8 GiB /
    2 GiB per step). At N > 1 the NAMED problem is sharded by coordinate ranges (strong scaling): every rank runs
    tlb_copy / tlb_eval_range on its own range, value = whole-problem bytes / max-over-ranks time."""
    out = []
    hbm = pk["hbm_gbs"]
    want = lambda name: only is None or name in only
    cpu_ok = rank == 0 and world == 1 and not args.no_cpu   # the CPU legs run at N = 1 only

    def entry(name, metric, workload, bytes_per_step, sec, steps, plan, kernel, extra=None):
        # bytes_per_step is the WHOLE problem's algorithmic bytes; at N > 1 each rank moved 1/N of them per step
        gbs = bytes_per_step * steps / sec / 1e9
        per_gpu = gbs / world
        tr, tr_src = traffic_for(name)
        e = {"name": name, "metric": metric, "value": gbs, "unit": "GB/s", "n_gpus": world,
             "scaling": "strong" if world > 1 else "n/a (1 GPU)", "steps": steps,
             "ms_per_step": sec / steps * 1e3, "config": {"workload": workload, "plan": plan},
             "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": hbm, "unit": "GB/s", "frac": per_gpu / hbm,
                          "traffic": tr, "traffic_source": tr_src, "kernel": kernel,
                          "peak_source": f"{pk['_source']} torch copy_",
                          "frac_of_nominal_8000": per_gpu / 8000.0, "algorithmic_bytes_per_launch": bytes_per_step / world}}
        if extra:
            e.update(extra)
        return e

    def copy_config(name, s, d, eb, workload, kernel, steps, warm, cpu_sample=None, e2e_steps=0, dtype=torch.int32, tv_threads=0):
        n = host.L(s).size
        src = torch.arange(host.L(s).lower().max_offset + 1, dtype=dtype, device="cuda")   # element-index bit patterns
        dst = torch.empty(host.L(d).lower().max_offset + 1, dtype=dtype, device="cuda")
        a = host.tensor_of(s, src)
        b = host.tensor_of(d, dst)
        i0, i1 = shard.copy_range(s, world, rank) if world > 1 else (0, 2**64 - 1)
        if tv_threads:   # the copy partitioned by the library-derived thread-value layout (every rank the whole problem)
            tv = host.copy_tv_auto(s, d, eb, tv_threads)
            sec = timed(torch, dist, world, lambda i: host.copy_tv(a, b, tv), steps, warm)
        else:
            sec = timed(torch, dist, world, lambda i: host.copy(a, b, i0, i1), steps, warm)
        plan = lib.tlb_last_plan().decode()
        extra = {}
        if world > 1:
            extra["shard"] = {"rank0_range": list(shard.copy_range(s, world, 0)), "how": "shard.copy_range: whole slices of the outermost mode per rank"}
        del src, dst
        torch.cuda.empty_cache()
        if e2e_steps:
            hs = torch.empty(host.L(s).lower().max_offset + 1, dtype=dtype).pin_memory()
            hs.random_(0, 2**31 - 1)
            hd = torch.empty(host.L(d).lower().max_offset + 1, dtype=dtype).pin_memory()
            ha_, hb_ = host.tensor_of(s, hs), host.tensor_of(d, hd)
            esec = wall_timed(torch, dist, world, lambda: host.copy_host(ha_, hb_), e2e_steps, 1)
            extra["e2e"] = {"value": 2.0 * eb * n * e2e_steps * world / esec / 1e9, "unit": "GB/s",
                            "h2d_bytes_per_step": hs.numel() * eb, "d2h_bytes_per_step": hd.numel() * eb, "steps": e2e_steps,
                            "ms_per_step": esec / e2e_steps * 1e3,
                            "api": "tlb_copy_host (pinned host buffers; every rank copies the whole problem: weak)" if world > 1
                                   else "tlb_copy_host (pinned host buffers)"}
            del hs, hd
        if cpu_ok and cpu_sample:
            extra["cpu_baseline"] = cpu_copy_baseline(*cpu_sample)
        out.append(entry(name, "copy_gbs", workload, 2 * n * eb, sec, steps, plan, kernel, extra))

    # C1
    if want("C1"):
        n = 8192
        copy_config("C1", f"({n},{n}):({n},1)", f"({n},{n}):(1,{n})", 4,
                    "fp32 8192x8192 transpose copy (8192,8192):(8192,1) -> (8192,8192):(1,8192) (configs[0])", "tiled_kernel", K, W,
                    cpu_sample=("(2048,2048):(8192,1)", "(2048,2048):(1,8192)", 4, "a 2048x2048 sub-block of C1 with the same strides (1/16 of the elements)"),
                    e2e_steps=max(3, min(K, 5)))
    # C3
    if want("C3"):
        T = 4096
        copy_config("C3", f"((8,128),(4,64),{T}):((1,2048),(8,32),262144)", f"((8,128),(4,64),{T}):((128,1),(65536,1024),262144)", 4,
                    "hierarchical permute copy ((8,128),(4,64)) x 4096 tiles, 4 GiB tensors, Swizzle<3,4,3> smem staging (configs[2])",
                    "tiled_kernel", max(3, K // 4), 3,
                    cpu_sample=("((8,128),(4,64),8):((1,2048),(8,32),262144)", "((8,128),(4,64),8):((128,1),(65536,1024),262144)", 4,
                                "8 of the 4096 tiles of C3 (1/512 of the elements)"),
                    e2e_steps=0 if args.quick else 2)
    # fallback plans: an Xor (swizzled) destination and a non-injective destination
    if want("Cx"):
        copy_config("Cx_xor_dst", "(128,8,65536):(1,128,1024)", "(128,8,65536):(f1,f144,f1024)", 4,
                    "2^26 fp32 elements into a Swizzle<3,4,3>-per-KiB destination (128,8,65536):(f1,f144,f1024)", "gather_run_kernel (Xor strides, one evaluation per 64-byte run, 256-bit accesses)",
                    max(3, K // 4), 3)
        copy_config("Cx_ragged_transpose", "(8000,6000):(6000,1)", "(8000,6000):(1,8000)", 4,
                    "fp32 8000x6000 transpose: rows are not whole 128-byte pieces nor whole tiles (whole-tile body on the staged plan + edge strips)",
                    "tiled_kernel (body) + gather_joint_kernel (edge strips)", max(3, K // 4), 3)
        copy_config("Cx_interleave", "(4,16777216):(1,4)", "(4,16777216):(16777216,1)", 4,
                    "AoS -> SoA: 2^24 fp32 4-vectors de-interleaved into four planar rows (register-permuting interleave plan, 256-bit accesses)",
                    "interleave_kernel<4, 4, true>", max(3, K // 4), 3)
        copy_config("Cx_non_injective_dst", "(8192,4096):(1,8192)", "(8192,4096):(1,8191)", 4,
                    "2^25 fp32 elements into a destination whose columns overlap by one cell (stride 8191 < 8192: last writer wins, tensor.hpp:198)",
                    "winner_kernel + ordered_kernel", max(3, K // 8), 2)
        # the paper's own way of partitioning a copy (local_partition by a thread-value layout): the C1 layouts
        # through tlb_copy_tv with the TV layout the library derives (max_common_vector + raked_product); the digit-permutation
        # TV layout composes with both tensors and the call runs the planner's staged plan in TV's order
        if world == 1:
            copy_config("Cx_tv_partitioned", "(8192,8192):(8192,1)", "(8192,8192):(1,8192)", 4,
                        "C1's transpose partitioned by the derived thread-value layout (256 threads): tlb_copy_tv = tlb_copy between src o TV and dst o TV",
                        "tiled_kernel", max(3, K // 2), 3, tv_threads=256)
        # a stride-0 (broadcast) destination mode: only the slice at its last coordinate survives, so the call is an 8192-element
        # copy; reported as elements of the reference's loop retired per second, not as bandwidth
        n_b = 8192 * 4096
        src_b = torch.arange(n_b, dtype=torch.int32, device="cuda")
        dst_b = torch.empty(8192, dtype=torch.int32, device="cuda")
        ab, bb = host.tensor_of("(8192,4096):(1,8192)", src_b), host.tensor_of("(8192,4096):(1,0)", dst_b)
        kb = max(3, K // 2)
        sec_b = timed(torch, dist, world, lambda i: host.copy(ab, bb), kb, 3)
        out.append({"name": "Cx_broadcast_dst", "metric": "copy_elements_per_s", "value": n_b * kb * world / sec_b, "unit": "elements/s", "n_gpus": world,
                    "scaling": "weak", "steps": kb, "ms_per_step": sec_b / kb * 1e3,
                    "config": {"workload": "2^25 fp32 elements into (8192,4096):(1,0): 4096 writers per cell, the last one wins (tensor.hpp:198); "
                                           "runs as the injective copy of the last column", "plan": lib.tlb_last_plan().decode()},
                    "roofline": None})
        del src_b, dst_b
    # C5: index maps of the 2^32-element divided layout, materialised in 2^28-element chunks (2 GiB)
    if want("C5"):
        Lt = "((128,64),(512,1024)):((65536,1),(8388608,64))"
        Rt = "(64,1024,128,512):(128,4194304,1,8192)"
        chunk = 2 ** 28
        steps5 = max(4, K // 2)
        c0, c1 = shard.even_split(chunk, world, rank, align=4096)    # this rank's slice of every chunk
        cn = c1 - c0
        buf = torch.empty(cn, dtype=torch.int64, device="cuda")
        note = ("write-only kernel: the denominator is the read+write copy peak, a pure write stream (torch fill_ of 2 GiB) "
                "measured 7533 GB/s on this pool, so frac may exceed 1")
        sec = timed(torch, dist, world, lambda i: host.eval_range(Lt, (i % 16) * chunk + c0, cn, buf), steps5, 3)
        extra = {"evals_per_s": chunk * steps5 / sec, "note": note}
        if cpu_ok:
            extra["cpu_baseline"] = cpu_eval_baseline(Lt, 2 ** 22)
        if not args.quick:
            hbuf = torch.empty(cn, dtype=torch.int64).pin_memory()
            esec = wall_timed(torch, dist, world, lambda: host.eval_range_host(Lt, 3 * chunk + c0, cn, hbuf), 2, 1)
            extra["e2e"] = {"value": chunk * 8 * 2 / esec / 1e9, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": cn * 8,
                            "steps": 2, "ms_per_step": esec / 2 * 1e3, "api": "tlb_eval_range_host (pinned host output)"}
            del hbuf
        out.append(entry("C5", "index_map_gbs", "L(i): index map of the 2^32-element zipped_divide layout, 2^28-element chunks, int64 out (configs[4])",
                         chunk * 8, sec, steps5, lib.tlb_last_plan().decode(), "eval_warp_kernel", extra))
        sec = timed(torch, dist, world, lambda i: host.eval_range(Rt, (i % 16) * chunk + c0, cn, buf), steps5, 3)
        out.append(entry("C5_rinv", "index_map_gbs", "R(k) = right_inverse(L)(k), 2^28-element chunks, int64 out (configs[4])",
                         chunk * 8, sec, steps5, lib.tlb_last_plan().decode(), "eval_warp_kernel",
                         {"evals_per_s": chunk * steps5 / sec, "note": note}))
        del buf
        # natural coordinates and back: idx2crd writes 4 leaves per index (32 B), crd2idx reads them and writes 8 B
        n5 = 2 ** 26
        q0, q1 = shard.even_split(n5, world, rank, align=4096)
        qn = q1 - q0
        crd = torch.empty(qn * 4, dtype=torch.int64, device="cuda")
        idx = torch.empty(qn, dtype=torch.int64, device="cuda")
        sec = timed(torch, dist, world, lambda i: host.idx2crd_range(Lt, (i % 64) * n5 + q0, qn, crd), steps5, 3)
        out.append(entry("C5_idx2crd", "index_map_gbs", "idx2crd: natural coordinates (4 leaves) of 2^26 indices per step, int64 out",
                         n5 * 32, sec, steps5, "idx2crd", "idx2crd_kernel<4>", {"evals_per_s": n5 * steps5 / sec}))
        sec = timed(torch, dist, world, lambda i: host.crd2idx_range(Lt, crd, qn, idx), steps5, 3)
        out.append(entry("C5_crd2idx", "index_map_gbs", "crd2idx of 2^26 natural coordinates per step (32 B read + 8 B written per index)",
                         n5 * 40, sec, steps5, "crd2idx", "crd2idx_kernel", {"evals_per_s": n5 * steps5 / sec}))
        del crd, idx
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        sec = timed(torch, dist, world, lambda i: host.rinv_check_range(Lt, Rt, (i % 16) * chunk + c0, cn, cnt), steps5, 3)
        torch.cuda.synchronize()
        out.append({"name": "C5_check", "metric": "checks_per_s", "value": chunk * steps5 / sec, "unit": "evaluations/s", "n_gpus": world,
                    "steps": steps5, "ms_per_step": sec / steps5 * 1e3, "mismatches": int(cnt.item()),
                    "config": {"workload": "L(R(k)) == k checked on device for 2^28 k per step (no output: compute bound)", "plan": "rinv_check"},
                    "roofline": None})
        torch.cuda.empty_cache()
    # C2 with C in the operands' type (bf16 C += A B^T, fp32 accumulation in TMEM, one rounding, bf16 reduction at L2): the
    # like-for-like workload of the cuBLAS bf16 -> bf16 figure that MEASURED_PEAKS.json and library_same_box quote
    if want("C2_bf16_c"):
        M2 = 4096
        sets16 = []
        g2 = torch.Generator(device="cuda").manual_seed(7)
        for _ in range(3):
            a16 = (torch.rand(M2 * M2, device="cuda", generator=g2) * 2 - 1).to(torch.bfloat16)
            b16 = (torch.rand(M2 * M2, device="cuda", generator=g2) * 2 - 1).to(torch.bfloat16)
            c16 = torch.zeros(M2 * M2, dtype=torch.bfloat16, device="cuda")
            sets16.append((host.tensor_of(f"({M2},{M2}):({M2},1)", a16.view(torch.int16), ranked=True),
                           host.tensor_of(f"({M2},{M2}):({M2},1)", b16.view(torch.int16), ranked=True),
                           host.tensor_of(f"({M2},{M2}):(1,{M2})", c16.view(torch.int16), ranked=True)))
        sec = timed(torch, dist, world, lambda i: host.gemm_bf16(*sets16[i % 3]), K, W)
        tf16 = 2.0 * M2 ** 3 * K * world / sec / 1e12
        per16 = 2.0 * M2 ** 3 / (sec / K) / 1e12
        tr, tr_src = traffic_for("C2_bf16_c")
        out.append({"name": "C2_bf16_c", "metric": "gemm_tflops", "value": tf16, "unit": "TFLOP/s", "ms_per_step": sec / K * 1e3,
                    "n_gpus": world, "scaling": "weak",
                    "config": {"workload": "C2 shape with C in bf16 (C += A B^T, fp32 accumulation in TMEM, bf16 L2 reduction): the output "
                                           "type of the cuBLAS figure the peak was measured with", "plan": lib.tlb_last_plan().decode()},
                    "roofline": {"bound": "tensor", "achieved": per16, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                                 "frac": per16 / pk["bf16_tflops"], "traffic": tr, "traffic_source": tr_src, "kernel": "umma_wide_kernel",
                                 "peak_source": f"{pk['_source']} burst cuBLAS bf16", "frac_of_nominal_2250": per16 / 2250.0,
                                 "algorithmic_flop_per_launch": 2.0 * M2 ** 3}})
        del sets16
        torch.cuda.empty_cache()
    # The other operand families of the paper's GEMM table: GETT-folded modes on tcgen05 through
    # rank-4/5 tensor maps, and BLIS strides (no unit stride: not TMA-addressable) on the tiled SIMT plan
    if want("Cg"):
        def gemm_family(name, la, lb, lc, workload, steps, kernel):
            Lx = host.L
            M_ = 1
            for e, *_ in Lx(la).modes[:Lx(la).top_leaves[0]]:
                M_ *= e
            N_ = 1
            for e, *_ in Lx(lb).modes[:Lx(lb).top_leaves[0]]:
                N_ *= e
            K_ = Lx(la).size // M_
            fsets = []
            for _ in range(2):
                a_ = torch.empty(Lx(la).lower().max_offset + 1, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
                b_ = torch.empty(Lx(lb).lower().max_offset + 1, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
                c_ = torch.zeros(Lx(lc).lower().max_offset + 1, dtype=torch.float32, device="cuda")
                fsets.append((host.tensor_of(la, a_.view(torch.int16), ranked=True), host.tensor_of(lb, b_.view(torch.int16), ranked=True),
                              host.tensor_of(lc, c_, ranked=True)))
            sec = timed(torch, dist, world, lambda i: host.gemm_bf16(*fsets[i % 2]), steps, 3)
            fl = 2.0 * M_ * N_ * K_
            per = fl / (sec / steps) / 1e12
            plan_ = lib.tlb_last_plan().decode()
            if not plan_.startswith("packed"):   # name the kernel the planner actually chose
                kernel = "umma_wide_kernel" if plan_.endswith("wide") else "umma_gemm_kernel"
            out.append({"name": name, "metric": "gemm_tflops", "value": fl * steps * world / sec / 1e12, "unit": "TFLOP/s", "n_gpus": world,
                        "scaling": "weak", "steps": steps, "ms_per_step": sec / steps * 1e3,
                        "config": {"workload": workload, "A": la, "B": lb, "C": lc, "plan": plan_},
                        "roofline": {"bound": "tensor", "achieved": per, "peak": pk["bf16_tflops"], "unit": "TFLOP/s", "frac": per / pk["bf16_tflops"],
                                     "traffic": None, "kernel": kernel, "peak_source": f"{pk['_source']} burst cuBLAS bf16",
                                     "frac_of_nominal_2250": per / 2250.0, "algorithmic_flop_per_launch": fl}})
            del fsets
            torch.cuda.empty_cache()
        gemm_family("Cg_gett_folded", "((128,32),(64,64)):((64,524288),(1,8192))", "((128,32),(64,64)):((64,524288),(1,8192))",
                    "(4096,4096):(1,4096)", "GETT: 4096^3 with m, n and k each folded into two leaves (rank-5 tensor maps), TN output", K,
                    "umma_wide_kernel")
        gemm_family("Cg_blis_strided", "(2048,2048):(3,6151)", "(2048,2048):(2,4099)", "(2048,2048):(5,10243)",
                    "BLIS: 2048^3 with general strides on every mode (no unit stride anywhere): packed by tlb_copy, tcgen05 on the "
                    "packed panels, C scattered back (the step times all five kernels)", max(3, K // 2), "copy kernels + umma_gemm_kernel")
        # CONV: fprop as a GEMM whose A is the im2col LAYOUT of the NHWC activations (no im2col buffer):
        # rows (q, p, n), k (c, s, r); 32 x 34 x 34 x 128 input, 3 x 3 filters, 1024 output channels
        gemm_family("Cg_conv_im2col", "((32,32,32),(128,3,3)):((128,4352,147968),(1,128,4352))", "(1024,1152):(1152,1)",
                    "(32768,1024):(1024,1)", "CONV fprop: 32x34x34x128 NHWC input, 3x3 filters, 1024 output channels, as a GEMM over the "
                    "im2col layout of the input (rank-5 tensor map: leaves q, p, n | c s, r), M 32768, N 1024, K 1152", K, "umma_wide_kernel")
    # C4: batched bf16 GEMM 64 x 8192^3, sharded by whole batches (= tile-id ranges) across the ranks (strong
    # scaling of the 64 batches; every rank owns its batches' operands, no data-path collective)
    if want("C4"):
        M = 8192
        b0, b1 = shard.batch_range(64, world, rank)
        nb = b1 - b0
        a = torch.empty(nb * M * M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
        b = torch.empty(nb * M * M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
        c = torch.zeros(nb * M * M, dtype=torch.float32, device="cuda")
        ta = host.tensor_of(f"({M},{M}):({M},1)", a.view(torch.int16), ranked=True)
        tb = host.tensor_of(f"({M},{M}):({M},1)", b.view(torch.int16), ranked=True)
        tc = host.tensor_of(f"({M},{M}):(1,{M})", c, ranked=True)
        k4 = 3
        n_l0 = lib.tlb_launch_count()
        sec = timed(torch, dist, world, lambda i: host.gemm_bf16_batched(ta, tb, tc, M * M, M * M, M * M, 0, nb), k4, 3)
        launches_c4 = int(lib.tlb_launch_count() - n_l0) // (k4 + 3)   # the call is cut into launches of ~8 waves (one per batch)
        flops = 2.0 * M * M * M * 64
        tf = flops * k4 / sec / 1e12
        per_gpu = 2.0 * M * M * M * nb / (sec / k4) / 1e12
        sustained = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        tr, tr_src = traffic_for("C4")
        out.append({"name": "C4", "metric": "gemm_tflops", "value": tf, "unit": "TFLOP/s", "ms_per_step": sec / k4 * 1e3,
                    "steps": k4, "scaling": "strong", "n_gpus": world,
                    "config": {"workload": "batched bf16 GEMM 64 x (8192^3), fp32 accumulate, batches sharded across ranks (configs[3])",
                               "batches_this_rank": nb, "plan": lib.tlb_last_plan().decode()},
                    "roofline": {"bound": "tensor", "achieved": per_gpu, "peak": sustained, "unit": "TFLOP/s",
                                 "frac": per_gpu / sustained, "traffic": tr, "traffic_source": tr_src, "kernel": "umma_wide_kernel",
                                 "peak_source": f"{pk['_source']} sustained cuBLAS bf16 (step >= 50 ms)",
                                 "frac_of_nominal_2250": per_gpu / 2250.0,
                                 "algorithmic_flop_per_launch": 2.0 * M * M * M, "launches_per_step": launches_c4,
                                 "traffic_note": "per 8192^3 batch = per launch (the call is cut into one launch per batch)"}})
        del a, b, c
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gemm-path", default="auto", choices=["auto", "1sm", "2sm"])
    ap.add_argument("--gemm-only", action="store_true", help="skip the other_configs lines (profiling runs)")
    ap.add_argument("--only", default="", help="comma-separated other_configs to run (C1,C3,Cx,C5,C2_bf16_c,Cg,C4): profiling runs")
    ap.add_argument("--quick", action="store_true", help="skip the multi-GiB pinned-host e2e legs of C3 / C5")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs (profiling runs)")
    ap.add_argument("--share-gpu", action="store_true", help="testing only: run the N ranks on cuda:0 over gloo when the box has fewer than N GPUs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    maybe_spawn(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
