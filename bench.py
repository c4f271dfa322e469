#!/usr/bin/env python
"""Benchmark of the layout-driven hot path (BASELINE.json: "copy GB/s & GEMM TFLOP/s (% of B200 roofline)
vs CPU ref").

    python bench.py --gpus N --steps K --warmup W            # our arm (libtlb.so, sm_100a)
    python bench.py --impl reference --gpus N ...            # the reference's own CPU implementation

One JSON line on stdout (rank 0). The headline workload is BASELINE.json configs[1] (C2: bf16 4096^3 TN GEMM,
fp32 accumulate); a "step" is one such GEMM per GPU (weak scaling: every rank owns one independent problem,
no collective on the data path). The copy / index-map configs (C1, C3, C5) are timed in the same run and
reported under "other_configs", each with its own HBM roofline.
"""
from __future__ import annotations

import argparse
import json
import os
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


# --------------------------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation (oracle/_ref when it was built, else the C port)
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
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms / 1e3


def traffic_for(config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full capture of the
    same workload (profiles/traffic.json, written by tools/ncu_summary.py); None when no capture exists."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        e = json.loads(p.read_text()).get(config)
        return e["dram_bytes_per_launch"] if e else None
    return None


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_02298_b200 import abi, host

    rank, world, local = dist_env()
    assert torch.cuda.is_available(), "bench.py needs a CUDA device: libtlb has no CPU fallback"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ.setdefault("TLB_GEMM_CLOCK", "1")  # the GEMM kernels stamp {clock64, globaltimer}: SM clock under load
    lib = abi.load()
    pk = peaks()
    K, W = args.steps, args.warmup

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
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic_for("C2"), "kernel": f"{'umma_wide_kernel' if plan.endswith('wide') else 'umma_gemm_kernel'} ({plan})",
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
    for _ in range(3):
        host.gemm_bf16_host(eta, etb, etc)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        host.gemm_bf16_host(eta, etb, etc)   # synchronous: returns after the D2H of C
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # verification gather (outside every timed region): one 64-bit checksum of C per rank over NCCL
    from paper_2603_02298_b200 import shard
    sums = shard.gather_checksums(shard.checksum64(sets[0][2][1][1]), device="cuda")
    verify = {"collective": "all_gather of per-rank C checksums (nccl)" if world > 1 else "none (1 GPU)",
              "ranks_reporting": len(sums), "all_nonzero": all(x != 0 for x in sums)}
    e2e = {"value": flops * ke * world / e2e_s / 1e12, "unit": "TFLOP/s",
           "h2d_bytes_per_step": (M * Kd + N * Kd) * 2 + M * N * 4, "d2h_bytes_per_step": M * N * 4,
           "steps": ke, "ms_per_step": e2e_s / ke * 1e3, "api": "tlb_gemm_bf16_host (pinned host buffers)"}
    # context, not a target: the vendor library on the same box, same shape and timing recipe (cuBLAS writes bf16 C and
    # does not read it; this path reads and writes fp32 C), and torch's copy_ on the C1 footprint
    library = None
    if rank == 0 and world == 1:
        lsets = [[(torch.rand(M, Kd, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2)] for _ in range(nsets)]
        lsec = timed(torch, dist, 1, lambda i: torch.matmul(lsets[i % nsets][0], lsets[i % nsets][1].t()), K, W)
        x_ = torch.empty(8192 * 8192, dtype=torch.float32, device="cuda")
        y_ = torch.empty_like(x_)
        csec = timed(torch, dist, 1, lambda i: y_.copy_(x_), K, W)
        library = {"cublas_bf16_4096_tflops": flops * K / lsec / 1e12, "torch_copy_512MiB_gbs": 2 * x_.numel() * 4 * K / csec / 1e9,
                   "note": "torch.matmul bf16->bf16 / torch copy_ timed in this process with the same recipe"}
        del lsets, x_, y_
    del ha, hb, hc, sets
    torch.cuda.empty_cache()

    other = []
    if not args.gemm_only:
        other = other_configs(torch, dist, world, lib, host, pk, K, W)

    if rank == 0 and world == 1:
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
                                     "samples": pc.get("samples")}
        del psets

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
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
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def other_configs(torch, dist, world, lib, host, pk, K, W):
    """C1 (8192^2 fp32 transpose), C3 (4 GiB hierarchical permute) and C5 (2^32 index map, 2^28-element chunks):
    same timing rules, HBM roofline. Inputs exceed L2 (512 MiB / 8 GiB / 2 GiB per step)."""
    out = []
    hbm = pk["hbm_gbs"]

    def entry(name, workload, bytes_per_step, sec, steps, plan, kernel, extra=None):
        gbs = bytes_per_step * steps * world / sec / 1e9
        per_gpu = bytes_per_step / (sec / steps) / 1e9
        e = {"name": name, "metric": "copy_gbs" if name != "C5" else "index_map_gbs", "value": gbs, "unit": "GB/s",
             "ms_per_step": sec / steps * 1e3, "config": {"workload": workload, "plan": plan},
             "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": hbm, "unit": "GB/s", "frac": per_gpu / hbm,
                          "traffic": traffic_for(name), "kernel": kernel, "peak_source": f"{pk['_source']} torch copy_",
                          "frac_of_nominal_8000": per_gpu / 8000.0, "algorithmic_bytes_per_launch": bytes_per_step}}
        if extra:
            e.update(extra)
        return e

    # C1
    n = 8192
    src = torch.arange(n * n, dtype=torch.int32, device="cuda")
    dst = torch.empty(n * n, dtype=torch.int32, device="cuda")
    a = host.tensor_of(f"({n},{n}):({n},1)", src)
    b = host.tensor_of(f"({n},{n}):(1,{n})", dst)
    sec = timed(torch, dist, world, lambda i: host.copy(a, b), K, W)
    out.append(entry("C1", "fp32 8192x8192 transpose copy (8192,8192):(8192,1) -> (8192,8192):(1,8192) (configs[0])",
                     2 * n * n * 4, sec, K, lib.tlb_last_plan().decode(), "tiled_kernel"))
    del src, dst
    # C3
    T = 4096
    s = f"((8,128),(4,64),{T}):((1,2048),(8,32),262144)"
    d = f"((8,128),(4,64),{T}):((128,1),(65536,1024),262144)"
    src = torch.empty(262144 * T, dtype=torch.int32, device="cuda")
    src.copy_(torch.arange(262144 * T, dtype=torch.int32, device="cuda"))
    dst = torch.empty(262144 * T, dtype=torch.int32, device="cuda")
    a = host.tensor_of(s, src)
    b = host.tensor_of(d, dst)
    k3 = max(3, K // 4)
    sec = timed(torch, dist, world, lambda i: host.copy(a, b), k3, 3)
    out.append(entry("C3", "hierarchical permute copy ((8,128),(4,64)) x 4096 tiles, 4 GiB tensors, Swizzle<3,4,3> smem staging (configs[2])",
                     2 * 262144 * T * 4, sec, k3, lib.tlb_last_plan().decode(), "tiled_kernel", {"steps": k3}))
    del src, dst
    torch.cuda.empty_cache()
    # C5: index maps of the 2^32-element divided layout, materialised in 2^28-element chunks (2 GiB)
    Lt = "((128,64),(512,1024)):((65536,1),(8388608,64))"
    chunk = 2 ** 28
    buf = torch.empty(chunk, dtype=torch.int64, device="cuda")
    sec = timed(torch, dist, world, lambda i: host.eval_range(Lt, (i % 16) * chunk, chunk, buf), max(4, K // 2), 3)
    steps5 = max(4, K // 2)
    out.append(entry("C5", "crd2idx / index map of the 2^32-element zipped_divide layout, 2^28-element chunks, int64 out (configs[4])",
                     chunk * 8, sec, steps5, "eval_range", "eval_warp_kernel",
                     {"steps": steps5, "evals_per_s": chunk * steps5 * world / sec,
                      "note": "write-only kernel: the denominator is the read+write copy peak, a pure write stream (torch fill_ "
                              "of 2 GiB) measured 7533 GB/s on this pool, so frac may exceed 1"}))
    del buf
    torch.cuda.empty_cache()
    # C2 with C in the operands' type (bf16 C += A B^T, fp32 accumulation in TMEM, one rounding, bf16 reduction at L2): the
    # like-for-like workload of the cuBLAS bf16 -> bf16 figure that MEASURED_PEAKS.json and library_same_box quote
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
    out.append({"name": "C2_bf16_c", "metric": "gemm_tflops", "value": tf16, "unit": "TFLOP/s", "ms_per_step": sec / K * 1e3,
                "config": {"workload": "C2 shape with C in bf16 (C += A B^T, fp32 accumulation in TMEM, bf16 L2 reduction): the output "
                                       "type of the cuBLAS figure the peak was measured with", "plan": lib.tlb_last_plan().decode()},
                "roofline": {"bound": "tensor", "achieved": per16, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                             "frac": per16 / pk["bf16_tflops"], "traffic": None, "kernel": "umma_wide_kernel",
                             "peak_source": f"{pk['_source']} burst cuBLAS bf16", "frac_of_nominal_2250": per16 / 2250.0,
                             "algorithmic_flop_per_launch": 2.0 * M2 ** 3}})
    del sets16
    torch.cuda.empty_cache()
    # C4: batched bf16 GEMM 64 x 8192^3, sharded by whole batches (= tile-id ranges) across the ranks (strong
    # scaling of the 64 batches; every rank owns its batches' operands, no data-path collective)
    from paper_2603_02298_b200 import shard
    M = 8192
    rank = dist.get_rank() if world > 1 else 0
    b0, b1 = shard.batch_range(64, world, rank)
    nb = b1 - b0
    a = torch.empty(nb * M * M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    b = torch.empty(nb * M * M, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
    c = torch.zeros(nb * M * M, dtype=torch.float32, device="cuda")
    ta = host.tensor_of(f"({M},{M}):({M},1)", a.view(torch.int16), ranked=True)
    tb = host.tensor_of(f"({M},{M}):({M},1)", b.view(torch.int16), ranked=True)
    tc = host.tensor_of(f"({M},{M}):(1,{M})", c, ranked=True)
    k4 = 3
    sec = timed(torch, dist, world, lambda i: host.gemm_bf16_batched(ta, tb, tc, M * M, M * M, M * M, 0, nb), k4, 3)
    flops = 2.0 * M * M * M * 64
    tf = flops * k4 / sec / 1e12
    per_gpu = 2.0 * M * M * M * nb / (sec / k4) / 1e12
    sustained = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    out.append({"name": "C4", "metric": "gemm_tflops", "value": tf, "unit": "TFLOP/s", "ms_per_step": sec / k4 * 1e3,
                "steps": k4, "scaling": "strong",
                "config": {"workload": "batched bf16 GEMM 64 x (8192^3), fp32 accumulate, batches sharded across ranks (configs[3])",
                           "batches_this_rank": nb, "plan": lib.tlb_last_plan().decode()},
                "roofline": {"bound": "tensor", "achieved": per_gpu, "peak": sustained, "unit": "TFLOP/s",
                             "frac": per_gpu / sustained, "traffic": traffic_for("C4"), "kernel": "umma_wide_kernel",
                             "peak_source": f"{pk['_source']} sustained cuBLAS bf16 (step >= 50 ms)",
                             "frac_of_nominal_2250": per_gpu / 2250.0,
                             "algorithmic_flop_per_launch": 2.0 * M * M * M * nb}})
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
    ap.add_argument("--gemm-only", action="store_true", help="skip the C1/C3/C5 lines (profiling runs)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (profiling runs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
