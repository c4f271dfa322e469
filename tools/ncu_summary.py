"""Summarises .ncu-rep captures into profiles/*.json / *.txt (run here, no GPU needed):

    python tools/ncu_summary.py <report.ncu-rep> <out_prefix> [kernel-substring ...]

Per launch: duration, DRAM bytes, DRAM / tensor-pipe / L2 utilisation, registers, grid. Also writes
profiles/traffic.json (dram read+write bytes per launch per kernel family) that bench.py reports as
roofline.traffic.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct_of_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__cycles_active.avg": "sm_cycles_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0,
              "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    want = sys.argv[3:]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        name = rec.get("Kernel Name", "")
        if want and not any(w in name for w in want):
            continue
        e = {"kernel": name.split("(")[0][-80:]}
        for k, short in KEYS.items():
            if k in rec and rec[k] != "":
                try:
                    val = float(rec[k].replace(",", ""))
                except ValueError:
                    continue
                unit = units[hdr.index(k)]
                if short in ("duration", "dram_read", "dram_write"):
                    val *= UNIT_SCALE.get(unit, 1.0)
                if short == "sm_clock":
                    val *= {"Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "GHz": 1e9, "MHz": 1e6}.get(unit, 1.0)
                e[short] = val
        if "dram_read" in e and "dram_write" in e:
            e["dram_bytes"] = e["dram_read"] + e["dram_write"]
            if e.get("duration"):
                e["dram_gbs"] = e["dram_bytes"] / e["duration"] / 1e9
        out.append(e)
    Path(prefix + ".json").write_text(json.dumps(out, indent=1))
    with open(prefix + ".txt", "w") as f:
        for e in out:
            f.write(" ".join(f"{k}={v:.6g}" if isinstance(v, float) else f"{k}={v}" for k, v in e.items()) + "\n")
    print(f"{len(out)} launches -> {prefix}.json/.txt")


if __name__ == "__main__":
    main()
