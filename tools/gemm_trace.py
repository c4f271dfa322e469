"""Reads a TLB_GEMM_TRACE dump and prints the per-CTA timeline summary (debug tool)."""
import sys
import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.int64)
grid, slots, cg, split = raw[:4]
t = raw[4:].reshape(grid, slots)
start = t[:, 0]
print(f"grid={grid} cg={cg} split={split}")
life = t[:, 120] - start
print("lifetime cycles: min %d  median %d  max %d" % (life.min(), np.median(life), life.max()))
print("setup (start->after sync): median %d" % np.median(t[:, 1] - start))
gt = t[:, 2]
print("globaltimer start spread (ns): %d" % (gt.max() - gt.min()))
for cta in (0, 1, grid // 2, grid - 1):
    print(f"-- cta {cta} smid {t[cta,3]} life {life[cta]}")
    for item in range(6):
        b = 8 + item * 10
        ev = t[cta, b:b + 8]
        if not ev.any():
            continue
        rel = [int(x - start[cta]) if x else -1 for x in ev]
        print(f"   item {item}: tma_first {rel[0]} tma_last {rel[1]} | mma tempty_ok {rel[2]} first_full {rel[3]} commit_issued {rel[4]}"
              f" | epi wait_start {rel[5]} tfull_ok {rel[6]} done {rel[7]}")
# aggregate: per item MMA span and epilogue span
for item in range(6):
    b = 8 + item * 10
    m = (t[:, b + 2] > 0) & (t[:, b + 4] > 0)
    if not m.any():
        continue
    mma = (t[m, b + 4] - t[m, b + 3])
    e = (t[:, b + 6] > 0) & (t[:, b + 7] > 0)
    epi = (t[e, b + 7] - t[e, b + 6]) if e.any() else np.array([0])
    lag = (t[e, b + 6] - t[e, b + 4])[t[e, b + 4] > 0] if e.any() else np.array([0])
    print(f"item {item}: n={m.sum()} mma issue span median {int(np.median(mma))} max {mma.max()} | epilogue median {int(np.median(epi))} max {epi.max()}"
          f" | commit->tfull_ok median {int(np.median(lag)) if len(lag) else -1}")

pw, mw, mi = t[:, 100], t[:, 101], t[:, 102]
if not (mi > 0).any():
    raise SystemExit(0)
lead = mi > 0
print("producer: cycles waiting on empty barriers  median %d" % np.median(pw[pw > 0]))
print("mma thread: waiting on full barriers median %d | issuing (wait-return -> commit issued) median %d" % (np.median(mw[lead]), np.median(mi[lead])))
