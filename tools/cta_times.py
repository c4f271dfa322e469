"""Reads a TLB_GEMM_CTA_TIMES dump: start / end spread of the CTAs of consecutive launches and the gaps between launches."""
import sys
import numpy as np
raw = np.fromfile(sys.argv[1], dtype=np.int64)
ring, slots, nxt = int(raw[0]), int(raw[1]), int(raw[2])
full = raw[4:].reshape(ring, slots)
t = full[:, :320].reshape(ring, 160, 2)
order = [(nxt - ring + i) % ring for i in range(ring)] if nxt >= ring else list(range(nxt))
prev_end = None
rows = []
for i in order[-12:]:
    x = t[i]
    live = x[:, 1] > 0
    st, en = x[live, 0], x[live, 1]
    s0 = st.min()
    rows.append((live.sum(), (st.max() - s0) / 1e3, (en.min() - s0) / 1e3, np.median(en - s0) / 1e3, (en.max() - s0) / 1e3,
                 (s0 - prev_end) / 1e3 if prev_end else float("nan")))
    prev_end = en.max()
print("ctas  start-spread  first-exit  median-exit  last-exit  gap-from-previous-launch (us)")
for r in rows:
    print("%4d  %10.2f  %10.2f  %10.2f  %9.2f  %8.2f" % r)

last = order[-1]
e = full[last, 320:320 + 60].reshape(12, 5)
if e.any():
    print("epilogue steps of CTA 0 / warp 0, cycles since the first chunk started: ld-issued  wait_read-done  tmem-data-ready  staged+fenced  tma-issued")
    b = e[0, 0]
    for c in range(12):
        if e[c, 0]:
            print("  chunk %2d: " % c + "  ".join("%7d" % (x - b) for x in e[c]))
