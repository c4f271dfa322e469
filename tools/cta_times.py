"""Reads a TLB_GEMM_CTA_TIMES dump: start / end spread of the CTAs of consecutive launches and the gaps between launches."""
import sys
import numpy as np
raw = np.fromfile(sys.argv[1], dtype=np.int64)
ring, slots, nxt = int(raw[0]), int(raw[1]), int(raw[2])
t = raw[4:].reshape(ring, slots // 2, 2)
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
