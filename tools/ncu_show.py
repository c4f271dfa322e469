import csv, sys
cols = {}
names = sys.argv[1:]
for f in names:
    try:
        rows = list(csv.reader(l for l in open(f"gpurun_out/ncu_{f}.csv") if l.startswith('"')))
    except OSError:
        continue
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        cols.setdefault(d["Metric Name"], {})[f] = d["Metric Value"]
        cols.setdefault("kernel", {})[f] = d["Kernel Name"][:28]
print(f'{"metric":62s}' + "".join(f"{n:>30s}" for n in names))
for m, v in cols.items():
    print(f"{m:62s}" + "".join(f'{v.get(n, "-"):>30s}' for n in names))
