"""Print an ncu --csv launch list (gpu__time_duration.sum) as one line per kernel launch; with
--last N only the last N launches (one repetition of the case)."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
ig, ib = h.index("Grid Size"), h.index("Block Size")
d = {}
for r in rows[1:]:
    e = d.setdefault(int(r[iid]), {"k": r[ik], "g": r[ig], "b": r[ib]})
    e[r[im]] = r[iv]
items = [d[k] for k in sorted(d)]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else len(items)
tot = 0.0
for it in items[-last:]:
    ns = float(it.get("gpu__time_duration.sum", "0").replace(",", ""))
    tot += ns
    print(f"  {it['k'][:60]:60s} {ns / 1e3:9.1f} us  grid {it['g']} block {it['b']}")
print(f"  total {tot / 1e3:.1f} us")
