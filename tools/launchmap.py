"""Join an ncu launch list (csv) with gs_describe() JSON: per pass kernel time, DRAM GB/s, registers.

    python tools/launchmap.py describe.json launches.csv
"""
import collections
import csv
import json
import re
import sys

desc = json.load(open(sys.argv[1]))
passes = {}
for li, L in enumerate(desc["levels"]):
    for side, b in enumerate(L["blocks"]):
        for pi, p in enumerate(b["passes"]):
            if p.get("jit", -1) >= 0:
                passes[p["jit"]] = (li, side, pi, p)
q = max(desc["q"])
rows = list(csv.reader(open(sys.argv[2])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
idx = {h: j for j, h in enumerate(rows[start])}
K = collections.OrderedDict()
for r in rows[start + 1:]:
    k = K.setdefault(r[idx["ID"]], {"name": r[idx["Kernel Name"]]})
    k[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0])
other = collections.defaultdict(lambda: [0, 0.0, 0.0])
for k in K.values():
    m = re.match(r"gsj_\d+_p(\d+)", k["name"])
    t = k.get("gpu__time_duration.sum", 0.0)  # ns
    by = k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
    if m:
        a = agg[int(m.group(1))]
        a[0] += 1; a[1] += t; a[2] += by; a[3] = k.get("launch__registers_per_thread", 0)
    else:
        o = other[k["name"].split("(")[0][:50]]
        o[0] += 1; o[1] += t; o[2] += by
tot = sum(a[1] for a in agg.values()) + sum(o[1] for o in other.values())
print(f"{'pass':>5} {'lvl':>3} {'s':>1} {'ops':>3} {'stages':<16} {'regs':>4} {'n':>3} {'ms':>8} {'share':>6} {'GB/s':>6}  tile")
for j in sorted(agg, key=lambda j: -agg[j][1]):
    n, t, by, regs = agg[j]
    li, side, pi, p = passes.get(j, (-1, -1, -1, {"ops": 0, "stages": [], "lbits": []}))
    tile = "".join("x" if i in p["lbits"] else "." for i in range(q))
    print(f"{j:5d} {li:3d} {side:1d} {p['ops']:3d} {str(p['stages']):<16} {int(regs):4d} {n:3d} {t / 1e6:8.2f} "
          f"{t / tot:6.3f} {by / t:6.0f}  {tile}")
for name, (n, t, by) in sorted(other.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:<50} n={n:4d} {t / 1e6:8.2f} ms share {t / tot:.3f} {by / max(t, 1e-9):6.0f} GB/s")
