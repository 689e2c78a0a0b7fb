"""Summarise an ncu launch list (csv) and an ncu --set full report into markdown.

    python tools/ncu_summary.py launches.csv [report.ncu-rep] > summary.md
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, recs = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            recs.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = d["Metric Value"]
    return list(recs.values())


def main():
    recs = launches(sys.argv[1])
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for m in recs:
        k = m["name"].split("(")[0].replace("void ", "")
        t = float(m.get("gpu__time_duration.sum", 0))
        b = float(m.get("dram__bytes_read.sum", 0)) + float(m.get("dram__bytes_write.sum", 0))
        tot[k][0] += 1
        tot[k][1] += t
        tot[k][2] += b
    all_t = sum(v[1] for v in tot.values())
    print(f"## Launch list `{sys.argv[1].split('/')[-1]}` ({len(recs)} launches, ncu cold-cache, serialised)\n")
    print("| kernel | launches | total us | share | DRAM GB | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t / 1e3:.1f} | {t / all_t:.1%} | {b / 1e9:.3f} | {b / max(t, 1):.0f} |")
    if len(sys.argv) > 2:
        raw = subprocess.run(["ncu", "-i", sys.argv[2], "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        hdr, units = rows[0], rows[1]
        keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
                "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__warps_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
        keys = [k for k in keys if k in hdr]
        print(f"\n## Full capture `{sys.argv[2].split('/')[-1]}`\n")
        print("| " + " | ".join(k.replace("__", " ").replace(".avg.pct_of_peak_sustained", " %")
                                for k in keys) + " |")
        print("|" + "---|" * len(keys))
        print("| " + " | ".join(units[hdr.index(k)] for k in keys) + " |")
        for r in rows[2:]:
            vals = [r[hdr.index(k)] for k in keys]
            vals[0] = vals[0].split("(")[0].replace("void ", "")
            print("| " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
