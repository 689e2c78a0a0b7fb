"""Per-launch DRAM traffic of the gate-pass kernel classes from an ncu launch list,
keyed by the schedule hash bench.py prints (roofline.schedule_hash).

    python tools/traffic.py <describe.json> <launches.csv> [profiles/traffic.json]

describe.json is ``bench.py --describe-out`` of the timed command (gs_describe +
schedule hash); launches.csv is the ncu launch list of the same command
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--clock-control none).  Launches of the specialised passes (gsj_<k>_p<pass>)
are split into the leaf level and the levels above it; the per-launch DRAM
bytes of each class are merged into profiles/traffic.json under the schedule
hash, which bench.py reads back as roofline.traffic for the identical schedule
(and reports null, loudly, for any other)."""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import launches  # noqa: E402


def main():
    desc = json.load(open(sys.argv[1]))
    path = sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "traffic.json")
    D = len(desc["levels"]) - 1
    level_of = {}
    for li, L in enumerate(desc["levels"]):
        for b in L["blocks"]:
            for p in b["passes"]:
                if p.get("jit", -1) >= 0:
                    level_of[p["jit"]] = li
    cls = {"upper_passes": [], "leaf": []}
    for m in launches(path):
        g = re.match(r"gsj_\d+_p(\d+)", m["name"])
        if not g:
            continue
        li = level_of.get(int(g.group(1)))
        if li is None:
            continue
        by = float(m.get("dram__bytes_read.sum", 0)) + float(m.get("dram__bytes_write.sum", 0))
        t = float(m.get("gpu__time_duration.sum", 0))
        cls["leaf" if li == D else "upper_passes"].append((by, t))
    rec = {"config": desc.get("config"), "window": desc.get("window"), "n_req": desc.get("n_req"),
           "source": os.path.basename(path) + " (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                     "dram__bytes_write.sum --clock-control none; cold-cache, serialised launches)"}
    for k, v in cls.items():
        if v:
            tot_b = sum(b for b, _ in v)
            tot_t = sum(t for _, t in v)
            rec[k] = {"dram_bytes_per_launch": tot_b / len(v), "launches": len(v),
                      "dram_gbs_serialised": tot_b / tot_t if tot_t else None}
    data = {}
    if os.path.exists(out):
        data = json.load(open(out))
    data = {k: v for k, v in data.items() if isinstance(v, dict) and "source" in v and "config" in v}
    data[desc["schedule_hash"]] = rec
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps({desc["schedule_hash"]: rec}))


if __name__ == "__main__":
    main()
