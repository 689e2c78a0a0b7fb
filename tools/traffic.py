"""Per-launch DRAM traffic of the gate-pass kernels from an ncu launch list.

    python tools/traffic.py <config> <launches.csv> [profiles/traffic.json]

The launch list is the bench command's own (tools/prof.sh: --metrics
dram__bytes_read.sum,dram__bytes_write.sum, warm cache, serialised); the
result is merged into profiles/traffic.json, which bench.py reads into
roofline.traffic for the same config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import launches  # noqa: E402


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "traffic.json")
    recs = [m for m in launches(path) if m["name"].startswith("gsj_") or "pass2_kernel" in m["name"]]
    tot = sum(float(m.get("dram__bytes_read.sum", 0)) + float(m.get("dram__bytes_write.sum", 0)) for m in recs)
    t = sum(float(m.get("gpu__time_duration.sum", 0)) for m in recs)
    data = {}
    if os.path.exists(out):
        data = json.load(open(out))
    data[cfg] = {"pass_dram_bytes_per_launch": tot / max(1, len(recs)), "pass_launches": len(recs),
                 "pass_dram_gbs_serialised": tot / t if t else None,
                 "source": os.path.basename(path) + " (ncu --cache-control none --clock-control none, "
                           "bench.py --config " + cfg + " --steps 2 --warmup 3)"}
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(data[cfg]))


if __name__ == "__main__":
    main()
