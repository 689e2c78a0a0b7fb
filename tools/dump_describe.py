"""Write gs_describe() of a config's program (device engine, JIT compiled) to a JSON file.

    python tools/dump_describe.py cfg5 out.json [key=value ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import Engine  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
circ, plan, req, pre = configs.build(name, n_req=4)
eng = Engine(device=0 if len(sys.argv) < 4 or "host" not in sys.argv[3:] else -1, dtype="c64")
for kv in sys.argv[3:]:
    if "=" in kv:
        k, v = kv.split("=")
        eng.set_option(k, int(v))
eng.load_program(lowered(circ, plan.cut))
with open(out, "w") as fh:
    json.dump(eng.describe(), fh)
