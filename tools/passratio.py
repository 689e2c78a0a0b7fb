"""Host-only estimate of passes per level: pass_bytes / pass_bytes_min over a bench window.

    python tools/passratio.py cfg5 [window] [key=value ...]
"""
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import Engine  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402

name = sys.argv[1]
window = int(sys.argv[2]) if len(sys.argv) > 2 else 64
circ, plan, req, pre = configs.build(name, n_req=4)
eng = Engine(device=-1, dtype="c64")
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    eng.set_option(k, int(v))
eng.load_program(lowered(circ, plan.cut))
eng.set_requests([0], [0])
st = eng.run(plan.x_p, pre[3 * window:4 * window], 0, plan.branch_space).stats
print(f"{name} window {window} {sys.argv[3:]}: nodes {st['n_nodes']} launches {st['n_pass_launches']} "
      f"pass/min {st['pass_bytes'] / st['pass_bytes_min']:.3f}")
