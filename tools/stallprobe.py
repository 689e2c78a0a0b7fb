"""Host wall time per queued gs_run vs device time per step (diagnostics for
slow outlier steps).  python tools/stallprobe.py [config] [steps]"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402
from paper_1807_10749_b200.plan import split_requests  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
window = {"cfg3": 256, "cfg4": 32}.get(name, 32)
circ, plan, req, pre = configs.build(name)
eng = ENGINES.get(0, "c64")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.set_stream(stream.cuda_stream)
eng.load_program(lowered(circ, plan.cut))
eng.set_requests(*split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req))
out = torch.zeros(2 * req.size, dtype=torch.float64, device="cuda")
nwin = pre.size // window
for s in range(3):
    eng.run(plan.x_p, pre[s * window:(s + 1) * window], 0, plan.branch_space, out_device_ptr=out.data_ptr(),
            want_host=False)
# synchronous calls: host enqueue time vs device time per step
rows = []
for s in range(steps):
    w = pre[(s % nwin) * window:((s % nwin) + 1) * window]
    t = time.perf_counter()
    st = eng.run(plan.x_p, w, 0, plan.branch_space, out_device_ptr=out.data_ptr(), want_host=False).stats
    rows.append(((time.perf_counter() - t) * 1e3, st["host_ms_enqueue"], st["host_ms_max_gap"], st["ms_total"]))
r = np.array(rows)
print(f"sync: wall median {np.median(r[:,0]):.3f} max {r[:,0].max():.3f} | enqueue median {np.median(r[:,1]):.3f} "
      f"max {r[:,1].max():.3f} | max gap median {np.median(r[:,2]):.3f} max {r[:,2].max():.3f} | device median "
      f"{np.median(r[:,3]):.3f} max {r[:,3].max():.3f}")
for i in np.where((r[:, 0] > 1.5 * np.median(r[:, 0])) | (r[:, 3] > 1.5 * np.median(r[:, 3])))[0][:15]:
    print("  slow step", i, np.round(r[i], 3))
eng.set_option("async_run", 1)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
host = []
torch.cuda.synchronize()
ev[0].record(stream)
for s in range(steps):
    w = pre[(s % nwin) * window:((s % nwin) + 1) * window]
    t = time.perf_counter()
    eng.run(plan.x_p, w, 0, plan.branch_space, out_device_ptr=out.data_ptr(), want_host=False)
    host.append((time.perf_counter() - t) * 1e3)
    ev[s + 1].record(stream)
torch.cuda.synchronize()
dev = np.array([ev[i].elapsed_time(ev[i + 1]) for i in range(steps)])
host = np.array(host)
print(f"{name}: device ms/step median {np.median(dev):.3f} max {dev.max():.3f} | host ms/call median "
      f"{np.median(host):.3f} max {host.max():.3f}")
bad = np.where(dev > 1.5 * np.median(dev))[0]
for i in bad[:20]:
    print(f"  step {i}: device {dev[i]:.3f} ms, host call {host[i]:.3f} ms, prev host {host[i-1] if i else 0:.3f}")
