"""Benchmark: Feynman paths/sec of the hybrid path sum on 1..8 B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (default ``--config cfg4``, BASELINE.json configs[3] -- the config
whose metric is quoted "paths sharded across 1/2/4/8 GPUs"): 6x7 grid,
depth 1+32+1, 21|21 cut, f = 0.01, 10^6 seeded bitstrings.  One *step* is
one batch of paths: every rank takes the next window of ``--window`` sorted
retained prefixes (x all 8 branches each) from its own contiguous slice of
the retained set, evolves them through the path tree on its GPU, gathers the
10^6 requested amplitudes into its complex128 partial, and the ranks
all-reduce the partials over NCCL.  Per-GPU work is fixed as N grows
(``scaling: weak``).

Every number is device-timed with CUDA events on the stream the engine
launches on (the torch current stream, handed to the library), max over
ranks.  ``e2e`` repeats the measurement through the public API
(``run_batched`` / ``run_batched_sharded``) with host buffers: request upload
and result download are inside its timed region.  ``--impl reference`` times
the reference algorithm (the CPU oracle -- a numpy restatement of the
reference's run_batched, because the reference is pure Python and cannot be
installed on the GPU box) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Feynman paths/sec (whole box)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--window", type=int, default=0, help="prefixes per GPU per step (0 = auto)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dtype", default="c64", choices=["c64", "c128"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=0)
    ap.add_argument("--opt", action="append", default=[], help="engine option key=value")
    ap.add_argument("--describe-out", default="", help="write gs_describe() + schedule hash here")
    ap.add_argument("--whole-job", action="store_true",
                    help="time the config's whole retained set in one public-API call (e2e, host buffers)")
    ap.add_argument("--no-single-core", action="store_true", help="skip the single-core CPU leg")
    return ap.parse_args()


def schedule_hash(desc: dict, window: int, n_req: int) -> str:
    """Key of the exact schedule being timed (the pass plan, leaf handling, window
    and request count); profiles/traffic.json holds ncu DRAM bytes per key."""
    import hashlib

    d = {k: v for k, v in desc.items() if k != "jit"}  # the jit field carries compile timings
    blob = json.dumps(d, sort_keys=True) + f"|{window}|{n_req}"
    return hashlib.sha256(blob.encode()).hexdigest()[:16]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


# prefixes per GPU per step (one run_batched call).  cfg4: 1,024 prefixes x 8 branches; the
# device rate is flat in the window (115.1k / 116.4k / 116.9k / 117.2k paths/s at 256 / 512 /
# 1,024 / 2,048, profiles/r02p_*), the public-API call's fixed cost (8 MB of requests up,
# 16 MB of amplitudes down) is amortised over 4x more paths than at 256 (e2e 104.7k -> 114.2k)
DEFAULT_WINDOW = {"cfg1": 16, "cfg1v2": 32, "cfg2": 32768, "cfg2v2": 32768, "cfg2h": 2048,
                  "cfg3": 256, "cfg3v2": 128, "cfg4": 1024, "cfg4v2": 512, "cfg5": 1, "cfg5v2": 1, "cfg5f": 1}


def describe(name, plan, window, n_req):
    from paper_1807_10749_b200.configs import CONFIGS

    s = CONFIGS[name]
    return (f"{name}: {s.rows}x{s.cols} grid, depth 1+{s.depth}+1 ({s.version}+final H), "
            f"{plan.cut.n_a}|{plan.cut.n_b} cut, f={s.fidelity:g}, {n_req} bitstrings; "
            f"step = {window} retained prefixes x {plan.branch_space} branches per GPU")


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    """nvidia-smi sampler started before the timed region; summary() keeps the
    samples whose timestamps fall inside [t0, t1] (the nearest one if none)."""

    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int, period_ms: int = 20):
        self.gpu = gpu_index
        self.period = period_ms
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            deadline = time.time() + 10
            while not self.rows and time.time() < deadline:  # wait for the first sample
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        import datetime

        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = time.time()
            self.rows.append((ts, f[1:]))

    def mark(self, begin: bool):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()
            time.sleep(2 * self.period / 1000.0)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        inside = [r for t, r in self.rows if self.t0 is not None and self.t0 <= t <= (self.t1 or t)]
        how = "during timed region"
        if not inside:
            mid = 0.5 * (self.t0 + self.t1) if self.t0 and self.t1 else time.time()
            inside = [min(self.rows, key=lambda tr: abs(tr[0] - mid))[1]]
            how = "nearest sample to the timed region"

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in inside if num(r[1]) is not None]
        mx = [num(r[2]) for r in inside if num(r[2]) is not None]
        reasons = sorted({self.NAMES[i] for r in inside for i in range(4)
                          if len(r) > 5 + i and r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "sampling": how}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of the reference's run_batched), forked over cores

def _cpu_job(args):
    name, prefixes, n_req = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import pathsum_oracle as oracle
    from paper_1807_10749_b200 import configs

    circ, plan, req, _ = configs.build(name, n_req=n_req)
    t = time.perf_counter()
    amps = oracle.run_batched(circ, plan, req, np.asarray(prefixes, dtype=np.int64))
    return time.perf_counter() - t, amps


def cpu_reference(name, prefixes, n_req, procs, pool=None):
    """Time the reference algorithm on `procs` processes, one prefix slice each."""
    import multiprocessing as mp

    slices = [s for s in np.array_split(np.asarray(prefixes), procs) if s.size]
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(len(slices))
    t = time.perf_counter()
    res = pool.map(_cpu_job, [(name, s, n_req) for s in slices])
    wall = time.perf_counter() - t
    if own:
        pool.close()
    total = sum(r[1] for r in res)
    return wall, total, len(slices)


# ---------------------------------------------------------------------------


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def main_whole_job(args):
    """The config's whole retained set in ONE public-API call (host requests in,
    host amplitudes out), timed by the host clock around the call; the device-side
    time of the same job is the engine's event time (stats ms_total)."""
    import torch

    from paper_1807_10749_b200 import configs
    from paper_1807_10749_b200.engine import ENGINES
    from paper_1807_10749_b200.pathsum import run_batched

    torch.cuda.set_device(0)
    name = args.config
    circ, plan, req, pre_all = configs.build(name)
    eng = ENGINES.get(0, args.dtype)
    for kv in args.opt:
        key, val = kv.split("=")
        eng.set_option(key, int(val))
    run_batched(circ, plan, req, prefixes=pre_all[:64])  # untimed: program load, JIT, buffers
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run_batched(circ, plan, req, prefixes=pre_all)
    wall = time.perf_counter() - t0
    paths = int(pre_all.size) * plan.branch_space
    line = {
        "metric": METRIC, "value": paths / wall, "unit": "paths/s", "n_gpus": 1, "steps": 1, "warmup": 1,
        "ms_per_step": 1e3 * wall, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c64 (fp32 complex states, fp64 accumulation)" if args.dtype == "c64" else "c128",
        "data": "synthetic: reference-generator circuit (seed 0), challenge_indices(seed 12345)",
        "config": {"workload": f"{name} whole job: all {pre_all.size} retained prefixes x {plan.branch_space} "
                               f"branches = {paths} paths, {req.size} bitstrings, one run_batched call",
                   "timer": "host wall clock around the public call (request upload, path tree, result "
                            "download into host memory)"},
        "e2e": {"value": paths / wall, "unit": "paths/s", "h2d_bytes_per_step": int(8 * req.size),
                "d2h_bytes_per_step": int(16 * req.size)},
        "amplitude_norm2": float(np.vdot(res.amps, res.amps).real),
        "whole_job_seconds": wall,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return main_reference(args)
    if args.whole_job:
        return main_whole_job(args)

    import torch
    import torch.distributed as dist

    from paper_1807_10749_b200 import configs
    from paper_1807_10749_b200.distributed import partition_prefixes, run_batched_sharded
    from paper_1807_10749_b200.engine import ENGINES
    from paper_1807_10749_b200.lowering import lowered
    from paper_1807_10749_b200.pathsum import run_batched
    from paper_1807_10749_b200.plan import split_requests

    world, rank, local = dist_setup(args)
    name = args.config
    circ, plan, req, pre_all = configs.build(name)
    window = args.window or DEFAULT_WINDOW.get(name, 8)
    n_steps_total = args.warmup + args.steps

    def rank_windows(r):
        """Step s of rank r: the s-th window of r's contiguous slice (wrapping if short)."""
        sl = partition_prefixes(pre_all, world, r)
        if sl.size < window:
            raise SystemExit(f"rank {r}: only {sl.size} prefixes for a window of {window}")
        n_win = sl.size // window
        return [sl[(s % n_win) * window:((s % n_win) + 1) * window] for s in range(n_steps_total)]

    windows = rank_windows(rank)
    all_windows = [rank_windows(r) for r in range(world)] if world > 1 else [windows]

    eng = ENGINES.get(local, args.dtype)
    for kv in args.opt:
        key, val = kv.split("=")
        eng.set_option(key, int(val))
    # a real (non-legacy) stream shared by torch and the engine: the CUDA events
    # below then bracket exactly the engine's launches
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    prog = lowered(circ, plan.cut)
    eng.load_program(prog)
    ia, ib = split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req)
    eng.set_requests(ia, ib)
    n_req = req.size
    out = torch.zeros(2 * n_req, dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step(s, stats_acc=None):
        flush.zero_()  # L2 flush between steps (the working set is >> L2 anyway)
        r = eng.run(plan.x_p, windows[s], 0, plan.branch_space, out_device_ptr=out.data_ptr(),
                    want_host=False)
        if world > 1:
            dist.all_reduce(out)
        if stats_acc is not None:
            stats_acc.append(r.stats)
        return r.stats

    for s in range(args.warmup):
        step(s)
    # one profiled step (events around every level) for the kernel split / roofline
    eng.set_option("profile", 1)
    prof = step(args.warmup % n_steps_total)
    eng.set_option("profile", 0)
    # steps are queued back to back: the host enumerates step s+1's path tree
    # while the device runs step s (stream order; results land in `out`)
    eng.set_option("async_run", 1)

    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stats = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local, int(os.environ.get("GS_BENCH_CLOCK_MS", "20")))
    if os.environ.get("GS_BENCH_NO_CLOCKS") != "1":  # diagnostics only: the JSON then says "unsampled"
        clk.start()
    torch.cuda.synchronize()
    clk.mark(True)
    e0.record(stream)
    for s in range(args.steps):
        step(args.warmup + s, stats)
    e1.record(stream)
    torch.cuda.synchronize()
    eng.set_option("async_run", 0)
    clk.mark(False)
    clk.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    paths_rank = sum(st["n_paths"] for st in stats)
    paths = paths_rank * world  # every rank processes the same window size
    value = paths / (ms / 1e3)

    # e2e through the public API with host buffers (request upload + result download inside)
    e2e = None
    if not args.no_e2e:
        def e2e_step(s):
            w = windows[s]
            if world > 1:
                union = np.concatenate([all_windows[r][s] for r in range(world)])
                run_batched_sharded(circ, plan, req, prefixes=union, dst=None, device=local, dtype=args.dtype)
            else:
                run_batched(circ, plan, req, prefixes=w, device=local, dtype=args.dtype)
            return w.size * plan.branch_space * world

        for s in range(min(args.warmup, 2)):  # untimed warm-up of the public-API path
            e2e_step(s)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_paths = 0
        for s in range(args.steps):
            e2e_paths += e2e_step(args.warmup + s)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": e2e_paths / el, "unit": "paths/s",
               "h2d_bytes_per_step": int(8 * n_req + 8 * window + stats[-1]["h2d_bytes"]),
               "d2h_bytes_per_step": int(16 * n_req), "timer": "host wall clock, max over ranks"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # roofline of the dominant kernel class, from the profiled step (CUDA events on the
    # engine's stream around every level): the gate passes above the leaf level (HBM
    # streaming) and the leaf level (the fused projected-leaf pass where it applies)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    desc = eng.describe()
    shash = schedule_hash(desc, window, n_req)
    if args.describe_out:
        with open(args.describe_out, "w") as fh:
            json.dump(dict(desc, schedule_hash=shash, config=name, window=window, n_req=n_req), fh)
    traffic_rec = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic_rec = json.load(fh).get(shash)
    except (OSError, ValueError):
        pass
    if traffic_rec is None:
        print(f"bench: no ncu DRAM capture for schedule {shash} in profiles/traffic.json; "
              f"roofline.traffic is null (tools/round_prof.sh records it)", file=sys.stderr)
    fused = bool(desc.get("proj_fused"))
    classes = {}
    ms_leaf = prof["ms_leaf"]
    n_leaf = max(0, prof["n_leaf_launches"])
    for cls, ms_c, by_c, n_c, kern in (
            ("upper_passes", prof["ms_pass"] - ms_leaf, prof["upper_bytes_alg"],
             prof["n_pass_launches"] - n_leaf, "gsj_* gate passes above the leaf level"),
            ("leaf", ms_leaf, prof["leaf_bytes_alg"], n_leaf,
             "gsj_* fused projected-leaf pass (leaf gates + projected gather)" if fused
             else "gsj_* leaf-level passes")):
        if n_c <= 0 or ms_c <= 0:
            continue
        per_launch_ms = ms_c / n_c
        ach = by_c / (ms_c / 1e3) / 1e9
        tr = (traffic_rec or {}).get(cls)
        classes[cls] = {
            "bound": "hbm", "kernel": kern, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "traffic": tr["dram_bytes_per_launch"] if tr else None,
            "traffic_vs_algorithmic": (tr["dram_bytes_per_launch"] / (by_c / n_c)) if tr and by_c else None,
            "algorithmic_bytes_per_launch": by_c / n_c, "avg_launch_ms": per_launch_ms, "launches": n_c,
            "share_of_step": ms_c / prof["ms_total"] if prof["ms_total"] else None,
        }
    if prof["ms_gather"] > 0:
        classes["gather"] = {"kernel": "reduce_kernel (fold of the fused pass's partials)" if fused
                             else "leaf gather + reduce", "ms": prof["ms_gather"],
                             "algorithmic_bytes": prof["gather_bytes"],
                             "achieved": prof["gather_bytes"] / (prof["ms_gather"] / 1e3) / 1e9,
                             "share_of_step": prof["ms_gather"] / prof["ms_total"] if prof["ms_total"] else None}
    dom = max((c for c in ("upper_passes", "leaf") if c in classes),
              key=lambda c: classes[c]["avg_launch_ms"] * classes[c]["launches"], default=None)
    roofline = dict(classes[dom]) if dom else {"bound": "hbm", "achieved": None, "peak": peak, "unit": "GB/s",
                                               "frac": None, "traffic": None}
    roofline.update({
        "class": dom, "peak_source": peak_src, "schedule_hash": shash,
        "traffic_source": (traffic_rec or {}).get("source"),
        "basis": "algorithmic bytes the schedule must move per launch: every parent state read once per "
                 "level chunk, every written state written once (later passes of a level read+write their "
                 "node); the fused leaf pass reads each parent once per side and writes one fp64 partial "
                 "per (request, 8-leaf group) -- no leaf state reaches HBM",
        "classes": classes,
    })
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "paths/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c64 (fp32 complex states, fp64 accumulation)" if args.dtype == "c64" else "c128",
        "data": "synthetic: reference-generator circuit (seed 0), challenge_indices(seed 12345)",
        "config": {
            "workload": describe(name, plan, window, n_req),
            "paths_per_gpu_per_step": int(paths_rank / max(1, args.steps)),
            "l2": "256 MB L2 flush before every step; working set (16 MB half-states x nodes) >> L2",
            "parallelism": f"path-sharded dp{world}, NCCL all-reduce of the complex128 partials",
        },
        "e2e": e2e,
        "roofline": roofline,
        "schedule_hash": shash,
        "gpu_launches": int(sum(st["n_launches"] for st in stats)),
        "clocks": clk.summary(),
        "nodes_per_step": int(np.mean([st["n_nodes"] for st in stats])),
        # per-path cost (BASELINE cfg5: "a fixed budget of 2^16 paths with per-path cost reported")
        "per_path": {"gpu_ms_per_path": 1e3 * world / value if value else None,
                     "budget_2p16_paths_s": 65536.0 / value if value else None},
    }
    if not args.no_cpu and world == 1:
        procs = args.cpu_procs or min(os.cpu_count() or 1, 32)
        sample = windows[args.warmup][: max(1, min(window, procs))]
        wall, _, used = cpu_reference(name, sample, n_req, min(procs, sample.size))
        cpu_paths = sample.size * plan.branch_space
        line["cpu_baseline"] = {
            "value": cpu_paths / wall, "unit": "paths/s", "cores": used, "kind": "port",
            "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
            "sample": f"{sample.size} prefixes x {plan.branch_space} branches of the same window, "
                      f"{used} forked processes, numpy restatement of reference run_batched",
        }
        if not args.no_single_core:  # one process, one thread: the reference's own per-core rate
            w1, _, _ = cpu_reference(name, sample[:1], n_req, 1)
            line["cpu_baseline"]["single_core"] = {
                "value": plan.branch_space / w1, "unit": "paths/s", "cores": 1,
                "sample": f"1 prefix x {plan.branch_space} branches, 1 process (OMP_NUM_THREADS=1)"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _ref_job(args):
    """One CPU process of the reference arm: the reference package's own
    run_batched (gridsim, from baseline/_ref) over a slice of prefixes."""
    name, prefixes, n_req = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from paper_1807_10749_b200 import configs
    from paper_1807_10749_b200.gridsim_engine import load_gridsim

    gc, gps = load_gridsim("circuit"), load_gridsim("pathsum")
    circ, plan, req, _ = configs.build(name, n_req=n_req)
    spec = configs.CONFIGS[name]
    with open(spec.circuit_file) as fh:
        rc = gc.parse_circuit(fh.read(), spec.rows, spec.cols)
    cut = gc.Cut(plan.cut.orientation, plan.cut.position, tuple(plan.cut.block_a), tuple(plan.cut.block_b))
    rplan = gps.SimPlan(cut, plan.fidelity, tuple(plan.radices), plan.x_p, plan.x_b, plan.d_p, plan.d_b,
                        plan.seed, plan.retained)
    t = time.perf_counter()
    amps = gps.run_batched(rc, rplan, req, prefixes=np.asarray(prefixes, dtype=np.int64)).amps
    return time.perf_counter() - t, amps


def main_reference(args):
    """Reference arm: the reference's CPU implementation of the path on all host cores.

    Where the reference package is installed (baseline/_ref, `gridsim`), each
    process runs its own ``gridsim.pathsum.run_batched`` (kind "reference");
    otherwise the numpy restatement in oracle/ (kind "port", bit-exact with it).
    A timed step is the workload's natural unit on every core: each process
    evaluates one retained prefix with all of its branches (the reference's
    per-prefix job, orchestrator.py:133-159, on its batched engine).  Warm-up
    steps only import and run small jobs (untimed).  Rank 0 alone runs under
    torchrun.
    """
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    from paper_1807_10749_b200 import configs
    from paper_1807_10749_b200.gridsim_engine import gridsim_available

    name = args.config
    circ, plan, req, pre_all = configs.build(name)
    kind = "reference" if gridsim_available() else "port"
    job = _ref_job if kind == "reference" else _cpu_job
    procs = args.cpu_procs or min(os.cpu_count() or 1, 64)
    pool = mp.get_context("fork").Pool(procs)
    for s in range(args.warmup):
        pool.map(job, [(name, pre_all[s:s + 1], 64)] * procs)
    times, paths = [], 0
    for s in range(args.steps):
        sample = pre_all[(s * procs) % max(1, pre_all.size - procs):][:procs]
        slices = [x for x in np.array_split(sample, procs) if x.size]
        t = time.perf_counter()
        pool.map(job, [(name, x, req.size) for x in slices])
        times.append(time.perf_counter() - t)
        paths += sample.size * plan.branch_space
    pool.close()
    total = sum(times)
    value = paths / total
    what = ("gridsim.pathsum.run_batched (the reference package, baseline/_ref)" if kind == "reference"
            else "numpy restatement of reference run_batched (oracle/)")
    line = {
        "metric": METRIC, "value": value, "unit": "paths/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "impl": "reference",
        "dtype": "c64 (numpy complex64 states, complex128 accumulation)",
        "data": "synthetic: reference-generator circuit (seed 0), challenge_indices(seed 12345)",
        "config": {"workload": describe(name, plan, procs, req.size) + " (CPU: one prefix per process)",
                   "parallelism": f"{procs} forked CPU processes"},
        "cpu_baseline": {"value": value, "unit": "paths/s", "cores": procs, "kind": kind,
                         "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
                         "sample": f"{procs} prefixes x {plan.branch_space} branches per step, {what}"},
        "e2e": {"value": value, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
