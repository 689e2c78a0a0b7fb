"""Generate the golden fixtures from the reference implementation itself.

Run in the build container only (it imports the read-only reference from
/root/reference, which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--heavy]

Writes
  paper_1807_10749_b200/data/circuits/*.txt  config circuits (reference generator + serializer)
  paper_1807_10749_b200/data/cfg5*_retained_head.npy  leading retained prefixes of cfg5
  tests/golden/plans.json     per config: cut, radices, split, retained (or its sha256)
  tests/golden/amps/*.npz     reference amplitudes: run_approx / run_batched windows in
                              complex64 and complex128 (DTYPE rebound),
                              run_path per-path contributions, run_full / naive_state
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF)
sys.path.insert(0, REF_TESTS)

import gridsim.pathsum as ps  # noqa: E402
import gridsim.statevec as sv  # noqa: E402
from gridsim.benchgen import GenSpec, generate  # noqa: E402
from gridsim.circuit import Cut, Gate, GateKind, circuit_hash, parse_circuit, serialize_circuit  # noqa: E402
from gridsim.validate import challenge_indices  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DATA = os.path.join(ROOT, "paper_1807_10749_b200", "data")
AMPS = os.path.join(HERE, "amps")

CFG = {  # name: (rows, cols, depth, version, fidelity, n_req, cut)
    "cfg1": (4, 4, 16, "v1", 1.0, 1024, None),
    "cfg1v2": (4, 4, 16, "v2", 1.0, 1024, None),
    "cfg2": (5, 5, 24, "v1", 1.0, 10**4, "staircase"),
    "cfg2v2": (5, 5, 24, "v2", 1.0, 10**4, "staircase"),
    "cfg2h": (5, 5, 24, "v1", 1.0, 10**4, None),
    "cfg3": (6, 6, 28, "v1", 0.1, 10**5, None),
    "cfg3v2": (6, 6, 28, "v2", 0.1, 10**5, None),
    "cfg4": (6, 7, 32, "v1", 0.01, 10**6, None),
    "cfg4v2": (6, 7, 32, "v2", 0.01, 10**6, None),
    "cfg5": (7, 8, 40, "v1", 0.005, 10**6, None),
    "cfg5v2": (7, 8, 40, "v2", 0.005, 10**6, None),
}
FSIM_SEED = 2024


def staircase():
    a = tuple(sorted(q for q in range(25) if q % 5 <= 1 or (q % 5 == 2 and q // 5 <= 1)))
    b = tuple(q for q in range(25) if q not in a)
    return Cut("s", 2, a, b)


def fsim(theta, phi):
    c, s = math.cos(theta), math.sin(theta)
    return np.array(
        [[1, 0, 0, 0], [0, c, -1j * s, 0], [0, -1j * s, c, 0], [0, 0, 0, np.exp(-1j * phi)]],
        dtype=np.complex128,
    )


def fsim_variant(circ, seed=FSIM_SEED):
    """Every CZ -> g2 fSim(theta, phi), theta/phi ~ U[0, 2pi) from default_rng(seed), gate order."""
    rng = np.random.default_rng(seed)
    gates = []
    for g in circ.gates:
        if g.kind is GateKind.CZ:
            th, ph = rng.uniform(0, 2 * np.pi, size=2)
            gates.append(Gate(g.cycle, GateKind.GENERIC_2Q, g.qubits, fsim(th, ph)))
        else:
            gates.append(Gate(g.cycle, g.kind, g.qubits))
    return type(circ)(circ.rows, circ.cols, gates)


def circ_file(r, c, d, ver, fs=False):
    return os.path.join(DATA, "circuits", f"{r}x{c}_d{d}_{ver}{'_fsim' if fs else ''}.txt")


def gen(r, c, d, ver):
    return generate(GenSpec(r, c, d, ver, include_final_h=True, seed=0))


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.int64).tobytes()).hexdigest()


class c128:
    """Rebind the reference DTYPE to complex128; use on fresh circuits."""

    def __enter__(self):
        self.saved = (ps.DTYPE, sv.DTYPE)
        ps.DTYPE = np.complex128
        sv.DTYPE = np.complex128

    def __exit__(self, *a):
        ps.DTYPE, sv.DTYPE = self.saved


def fresh(circ):
    return parse_circuit(serialize_circuit(circ), circ.rows, circ.cols)


def write_circuits():
    os.makedirs(os.path.join(DATA, "circuits"), exist_ok=True)
    hashes = {}
    for name, (r, c, d, ver, *_rest) in CFG.items():
        circ = gen(r, c, d, ver)
        with open(circ_file(r, c, d, ver), "w") as fh:
            fh.write(serialize_circuit(circ))
        hashes[name] = circuit_hash(circ)
    f5 = fsim_variant(gen(7, 8, 40, "v1"))
    with open(circ_file(7, 8, 40, "v1", True), "w") as fh:
        fh.write(serialize_circuit(f5))
    hashes["cfg5f"] = circuit_hash(f5)
    return hashes


def plans(hashes):
    out = {}
    for name, (r, c, d, ver, f, n_req, cutname) in CFG.items():
        circ = gen(r, c, d, ver)
        cut = staircase() if cutname == "staircase" else None
        t = time.time()
        plan = ps.make_plan(circ, fidelity=f, seed=0, cut=cut, workers=1)
        ret = plan.retained
        rec = {
            "circuit_hash": hashes[name],
            "cut": [plan.cut.orientation, plan.cut.position, list(plan.cut.block_a), list(plan.cut.block_b)],
            "radices": list(plan.radices),
            "x_p": plan.x_p, "x_b": plan.x_b, "d_p": plan.d_p, "d_b": plan.d_b,
            "n_retained": int(ret.size), "retained_sha256": sha(ret),
            "retained_head": [int(v) for v in ret[:64]],
            "retained_tail": [int(v) for v in ret[-64:]],
            "plan_seconds": round(time.time() - t, 2),
        }
        if ret.size <= 20000:
            rec["retained"] = [int(v) for v in ret]
        if name.startswith("cfg5"):
            budget = 1 << 16
            head = ret[: math.ceil(budget / plan.branch_space)]
            np.save(os.path.join(DATA, f"{name}_retained_head.npy"), head)
        # workers>1 changes the default split; record one case for the planner tests
        if name in ("cfg1", "cfg3"):
            p8 = ps.make_plan(circ, fidelity=f, seed=0, cut=cut, workers=8)
            rec["workers8"] = {"x_p": p8.x_p, "x_b": p8.x_b}
        req = challenge_indices(circ.n_qubits, n_req, 12345)
        rec["requests_sha256"] = sha(req)
        rec["requests_head"] = [int(v) for v in req[:16]]
        ia, ib = ps.split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req[:256])
        rec["split_head"] = [[int(a) for a in ia], [int(b) for b in ib]]
        out[name] = rec
        print(name, "x", plan.x, "x_p", plan.x_p, "ret", ret.size, rec["plan_seconds"], "s", flush=True)
    # fSim cfg5 variant: reference-native 256 x 256 window
    f5 = fsim_variant(gen(7, 8, 40, "v1"))
    p = ps.make_plan(f5, fidelity=256 / 4**31, x_p=31, x_b=4, seed=0)
    out["cfg5f"] = {
        "circuit_hash": hashes["cfg5f"], "radices": list(p.radices), "x_p": p.x_p, "x_b": p.x_b,
        "d_p": p.d_p, "d_b": p.d_b, "n_retained": int(p.retained.size),
        "retained": [int(v) for v in p.retained], "retained_sha256": sha(p.retained),
        "cut": [p.cut.orientation, p.cut.position, list(p.cut.block_a), list(p.cut.block_b)],
    }
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def save(case, **arrays):
    os.makedirs(AMPS, exist_ok=True)
    np.savez_compressed(os.path.join(AMPS, f"{case}.npz"), **arrays)
    print("wrote", case, {k: getattr(v, "shape", v) for k, v in arrays.items()}, flush=True)


def small_cases():
    from oracles import naive_state

    # 2-qubit known answer (test_pathsum.py:160-174)
    circ = parse_circuit("2\n0 h 0\n0 h 1\n1 cz 0 1\n", rows=1, cols=2)
    plan = ps.make_plan(circ, x_p=1, x_b=0)
    idx = np.arange(4, dtype=np.int64)
    save("cz2", text=serialize_circuit(circ), requests=idx, x_p=1, x_b=0,
         amps_c64=ps.run_approx(circ, plan, idx).amps,
         path0=ps.run_prefix_tree(circ, plan, 0, idx).amps,
         path1=ps.run_prefix_tree(circ, plan, 1, idx).amps)

    cases = {
        "s3x4v2": (generate(GenSpec(3, 4, 14, "v2", seed=6)), None),
        "s3x4v1": (generate(GenSpec(3, 4, 14, "v1", seed=6)), None),
        "s4x4v2": (generate(GenSpec(4, 4, 12, "v2", seed=6)), None),
        "stair3x4": (generate(GenSpec(3, 4, 10, "v2", seed=2)),
                     Cut("s", 9, (0, 1, 2, 4, 5, 8), (3, 6, 7, 9, 10, 11))),
        "iswap2x3": (generate(GenSpec(2, 3, 8, "v2", seed=0, two_qubit=GateKind.ISWAP)), None),
        "iswap3x3": (generate(GenSpec(3, 3, 10, "v1", seed=4, two_qubit=GateKind.ISWAP)), None),
        "fsim3x4": (fsim_variant(generate(GenSpec(3, 4, 10, "v2", seed=3)), seed=7), None),
        "fsim2x4": (fsim_variant(generate(GenSpec(2, 4, 12, "v1", seed=5)), seed=11), None),
    }
    for name, (circ, cut) in cases.items():
        idx = np.arange(1 << circ.n_qubits, dtype=np.int64)
        plan = ps.make_plan(circ, fidelity=1.0, cut=cut)
        a64 = ps.run_approx(circ, plan, idx).amps
        with c128():
            fc = fresh(circ)
            a128 = ps.run_approx(fc, ps.make_plan(fc, fidelity=1.0, cut=cut), idx).amps
        n_paths = len(plan.retained) * plan.branch_space
        pids = np.unique(np.random.default_rng(1).integers(0, n_paths, size=6))
        path_amps = np.stack([ps.run_path(circ, plan, int(p), idx).amps for p in pids])
        save(name, text=serialize_circuit(circ), requests=idx,
             cut=np.array(cut.block_a if cut else [], dtype=np.int64),
             x_p=plan.x_p, x_b=plan.x_b, amps_c64=a64, amps_c128=a128,
             exact=naive_state(circ), path_ids=pids, path_amps=path_amps)


def config_cases():
    # (name, n_prefix window or None=all, n_req cap, c128 window)
    jobs = [
        ("cfg1", None, None, None),
        ("cfg1v2", None, None, None),
        ("cfg2", 256, None, 32),
        ("cfg2v2", 128, None, None),
        ("cfg2h", 128, None, 16),
        ("cfg3", 3, 4096, 1),
        ("cfg3v2", 2, 4096, None),
        ("cfg4", 2, 4096, None),
    ]
    for name, win, req_cap, win128 in jobs:
        r, c, d, ver, f, n_req, cutname = CFG[name]
        circ = gen(r, c, d, ver)
        cut = staircase() if cutname == "staircase" else None
        plan = ps.make_plan(circ, fidelity=f, seed=0, cut=cut, workers=1)
        req = challenge_indices(circ.n_qubits, n_req, 12345)
        if req_cap:
            req = req[:req_cap]
        pre = plan.retained if win is None else plan.retained[:win]
        t = time.time()
        a64 = ps.run_batched(circ, plan, req, prefixes=pre).amps
        t64 = time.time() - t
        arrays = dict(requests=req, prefixes=pre, amps_c64=a64, seconds_c64=t64)
        if name.startswith("cfg1"):
            with c128():
                fc = fresh(circ)
                p2 = ps.make_plan(fc, fidelity=f, seed=0, cut=cut, workers=1)
                arrays["amps_c128"] = ps.run_batched(fc, p2, req).amps
            arrays["full_c64"] = sv.fetch_amplitudes(sv.run_full(circ), req).amps
            n_paths = len(plan.retained) * plan.branch_space
            pids = np.unique(np.random.default_rng(2).integers(0, n_paths, size=8))
            arrays["path_ids"] = pids
            arrays["path_amps"] = np.stack([ps.run_path(circ, plan, int(p), req).amps for p in pids])
            # a truncated plan (f = 0.25) over the same circuit
            pq = ps.make_plan(circ, fidelity=0.25, seed=5, cut=cut, workers=1)
            arrays["f025_retained"] = pq.retained
            arrays["f025_amps"] = ps.run_approx(circ, pq, req).amps
        elif win128:
            with c128():
                fc = fresh(circ)
                p2 = ps.make_plan(fc, fidelity=f, seed=0, cut=cut, workers=1)
                pre128 = p2.retained[:win128]
                arrays["prefixes_c128"] = pre128
                arrays["amps_c128"] = ps.run_batched(fc, p2, req, prefixes=pre128).amps
        if name in ("cfg2", "cfg3"):
            n_paths = len(pre) * plan.branch_space
            pids = np.unique(np.random.default_rng(3).integers(0, n_paths, size=3))
            pids = np.array([int(pre[p // plan.branch_space]) * plan.branch_space
                             + p % plan.branch_space for p in pids], dtype=np.int64)
            arrays["path_ids"] = pids
            arrays["path_amps"] = np.stack([ps.run_path(circ, plan, int(p), req).amps for p in pids])
        save(name, **arrays)


def full_state_cases():
    """Exact amplitudes of config 2 at its 10^4 requests (run_full, DTYPE rebound to c128)."""
    r, c, d, ver, f, n_req, _ = CFG["cfg2"]
    req = challenge_indices(r * c, n_req, 12345)
    with c128():
        circ = fresh(gen(r, c, d, ver))
        t = time.time()
        state = sv.run_full(circ)
        exact = state.amps[req].astype(np.complex128)
    save("cfg2_full", requests=req, exact=exact, seconds=time.time() - t)


def _heavy_plan(name):
    base = gen(7, 8, 40, "v1")
    if name == "cfg5f":
        circ = fsim_variant(base)
        plan = ps.make_plan(circ, fidelity=256 / 4**31, x_p=31, x_b=4, seed=0)
        return circ, plan, plan.retained
    circ = base
    head = np.load(os.path.join(DATA, "cfg5_retained_head.npy"))
    from gridsim.pathsum import SimPlan
    p0 = ps.make_plan(circ, fidelity=1e-30, seed=0)
    plan = SimPlan(p0.cut, 0.005, p0.radices, p0.x_p, p0.x_b, p0.d_p, p0.d_b, 0, head)
    return circ, plan, head


HEAVY_BRANCHES = {"cfg5": (0, 3), "cfg5f": (0, 3)}
HEAVY_NREQ = 2048


def heavy_one(name, branch):
    """One reference run_path at 28|28 (about 30-50 CPU-minutes, ~10 GB): the path
    (first retained prefix, branch) of cfg5 / cfg5f, saved as a part file."""
    circ, plan, pre = _heavy_plan(name)
    req = challenge_indices(circ.n_qubits, 10**6, 12345)[:HEAVY_NREQ]
    pid = int(pre[0]) * plan.branch_space + branch
    t = time.time()
    amps = ps.run_path(circ, plan, pid, req).amps
    os.makedirs(os.path.join(AMPS, "_parts"), exist_ok=True)
    np.savez(os.path.join(AMPS, "_parts", f"{name}_{branch}.npz"), requests=req, path_id=pid,
             amps=amps, seconds=time.time() - t, digits=np.array(ps.path_digits(pid, plan.radices)))
    print(name, branch, "path", pid, "took", round(time.time() - t, 1), "s", flush=True)


def heavy_merge(name):
    parts = [np.load(os.path.join(AMPS, "_parts", f"{name}_{b}.npz")) for b in HEAVY_BRANCHES[name]]
    save(name, requests=parts[0]["requests"],
         path_ids=np.array([int(p["path_id"]) for p in parts], dtype=np.int64),
         path_amps=np.stack([p["amps"] for p in parts]),
         seconds=np.array([float(p["seconds"]) for p in parts]))


def heavy_cases(which=("cfg5", "cfg5f")):
    """cfg5 / cfg5f per-path reference amplitudes at 28|28 (hours of CPU; 2 GiB
    half-states). Each path runs in its own process (``--heavy-one name:branch``)
    so they can run side by side; ``--heavy-merge`` writes amps/<name>.npz."""
    for name in which:
        for b in HEAVY_BRANCHES[name]:
            heavy_one(name, b)
        heavy_merge(name)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--heavy", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--heavy-one", default="")
    ap.add_argument("--heavy-merge", default="")
    args = ap.parse_args()
    if args.heavy_one:
        nm, br = args.heavy_one.split(":")
        heavy_one(nm, int(br))
        sys.exit(0)
    if args.heavy_merge:
        for nm in args.heavy_merge.split(","):
            heavy_merge(nm)
        sys.exit(0)
    if args.heavy:
        heavy_cases(tuple(args.only.split(",")) if args.only else ("cfg5", "cfg5f"))
        sys.exit(0)
    steps = args.only.split(",") if args.only else ["circuits", "small", "configs", "full"]
    if "circuits" in steps:
        h = write_circuits()
        plans(h)
    if "small" in steps:
        small_cases()
    if "configs" in steps:
        config_cases()
    if "full" in steps:
        full_state_cases()
