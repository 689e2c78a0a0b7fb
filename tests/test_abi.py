"""The C ABI library: loads, exports every declared symbol, and its host-side
planning (path-tree enumeration, pass scheduling, error mapping) is exercised
through host-only contexts (device = -1: no kernels, no GPU needed)."""
import os
import re

import numpy as np
import pytest

from paper_1807_10749_b200 import CircuitError, configs, make_plan, split_requests
from paper_1807_10749_b200.lowering import lowered

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_1807_10749_b200 import engine

    with open(os.path.join(ROOT, "include", "gridsim_b200.h")) as fh:
        header = fh.read()
    declared = set(re.findall(r"\b(gs_[a-z_]+)\s*\(", header))
    assert declared == set(engine.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(engine.LIB, name), name
    assert engine.LIB.gs_abi_version() == 2


def host_engine(dtype="c64"):
    from paper_1807_10749_b200.engine import Engine

    return Engine(device=-1, dtype=dtype)


def expected_nodes(circ, plan, prefixes, branch_lo=0, branch_hi=None):
    """Distinct digit prefixes per level (the path tree), counted in Python."""
    radices = plan.radices
    prog = lowered(circ, plan.cut)
    cyc = prog.cross_cycle
    ends = [k + 1 for k in range(len(cyc)) if k + 1 == len(cyc) or cyc[k + 1] != cyc[k]]
    bs = plan.branch_space
    branch_hi = bs if branch_hi is None else branch_hi
    paths = [int(p) * bs + b for p in sorted(prefixes) for b in range(branch_lo, branch_hi)]
    total = 1  # root
    for li, e in enumerate(ends):
        suffix = int(np.prod(radices[e:], dtype=object)) if e < len(radices) else 1
        keys = [p // suffix for p in paths]
        total += len(keys) if li == len(ends) - 1 else len(set(keys))
    return total, len(paths), len(ends) + 1


@pytest.mark.parametrize("name", ["cfg1", "cfg1v2", "cfg2", "cfg3"])
def test_dry_run_tree_counts(name):
    circ, plan, req, pre = configs.build(name, n_req=16)
    if name == "cfg3":
        pre = pre[:300]
    eng = host_engine()
    eng.load_program(lowered(circ, plan.cut))
    ia, ib = split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req)
    eng.set_requests(ia, ib)
    st = eng.run(plan.x_p, pre, 0, plan.branch_space).stats
    nodes, leaves, levels = expected_nodes(circ, plan, pre)
    assert st["n_paths"] == leaves
    assert st["n_nodes"] == nodes
    assert st["n_levels"] == levels
    # a branch sub-range and another split enumerate the same leaves
    st2 = eng.run(plan.x_p, pre[:3], 1, plan.branch_space).stats
    assert st2["n_paths"] == 3 * (plan.branch_space - 1)
    p0 = make_plan(circ, x_p=0, cut=plan.cut) if plan.x <= 20 else None
    if p0 is not None:
        st3 = eng.run(0, [0], 0, p0.branch_space).stats
        assert st3["n_paths"] == p0.branch_space


def test_dry_run_duplicates_and_unsorted():
    circ, plan, req, _ = configs.build("cfg1v2", n_req=4)
    eng = host_engine()
    eng.load_program(lowered(circ, plan.cut))
    eng.set_requests(*split_requests(16, plan.cut.block_a, plan.cut.block_b, req))
    pre = np.array([5, 3, 5, 9], dtype=np.int64)
    st = eng.run(plan.x_p, pre, 0, plan.branch_space).stats
    assert st["n_paths"] == 4 * plan.branch_space
    flat = make_plan(circ, x_b=0)
    st = eng.run(flat.x_p, np.array([7, 7, 2]), 0, 1).stats
    assert st["n_paths"] == 3


def test_error_mapping():
    circ, plan, req, _ = configs.build("cfg1", n_req=4)
    eng = host_engine()
    with pytest.raises(RuntimeError):
        eng.run(plan.x_p, plan.retained, 0, plan.branch_space)  # no program
    eng.load_program(lowered(circ, plan.cut))
    with pytest.raises(IndexError):
        eng.set_requests(np.array([256]), np.array([0]))
    eng.set_requests(np.array([0, 1]), np.array([2, 3]))
    with pytest.raises(CircuitError):
        eng.run(plan.x + 1, [0], 0, 1)
    with pytest.raises(ValueError):
        eng.run(plan.x_p, [plan.prefix_space], 0, plan.branch_space)
    with pytest.raises(ValueError):
        eng.run(plan.x_p, [0], 0, plan.branch_space + 1)
    with pytest.raises(ValueError):
        eng.set_option("no_such_option", 1)
    with pytest.raises(ValueError):
        eng.set_option("tile_bits", 40)


@pytest.mark.parametrize("tile_bits", [4, 5, 8, 13])
def test_scheduler_covers_all_ops(tile_bits):
    """Smaller tiles split levels into more passes; every op is still scheduled once."""
    circ, plan, req, pre = configs.build("cfg2", n_req=4)
    eng = host_engine()
    eng.set_option("tile_bits", tile_bits)
    eng.load_program(lowered(circ, plan.cut))
    eng.set_requests(np.array([0]), np.array([0]))
    st = eng.run(plan.x_p, pre[:64], 0, plan.branch_space).stats
    assert st["n_paths"] == 64 * plan.branch_space
    assert st["n_pass_launches"] >= 2 * st["n_levels"]


def test_set_requests_global_validation():
    circ, plan, req, _ = configs.build("cfg1", n_req=8)
    eng = host_engine()
    eng.load_program(lowered(circ, plan.cut))
    eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
    assert eng.n_req == req.size
    with pytest.raises(IndexError):
        eng.set_requests_global(np.array([1 << 16]), 16, plan.cut.block_a, plan.cut.block_b)
    with pytest.raises(IndexError):
        eng.set_requests_global(np.array([-1]), 16, plan.cut.block_a, plan.cut.block_b)
    with pytest.raises(ValueError):
        eng.set_requests_global(req, 15, plan.cut.block_a, plan.cut.block_b)
    with pytest.raises(ValueError):
        eng.set_requests_global(req, 16, plan.cut.block_a, plan.cut.block_a)


def test_run_batched_host_only():
    """gs_run_batched = set_requests_global + run: same tree, same validation."""
    circ, plan, req, pre = configs.build("cfg1", n_req=64)
    eng = host_engine()
    eng.load_program(lowered(circ, plan.cut))
    ba, bb = plan.cut.block_a, plan.cut.block_b
    r = eng.run_batched(req, circ.n_qubits, ba, bb, plan.x_p, pre[:5], 0, plan.branch_space)
    assert r.stats["n_paths"] == 5 * plan.branch_space
    assert eng.n_req == req.size
    # the requests stay loaded for plain runs
    assert eng.run(plan.x_p, pre[:2], 0, plan.branch_space).stats["n_paths"] == 2 * plan.branch_space
    bad = req.copy()
    bad[-1] = 1 << circ.n_qubits
    with pytest.raises(IndexError):
        eng.run_batched(bad, circ.n_qubits, ba, bb, plan.x_p, pre[:5], 0, plan.branch_space)
    with pytest.raises(RuntimeError):  # a failed call leaves no requests loaded
        eng.run(plan.x_p, pre[:2], 0, plan.branch_space)
    with pytest.raises(ValueError):
        eng.run_batched(req, circ.n_qubits, ba, ba, plan.x_p, pre[:5], 0, plan.branch_space)
    with pytest.raises(ValueError):  # bad prefix: workers joined, error reported
        eng.run_batched(req, circ.n_qubits, ba, bb, plan.x_p, [plan.prefix_space], 0, plan.branch_space)
    r = eng.run_batched(np.array([], dtype=np.int64), circ.n_qubits, ba, bb, plan.x_p, pre[:1], 0, 1)
    assert r.amps.shape == (0,)


def _gf2_rank(vectors):
    rows, rank = list(vectors), 0
    for bit in range(32):
        piv = next((i for i in range(rank, len(rows)) if (rows[i] >> bit) & 1), None)
        if piv is None:
            continue
        rows[rank], rows[piv] = rows[piv], rows[rank]
        for i in range(len(rows)):
            if i != rank and (rows[i] >> bit) & 1:
                rows[i] ^= rows[rank]
        rank += 1
    return rank


def test_pauli_sibling_planning_host_only():
    """Planning of the Pauli-sibling leaves on host-only contexts:
    which leaf sides are Pauli-compatible, which form is planned, and the parked
    tile's address map (invertible over GF(2), branch-gate flips on address bits
    0..2, conflict-free park stores)."""
    want = {  # name: (pauli_sides, fused Pauli pass planned, psib_side)
        "cfg4": ([1, 1], True, -1),    # CZ cut, v1 rules: I/Z side fused with the projected gather
        "cfg3v2": ([1, 1], True, -1),
        "cfg3": ([0, 0], False, -1),   # a T behind an X^1/2 in the leaf level: not Pauli-compatible
        "cfg5": ([0, 1], False, 1),    # 28|28: path-major gathers read side B's leaves as Pauli images
        "cfg2h": ([1, 1], False, 1),
    }
    for name, (sides, fused, psib) in want.items():
        circ, plan, _, _ = configs.build(name, n_req=4)
        eng = host_engine()
        eng.load_program(lowered(circ, plan.cut))
        d = eng.describe()
        assert d["pauli_sides"] == sides, name
        assert (d["pauli"] is not None) == fused, name
        assert d["psib_side"] == psib, name
        if not fused:
            continue
        leaf = d["levels"][-1]["blocks"][1 - d["proj_side"]]["passes"]
        assert len(leaf) == 1 and leaf[0]["k"] == leaf[0]["K"]  # one pass, no slot bits
        assert all(not tok.startswith("dx") for tok in leaf[0]["opl"].split())  # no cross terms in it
        K, lbits = leaf[0]["k"], leaf[0]["lbits"]
        lcol = d["pauli"]["lcol"][:K]
        assert _gf2_rank(lcol) == K  # L is invertible
        assert d["pauli"]["conflicts"] == 1
        gates = d["pauli"]["gates"]
        for b in range(min(3, len(gates))):  # sibling bit b <-> the b-th last cross gate: L f_b = e_b
            f = gates[len(gates) - 1 - b]["f"]
            lf = 0
            for j, sb in enumerate(lbits):
                if (f >> sb) & 1:
                    lf ^= lcol[j]
            assert lf == 1 << b, (name, b)
        for g in gates:  # every flip / sign bit is a tile bit of the pass
            assert all(((g["f"] | g["z"]) >> sb) & 1 == 0 for sb in range(circ.n_qubits) if sb not in lbits)
    # option off: the 8-slot form
    circ, plan, _, _ = configs.build("cfg4", n_req=4)
    eng = host_engine()
    eng.set_option("pf_pauli", 0)
    eng.load_program(lowered(circ, plan.cut))
    d = eng.describe()
    assert d["pauli"] is None and d["levels"][-1]["blocks"][1]["passes"][0]["K"] == 13
    assert d["levels"][-1]["blocks"][1]["passes"][0]["k"] == 10
