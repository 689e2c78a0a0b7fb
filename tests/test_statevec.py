"""Full state-vector engine (reference run_full, statevec.py:410-446) -- SURVEY §8(f) row 1.

CPU tests: the uncut program loads and schedules on a host-only context, the
budget / index errors.  GPU tests: the GPU state equals the reference's exact
states (tests/golden/amps: `exact` = reference run_full/naive_state at the
requested indices) on CZ, iSWAP, fSim and 25-qubit circuits.
"""
import numpy as np
import pytest

from conftest import load_amps, rel_l2, small_case
from paper_1807_10749_b200 import configs
from paper_1807_10749_b200.lowering import lowered
from paper_1807_10749_b200.statevec import (
    MemoryBudgetError,
    StateBlock,
    fetch_amplitudes,
    full_cut,
    run_full,
)


def _host_engine():
    from paper_1807_10749_b200.engine import Engine

    return Engine(device=-1, dtype="c64")


def test_uncut_program_schedules_on_host():
    circ, plan, _, _ = configs.build("cfg1", n_req=4)
    prog = lowered(circ, full_cut(circ))
    assert (prog.n_a, prog.n_b, prog.n_cross) == (16, 0, 0)
    eng = _host_engine()
    eng.load_program(prog)
    d = eng.describe()
    assert len(d["levels"]) == 1
    a, b = d["levels"][0]["blocks"]
    assert len(b["passes"]) == 0 and len(a["passes"]) >= 1
    assert sum(p["ops"] for p in a["passes"]) == prog.n_ops
    r = eng.run_full()
    assert r.amps.shape == (1 << 16,) and r.stats["n_pass_launches"] == len(a["passes"])
    with pytest.raises(Exception):
        eng.set_requests([0], [0])
        eng.run(0, [0], 0, 1)  # the path sum refuses an uncut program


def test_cut_program_refuses_run_full():
    circ, plan, _, _ = configs.build("cfg1", n_req=4)
    eng = _host_engine()
    eng.load_program(lowered(circ, plan.cut))
    with pytest.raises(ValueError):
        eng.run_full()


def test_budget_and_index_errors():
    circ, _, _, _ = configs.build("cfg1", n_req=4)
    with pytest.raises(MemoryBudgetError):
        run_full(circ, mem_limit=1000)
    st = StateBlock.zero_state(3)
    assert st.norm_squared() == 1.0
    b = fetch_amplitudes(st, [0, 7])
    assert b.amps.dtype == np.complex128 and b.amps[0] == 1
    with pytest.raises(IndexError):
        fetch_amplitudes(st, [8])


SMALL = ["s3x4v2", "s3x4v1", "s4x4v2", "stair3x4", "iswap2x3", "iswap3x3", "fsim3x4", "fsim2x4"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SMALL)
def test_run_full_matches_exact(case):
    circ, _, _, g = small_case(case)
    st = run_full(circ)
    assert st.amps.dtype == np.complex64 and st.amps.size == 1 << circ.n_qubits
    assert rel_l2(fetch_amplitudes(st, g["requests"]).amps, g["exact"]) <= 1e-5
    st2 = run_full(circ, dtype="c128")
    assert rel_l2(st2.amps[g["requests"]], g["exact"]) <= 1e-10
    assert abs(st.norm_squared() - 1.0) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "cfg1v2"])
def test_run_full_matches_reference_run_full(name):
    g = load_amps(name)
    circ, _, _, _ = configs.build(name, n_req=4)
    st = run_full(circ)
    assert rel_l2(st.amps[g["requests"]], g["full_c64"]) <= 1e-5


@pytest.mark.gpu
def test_run_full_25_qubits():
    """config 2 (5x5, 1+24+1): the GPU full state equals the reference's exact
    25-qubit state at the 10^4 requested indices, and is normalised."""
    g = load_amps("cfg2_full")
    circ, _, _, _ = configs.build("cfg2", n_req=4)
    st = run_full(circ)
    assert rel_l2(st.amps[g["requests"]], g["exact"]) <= 1e-5
    assert abs(st.norm_squared() - 1.0) <= 1e-4
