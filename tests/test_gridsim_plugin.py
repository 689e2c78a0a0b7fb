"""The drop-in boundary: the reference package's own objects and engine hook.

``gridsim.pathsum.run_approx(engine=...)`` (``pathsum.py:419-443``) is the
reference's extension point.  CPU: a ``gridsim`` circuit/cut/plan lowers to
exactly the arrays our own parse of the same text lowers to, and
``install`` / ``uninstall`` swap the functions in every ``gridsim`` module
that bound them.  GPU: ``gridsim.pathsum.run_approx(..., engine="b200")`` on
the reference's objects matches the reference's own engine and the golden
amplitudes; with ``default=True`` the reference's unmodified callers
(``validate.claimant_round``) run on the device.

``gridsim`` comes from the offline install under ``baseline/_ref`` (it travels
to the GPU box with the repo); the tests skip only where it is absent.
"""
import numpy as np
import pytest

from conftest import load_amps, rel_l2, small_case
from paper_1807_10749_b200 import configs
from paper_1807_10749_b200.gridsim_engine import gridsim_available, load_gridsim

pytestmark = pytest.mark.skipif(not gridsim_available(), reason="gridsim not installed")


def _ref_objects(name):
    """(gridsim circuit, gridsim plan, requests, our circuit, our plan) for a config."""
    gc = load_gridsim("circuit")
    gps = load_gridsim("pathsum")
    circ, plan, req, _ = configs.build(name)
    with open(configs.CONFIGS[name].circuit_file) as fh:
        text = fh.read()
    rc = gc.parse_circuit(text, circ.rows, circ.cols)
    cut = plan.cut
    rcut = gc.Cut(cut.orientation, cut.position, tuple(cut.block_a), tuple(cut.block_b))
    spec = configs.CONFIGS[name]
    rplan = gps.make_plan(rc, fidelity=spec.fidelity, x_p=spec.x_p, x_b=spec.x_b, seed=0, cut=rcut,
                          workers=1)
    return rc, rplan, req, circ, plan


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_gridsim_objects_lower_identically(name):
    from paper_1807_10749_b200.lowering import lower_circuit

    rc, rplan, _, circ, plan = _ref_objects(name)
    assert np.array_equal(rplan.retained, plan.retained)
    assert tuple(rplan.radices) == tuple(plan.radices)
    mine = lower_circuit(circ, plan.cut)
    theirs = lower_circuit(rc, rplan.cut)
    for field in mine.__dataclass_fields__:
        a, b = getattr(mine, field), getattr(theirs, field)
        assert np.array_equal(np.asarray(a), np.asarray(b)), field


def test_gridsim_fsim_and_iswap_gates_lower_identically():
    from paper_1807_10749_b200.circuit import serialize_circuit
    from paper_1807_10749_b200.lowering import lower_circuit

    gc = load_gridsim("circuit")
    for case in ("fsim3x4", "iswap3x3"):
        circ, plan, _, _ = small_case(case)
        rc = gc.parse_circuit(serialize_circuit(circ), circ.rows, circ.cols)
        rcut = gc.Cut(plan.cut.orientation, plan.cut.position, plan.cut.block_a, plan.cut.block_b)
        a, b = lower_circuit(circ, plan.cut), lower_circuit(rc, rcut)
        assert np.array_equal(a.coef, b.coef) and np.array_equal(a.term_kind_a, b.term_kind_a)
        assert np.array_equal(a.op_kind, b.op_kind) and np.array_equal(a.cross_rank, b.cross_rank)


def test_circuit_hash_and_text_are_interchangeable():
    from paper_1807_10749_b200.circuit import circuit_hash, serialize_circuit

    gc = load_gridsim("circuit")
    for name in ("cfg1", "cfg5f"):
        spec = configs.CONFIGS[name]
        circ = configs.load_circuit(spec)
        rc = gc.parse_circuit(serialize_circuit(circ), spec.rows, spec.cols)
        assert gc.serialize_circuit(rc) == serialize_circuit(circ)
        assert gc.circuit_hash(rc) == circuit_hash(circ)
        assert gc.choose_cut(rc).block_a == configs.build(name, n_req=4)[1].cut.block_a or \
            spec.cut != "default"


def test_install_routes_every_binding_and_uninstall_restores():
    from paper_1807_10749_b200 import gridsim_engine as ge

    ps, gv, orch = load_gridsim("pathsum"), load_gridsim("validate"), load_gridsim("orchestrator")
    ref = (ps.run_approx, gv.run_approx, ps.run_batched, orch.run_prefix_tree, gv.run_full)
    rc, rplan, req, _, _ = _ref_objects("cfg1")
    with pytest.raises(ValueError):
        ps.run_approx(rc, rplan, req[:4], engine="b200")  # not registered yet: the reference's error
    ge.install()
    try:
        assert ps.run_approx is not ref[0] and gv.run_approx is ps.run_approx
        assert ps.run_batched is ref[2]  # default=False leaves the reference default engine alone
        with pytest.raises(ValueError):
            ps.run_approx(rc, rplan, req[:4], engine="nope")
        ge.install(default=True)
        assert ps.run_batched is not ref[2] and orch.run_prefix_tree is not ref[3]
        assert gv.run_full is not ref[4]
    finally:
        ge.uninstall()
    assert (ps.run_approx, gv.run_approx, ps.run_batched, orch.run_prefix_tree, gv.run_full) == ref
    with ge.routed_to_device():
        assert ps.run_batched is not ref[2]
    assert ps.run_batched is ref[2] and not ge.installed()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "cfg1v2"])
def test_gridsim_run_approx_engine_b200(name):
    from paper_1807_10749_b200 import gridsim_engine as ge

    ps, sv = load_gridsim("pathsum"), load_gridsim("statevec")
    rc, rplan, req, _, _ = _ref_objects(name)
    ge.install()
    try:
        got = ps.run_approx(rc, rplan, req, engine="b200")
        cpu = ps.run_approx(rc, rplan, req)  # the reference's own batched engine
    finally:
        ge.uninstall()
    assert isinstance(got, sv.AmplitudeBatch)
    assert np.array_equal(got.indices, req)
    assert rel_l2(got.amps, cpu.amps) <= 1e-5
    assert rel_l2(got.amps, load_amps(name)["amps_c64"]) <= 1e-5


@pytest.mark.gpu
def test_gridsim_run_batched_prefix_hook_on_device():
    from paper_1807_10749_b200 import gridsim_engine as ge

    ps = load_gridsim("pathsum")
    rc, rplan, _, _, _ = _ref_objects("cfg3")
    g = load_amps("cfg3")
    with ge.routed_to_device():
        got = ps.run_batched(rc, rplan, g["requests"], prefixes=g["prefixes"])
    assert rel_l2(got.amps, g["amps_c64"]) <= 1e-5


@pytest.mark.gpu
def test_gridsim_claimant_round_on_device():
    """The reference's claimant round, unmodified, with its run_approx routed to the B200."""
    from paper_1807_10749_b200 import gridsim_engine as ge

    gv = load_gridsim("validate")
    rc, _, _, _, _ = _ref_objects("cfg1")
    ch = gv.issue_challenge(rc, k=256, seed=3, f1=0.2)
    cpu = gv.claimant_round(rc, ch, engine="hybrid", fidelity=0.5, seed=4)
    with ge.routed_to_device():
        dev = gv.claimant_round(rc, ch, engine="hybrid", fidelity=0.5, seed=4)
        exact = gv.claimant_round(rc, ch, engine="exact")
    assert rel_l2(dev.amps, cpu.amps) <= 1e-5
    assert rel_l2(exact.amps, gv.claimant_round(rc, ch, engine="exact").amps) <= 1e-5
