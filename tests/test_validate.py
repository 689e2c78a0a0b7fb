"""Verifier / claimant rounds against the reference's
own rounds, recorded by ``tests/golden/make_validate_golden.py`` on the
reference test's circuits (``test_validate.py:23-36``).

CPU: challenge bookkeeping and the verifier cut.  GPU: every round simulates
on the device (path sum + full state) and scores on the device; the retained
fraction and pass decision are exact, f_e within 1e-5 of the reference
(complex64 amplitudes, fp64 overlap).
"""
import json
import os

import numpy as np
import pytest

from paper_1807_10749_b200 import parse_circuit
from paper_1807_10749_b200.validate import (
    Challenge, ValidationError, calibrate_delta, challenge_indices, claimant_round, issue_challenge,
    read_challenge, verifier_cut, verifier_round, write_challenge,
)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "validate.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def circuit(golden):
    return parse_circuit(golden["circuit"])


def test_verifier_cut_matches_reference(golden, circuit):
    vc = verifier_cut(circuit)
    g = golden["verifier_cut"]
    assert (vc.orientation, vc.position) == (g["orientation"], g["position"])
    assert list(vc.block_a) == g["a"] and list(vc.block_b) == g["b"]


def test_challenge_round_trip_keeps_secret(circuit, tmp_path):
    ch = issue_challenge(circuit, k=64, seed=4, f1=0.1)
    path = tmp_path / "ch.json"
    write_challenge(path, ch)
    assert "f1" not in json.loads(path.read_text())
    back = read_challenge(path)
    assert back.f1 is None and back.public_dict() == ch.public_dict()
    (tmp_path / "bad.json").write_text("{}")
    with pytest.raises(ValidationError):
        read_challenge(tmp_path / "bad.json")


def test_challenge_validation(circuit):
    with pytest.raises(ValidationError):
        Challenge("h", 0, 1, 0.1)
    with pytest.raises(ValidationError):
        Challenge("h", 4, 1, -0.1)
    with pytest.raises(ValidationError):
        Challenge("h", 4, 1, 0.5, f1=0.1)
    with pytest.raises(ValidationError):
        issue_challenge(circuit, k=(1 << circuit.n_qubits) + 1)
    assert np.array_equal(challenge_indices(4, 16, 3), np.arange(16))


@pytest.mark.gpu
def test_rounds_match_reference(golden, circuit):
    vcut = verifier_cut(circuit)
    delta = golden["delta"]
    for r in golden["rounds"]:
        ch = issue_challenge(circuit, k=2048, delta=delta, seed=r["seed"], f1=r["f1"])
        resp = claimant_round(circuit, ch, engine=r["engine"], fidelity=r["fidelity"], seed=r["claimant_seed"])
        res = verifier_round(circuit, ch, resp, path_seed=r["path_seed"], cut=vcut)
        assert res.f1_realized == r["f1_realized"]
        assert res.f_e == pytest.approx(r["f_e"], abs=1e-5)
        assert res.passed == r["passed"]


@pytest.mark.gpu
def test_calibrated_delta_matches_reference(golden, circuit):
    delta = calibrate_delta(circuit, k=2048, rounds=6, seed=5, cut=verifier_cut(circuit))
    assert delta == pytest.approx(golden["delta"], abs=1e-4)
    assert delta < 0.05


@pytest.mark.gpu
def test_round_errors(golden, circuit):
    vcut = verifier_cut(circuit)
    other = parse_circuit(golden["other"])
    ch = issue_challenge(circuit, k=64, seed=1)
    public = Challenge(ch.circuit_hash, ch.k, ch.index_seed, ch.delta)
    response = claimant_round(circuit, public, engine="exact")
    with pytest.raises(ValidationError):
        verifier_round(circuit, public, response, path_seed=1, cut=vcut)
    with pytest.raises(ValidationError):
        claimant_round(other, ch, engine="exact")
    with pytest.raises(ValidationError):
        verifier_round(other, ch, response, path_seed=1)
    with pytest.raises(ValidationError):
        claimant_round(circuit, ch, engine="prayer")
    a = verifier_round(circuit, ch, response, path_seed=55, cut=vcut)
    b = verifier_round(circuit, ch, response, path_seed=55, cut=vcut)
    assert a == b
