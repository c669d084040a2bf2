"""Pins for the oracle's routing (row a7): Alg. 1 lines 8-13,
route(i), the Llama-3.2-1B worked values."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden_counts():
    rows = []
    for line in open(os.path.join(GOLD, "threshold_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        parts = line.split()
        rows.append((float(parts[0]), int(parts[1]), [int(v) for v in parts[2:]]))
    return rows


def test_paper_threshold_table(orc):
    text = open(os.path.join(GOLD, "llama32_1b_profile.json")).read()
    scores, tau, routes = orc.routes_from_profile(text)
    assert tau == 0.7 and len(scores) == 16
    for t, count, which in _golden_counts():
        r = orc.route_layers(scores, t)
        assert sum(r) == count, (t, r)
        if which:
            assert [i for i, v in enumerate(r) if v == orc.W4A16] == which


def test_golden_routes_at_default_tau(orc):
    # with tau = 0.7 one layer (the last, L15 0-based) goes to W4A16
    text = open(os.path.join(GOLD, "llama32_1b_profile.json")).read()
    _, _, routes = orc.routes_from_profile(text)
    assert routes == [0] * 15 + [1]


def test_raw_scores_renormalise_to_same_routes(orc):
    obj = json.load(open(os.path.join(GOLD, "llama32_1b_profile.json")))
    del obj["scores"]
    s, tau, routes = orc.routes_from_profile(json.dumps(obj))
    assert routes == [0] * 15 + [1]
    assert min(s) == 0.0 and max(s) == 1.0
    assert 0.69 < s[1] < 0.7                    # L1 sits just below tau


def test_minmax_spec_examples(orc):
    # S:149-151
    assert orc.minmax_normalize([1, 2, 3]) == [0.0, 0.5, 1.0]
    assert orc.minmax_normalize([5, 5, 5]) == [0.0, 0.0, 0.0]
    assert orc.minmax_normalize([0, 10]) == [0.0, 1.0]


def test_degenerate_all_w4a8(orc):
    # Alg. 1 line 9-10: max - min < eps -> all s^ = 0 -> every layer W4A8
    text = json.dumps({"raw_scores": [3.0] * 16, "epsilon": 1e-9})
    s, tau, r = orc.routes_from_profile(text)
    assert s == [0.0] * 16 and r == [0] * 16
    text = json.dumps({"raw_scores": [3.0, 3.0 + 1e-12], "epsilon": 1e-9})
    assert orc.routes_from_profile(text)[2] == [0, 0]


def test_tie_at_tau_goes_w4a16(orc):
    # P:557 "uses W4A16 if s^_i >= tau"
    assert orc.route_layers([0.7, 0.6999999], 0.7) == [1, 0]


def test_monotone_in_tau(orc):
    rng = np.random.default_rng(0)
    s = list(rng.uniform(0, 1, 32))
    prev = None
    for t in np.linspace(0, 1.2, 61):
        r = orc.route_layers(s, t)
        if prev is not None:
            assert all(a >= b for a, b in zip(prev, r))
        prev = r


@pytest.mark.parametrize("bad", [
    "[1,2,3]",
    "{\"tau\": 0.5}",
    "{\"scores\": [0.1, 1.5]}",
    "{\"scores\": [0.1, 0.2], \"num_layers\": 3}",
    "{\"scores\": [0.1, ",
])
def test_malformed_profiles_rejected(orc, bad):
    with pytest.raises((orc.OracleError, ValueError)):
        orc.routes_from_profile(bad)
