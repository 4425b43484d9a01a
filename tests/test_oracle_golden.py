"""Pin the CPU semantics oracle against traces produced by the real reference
EmulatedWorker (tests/golden/worker_traces.json, made by oracle/make_golden.py)."""

import json
import os

import pytest

from helpers import run_oracle, scenario

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worker_traces.json")
TRACES = json.load(open(GOLDEN))


@pytest.mark.parametrize("trace", TRACES, ids=lambda t: f"seed{t['seed']}")
def test_oracle_reproduces_reference_trace(trace):
    got = run_oracle(scenario(trace["seed"]))
    assert got["results"] == trace["results"]
    assert got["final"] == trace["final"]


def test_golden_covers_every_status():
    statuses = {r[1] for t in TRACES for r in t["results"]}
    assert statuses == {1, 2, 3, 4, 5}
