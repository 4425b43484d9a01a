"""The native executor (libcw engine, sim mode) against the reference: bit-exact
statuses, start/end/device_duration and PageCache pages_free on every result,
and the final resident sets (SURVEY §4 differential test (1))."""

import json
import os

import pytest

from helpers import run_engine, run_oracle, scenario

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worker_traces.json")
TRACES = json.load(open(GOLDEN))


@pytest.mark.parametrize("trace", TRACES, ids=lambda t: f"seed{t['seed']}")
def test_engine_reproduces_reference_trace(trace):
    got = run_engine(scenario(trace["seed"]))
    assert got["results"] == trace["results"]
    assert got["final"] == trace["final"]


@pytest.mark.parametrize("seed", range(1000, 1150))
def test_engine_matches_oracle_on_fresh_scenarios(seed):
    sc = scenario(seed)
    assert run_engine(sc) == run_oracle(sc)


def test_page_conservation_and_window_compliance():
    # SPEC.md:236-241 invariants over many scenarios.
    for seed in range(2000, 2060):
        sc = scenario(seed)
        got = run_engine(sc)
        acts = {d["action_id"]: d for d in sc["deliveries"]}
        for aid, status, start, end, dur, free in got["results"]:
            a = acts[aid]
            if status == 1 and a["kind"] != 2:
                assert a["earliest"] <= start <= a["latest"]
                assert end >= start
            if status != 1:
                assert dur == 0
            if free >= 0:
                assert 0 <= free <= sc["pages"]
        for g, (free, res) in enumerate(got["final"]):
            assert free + sum(p for _, p in res) == sc["pages"]


def test_exec_intervals_never_overlap():
    for seed in range(3000, 3040):
        sc = scenario(seed)
        got = run_engine(sc)
        acts = {d["action_id"]: d for d in sc["deliveries"]}
        spans = {}
        for aid, status, start, end, dur, _ in got["results"]:
            a = acts[aid]
            if status == 1 and a["kind"] == 3:
                spans.setdefault(a["gpu"], []).append((start, start + dur))
        for g, iv in spans.items():
            iv.sort()
            for (s0, e0), (s1, e1) in zip(iv, iv[1:]):
                assert s1 >= e0
