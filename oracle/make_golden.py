"""Generate golden fixtures from the REAL reference — TEST INFRASTRUCTURE ONLY.

Runs only in the build container, where the read-only reference lives at
/root/reference; its outputs are committed under tests/golden/ so the GPU box
(which has no reference) and the CPU tests can check against them.

    python oracle/make_golden.py

Fixtures:
  worker_traces.json  per scenario (oracle/scenarios.py): every ActionResult the
                      reference EmulatedWorker emits under SimLoop, in emission
                      order, with the action's GPU pages_free at emission, plus
                      the final resident set of every GPU.
  wire_frames.json    fuzzed messages of all five kinds encoded by
                      sloserve.protocol.encode_message (hex), incl. the SPEC
                      known-answer sizes (38-byte Unload).
  catalog.json        pages_needed and canonical dumps for the reference catalog
                      (profiles.py:109-111, 284-312, 322-374).
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = "/root/reference/pkg/src"
OUT = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, REPO)

from sloserve import profiles, protocol  # noqa: E402
from sloserve.protocol import Action, ActionKind  # noqa: E402
from sloserve.timebase import SimLoop  # noqa: E402
from sloserve.worker import EmulatedWorker  # noqa: E402

from oracle.scenarios import scenario  # noqa: E402

N_SCENARIOS = 40


def run_reference(sc: dict) -> dict:
    catalog = profiles.loads_catalog(sc["catalog"])
    loop = SimLoop()
    results = []
    holder = {}

    def send_result(r):
        w = holder["w"]
        act = holder["acts"][r.action_id]
        free = w.gpus[act.gpu_index].pages.pages_free if act.gpu_index < len(w.gpus) else -1
        results.append([r.action_id, int(r.status), r.start, r.end, r.device_duration, free])

    w = EmulatedWorker(0, catalog, loop, send_result, gpu_count=sc["gpu_count"],
                       pages_per_gpu=sc["pages"], io_capacity=sc["io_capacity"],
                       keep_records=False)
    holder["w"] = w
    holder["acts"] = {}
    for d in sc["deliveries"]:
        batch = tuple(range(d["batch"])) if d["kind"] == 3 else ()
        a = Action(d["action_id"], ActionKind(d["kind"]), d["model_id"], d["earliest"],
                   d["latest"], batch, d["gpu"])
        holder["acts"][a.action_id] = a
        loop.call_at(d["t"], w.on_action, a)
    loop.run_until(sc["horizon"])
    final = [[g.pages.pages_free, sorted([m, p] for m, p in g.pages.resident.items())]
             for g in w.gpus]
    return {"results": results, "final": final}


def wire_fixtures(n: int = 300) -> list:
    rng = random.Random(7)
    out = []
    for i in range(n):
        k = i % 5
        if k == 0:
            kind = rng.choice([1, 2, 3])
            e = rng.randrange(-2**40, 2**40)
            batch = tuple(rng.randrange(2**64) for _ in range(rng.randint(1, 16))) if kind == 3 else ()
            msg = Action(rng.randrange(2**64), ActionKind(kind), rng.randrange(2**32), e,
                         e + rng.randrange(2**40), batch, rng.randrange(2**16),
                         rng.randrange(2**40) if kind == 3 else 0)
            fields = dict(type="action", action_id=msg.action_id, kind=kind,
                          model_id=msg.model_id, earliest=msg.earliest, latest=msg.latest,
                          batch=list(batch), gpu_index=msg.gpu_index,
                          expected_duration=msg.expected_duration)
        elif k == 1:
            st = rng.randint(1, 5)
            s = rng.randrange(-2**40, 2**40)
            msg = protocol.ActionResult(rng.randrange(2**64), protocol.ResultStatus(st), s,
                                        s + rng.randrange(2**30),
                                        rng.randrange(2**30) if st == 1 else 0)
            fields = dict(type="result", action_id=msg.action_id, status=st, start=msg.start,
                          end=msg.end, device_duration=msg.device_duration)
        elif k == 2:
            payload = bytes(rng.randrange(256) for _ in range(rng.randint(0, 40)))
            msg = protocol.InferenceRequest(rng.randrange(2**64), rng.randrange(2**32),
                                            rng.randrange(1, 2**40), rng.randrange(2**40),
                                            rng.randrange(2**30), payload)
            fields = dict(type="request", request_id=msg.request_id, model_id=msg.model_id,
                          slo=msg.slo, arrival=msg.arrival, input_size=msg.input_size,
                          payload=payload.hex())
        elif k == 3:
            msg = protocol.InferenceResponse(rng.randrange(2**64),
                                             protocol.ResponseStatus(rng.randint(1, 3)),
                                             rng.randrange(-2**40, 2**40), rng.random() < 0.5)
            fields = dict(type="response", request_id=msg.request_id, status=int(msg.status),
                          latency=msg.latency, cold_start=msg.cold_start)
        else:
            models = tuple(rng.randrange(2**32) for _ in range(rng.randint(0, 12)))
            msg = protocol.WorkerHandshake(rng.randrange(2**32), rng.randint(1, 8),
                                           rng.randrange(1, 2**40), models)
            fields = dict(type="handshake", worker_id=msg.worker_id, gpu_count=msg.gpu_count,
                          pages_total=msg.pages_total, models=list(models))
        out.append({"fields": fields, "hex": protocol.encode_message(msg).hex()})
    # SPEC.md:136 known answer: Unload{0,0,0,0} is a 38-byte frame.
    kat = protocol.encode_message(Action(0, ActionKind.UNLOAD, 0, 0, 0))
    out.append({"fields": dict(type="action", action_id=0, kind=2, model_id=0, earliest=0,
                               latest=0, batch=[], gpu_index=0, expected_duration=0),
                "hex": kat.hex(), "kat_len": len(kat)})
    return out


def catalog_fixture() -> dict:
    cat = profiles.reference_catalog()
    profiles.replicate_model(cat, "resnet50", 3)
    return {
        "text": profiles.REFERENCE_CATALOG,
        "pages_needed": [cat.pages_needed(m) for m in cat.model_ids()],
        "dumps": profiles.dumps_catalog(cat),
        "names": [e.replica_of for e in cat.entries],
    }


def main():
    os.makedirs(OUT, exist_ok=True)
    traces = []
    for seed in range(N_SCENARIOS):
        sc = scenario(seed)
        traces.append({"seed": seed, **run_reference(sc)})
    with open(os.path.join(OUT, "worker_traces.json"), "w") as f:
        json.dump(traces, f, separators=(",", ":"))
    with open(os.path.join(OUT, "wire_frames.json"), "w") as f:
        json.dump(wire_fixtures(), f, indent=0)
    with open(os.path.join(OUT, "catalog.json"), "w") as f:
        json.dump(catalog_fixture(), f, indent=1)
    n = sum(len(t["results"]) for t in traces)
    print(f"wrote {len(traces)} traces ({n} results), wire and catalog fixtures to {OUT}")


if __name__ == "__main__":
    main()
