"""Shared test helpers: run a scenario (oracle/scenarios.py) through the
native engine in sim mode and through the CPU oracle."""

from oracle import scenarios, worker_oracle
from paper_2006_02464_b200 import catalog as catalog_mod
from paper_2006_02464_b200.wire import Action, ActionKind
from paper_2006_02464_b200.worker import Engine


def run_engine(sc: dict) -> dict:
    cat = catalog_mod.parse(sc["catalog"])
    eng = Engine(cat, mode="sim", worker_id=0, gpu_count=sc["gpu_count"], pages_per_gpu=sc["pages"],
                 io_capacity=sc["io_capacity"])
    try:
        for d in sc["deliveries"]:
            batch = tuple(range(d["batch"])) if d["kind"] == 3 else ()
            eng.submit(Action(d["action_id"], ActionKind(d["kind"]), d["model_id"], d["earliest"],
                              d["latest"], batch, d["gpu"]), at=d["t"])
        eng.sim_run(sc["horizon"])
        results = []
        while True:
            r = eng.poll(0)
            if not r:
                break
            results += [[a, s, st, en, du, free] for a, s, st, en, du, _ref, free, _k in r]
        final = []
        for g in range(sc["gpu_count"]):
            free, res = eng.pages(g)
            final.append([free, [list(x) for x in res]])
        return {"results": results, "final": final}
    finally:
        eng.close()


def run_oracle(sc: dict) -> dict:
    cat = catalog_mod.parse(sc["catalog"])
    profs = [worker_oracle.Profile(p.weights_bytes, p.weights_transfer_ns, dict(p.exec_ns),
                                   p.input_bytes, p.output_bytes, p.input_ns, p.output_ns)
             for p in cat.models]
    w = worker_oracle.OracleWorker(profs, sc["gpu_count"], sc["pages"], sc["io_capacity"],
                                   cat.page_bytes)
    for d in sc["deliveries"]:
        w.deliver(d["t"], worker_oracle.Act(d["action_id"], d["kind"], d["model_id"],
                                            d["earliest"], d["latest"], d["batch"], d["gpu"]))
    w.run_until(sc["horizon"])
    final = []
    for g in range(sc["gpu_count"]):
        free, held = w.pages_state(g)
        final.append([free, [list(x) for x in held]])
    return {"results": [list(r) for r in w.results], "final": final}


scenario = scenarios.scenario
