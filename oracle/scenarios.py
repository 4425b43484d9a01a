"""Seeded action-sequence scenarios for worker-semantics parity — TEST INFRASTRUCTURE.

Each scenario is a catalog, a worker shape (GPUs, pages, IOCache bytes) and a
list of (delivery time, action) pairs covering every branch of the reference
executor: MALFORMED (unknown model / GPU / batch size), tight and missed
windows, IOCache blocking, OUT_OF_PAGES, MODEL_NOT_LOADED, LOAD of a resident
model, UNLOAD idempotence, and executor ordering by `earliest`.
"""

from __future__ import annotations

import random

MS = 1_000_000

BASE_CATALOG = """\
page_bytes 16777216
model resnet18
weights_bytes 46700000
weights_transfer_ns 3810000
io_ns 50000 50000
io_bytes 602000 4000
batch 1 1270000
batch 2 1860000
batch 4 2730000
batch 8 4060000
batch 16 7020000
model resnet50
weights_bytes 102300000
weights_transfer_ns 8330000
io_ns 50000 50000
io_bytes 602000 4000
batch 1 2610000
batch 2 3780000
batch 4 5610000
batch 8 9130000
batch 16 15670000
"""


def scenario(seed: int) -> dict:
    rng = random.Random(seed)
    copies = rng.randint(1, 5)
    catalog = BASE_CATALOG + f"replicas resnet50 {copies}\n"
    n_models = 2 + copies
    gpu_count = rng.choice([1, 1, 2])
    pages = rng.randint(4, 40)
    io_capacity = rng.choice([512 * 1024 * 1024, 20 * 606000, 5 * 606000])
    n_actions = rng.randint(10, 150)
    t = 0
    deliveries = []
    for i in range(n_actions):
        t += rng.choice([0, 0, 50_000, 300_000, 1 * MS, 3 * MS])
        r = rng.random()
        kind = 3 if r < 0.6 else (1 if r < 0.85 else 2)
        model = rng.randrange(n_models)
        if rng.random() < 0.03:
            model = n_models + rng.randrange(3)
        gpu = rng.randrange(gpu_count)
        if rng.random() < 0.03:
            gpu = gpu_count
        earliest = max(0, t + rng.choice([-MS, 0, 0, 200_000, 2 * MS, 5 * MS]))
        latest = earliest + rng.choice([0, 500_000, 2 * MS, 10 * MS, 40 * MS, 1000 * MS])
        batch = 0
        if kind == 3:
            batch = rng.choice([1, 2, 4, 8, 16, 16, 3] if rng.random() < 0.05 else
                               [1, 2, 4, 8, 16])
        deliveries.append(dict(t=t, action_id=1000 + i, kind=kind, model_id=model, gpu=gpu,
                               earliest=earliest, latest=latest, batch=batch))
    return dict(seed=seed, catalog=catalog, gpu_count=gpu_count, pages=pages,
                io_capacity=io_capacity, deliveries=deliveries, horizon=t + 10_000 * MS)
