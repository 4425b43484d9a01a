"""Model catalog for the B200 worker: the reference's profile-file grammar
(pkg/src/sloserve/profiles.py:10-22) restated, so the worker reads the same
catalog files as the reference controller and assigns the same dense model ids.

    page_bytes <int>            optional header (default 16 MiB)
    model <name>                profile record
      weights_bytes <int>
      weights_transfer_ns <int>
      io_ns <in_ns> <out_ns>    default 50000 50000
      io_bytes <in_B> <out_B>   default 0 0
      batch <size> <exec_ns>    one per supported batch size
    replicas <name> <count>     <count> more ids sharing <name>'s profile

The worker consumes, per model id: the base name (which network / weights blob
it is), pages_needed = max(1, ceil(weights_bytes / page_bytes)) for bit-exact
page accounting (profiles.py:109-111), the supported batch sizes (MALFORMED
check, worker.py:206-208), the IO sizes for the IOCache gauge (worker.py:210),
and the profiled durations, which drive only the sim-mode device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

PAGE_BYTES = 16 * 1024 * 1024
IO_NS = 50_000


class CatalogError(ValueError):
    pass


@dataclass(frozen=True)
class Profile:
    name: str
    weights_bytes: int
    weights_transfer_ns: int
    exec_ns: dict                      # batch size -> ns
    input_bytes: int = 0
    output_bytes: int = 0
    input_ns: int = IO_NS
    output_ns: int = IO_NS

    @property
    def batch_sizes(self) -> tuple[int, ...]:
        return tuple(sorted(self.exec_ns))

    def pages(self, page_bytes: int) -> int:
        return max(1, math.ceil(self.weights_bytes / page_bytes))

    def check(self) -> None:
        bs = self.batch_sizes
        if self.weights_bytes <= 0 or self.weights_transfer_ns <= 0:
            raise CatalogError(f"{self.name}: weights size/transfer must be > 0")
        if self.input_ns <= 0 or self.output_ns <= 0 or self.input_bytes < 0 or self.output_bytes < 0:
            raise CatalogError(f"{self.name}: bad io fields")
        if not bs or bs[0] <= 0:
            raise CatalogError(f"{self.name}: batch sizes must be positive")
        for lo, hi in zip(bs, bs[1:]):
            a, b = self.exec_ns[lo], self.exec_ns[hi]
            if b < a or b * lo > a * hi:
                raise CatalogError(f"{self.name}: exec durations not monotone / "
                                   "per-request cost grows with batch size")
        if any(self.exec_ns[b] <= 0 for b in bs):
            raise CatalogError(f"{self.name}: exec durations must be > 0")


@dataclass
class Catalog:
    page_bytes: int = PAGE_BYTES
    models: list[Profile] = field(default_factory=list)   # index = model id
    base: list[str] = field(default_factory=list)          # base profile name per id

    def __len__(self) -> int:
        return len(self.models)

    def pages_needed(self, model_id: int) -> int:
        return self.models[model_id].pages(self.page_bytes)

    def has_model(self, model_id: int) -> bool:
        return 0 <= model_id < len(self.models)

    def model_ids(self) -> range:
        return range(len(self.models))

    def bases(self) -> list[str]:
        seen: dict[str, None] = {}
        for b in self.base:
            seen.setdefault(b, None)
        return list(seen)

    def replicate(self, name: str, copies: int) -> "Catalog":
        prof = next((p for p, b in zip(self.models, self.base) if b == name), None)
        if prof is None:
            raise CatalogError(f"unknown base model {name!r}")
        self.models += [prof] * copies
        self.base += [name] * copies
        return self


def parse(text: str) -> Catalog:
    cat = Catalog()
    named: dict[str, Profile] = {}
    rec: dict | None = None

    def close():
        nonlocal rec
        if rec is None:
            return
        for key in ("weights_bytes", "weights_transfer_ns"):
            if key not in rec:
                raise CatalogError(f"model {rec['name']!r} missing {key}")
        if not rec["batch"]:
            raise CatalogError(f"model {rec['name']!r} has no batch lines")
        io_ns = rec.get("io_ns", (IO_NS, IO_NS))
        io_b = rec.get("io_bytes", (0, 0))
        p = Profile(rec["name"], rec["weights_bytes"], rec["weights_transfer_ns"],
                    dict(rec["batch"]), io_b[0], io_b[1], io_ns[0], io_ns[1])
        if [b for b, _ in rec["batch"]] != sorted({b for b, _ in rec["batch"]}):
            raise CatalogError(f"{p.name}: batch sizes must be strictly increasing")
        p.check()
        if p.name in named:
            raise CatalogError(f"duplicate model name {p.name!r}")
        named[p.name] = p
        cat.models.append(p)
        cat.base.append(p.name)
        rec = None

    for n, raw in enumerate(text.splitlines(), 1):
        words = raw.split("#", 1)[0].split()
        if not words:
            continue
        key, args = words[0], words[1:]
        try:
            if key == "page_bytes":
                close()
                cat.page_bytes = int(args[0])
                if cat.page_bytes <= 0:
                    raise CatalogError("page_bytes must be > 0")
            elif key == "model":
                close()
                rec = {"name": args[0], "batch": []}
            elif key == "replicas":
                close()
                name, count = args[0], int(args[1])
                if name not in named or count < 0:
                    raise CatalogError(f"bad replicas line for {name!r}")
                cat.models += [named[name]] * count
                cat.base += [name] * count
            elif rec is None:
                raise CatalogError(f"{key} outside a model record")
            elif key in ("weights_bytes", "weights_transfer_ns"):
                rec[key] = int(args[0])
            elif key in ("io_ns", "io_bytes"):
                rec[key] = (int(args[0]), int(args[1]))
            elif key == "batch":
                rec["batch"].append((int(args[0]), int(args[1])))
            else:
                raise CatalogError(f"unknown directive {key!r}")
        except (IndexError, ValueError) as exc:
            raise CatalogError(f"line {n}: {exc}") from None
    close()
    return cat


def load(path: str) -> Catalog:
    with open(path, encoding="utf-8") as f:
        return parse(f.read())


def from_reference(ref_catalog) -> Catalog:
    """Adopt an already-parsed reference `ModelCatalog` (in-process drop-in)."""
    cat = Catalog(page_bytes=ref_catalog.page_size)
    for e in ref_catalog.entries:
        p = e.profile
        cat.models.append(Profile(p.model_name, p.weights_size, p.weights_transfer,
                                  dict(p.exec_duration), p.input_size, p.output_size,
                                  p.input_transfer, p.output_transfer))
        cat.base.append(e.replica_of)
    return cat


def dumps(cat: Catalog) -> str:
    """Canonical text (profile at first use, runs of copies as `replicas`)."""
    lines = [f"page_bytes {cat.page_bytes}"]
    seen: set[str] = set()
    i = 0
    while i < len(cat.models):
        name, p = cat.base[i], cat.models[i]
        if name not in seen:
            seen.add(name)
            lines += [f"model {name}", f"weights_bytes {p.weights_bytes}",
                      f"weights_transfer_ns {p.weights_transfer_ns}",
                      f"io_ns {p.input_ns} {p.output_ns}",
                      f"io_bytes {p.input_bytes} {p.output_bytes}"]
            lines += [f"batch {b} {p.exec_ns[b]}" for b in p.batch_sizes]
            i += 1
            continue
        j = i
        while j < len(cat.models) and cat.base[j] == name:
            j += 1
        lines.append(f"replicas {name} {j - i}")
        i = j
    return "\n".join(lines) + "\n"
