"""Catalog grammar: same model ids, pages_needed and canonical text as the
reference parser (tests/golden/catalog.json; profiles.py:109-111, 284-312)."""

import json
import os

import pytest

from paper_2006_02464_b200 import catalog

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "catalog.json")))


def test_reference_catalog_pages_and_dump():
    cat = catalog.parse(G["text"]).replicate("resnet50", 3)
    assert [cat.pages_needed(m) for m in cat.model_ids()] == G["pages_needed"]
    assert cat.base == G["names"]
    assert catalog.dumps(cat) == G["dumps"]
    assert catalog.dumps(catalog.parse(G["dumps"])) == G["dumps"]


def test_spec_known_answers():
    cat = catalog.parse(G["text"])
    ids = {n: i for i, n in enumerate(cat.base)}
    assert cat.pages_needed(ids["resnet50"]) == 7      # SPEC.md:205 (102.3 MB / 16 MiB)
    assert cat.pages_needed(ids["resnet18"]) == 3
    assert cat.models[ids["resnet50"]].exec_ns[16] == 15_670_000


@pytest.mark.parametrize("text", [
    "model a\nweights_bytes 10\nweights_transfer_ns 5\nbatch 1 10\nbatch 2 9\n",    # decreasing
    "model a\nweights_bytes 10\nweights_transfer_ns 5\nbatch 1 10\nbatch 2 30\n",   # per-req worse
    "model a\nweights_bytes 10\nbatch 1 10\n",                                     # missing field
    "weights_bytes 10\n",                                                          # outside record
    "model a\nweights_bytes 10\nweights_transfer_ns 5\nbatch 1 10\nreplicas b 2\n",
    "page_bytes 0\n",
    "model a\nweights_bytes 10\nweights_transfer_ns 5\nbogus 1\n",
])
def test_invalid_catalogs_rejected(text):
    with pytest.raises(catalog.CatalogError):
        catalog.parse(text)
