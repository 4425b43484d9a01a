"""Model artifacts (.cwm, artifact.py): the blob a LOAD copies, its page map and arch name
round-trip through a file bit for bit; a torchvision-named state dict packs to the same
blob the worker builds from the same parameters; damaged files are refused."""

import os

import numpy as np
import pytest

from paper_2006_02464_b200 import arch, artifact, cli


@pytest.fixture(scope="module")
def r18():
    spec = arch.build_arch("resnet18")
    params = arch.make_params(spec, seed=3)
    return spec, params, arch.pack_blob(spec, arch.fold(spec, params))


def test_round_trip(r18, tmp_path):
    spec, params, blob = r18
    p = str(tmp_path / "m.cwm")
    artifact.save(p, "resnet18", blob)
    name, b2 = artifact.load(p)
    assert name == "resnet18" and b2.pages == blob.pages and b2.page_bytes == blob.page_bytes
    assert b2.locs == [tuple(l) for l in blob.locs]
    assert np.array_equal(b2.data, blob.data)


def test_state_dict_packs_like_the_worker(r18):
    spec, params, blob = r18
    b2 = artifact.from_state_dict("resnet18", params)
    assert np.array_equal(b2.data, blob.data) and b2.locs == blob.locs


def test_missing_tensor_refused(r18):
    _, params, _ = r18
    sd = dict(params)
    sd.pop("layer2.0.bn1.running_var")
    with pytest.raises(artifact.ArtifactError, match="running_var"):
        artifact.from_state_dict("resnet18", sd)


def test_damaged_files_refused(r18, tmp_path):
    _, _, blob = r18
    p = str(tmp_path / "m.cwm")
    artifact.save(p, "resnet18", blob)
    raw = bytearray(open(p, "rb").read())
    bad = bytearray(raw)
    bad[-100] ^= 0xFF
    open(p, "wb").write(bytes(bad))
    with pytest.raises(artifact.ArtifactError, match="checksum"):
        artifact.load(p)
    open(p, "wb").write(bytes(raw[:-1000]))
    with pytest.raises(artifact.ArtifactError, match="truncated"):
        artifact.load(p)
    open(p, "wb").write(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(artifact.ArtifactError, match="not a CWM1"):
        artifact.load(p)


def test_cli_pack_from_npz(r18, tmp_path):
    spec, params, blob = r18
    npz = str(tmp_path / "sd.npz")
    np.savez(npz, **params)
    out = str(tmp_path / "resnet18.cwm")
    assert cli.main(["pack", "--arch", "resnet18", "--state-dict", npz, "--out", out]) == 0
    name, b2 = artifact.load(out)
    assert name == "resnet18" and np.array_equal(b2.data, blob.data)
    assert os.path.getsize(out) >= blob.data.size
