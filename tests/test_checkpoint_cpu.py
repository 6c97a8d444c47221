"""Checkpoint files (the GSPL f32 checkpoint writer and model.dogs).

The native codec (host/checkpoint_io.cpp through libbsgpu.so, no device needed) is
compared byte for byte with the oracle's restatement of scene_io.cpp
(oracle/scene_format.py), and given the malformed inputs of the reference's
own format tests (test_image_scene.cpp:170-240), each of which must raise
the same FormatErrorCode.
"""
import os
import struct
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import scene_format as sf  # noqa: E402
from paper_2405_13943_b200 import api  # noqa: E402


def random_cloud(n, fd, seed=0, start_id=0):
    g = np.random.default_rng(seed)
    ids = np.sort(g.choice(10 * n + 10, n, replace=False)).astype(np.uint64) + np.uint64(start_id)
    q = g.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return dict(ids=ids, pos=g.normal(size=(n, 3)) * 7.3, rot=q, ls=g.normal(size=(n, 3)) - 3.0,
                feat=g.uniform(-1, 1, size=(n, fd)), op=g.normal(size=n))


def sample_views():
    return [dict(id=3, fx=120.5, fy=121.25, cx=32.0, cy=24.0, width=64, height=48, q=(0.9, 0.1, -0.3, 0.2),
                 t=(0.5, -1.0, 4.0), path="gt/view_00003.ppm"),
            dict(id=7, fx=80.0, fy=80.0, cx=16.0, cy=16.0, width=32, height=32, q=(1.0, 0.0, 0.0, 0.0),
                 t=(0.0, 0.0, 0.0), path="")]


def sample_points():
    return [dict(pos=(0.25, -1.5, 3.0), rgb=(255, 0, 17)), dict(pos=(1e-3, 2.0, -7.0), rgb=(1, 2, 3))]


@pytest.fixture(scope="module", autouse=True)
def lib():
    api.load_library()


@pytest.mark.parametrize("fd", [3, 12])
def test_save_model_bytes_match_reference_layout(tmp_path, fd):
    c = random_cloud(257, fd, seed=fd)
    p = tmp_path / "model.dogs"
    api.save_model(str(p), c)
    assert p.read_bytes() == sf.encode_model(c)


@pytest.mark.parametrize("fd", [3, 12])
def test_load_checkpoint_is_exact_narrowing_and_reencode_is_identical(tmp_path, fd):
    c = random_cloud(100, fd, seed=10 + fd)
    p = tmp_path / "model.dogs"
    api.save_model(str(p), c)
    back = api.load_checkpoint(str(p))
    ref = sf.narrow(c)
    assert np.array_equal(back["ids"], c["ids"])
    for k in ("pos", "rot", "ls", "feat", "op"):
        assert np.array_equal(np.asarray(back[k]).reshape(-1), np.asarray(ref[k]).reshape(-1)), k
    # narrowing is idempotent: a second save is bit-identical (test_image_scene.cpp:159-162)
    p2 = tmp_path / "again.dogs"
    api.save_model(str(p2), back)
    assert p2.read_bytes() == p.read_bytes()


def test_decode_reads_checkpoint_past_cams_and_pnts_sections():
    c = random_cloud(33, 3, seed=5)
    data = sf.encode_scene(sample_views(), sample_points(), sf.narrow(c))
    back = api.decode_checkpoint(data)
    ref = sf.decode_checkpoint(data)
    assert np.array_equal(back["ids"], ref["ids"])
    for k in ("pos", "rot", "ls", "feat", "op"):
        assert np.array_equal(np.asarray(back[k]).reshape(-1), np.asarray(ref[k]).reshape(-1))


def test_empty_model_and_missing_checkpoint(tmp_path):
    empty = dict(ids=np.zeros(0, np.uint64), pos=np.zeros((0, 3)), rot=np.zeros((0, 4)), ls=np.zeros((0, 3)),
                 feat=np.zeros((0, 3)), op=np.zeros(0))
    p = tmp_path / "empty.dogs"
    api.save_model(str(p), empty)
    assert p.read_bytes() == sf.encode_model(empty)
    assert len(api.load_checkpoint(str(p))["ids"]) == 0
    with pytest.raises(api.InvalidArgument):
        api.decode_checkpoint(sf.encode_scene(sample_views(), sample_points(), None))


def malformed_cases():
    """The reference's malformed containers (test_image_scene.cpp:170-240)."""
    c = sf.narrow(random_cloud(6, 3, seed=2))
    good = sf.encode_scene(sample_views(), sample_points(), c)
    cases = {}
    b = bytearray(good); b[0] = ord("X"); cases["bad_magic"] = (bytes(b), "BadMagic")
    b = bytearray(good); b[4] += 1; cases["bad_version"] = (bytes(b), "UnsupportedVersion")
    b = bytearray(good); b[8] = ord("Z"); cases["unknown_tag"] = (bytes(b), "UnknownSection")
    cases["truncated"] = (good[:-3], "TruncatedSection")
    cases["trailing_byte"] = (good + b"\x00", "TruncatedBuffer")
    # duplicate: append a second copy of the GSPL section
    off, gspl = 8, None
    while off + 12 <= len(good):
        (ln,) = struct.unpack_from("<Q", good, off + 4)
        if good[off:off + 4] == b"GSPL":
            gspl = good[off:off + 12 + ln]
        off += 12 + ln
    cases["duplicate_gspl"] = (good + gspl, "BadHeader")
    cases["tiny"] = (b"DO", "TruncatedBuffer")
    swapped = dict(c)
    swapped["ids"] = c["ids"].copy()
    swapped["ids"][[0, 1]] = swapped["ids"][[1, 0]]
    cases["non_monotone_ids"] = (sf.encode_scene(checkpoint=swapped), "NonMonotoneIds")
    # feature width 5 and a count that cannot fit the payload
    g = bytearray(sf.encode_scene(checkpoint=c))
    gs = g.index(b"GSPL") + 12
    bad_fd = bytearray(g); struct.pack_into("<I", bad_fd, gs + 8, 5); cases["bad_feature_width"] = (bytes(bad_fd), "BadHeader")
    big = bytearray(g); struct.pack_into("<Q", big, gs, 1 << 40); cases["count_overflow"] = (bytes(big), "CountOverflow")
    # a section with bytes after its payload
    extra = sf.section(b"PNTS", sf.pnts_payload(sample_points()) + b"\x01")
    cases["section_trailing"] = (b"DOGS" + struct.pack("<I", 1) + extra, "TruncatedSection")
    return cases


@pytest.mark.parametrize("name", sorted(malformed_cases()))
def test_malformed_containers_raise_the_reference_code(name):
    data, code = malformed_cases()[name]
    with pytest.raises(sf.OracleFormatError) as ref:
        sf.decode_checkpoint(data)
    assert ref.value.code == code  # the oracle restates the reference
    with pytest.raises(api.FormatError) as e:
        api.decode_checkpoint(data)
    assert e.value.code == code
