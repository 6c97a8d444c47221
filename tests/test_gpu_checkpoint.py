"""GPU: the device GSPL checkpoint encoder (bsg_encode_gspl, csrc/checkpoint.cu)
against the oracle's restatement of scene_io.cpp:48-59, byte for byte, for a
freshly uploaded cloud, after training steps, after densification (rows
added / removed) and at the bench scale; and the model.dogs of run_simulated."""
import os
import struct
import sys

import numpy as np
import pytest

from gpu_helpers import dev_cam, gpu, new_block
from paper_2405_13943_b200 import api
from refcases import HostCloud

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import scene_format as sf  # noqa: E402

pytestmark = gpu


def _dict(c):
    return dict(ids=c["ids"], pos=c["pos"], rot=c["rot"], ls=c["ls"], feat=c["feat"], op=c["op"])


def _random_cloud(n, fd, seed):
    g = np.random.default_rng(seed)
    q = g.normal(size=(n, 4))
    ids = np.sort(g.choice(5 * n, n, replace=False)).astype(np.uint64)
    return HostCloud(ids, g.normal(size=(n, 3)) * 3, q / np.linalg.norm(q, axis=1, keepdims=True),
                     g.normal(size=(n, 3)) - 2, g.uniform(-1, 1, size=(n, fd)), g.normal(size=n))


@pytest.mark.parametrize("fd", [3, 12])
def test_device_gspl_equals_reference_encoding_of_narrowed_cloud(fd):
    hc = _random_cloud(301, fd, fd)
    b = new_block(hc)
    got = b.encode_gspl()
    want = sf.gspl_payload(sf.narrow(dict(ids=hc.ids, pos=hc.pos, rot=hc.rot, ls=hc.ls, feat=hc.feat, op=hc.op)))
    assert got == want
    b.close()


def test_device_gspl_after_training_and_densify():
    import _oracle as orc
    from test_gpu_train import toy_scene
    s, init = toy_scene(seed=4, gaussians=60)
    b = new_block(init)
    b.set_views([dev_cam(v) for v in s.views], s.images())
    b.trainer_init(api.trainer_config(iterations=40, densify={"enabled": 1, "interval": 10, "stop_iteration": 40,
                                                              "grad_threshold": 1e-7}))
    b.train_steps(orc.view_sequence(1, 0, len(s.views), 25))
    c = b.download_cloud()
    got = b.encode_gspl()
    assert got == sf.gspl_payload(_dict(c))  # device values are f32: narrowing is the identity
    n, fd = struct.unpack_from("<QI", got)
    assert n == len(c["ids"]) and fd == 3
    b.close()


def test_device_gspl_bench_scale_roundtrip(tmp_path):
    """2M rows (BASELINE configs[1] size): device encoding == host encoding of
    the downloaded cloud, and the written model decodes back exactly."""
    g = np.random.default_rng(9)
    n = 2_000_000
    b = api.Block(0, 3)
    ids = np.arange(n, dtype=np.uint64) * np.uint64(3)
    q = g.normal(size=(n, 4))
    b.upload_cloud(ids, g.normal(size=(n, 3)) * 50, q / np.linalg.norm(q, axis=1, keepdims=True),
                   g.normal(size=(n, 3)) - 2, g.uniform(size=(n, 3)), g.normal(size=n))
    got = b.encode_gspl()
    c = b.download_cloud()
    assert got == sf.gspl_payload(_dict(c))
    p = tmp_path / "model.dogs"
    api.save_model(str(p), c)
    data = p.read_bytes()
    assert data[-len(got):] == got  # the GSPL section is the container's last
    back = api.load_checkpoint(str(p))
    assert np.array_equal(back["ids"], c["ids"]) and np.array_equal(back["op"], c["op"])
    b.close()


def test_run_simulated_model_roundtrips_through_model_dogs(tmp_path):
    from test_gpu_distributed import desk_scene, run_both
    s, init = desk_scene()
    _, _, model, _ = run_both(s, init, 2, 20, 10, 1.6)
    p = tmp_path / "model.dogs"
    api.save_model(str(p), model)
    assert p.read_bytes() == sf.encode_model(model)
    back = api.load_checkpoint(str(p))
    ref = sf.narrow(model)
    for k in ("pos", "rot", "ls", "feat", "op"):
        assert np.array_equal(np.asarray(back[k]).reshape(-1), np.asarray(ref[k]).reshape(-1))
