"""The native host planner (libbsgpu.so, host/plan.cpp) against the oracle's
split_recursive + expand_and_assign (splitter.cpp:48-201): block membership,
shared sets, view assignment and boxes must be bit-exact (north star). CPU only."""
import numpy as np
import pytest

import _oracle as orc
from paper_2405_13943_b200 import api
from paper_2405_13943_b200.scene import aerial_scene, look_at
from refcases import HostCloud


def oracle_partition(cloud, cams, k, scale):
    return orc.split_and_assign(cloud.pos, k, cams, cloud.oracle(), scale, 1, False)


def to_oracle_cam(c):
    oc = orc.look_at([0, 5, 0], [0, 0, 1], [0, 1, 0], 1, 1, 0, 0, 2, 2)  # placeholder, overwritten below
    oc.fx, oc.fy, oc.cx, oc.cy = c.fx, c.fy, c.cx, c.cy
    oc.set_rotation_quat(list(c.q))
    oc.t = list(c.t)
    oc.width, oc.height = c.width, c.height
    return oc


@pytest.mark.parametrize("n,k,scale", [(1000, 2, 1.4), (5000, 4, 1.4), (20000, 8, 1.4), (20000, 8, 2.0), (3000, 3, 1.0)])
def test_planner_bit_exact(n, k, scale):
    cloud, cams = aerial_scene(n, 64, 48, 16, 100.0, seed=n + k)
    hc = HostCloud(cloud["ids"], cloud["pos"], cloud["rot"], cloud["ls"], cloud["feat"], cloud["op"])
    ocams = [to_oracle_cam(c) for c in cams]
    centers = np.array([c.center() for c in cams])
    np.testing.assert_array_equal(centers, np.array([oc.center() for oc in ocams]))
    plan = api.Plan(hc.ids, hc.pos, centers, k, scale)
    want = oracle_partition(hc, ocams, k, scale)
    boxes = plan.boxes()
    for key in ("core_min", "core_max", "exp_min", "exp_max"):
        np.testing.assert_array_equal(boxes[key], want[key])
    for b in range(k):
        ids, views = plan.block(b)
        assert list(ids) == list(want["block_gaussians"][b])
        assert list(views) == list(want["block_views"][b])
    sids, cnt, first = plan.shared()
    assert list(sids) == sorted(want["shared"].keys())
    for s, gid in enumerate(sids):
        owners = want["shared"][int(gid)]
        assert cnt[s] == len(owners) and first[s] == owners[0]
    # per-block slot tables
    for b in range(k):
        ids, _ = plan.block(b)
        rows, slots, fo = plan.block_shared(b)
        assert np.all(sids[slots] == ids[rows])
        assert np.all(fo == (first[slots] == b))


def test_planner_rejects_bad_input():
    with pytest.raises(api.InvalidArgument):
        api.Plan(np.arange(3, dtype=np.uint64), np.zeros((3, 3)), np.zeros((0, 3)), 4, 1.4)
    with pytest.raises(api.InvalidArgument):
        api.Plan(np.arange(3, dtype=np.uint64), np.zeros((3, 3)), np.zeros((0, 3)), 2, 0.5)


def test_look_at_matches_oracle():
    c = look_at([3.0, 30.0, -2.0], [5.0, 0.0, 1.0], [0, 1, 0], 800, 800, 512, 384, 1024, 768)
    o = orc.look_at([3.0, 30.0, -2.0], [5.0, 0.0, 1.0], [0, 1, 0], 800, 800, 512, 384, 1024, 768)
    assert list(c.q) == list(o.q)
    np.testing.assert_array_equal(c.R, o.R)
    np.testing.assert_array_equal(c.t, np.array(o.t))


def desk_scene():
    from refcases import HostCloud as HC
    sc = orc.SynthConfig()
    sc.seed, sc.gaussians, sc.cameras, sc.image_size, sc.extent = 42, 200, 24, 96, 10.0
    s = orc.generate_scene(sc)
    p, c = s.points()
    init = HC.from_oracle(orc.init_cloud_from_points(p, c, 0, 0.1)).narrowed()
    s.has_checkpoint = True
    s.checkpoint = init.oracle()
    return s, init


def test_planner_matches_oracle_plan():
    s, init = desk_scene()
    tc = orc.TrainerConfig()
    plan = orc.plan_cluster(s, 4, 1.4, 8, tc)
    centers = np.array([v.center() for v in s.views])
    p = api.Plan(init.ids, init.pos, centers, 4, 1.4)
    for b in range(4):
        ids, views = p.block(b)
        assert list(ids) == plan.shard_ids(b)
        assert [v for v in views if v % 8 != 0] == plan.shard_views(b)
        rows, slots, first = p.block_shared(b)
        sids, _, _ = p.shared()
        assert list(sids[slots]) == plan.shard_shared(b)


@pytest.mark.parametrize("seed,block,n_views,steps", [(1, 0, 6, 20), (7, 3, 28, 100), (42, 1, 1, 5),
                                                      (123456789, 7, 64, 300), (0, 31, 96, 200)])
def test_host_trainer_view_order_matches_reference(seed, block, n_views, steps):
    """S20 (trainer.cpp:116-118,250-252): the C++ host BlockTrainer's view
    order (bsg_view_sequence runs the trainer's own draw_views) against the
    oracle's Rng::shuffle restatement, and that against the oracle
    BlockTrainer's actual train_step draws."""
    got = list(api.view_sequence(seed, block, n_views, steps))
    assert got == list(orc.view_sequence(seed, block, n_views, steps))


def test_oracle_trainer_draws_the_restated_sequence():
    sc = orc.SynthConfig()
    sc.seed, sc.gaussians, sc.cameras, sc.image_size, sc.extent = 3, 30, 5, 16, 4.0
    s = orc.generate_scene(sc)
    p, c = s.points()
    init = orc.init_cloud_from_points(p, c, 0, 0.1)
    tc = orc.TrainerConfig()
    tc.iterations, tc.seed = 20, 11
    tc.densify_enabled = False
    t = orc.BlockTrainer(2, init, s.views, s.images(), [], init.size(), tc)
    seq = list(api.view_sequence(11, 2, len(s.views), 12))
    for k in range(12):
        t.train_step()
        assert t.last_view() == seq[k]


def test_view_sequence_rejects_empty_views():
    with pytest.raises(api.InvalidArgument):
        api.view_sequence(1, 0, 0, 3)
