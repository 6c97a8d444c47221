"""Test fixtures restated from the reference's own unit tests.

Each builder cites the reference test helper it mirrors. Random fixtures draw
from the oracle's `Rng` (mt19937_64 with the reference's hand-rolled
distributions, math.hpp:74-135); multi-argument `Vec3(...)` constructors of rng
calls are drawn right to left, as GCC evaluates them (see oracle/orc.cpp).
"""
import math

import numpy as np

import _oracle as orc

SH0 = 0.28209479177387814


def logit(p):
    return math.log(p / (1.0 - p))


class HostCloud:
    """Plain numpy SoA cloud (ids ascending), convertible to oracle / device."""

    def __init__(self, ids, pos, rot, ls, feat, op):
        self.ids = np.ascontiguousarray(ids, dtype=np.uint64)
        self.pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        self.rot = np.ascontiguousarray(rot, dtype=np.float64).reshape(-1, 4)
        self.ls = np.ascontiguousarray(ls, dtype=np.float64).reshape(-1, 3)
        n = len(self.ids)
        self.feat = np.ascontiguousarray(feat, dtype=np.float64).reshape(n, -1) if n else np.zeros((0, 3))
        self.op = np.ascontiguousarray(op, dtype=np.float64).reshape(-1)

    @property
    def n(self):
        return len(self.ids)

    @property
    def fd(self):
        return self.feat.shape[1]

    def oracle(self):
        return orc.Cloud(self.ids, self.pos, self.rot, self.ls, self.feat, self.op)

    @staticmethod
    def from_oracle(c):
        d = c.dict()
        return HostCloud(d["ids"], d["pos"], d["rot"], d["ls"], d["feat"], d["op"])

    def narrowed(self):
        """Parameters rounded to f32 (the device storage type) and widened back."""
        f = lambda a: a.astype(np.float32).astype(np.float64)
        return HostCloud(self.ids, f(self.pos), f(self.rot), f(self.ls), f(self.feat), f(self.op))

    def copy(self):
        return HostCloud(self.ids.copy(), self.pos.copy(), self.rot.copy(), self.ls.copy(), self.feat.copy(), self.op.copy())


def empty_cloud(fd=3):
    return HostCloud(np.zeros(0, np.uint64), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros((0, fd)), np.zeros(0))


def axis_camera(f, c, size):
    """test_renderer.cpp:18-24: identity pose, camera at the origin."""
    cam = orc.Camera()
    cam.fx = cam.fy = f
    cam.cx = cam.cy = c
    cam.width = cam.height = size
    cam.set_rotation_quat([1.0, 0.0, 0.0, 0.0])
    cam.t = [0.0, 0.0, 0.0]
    return cam


def ref_camera(size=24):
    """test_renderer.cpp:55-58."""
    return orc.look_at([0.3, 0.4, -6.0], [0.05, -0.05, 0.0], [0.0, 1.0, 0.0], 1.1 * size, 1.1 * size,
                       size / 2.0, size / 2.0, size, size)


def splat_at(rows, gid, pos, rgb, opacity, log_scale=-1.0):
    """test_renderer.cpp:26-36 (appends one row to a list of tuples)."""
    rows.append((gid, list(pos), [1.0, 0.0, 0.0, 0.0], [log_scale] * 3, [c / SH0 for c in rgb], logit(opacity)))


def cloud_from_rows(rows, fd=3):
    if not rows:
        return empty_cloud(fd)
    ids, pos, rot, ls, feat, op = zip(*rows)
    return HostCloud(np.array(ids, np.uint64), np.array(pos), np.array(rot), np.array(ls), np.array(feat), np.array(op))


def _vec3_rtl(f):
    z = f()
    y = f()
    x = f()
    return [x, y, z]


def random_cloud(n, seed, spread=1.5):
    """test_renderer.cpp:38-53."""
    rng = orc.Rng(seed)
    rows = []
    for i in range(n):
        pos = _vec3_rtl(lambda: rng.uniform_range(-spread, spread))
        q = rng.random_unit_quat()
        ls = _vec3_rtl(lambda: rng.uniform_range(-2.5, -0.8))
        feat = [rng.uniform_range(0, 3) for _ in range(3)]
        op = rng.uniform_range(-1.5, 2.0)
        rows.append((i, pos, q, ls, feat, op))
    return cloud_from_rows(rows)


def grad_check_cloud(rng):
    """acceptance_main.cpp:51-65."""
    rows = []
    for i in range(8):
        z = rng.uniform_range(-1.0, 1.0)
        y = rng.uniform_range(-1.2, 1.2)
        x = rng.uniform_range(-1.2, 1.2)
        q = rng.random_unit_quat()
        ls = _vec3_rtl(lambda: rng.uniform_range(-2.5, -0.8))
        feat = [rng.uniform_range(0, 3) for _ in range(3)]
        op = rng.uniform_range(-1.5, 2.0)
        rows.append((i, [x, y, z], q, ls, feat, op))
    return cloud_from_rows(rows)


def random_bundle(ids, seed):
    """test_admm.cpp:26-40."""
    rng = orc.Rng(seed)
    rows = []
    for gid in ids:
        pos = _vec3_rtl(rng.normal)
        q = rng.random_unit_quat()
        ls = _vec3_rtl(rng.normal)
        feat = [rng.normal() for _ in range(3)]
        op = rng.normal()
        rows.append((gid, pos, q, ls, feat, op))
    return cloud_from_rows(rows)


def scalar_cloud(gid, opacity_value):
    """test_admm.cpp:15-24: only the opacity logit is non-zero."""
    return cloud_from_rows([(gid, [0, 0, 0], [1.0, 0, 0, 0], [0, 0, 0], [0, 0, 0], opacity_value)])


def random_image(w, h, seed):
    """test_ssim.cpp:53-58."""
    rng = orc.Rng(seed)
    return np.array([rng.uniform() for _ in range(3 * w * h)]).reshape(h, w, 3)


def aerial_scene(n, width, height, n_views, extent, seed, sh_degree=0):
    """Synthetic Mill-19-like block (SURVEY §8(d) cfg 2-5): uniform positions in
    the reference's 5:1:5 box, isotropic scales r = (E/sqrt(N))*U(0.3,1),
    features U(0.05,0.95)/SH0, opacity logit(U(0.4,0.9)), cameras on a jittered
    aerial grid at altitude 0.3E tilted ~30 degrees. Vectorised numpy (seeded);
    not a reference fixture, so no Rng stream parity is needed."""
    g = np.random.default_rng(seed)
    half = extent / 2
    pos = np.stack([g.uniform(-half, half, n), g.uniform(-half / 5, half / 5, n), g.uniform(-half, half, n)], 1)
    q = g.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1
    r = (extent / math.sqrt(n)) * g.uniform(0.3, 1.0, n)
    ls = np.repeat(np.log(r)[:, None], 3, 1)
    fd = 12 if sh_degree >= 1 else 3
    feat = np.zeros((n, fd))
    feat[:, :3] = g.uniform(0.05, 0.95, (n, 3)) / SH0
    op = np.log(1 / (1 / g.uniform(0.4, 0.9, n) - 1))
    cloud = HostCloud(np.arange(n, dtype=np.uint64), pos, q, ls, feat, op)
    cams = []
    side = int(math.ceil(math.sqrt(n_views)))
    alt = 0.3 * extent
    f = 0.8 * width
    for v in range(n_views):
        gx, gz = v % side, v // side
        cx = -half + (gx + 0.5) * extent / side + g.uniform(-0.05, 0.05) * extent / side
        cz = -half + (gz + 0.5) * extent / side + g.uniform(-0.05, 0.05) * extent / side
        yaw = g.uniform(0, 2 * math.pi)
        d = alt * math.tan(math.radians(30))
        target = [cx + d * math.cos(yaw), 0.0, cz + d * math.sin(yaw)]
        cam = orc.look_at([cx, alt, cz], target, [0.0, 1.0, 0.0], f, f, width / 2, height / 2, width, height)
        cam.view_id = v
        cams.append(cam)
    return cloud, cams


def dapprox(a, b, eps):
    """doctest::Approx(b).epsilon(eps) == a  (scale 1): |a-b| < eps*(1+max(|a|,|b|))."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))
