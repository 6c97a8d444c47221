"""Host-side scene plumbing for the benchmark configurations (not the hot path).

`look_at` restates camera.hpp:42-58 (including the quaternion round trip of
math.hpp:48-69) so cameras built here are bit-identical to the reference's.
`aerial_scene` is the synthetic "Mill-19-like" generator of SURVEY §8(d)
(cfg 2-5): Gaussians uniform in the reference's 5:1:5 box (synth.cpp:27-28
proportions, rescaled), isotropic scales r = (E/sqrt(N)) U(0.3, 1),
features U(0.05, 0.95)/SH0, opacity logit(U(0.4, 0.9)) (synth.cpp:30-37
distributions), views on a jittered aerial grid at altitude 0.3E looking 5
degrees off nadir (never straight down: look_at degenerates, camera.hpp:45-46).
"""
import math

import numpy as np

SH0 = 0.28209479177387814


def _normalized(v):
    return v / math.sqrt(float((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]))


def quat_to_rotation(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def rotation_to_quat(r):
    t = (r[0, 0] + r[1, 1]) + r[2, 2]
    if t > 0.0:
        s = math.sqrt(t + 1.0) * 2.0
        q = [0.25 * s, (r[2, 1] - r[1, 2]) / s, (r[0, 2] - r[2, 0]) / s, (r[1, 0] - r[0, 1]) / s]
    elif r[0, 0] > r[1, 1] and r[0, 0] > r[2, 2]:
        s = math.sqrt(1.0 + r[0, 0] - r[1, 1] - r[2, 2]) * 2.0
        q = [(r[2, 1] - r[1, 2]) / s, 0.25 * s, (r[0, 1] + r[1, 0]) / s, (r[0, 2] + r[2, 0]) / s]
    elif r[1, 1] > r[2, 2]:
        s = math.sqrt(1.0 + r[1, 1] - r[0, 0] - r[2, 2]) * 2.0
        q = [(r[0, 2] - r[2, 0]) / s, (r[0, 1] + r[1, 0]) / s, 0.25 * s, (r[1, 2] + r[2, 1]) / s]
    else:
        s = math.sqrt(1.0 + r[2, 2] - r[0, 0] - r[1, 1]) * 2.0
        q = [(r[1, 0] - r[0, 1]) / s, (r[0, 2] + r[2, 0]) / s, (r[1, 2] + r[2, 1]) / s, 0.25 * s]
    n = math.sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3])
    q = [v / n for v in q] if n != 0 else [1.0, 0.0, 0.0, 0.0]
    return [-v for v in q] if q[0] < 0 else q


class Camera:
    """CameraView (camera.hpp:14-37)."""

    def __init__(self, fx, fy, cx, cy, q, t, width, height, view_id=0):
        self.fx, self.fy, self.cx, self.cy = float(fx), float(fy), float(cx), float(cy)
        self.q = list(q)
        self.R = quat_to_rotation(self.q)
        self.t = np.asarray(t, dtype=np.float64)
        self.width, self.height = int(width), int(height)
        self.view_id = view_id

    def center(self):
        R, t = self.R, self.t
        return np.array([-((R[0, k] * t[0] + R[1, k] * t[1]) + R[2, k] * t[2]) for k in range(3)])

    def device(self):
        from .api import make_camera
        return make_camera(self.fx, self.fy, self.cx, self.cy, self.R, self.t, self.width, self.height)


def look_at(position, target, world_up, fx, fy, cx, cy, width, height):
    """camera.hpp:42-58."""
    p = np.asarray(position, dtype=np.float64)
    forward = _normalized(np.asarray(target, dtype=np.float64) - p)
    right = _normalized(np.cross(forward, np.asarray(world_up, dtype=np.float64)))
    down = np.cross(forward, right)
    q = rotation_to_quat(np.stack([right, down, forward]))
    R = quat_to_rotation(q)
    t = np.array([-((R[i, 0] * p[0] + R[i, 1] * p[1]) + R[i, 2] * p[2]) for i in range(3)])
    return Camera(fx, fy, cx, cy, q, t, width, height)


def aerial_scene(n, width, height, n_views, extent, seed, sh_degree=0, tilt_deg=5.0):
    """Returns (cloud dict of numpy arrays, list of Camera).

    tilt_deg: angle of the optical axis off nadir. The reference culls only
    z <= near and empty rects (renderer.cpp:124,130-132; no frustum guard
    band), so a Gaussian lying near a camera's z = 0 plane projects to a
    footprint clamped to the whole image and composites first in every pixel.
    At 30 degrees the camera plane cuts the scene slab ~35 m away and such
    near-plane splats dominate every tile list (x30 pairs); at 5 degrees the
    plane clears the slab (min depth ~19 m), which is the drone-survey regime
    of Mill-19. The degenerate regime stays covered by the parity tests."""
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
    cloud = dict(ids=np.arange(n, dtype=np.uint64), pos=pos, rot=q, ls=ls, feat=feat, op=op)
    cams = []
    side = int(math.ceil(math.sqrt(n_views)))
    alt = 0.3 * extent
    f = 0.8 * width
    for v in range(n_views):
        gx, gz = v % side, v // side
        cx = -half + (gx + 0.5) * extent / side + g.uniform(-0.05, 0.05) * extent / side
        cz = -half + (gz + 0.5) * extent / side + g.uniform(-0.05, 0.05) * extent / side
        yaw = g.uniform(0, 2 * math.pi)
        d = alt * math.tan(math.radians(tilt_deg))
        target = [cx + d * math.cos(yaw), 0.0, cz + d * math.sin(yaw)]
        cam = look_at([cx, alt, cz], target, [0.0, 1.0, 0.0], f, f, width / 2, height / 2, width, height)
        cam.view_id = v
        cams.append(cam)
    return cloud, cams


def perturbed_init(cloud, seed, init_opacity=0.1):
    """Training start for a synthetic block: jittered positions, grey colour and
    the reference's initial opacity (trainer.hpp:57, init_cloud_from_points)."""
    g = np.random.default_rng(seed + 1)
    r = np.exp(cloud["ls"][:, 0])
    out = {k: v.copy() for k, v in cloud.items()}
    out["pos"] = cloud["pos"] + g.normal(size=cloud["pos"].shape) * r[:, None]
    out["feat"][:, :3] = 0.5 / SH0
    out["op"][:] = math.log(init_opacity / (1 - init_opacity))
    return out
