"""Acceptance criterion 1 (acceptance_main.cpp:67-129) through the device:
prints, for every checked parameter, the device gradient, the FP64 central
differences at h = 1e-5, 1e-6, 1e-7 and whether the reference's rule
(err <= 1e-6 or rel <= 1e-3 at some h) holds. Diagnostic for the FD test."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    sys.path.insert(0, p)
import _oracle as orc  # noqa: E402
from gpu_helpers import dev_cam, new_block  # noqa: E402
from refcases import grad_check_cloud  # noqa: E402

rows = []
for s in range(50):
    rng = orc.Rng(1000 + s)
    c = grad_check_cloud(rng).narrowed()
    ez = 5.5
    ey = rng.uniform_range(-0.5, 0.5)
    ex = rng.uniform_range(-0.5, 0.5)
    cam = orc.look_at([ex, ey, ez], [0, 0, 0], [0, 1, 0], 14, 14, 8, 8, 16, 16)
    gt = np.array([rng.uniform() for _ in range(16 * 16 * 3)]).reshape(16, 16, 3)
    got = new_block(c).render_backward(dev_cam(cam), gt)
    want = orc.render_backward(c.oracle(), cam, gt, orc.RenderConfig())
    for name, gname in (("pos", "g_pos"), ("rot", "g_rot"), ("ls", "g_ls"), ("feat", "g_feat"), ("op", "g_op")):
        arr = getattr(c, name)
        for idx in np.ndindex(arr.shape):
            fds = []
            for h in (1e-5, 1e-6, 1e-7):
                up, dn = c.copy(), c.copy()
                getattr(up, name)[idx] += h
                getattr(dn, name)[idx] -= h
                fds.append((orc.loss_value(orc.render(up.oracle(), cam, orc.RenderConfig())[0], gt, 0.2) -
                            orc.loss_value(orc.render(dn.oracle(), cam, orc.RenderConfig())[0], gt, 0.2)) / (2 * h))
            g = float(got[gname][idx])
            w = float(want[gname][idx])
            rows.append(dict(seed=s, p=name, idx=[int(i) for i in idx], g=g, g64=w, fd=fds))
print(json.dumps(rows))
