import sys, os
sys.path[:0] = ['/root/repo', '/root/repo/tests', '/root/repo/oracle']
import numpy as np
import _oracle as orc
from gpu_helpers import dev_cam, new_block
from test_gpu_raster import CASES, grad_close
name, cloud, cam = [c for c in CASES if c[0] == 'aerial0'][0]
rng = np.random.default_rng(3)
gt = rng.uniform(0, 1, (cam.height, cam.width, 3))
want = orc.render_backward(cloud.oracle(), cam, gt, orc.RenderConfig())
proj = orc.project(cloud.oracle(), cam, orc.RenderConfig())
grazing = proj["visible"].astype(bool) & (proj["depth"] < 1.0)
print("grazing splats:", grazing.sum())
b = new_block(cloud)
for it in range(10):
    got = b.render_backward(dev_cam(cam), gt)
    e = grad_close({k: (v[grazing] if k.startswith("g_") else v) for k, v in got.items()},
                   {k: (v[grazing] if k.startswith("g_") else v) for k, v in want.items()}, 1e-3)
    e2 = grad_close({k: (v[~grazing] if k.startswith("g_") else v) for k, v in got.items()},
                   {k: (v[~grazing] if k.startswith("g_") else v) for k, v in want.items()}, 1e-3)
    print({k: round(v, 4) for k, v in e.items()}, {k: round(v, 6) for k, v in e2.items()})
