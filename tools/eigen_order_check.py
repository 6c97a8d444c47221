"""How much the integer contract depends on the FP64 summation order of the
reference's Eigen expressions.

The oracle and the device evaluate 3-term sums left to right, (e0+e1)+e2, and
the quaternion norm as ((w2+x2)+y2)+z2. Eigen's completely unrolled,
non-vectorised redux splits the range in halves: e0+(e1+e2) for 3 terms,
(e0+e1)+(e2+e3) for 4; its vectorised paths (SSE2 packets of two doubles)
give (e0+e1)+e2 again -- which one a given expression takes depends on the
Eigen version, the flags and the expression's storage order, and no Eigen is
installed here to settle it. This tool evaluates the projection of
renderer.cpp:121-134 / cloud.cpp:162-167 (camera.hpp:23-36) vectorised in
numpy FP64 (no FMA, like the oracle's -ffp-contract=off) under both orders
on the bench's scenes, and counts how many of the integer outputs differ:
visibility, footprint rects, the (depth, index) compositing order -- and,
for scale, how many FP64 depths differ in their last bits.

usage: python tools/eigen_order_check.py [--out profiles/eigen_order_check.json]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_13943_b200.scene import aerial_scene  # noqa: E402


def s3(a, b, c, order):
    return (a + b) + c if order == "left" else a + (b + c)


def s4(a, b, c, d, order):
    return ((a + b) + c) + d if order == "left" else (a + b) + (c + d)


def project(cl, cam, order, near=0.01, dil=0.3, ext=3.0):
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # the device's FP32 storage
    p, q, ls = f32(cl["pos"]), f32(cl["rot"]), f32(cl["ls"])
    R, t = np.asarray(cam.R, np.float64), np.asarray(cam.t, np.float64)
    pc = [s3(R[r, 0] * p[:, 0], R[r, 1] * p[:, 1], R[r, 2] * p[:, 2], order) + t[r] for r in range(3)]
    z = pc[2]
    qn = np.sqrt(s4(q[:, 0] ** 2, q[:, 1] ** 2, q[:, 2] ** 2, q[:, 3] ** 2, order))
    w, x, y, zq = (q[:, k] / qn for k in range(4))
    Rq = [[1 - 2 * (y * y + zq * zq), 2 * (x * y - w * zq), 2 * (x * zq + w * y)],
          [2 * (x * y + w * zq), 1 - 2 * (x * x + zq * zq), 2 * (y * zq - w * x)],
          [2 * (x * zq - w * y), 2 * (y * zq + w * x), 1 - 2 * (x * x + y * y)]]
    s = np.exp(ls)
    M = [[Rq[a][b] * s[:, b] for b in range(3)] for a in range(3)]
    S = [[s3(M[a][0] * M[b][0], M[a][1] * M[b][1], M[a][2] * M[b][2], order) for b in range(3)] for a in range(3)]
    mx = cam.fx * pc[0] / z + cam.cx
    my = cam.fy * pc[1] / z + cam.cy
    iz = 1.0 / z
    iz2 = iz * iz
    J = [[cam.fx * iz, 0.0 * iz, -cam.fx * pc[0] * iz2], [0.0 * iz, cam.fy * iz, -cam.fy * pc[1] * iz2]]
    A = [[s3(J[r][0] * R[0, k], J[r][1] * R[1, k], J[r][2] * R[2, k], order) for k in range(3)] for r in range(2)]
    T = [[s3(A[r][0] * S[0][k], A[r][1] * S[1][k], A[r][2] * S[2][k], order) for k in range(3)] for r in range(2)]
    C = [[s3(T[r][0] * A[c][0], T[r][1] * A[c][1], T[r][2] * A[c][2], order) + (dil if r == c else 0.0)
          for c in range(2)] for r in range(2)]
    mid = 0.5 * (C[0][0] + C[1][1])
    det = C[0][0] * C[1][1] - C[0][1] * C[1][0]
    lam = mid + np.sqrt(np.maximum(0.0, mid * mid - det))
    rad = ext * np.sqrt(lam)
    with np.errstate(all="ignore"):
        x0 = np.maximum(0, np.clip(np.ceil(mx - rad), -2 ** 30, 2 ** 30)).astype(np.int64)
        x1 = np.minimum(cam.width - 1, np.clip(np.floor(mx + rad), -2 ** 30, 2 ** 30)).astype(np.int64)
        y0 = np.maximum(0, np.clip(np.ceil(my - rad), -2 ** 30, 2 ** 30)).astype(np.int64)
        y1 = np.minimum(cam.height - 1, np.clip(np.floor(my + rad), -2 ** 30, 2 ** 30)).astype(np.int64)
    vis = (z > near) & (x0 <= x1) & (y0 <= y1)
    rect = np.stack([x0, x1, y0, y1], 1)
    idx = np.nonzero(vis)[0]
    order_idx = idx[np.lexsort((idx, z[idx]))]
    return vis, rect, z, order_idx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "eigen_order_check.json"))
    args = ap.parse_args()
    rows = []
    for name, n, w, h, views, tilt in (("cfg2", 2_000_000, 1024, 768, 4, 5.0), ("cfg2_tilt30", 2_000_000, 1024, 768, 4, 30.0),
                                       ("cfg3", 6_000_000, 1600, 1066, 2, 5.0)):
        cloud, cams = aerial_scene(n, w, h, 64 if name.startswith("cfg2") else 96, 100.0, 42, tilt_deg=tilt)
        for v in range(views):
            cam = cams[v]
            va, ra, za, oa = project(cloud, cam, "left")
            vb, rb, zb, ob = project(cloud, cam, "eigen")
            both = va & vb
            r = {"scene": name, "view": v, "gaussians": n, "visible": int(va.sum()),
                 "visibility_differs": int((va != vb).sum()),
                 "rects_differ": int((ra[both] != rb[both]).any(1).sum()),
                 "depth_bits_differ": int((za[both].view(np.uint64) != zb[both].view(np.uint64)).sum()),
                 "order_positions_differ": int((oa != ob).sum()) if len(oa) == len(ob) else None}
            rows.append(r)
            print(json.dumps(r), flush=True)
    doc = {"what": "integer outputs of the projection under (e0+e1)+e2 (oracle, device) vs Eigen's unrolled "
                   "e0+(e1+e2) / (e0+e1)+(e2+e3) summation, FP64 numpy, FP32-stored parameters", "rows": rows}
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
