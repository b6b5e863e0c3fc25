"""Generates the committed golden fixtures from the ORACLE (the unmodified reference sources
compiled with the Philox RNG seam, oracle/Makefile). Run in the build container, where
/root/reference exists:

    python tests/golden/make_golden.py

Fixtures (small, deterministic):
  traversal_c1.npz   10,000 rays on the C1 scene (camera + surface-origin rays):
                     Scene::intersect primitive ids and hit t (proj/src/scene.cpp:127-168)
  bdpt_caustic.npz   render_bdpt (unmodified reference) of the 12x12 caustic box, 3 spp, seed 11
  proxy_caustic.npz  restated render_proxy_bdpt loop: per-pass per-pixel values, pool entries
                     and reciprocal estimates of the 12x12 caustic box, 3 passes, seed 5
  recip_twopoint.npz reciprocal estimator on the reference's two-point fixture, B = 6 and 1.9
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle as orc  # noqa: E402
from paper_2503_23412_b200 import scenes  # noqa: E402

PROXY_PARAMS = {"pretrace_paths": 2000, "light_walks": 2000}


def camera_rays(sc, n, rng):
    cam = sc.camera
    pos = np.array(cam.position)
    fwd = np.array(cam.look_at) - pos
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, cam.up)
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    th = np.tan(np.radians(cam.fov_y) / 2)
    sx = (2 * rng.random(n) - 1) * th * cam.width / cam.height
    sy = (1 - 2 * rng.random(n)) * th
    d = fwd + sx[:, None] * right + sy[:, None] * up
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([np.broadcast_to(pos, (n, 3)), d], axis=1)


def main():
    rng = np.random.default_rng(2024)
    c1 = scenes.cornell_c1(64)
    o = orc.OracleScene(c1.to_json())
    r0 = camera_rays(c1, 5000, rng)
    p0, t0 = o.intersect(r0)
    ok = p0 >= 0
    pts = r0[ok, :3] + t0[ok, None] * r0[ok, 3:]
    d = rng.normal(size=pts.shape)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = np.concatenate([r0, np.concatenate([pts, d], axis=1)[:5000]])
    prim, t = o.intersect(rays)
    np.savez_compressed(os.path.join(HERE, "traversal_c1.npz"), rays=rays, prim=prim, t=t)

    cb = scenes.caustic_box(12)
    ob = orc.OracleScene(cb.to_json())
    np.savez_compressed(os.path.join(HERE, "bdpt_caustic.npz"), image=ob.render_bdpt(3, 11), spp=3, seed=11)

    img, run = ob.render(3, 5, params=PROXY_PARAMS, threads=4, trace=True)
    np.savez_compressed(os.path.join(HERE, "proxy_caustic.npz"), image=img, pass_val=run.pass_val,
                        pool_n=run.pool_n, pool_raw=run.pool_raw, pool_walk=run.pool_walk, pool_end=run.pool_end,
                        pool_inv_p=run.pool_inv_p, spp=3, seed=5)

    e6, c6, t6 = orc.recip_twopoint(2000, 6.0, 10000, 1)
    e19, c19, t19 = orc.recip_twopoint(300, 1.9, 10000, 8)
    np.savez_compressed(os.path.join(HERE, "recip_twopoint.npz"), est6=e6, cost6=c6, est19=e19, cost19=c19,
                        trunc19=t19)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
