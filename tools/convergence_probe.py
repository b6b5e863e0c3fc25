"""Probe: GPU PT as the converged reference; relMSE of proxy-BDPT renders vs spp."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer, render_pt


def relmse(x, r, eps=1e-2):
    return float(np.mean((x - r) ** 2 / (r ** 2 + eps)))


for name, sc in (("c1_32", scenes.cornell_c1(32, max_depth=8)), ("c2_32", scenes.cornell_c2(32, max_depth=10)),
                 ("caustic_box16", scenes.caustic_box(16))):
    t = time.time(); ref = render_pt(sc, 1024, 1, chunks=256); t1 = time.time() - t
    ref2 = render_pt(sc, 1024, 2, chunks=256)
    print(f"{name}: PT 262144 spp {t1:.1f}s mean {ref.mean():.5f}; PT-vs-PT relMSE {relmse(ref2, ref):.3e}", flush=True)
    with ProxyRenderer(sc, 7, ProxyParams()) as r:
        done = 0
        for spp in (16, 64, 256, 1024, 4096):
            t = time.time(); r.render_passes(spp - done); done = spp; dt = time.time() - t
            img = r.mean()
            e = relmse(img, ref)
            bias = (img.mean() - ref.mean()) / ref.mean()
            print(f"  proxy-bdpt {spp:5d} spp: relMSE {e:.3e}  relMSE*spp {e*spp:.3f}  mean rel diff {bias:+.2e} ({dt:.1f}s)",
                  flush=True)
