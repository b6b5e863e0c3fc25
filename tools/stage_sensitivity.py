"""Pass-time sensitivity to the Stage-1 load (debugging aid, NOT a valid configuration):
times C2 passes with the default ProxyParams and with Stage 1 artificially reduced."""
import sys
import time
import torch  # noqa: F401  (CUDA context like bench.py)
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

sc = scenes.cornell_c2()
for name, kw in [("default", {}), ("repeats=1", {"recip_repeats": 1}), ("budget=100", {"pool_budget": 100}),
                 ("budget=1", {"pool_budget": 1}), ("proxy off", {"enabled": False})]:
    r = ProxyRenderer(sc, seed=1, params=ProxyParams(light_walks=262144, **kw))
    r.set_pass_limit(16)
    r.render_passes(8)
    r.set_pass_limit(40)
    t, _ = r.timing()
    r.render_passes(32)
    t, _ = r.timing()
    print(f"{name:12s} {t[6] / 32:.3f} ms/pass  stage1 {t[0]:.1f} recip {t[1]:.1f}")
    r.close()
