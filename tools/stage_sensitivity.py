"""Pass-time sensitivity to the Stage-1 load (debugging aid, NOT a valid configuration):
times passes with the default ProxyParams and with Stage 1 artificially reduced.
Usage: python tools/stage_sensitivity.py [C2|C4]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (CUDA context like bench.py)
import bench
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
sc, walks = bench.make_scene(cfg)
npass = 16 if cfg in ("C3", "C4") else 32
for name, kw in [("default", {}), ("repeats=1", {"recip_repeats": 1}), ("budget=100", {"pool_budget": 100}),
                 ("budget=1", {"pool_budget": 1}), ("walks/8", {"light_walks": max(1, walks // 8)}),
                 ("proxy off", {"enabled": False})]:
    kw.setdefault("light_walks", walks)
    r = ProxyRenderer(sc, seed=1, params=ProxyParams(**kw))
    r.set_pass_limit(16)
    r.render_passes(8)
    r.set_pass_limit(16 + npass)
    r.render_passes(npass)
    t, _ = r.timing()
    print(f"{cfg} {name:12s} {t[6] / npass:.3f} ms/pass  stage1 {t[0]:.1f} recip {t[1]:.1f}", flush=True)
    r.close()
