"""Reciprocal-run cost distribution and per-round evaluation counts on a config (PXG_PROFILE
output of one context; debugging aid). Usage: PXG_PROFILE=1 python tools/recip_dist.py C4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
sc, walks = bench.make_scene(cfg)
r = ProxyRenderer(sc, seed=1, params=ProxyParams(light_walks=walks))
r.set_pass_limit(24)
r.render_passes(24)
r.close()
