"""e2e breakdown on C2 (debugging aid): context creation phases (PXG_PROFILE), one full
render_proxy_bdpt(64 spp) call with the per-pass callback, and the same passes timed inside a
warm context."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer, render_proxy_bdpt

sc = scenes.cornell_c2(512)
p = ProxyParams(light_walks=262144)
render_proxy_bdpt(sc, 2, 1, p, pass_done=lambda d, im: True)
for trial in range(2):
    t0 = time.perf_counter()
    render_proxy_bdpt(sc, 64, 7 + trial, p, pass_done=lambda d, im: True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    r = ProxyRenderer(sc, 3, p)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r.set_pass_limit(64)
    r.render_passes(64)
    t3 = time.perf_counter()
    r.close()
    t4 = time.perf_counter()
    print(f"e2e {1e3*(t1-t0):.1f} ms | create {1e3*(t2-t1):.1f} | 64 passes {1e3*(t3-t2):.1f} | destroy {1e3*(t4-t3):.1f}", flush=True)
