"""render_proxy_bdpt(C2, 64 spp) wall time: with the per-pass mean read-back callback, without
it, and context creation alone (debugging aid)."""
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
    for name, cb in (("callback", lambda d, im: True), ("no callback", None)):
        t0 = time.perf_counter()
        render_proxy_bdpt(sc, 64, 7 + trial, p, pass_done=cb)
        torch.cuda.synchronize()
        print(f"{name}: {1e3 * (time.perf_counter() - t0):.1f} ms")
    t0 = time.perf_counter()
    r = ProxyRenderer(sc, 3, p)
    t1 = time.perf_counter()
    r.close()
    print(f"create {1e3 * (t1 - t0):.1f} ms")
