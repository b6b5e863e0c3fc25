"""e2e variance probe: the bench's order (main context, measurement, close), then repeated
public-API renders with a create / passes / close breakdown (debugging aid)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer, render_proxy_bdpt

sc = scenes.cornell_c2(512)
p = ProxyParams(light_walks=262144)
r = ProxyRenderer(sc, 1, p)
r.set_pass_limit(16)
r.render_passes(8)
r.set_pass_limit(40)
r.render_passes(16)
if len(sys.argv) > 1:
    r.set_pass_limit(-1)
    r.measure_traversal(2)
r.close()
render_proxy_bdpt(sc, 1, 1000, p, pass_done=lambda d, im: True)
for trial in range(6):
    t0 = time.perf_counter()
    q = ProxyRenderer(sc, 2000 + trial, p)
    t1 = time.perf_counter()
    q.set_pass_limit(16)
    q.render_passes_async(1)
    q.snapshot(0)
    for k in range(1, 17):
        if k < 16:
            q.render_passes_async(1)
            q.snapshot(k & 1)
        img = q.read_snapshot((k - 1) & 1)
    t2 = time.perf_counter()
    q.close()
    t3 = time.perf_counter()
    print(f"trial {trial}: create {1e3 * (t1 - t0):.1f} passes {1e3 * (t2 - t1):.1f} close {1e3 * (t3 - t2):.1f} ms")
