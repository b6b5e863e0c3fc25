"""Breaks the end-to-end render_proxy_bdpt time into create / passes / read-back / destroy."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

sc = scenes.cornell_c2(512)
p = ProxyParams(light_walks=262144)
for trial in range(3):
    t0 = time.perf_counter()
    r = ProxyRenderer(sc, 5 + trial, p)
    t1 = time.perf_counter()
    r.set_pass_limit(16)
    tr, tm = 0.0, 0.0
    for k in range(16):
        a = time.perf_counter(); r.render_passes(1); b = time.perf_counter(); m = r.mean(); c = time.perf_counter()
        tr += b - a; tm += c - b
    t2 = time.perf_counter()
    r.close()
    t3 = time.perf_counter()
    print(f"trial {trial}: create {1e3*(t1-t0):.1f} ms, passes {1e3*tr:.1f} ms, mean readback {1e3*tm:.1f} ms, destroy {1e3*(t3-t2):.1f} ms")

# the public API path bench.py times (pipelined pass_done callback)
from paper_2503_23412_b200.render import render_proxy_bdpt
for trial in range(3):
    t0 = time.perf_counter()
    img = render_proxy_bdpt(sc, 16, 2000 + trial, p, pass_done=lambda d, im: True)
    print(f"render_proxy_bdpt trial {trial}: {1e3 * (time.perf_counter() - t0):.1f} ms")
