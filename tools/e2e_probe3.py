"""Per-pass host timeline of the pipelined public-API loop (debugging aid)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer, render_proxy_bdpt

sc = scenes.cornell_c2(512)
p = ProxyParams(light_walks=262144)
NP = int(sys.argv[1]) if len(sys.argv) > 1 else 32
render_proxy_bdpt(sc, 2, 1000, p, pass_done=lambda d, im: True)
for trial in range(2):
    t0 = time.perf_counter()
    q = ProxyRenderer(sc, 2000 + trial, p)
    t1 = time.perf_counter()
    q.set_pass_limit(NP)
    q.render_passes_async(1)
    q.snapshot(0)
    marks = []
    for k in range(1, NP + 1):
        if k < NP:
            q.render_passes_async(1)
            q.snapshot(k & 1)
        a = time.perf_counter()
        img = q.read_snapshot((k - 1) & 1)
        b = time.perf_counter()
        marks.append((b - t1, b - a))
    q.close()
    print(f"trial {trial}: create {1e3 * (t1 - t0):.1f} ms")
    print("  pass done at (ms):", " ".join(f"{1e3 * m[0]:.0f}" for m in marks))
    print("  read wait (ms):   ", " ".join(f"{1e3 * m[1]:.1f}" for m in marks))
