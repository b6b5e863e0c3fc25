"""Context-creation phases on C2 (PXG_PROFILE=1 prints them; debugging aid)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

sc = scenes.cornell_c2(512)
p = ProxyParams(light_walks=262144)
for trial in range(3):
    t0 = time.perf_counter()
    r = ProxyRenderer(sc, 3, p)
    t1 = time.perf_counter()
    r.close()
    print(f"trial {trial}: create {1e3 * (t1 - t0):.1f} ms", flush=True)
