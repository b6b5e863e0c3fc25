"""Traversal measurement probe on C2: repeated pxg_measure_traversal calls (debugging aid)."""
import time
import numpy as np
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyRenderer

sc = scenes.cornell_c2()
r = ProxyRenderer(sc, seed=1)
r.render_passes(8)
for it in range(4):
    t0 = time.time()
    m = r.measure_traversal(2)
    print("measure", it, m, "wall", round(time.time() - t0, 3))
