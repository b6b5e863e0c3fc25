"""Reciprocal-run profile on C2: per-round active runs, and the distribution of run costs
(nodes evaluated per run) over a few passes. Debugging aid (GPU)."""
import sys
import numpy as np
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyRenderer

sc = scenes.cornell_c2()
r = ProxyRenderer(sc, seed=1)
r.render_passes(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
t = r.timing()
print("timing", t)
