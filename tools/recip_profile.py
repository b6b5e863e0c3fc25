"""Stage timeline on C2 (pxg_read_timing of a 16-pass call after 8 warm-up passes):
t[0] Stage-1 batch wall time, t[1] reciprocal rounds, t[2] sub-path trace, t[3] connections
+ MIS, t[4] proxy connection, t[5] gate + film + gamma (t[2..5]: last pass of each batch),
t[6] whole call. With PXG_PROFILE=1 also the per-round reciprocal schedule (debugging aid)."""
import sys
import numpy as np
from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

sc = scenes.cornell_c2()
r = ProxyRenderer(sc, seed=1, params=ProxyParams(light_walks=262144))
r.set_pass_limit(16)
r.render_passes(8)
r.set_pass_limit(32)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
r.render_passes(n)
t, cnt = r.timing()
print("stage1 %.2f recip %.2f | last pass: trace %.3f conn %.3f proxy %.3f gate %.3f | call %.2f ms (%.3f ms/pass) launches %d"
      % (t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[6] / n, cnt[0]))
