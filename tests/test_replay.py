"""Replay parity (SURVEY §8c mode ii, row a29): the device's own vertices of a pass, dumped
through pxg_dump_paths, rescored by the reference's functions in oracle/_ref/liboracle.so:

* standard strategies: weighted_bdpt_value (proj/src/proxy.cpp:621-643) over the dumped eye
  and light sub-paths with the pass's statistics snapshot -> the device's per-pixel sum;
* proxy connections: proxy_pdf_components (proj/src/proxy.cpp:321-378) of the device's
  retraced block -> the device's prefix density (1e-12, the reference's own bar at
  proj/tests/test_proxy.cpp:747-748) and sample-time retrace density (1e-6, the bar at
  proj/tests/test_proxy.cpp:724-726); dropout's subspace labels (exact); the proxy_connect
  value formed after the retrace (proj/src/proxy.cpp:562-602) -> the device's value (1e-4).

Unlike the trajectory tests this needs no shared random streams: it separates arithmetic error
from trajectory divergence (SURVEY §7 hard part 1). No failure budget.
"""
import numpy as np
import pytest

from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4      # per-path value (north star)
PREFIX_TOL = 1e-12  # proj/tests/test_proxy.cpp:747-748 (a prefix whose interior vertices are diffuse)
RETRACE_TOL = 1e-6  # proj/tests/test_proxy.cpp:724-726 ("near-mirror lobes evaluate to ~1e7, so recomputing the
#                     density loses a few ulps"): also the bar of a prefix recomputed through a GGX lobe


def rel_err(a, b):
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)


REPLAY_SCENES = {
    "caustic_box": (lambda: scenes.caustic_box(24), {"pretrace_paths": 4000, "light_walks": 4000}, 4, None),
    "glass_slab": (lambda: scenes.glass_slab(24), {"pretrace_paths": 4000, "light_walks": 4000}, 4, None),
    "c2_small": (lambda: scenes.cornell_c2(48, max_depth=10), {"pretrace_paths": 4000, "light_walks": 8000}, 3, None),
    "c3_small": (lambda: scenes.lens_room_c3(32, max_depth=12), {"pretrace_paths": 4000, "light_walks": 8000}, 3,
                 None),
    "c1_depth16": (lambda: scenes.cornell_c1(24, max_depth=16), {"pretrace_paths": 4000, "light_walks": 8000}, 3,
                   None),
    # BASELINE configs at full size: C2 512x512 (every pixel) and C4 1920x1080 (a 1/8 row band)
    "C2_full": (lambda: scenes.cornell_c2(512), {}, 2, None),
    "C4_full_band": (lambda: scenes.procedural_c4(1920, 1080), {}, 1, (1920 * 540, 1920 * 675)),
}


@pytest.mark.parametrize("name", list(REPLAY_SCENES))
def test_replay_rescoring_matches_device(pxg, oracle, name, parity_report):
    make, pd, passes, rng = REPLAY_SCENES[name]
    sc = make()
    o = oracle.OracleScene(sc.to_json())
    rec = {"scene": name, "pixels": 0, "passes": passes, "bdpt_over_tol": 0, "bdpt_max_rel": 0.0,
           "proxy_paths": 0, "prefix_max_rel": 0.0, "prefix_glossy_max_rel": 0.0, "retrace_max_rel": 0.0,
           "label_mismatch": 0,
           "c_over_tol": 0, "c_max_rel": 0.0, "c_nonzero": 0, "zero_c_without_retrace": True}
    lobed = np.array([m.metallic > 0.0 or m.transmission > 0.0 for m in sc.materials])  # a GGX lobe is sampled
    with ProxyRenderer(sc, 11, ProxyParams(**pd)) as r:
        r.set_pass_limit(passes)
        for p in range(passes):
            r.render_passes(1)
            lo, hi = rng if rng else (0, r.n)
            recs, eye, light, proxy, stats = r.dump_paths(lo, hi)
            rec["pixels"] = hi - lo
            # standard strategies
            bd = o.replay_bdpt(eye, recs["n_eye"], light, recs["n_light"], stats, threads=16)
            e = rel_err(recs["bdpt"], bd)
            rec["bdpt_over_tol"] += int(np.count_nonzero((e > REL_TOL).any(axis=1)))
            rec["bdpt_max_rel"] = max(rec["bdpt_max_rel"], float(e.max()))
            # proxy connections with an accepted retrace
            acc = (recs["flags"] & 16) != 0
            picked = (recs["flags"] & 4) != 0
            rec["zero_c_without_retrace"] &= bool(np.all(recs["c"][picked & ~acc] == 0.0))
            if not acc.any():
                continue
            a = recs[acc]
            out = o.replay_proxy(eye[acc], a["tp"], proxy[acc], a["u"], a["n_prefix"], a["cdir"], a["has_cdir"],
                                 a["prefix_pdf"], a["inverse_p"], stats, threads=16)
            rec["proxy_paths"] += int(acc.sum())
            # proxy_pdf_components recomputes the prefix density from positions: through the
            # interior prefix vertices' BSDF lobes, so a GGX lobe on the way amplifies rounding
            pe = rel_err(a["prefix_pdf"], out["prefix_pdf"])
            pv = proxy[acc]
            interior = (np.arange(pv.shape[1])[None, :] >= 1) & (np.arange(pv.shape[1])[None, :] < a["n_prefix"][:, None] - 1)
            glossy = (interior & lobed[np.maximum(pv["material"], 0)]).any(axis=1)
            if (~glossy).any():
                rec["prefix_max_rel"] = max(rec["prefix_max_rel"], float(pe[~glossy].max()))
            if glossy.any():
                rec["prefix_glossy_max_rel"] = max(rec["prefix_glossy_max_rel"], float(pe[glossy].max()))
            rec["retrace_max_rel"] = max(rec["retrace_max_rel"],
                                         float(rel_err(a["retrace_density"], out["retrace_density"]).max()))
            rec["label_mismatch"] += int(np.count_nonzero((a["s_label"] != out["s_label"]) |
                                                          (a["c_label"] != out["c_label"])))
            ec = rel_err(a["c"], out["c"])
            rec["c_over_tol"] += int(np.count_nonzero((ec > REL_TOL).any(axis=1)))
            rec["c_max_rel"] = max(rec["c_max_rel"], float(ec.max()))
            rec["c_nonzero"] += int(np.count_nonzero((a["c"] != 0).any(axis=1)))
    parity_report("replay", rec)
    print(rec)
    assert rec["bdpt_over_tol"] == 0
    assert rec["prefix_max_rel"] <= PREFIX_TOL
    assert rec["prefix_glossy_max_rel"] <= RETRACE_TOL
    assert rec["retrace_max_rel"] <= RETRACE_TOL
    assert rec["label_mismatch"] == 0
    assert rec["c_over_tol"] == 0
    assert rec["zero_c_without_retrace"]
    # glass_slab's u = 2 retraces are accepted about once per 10 passes at this size (the restated
    # loop agrees: no accepted retrace in these 4 passes), so it only pins the standard strategies
    # and the zero-without-retrace rule
    if name in ("caustic_box", "c2_small", "C2_full"):
        assert rec["proxy_paths"] > 0 and rec["c_nonzero"] > 0


def test_dump_paths_rejects_bad_range(pxg):
    sc = scenes.caustic_box(8)
    with ProxyRenderer(sc, 3, ProxyParams(pretrace_paths=2000, light_walks=1000)) as r:
        r.render_passes(1)
        with pytest.raises(Exception):
            r.dump_paths(0, r.n + 1)
        recs, eye, light, proxy, stats = r.dump_paths(5, 5)
        assert recs.shape == (0,)
