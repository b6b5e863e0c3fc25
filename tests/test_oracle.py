"""CPU tests: pin the oracle (the compiled reference + restated loop) and the host logic.

The oracle is checked against (1) the Random123 known-answer vectors of Philox4x32-10, (2)
the UNMODIFIED reference renderers compiled from /root/reference (bitwise), and (3) the
reference's own closed-form fixtures (proj/tests/test_recip.cpp:16-18,74-152).
"""
import json

import numpy as np
import pytest

from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.scene import SceneError, load_scene_from_string


def philox_word(c, k):
    """Philox4x32-10 restated in Python (Salmon et al. 2011), all four words."""
    M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
    c = list(c)
    k = list(k)
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [(p1 >> 32) ^ c[1] ^ k[0], p1 & 0xFFFFFFFF, (p0 >> 32) ^ c[3] ^ k[1], p0 & 0xFFFFFFFF]
        k = [(k[0] + W0) & 0xFFFFFFFF, (k[1] + W1) & 0xFFFFFFFF]
    return c


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32_10
    assert philox_word((0, 0, 0, 0), (0, 0)) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert philox_word((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert philox_word((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0)) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


@pytest.mark.parametrize("seed,kind,sub,stream", [(0, 0, 0, 0), (7, 0, 0, 12345), (3, 4, 0x205, (5 << 32) | 77),
                                                  (2**64 - 1, 5, 0xFFFFFF, 2**64 - 1)])
def test_oracle_streams_are_philox(oracle, seed, kind, sub, stream):
    got = oracle.rng_draws(seed, kind, sub, stream, 16)
    tag = (kind << 24) | sub
    want = [philox_word((i, tag, stream & 0xFFFFFFFF, stream >> 32), (seed & 0xFFFFFFFF, seed >> 32))[0]
            for i in range(16)]
    assert got.tolist() == want


SMALL = {
    "caustic_box": lambda: scenes.caustic_box(12),
    "sphere_room": lambda: scenes.sphere_room(12),
    "glass_slab": lambda: scenes.glass_slab(10),
    "c1_small": lambda: scenes.cornell_c1(16, max_depth=8, subdiv=2),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_restated_loop_equals_reference_bdpt_bitwise(oracle, name):
    """proxy off => the restated loop is bitwise the unmodified reference render_bdpt
    (the reference's own invariant, proj/tests/test_proxy.cpp:1053-1079)."""
    sc = SMALL[name]()
    o = oracle.OracleScene(sc.to_json())
    ref = o.render_bdpt(3, 11)
    img, _ = o.render(3, 11, params={"enabled": 0}, threads=4)
    assert np.array_equal(ref, img)


def test_restated_loop_equals_reference_on_diffuse_scene(oracle):
    """No specular material: the proxy machinery never activates, so the restated loop with
    proxy ON equals both unmodified reference renderers bitwise."""
    o = oracle.OracleScene(scenes.diffuse_box(10).to_json())
    ref_b = o.render_bdpt(3, 5)
    ref_p, raw, kept = o.render_proxy_ref(3, 5, params={"pretrace_paths": 1000})
    img, _ = o.render(3, 5, params={"pretrace_paths": 1000}, threads=4)
    assert raw == 0 and kept == 0
    assert np.array_equal(ref_b, ref_p) and np.array_equal(ref_b, img)


def test_restated_loop_deterministic_across_threads(oracle):
    o = oracle.OracleScene(scenes.caustic_box(12).to_json())
    p = {"pretrace_paths": 2000, "light_walks": 2000}
    a, ra = o.render(3, 1, params=p, threads=1, trace=True)
    b, rb = o.render(3, 1, params=p, threads=8, trace=True)
    assert np.array_equal(a, b)
    assert np.array_equal(ra.pool_inv_p, rb.pool_inv_p)
    assert np.array_equal(ra.gamma_rows, rb.gamma_rows)
    assert np.array_equal(ra.diag, rb.diag)


def test_restated_loop_agrees_with_reference_in_distribution(oracle):
    """The documented stream deviations change trajectories, not the estimator: 48 renders of
    64 spp by the restated loop (Philox, re-keyed streams) and 48 by the unmodified reference
    render_proxy_bdpt (PCG32 as shipped) are one distribution: medians of the mean image luminance within 10%
    (3.5 standard errors; round 1 accepted a flat 20% on the mean of 4 renders) and a
    Mann-Whitney U test; the caustic estimator is heavy-tailed
    (proj/tests/test_proxy.cpp:1125-1131), which rank statistics do not mind."""
    from scipy.stats import mannwhitneyu
    sc = scenes.caustic_box(8)
    o = oracle.OracleScene(sc.to_json())
    opcg = oracle.OracleScene(sc.to_json(), variant="pcg")
    p = {"pretrace_paths": 2000, "light_walks": 3000}
    lum = np.array([0.2126, 0.7152, 0.0722])
    n = 48
    a = np.array([(o.render(64, 100 + s, params=p, threads=8)[0] @ lum).mean() for s in range(n)])
    b = (opcg.render_proxy_ref_mt(64, 200, n, p, all_images=True) @ lum).mean(axis=(1, 2))
    # the estimator is heavy-tailed (single rare samples move a render's mean by 10x its spread), so
    # the comparison is on robust statistics: medians (standard error ~2% each) and rank sums
    assert abs(np.median(a) / np.median(b) - 1.0) <= 0.10, (np.median(a), np.median(b))
    assert mannwhitneyu(a, b).pvalue > 0.005


def test_recip_two_point_closed_forms(oracle):
    """proj/tests/test_recip.cpp:74-82,139-152: mean 1/4, variance 5/432, mean cost 1.5 at B = 6."""
    est, cost, tr = oracle.recip_twopoint(200000, 6.0)
    se = est.std(ddof=1) / np.sqrt(est.size)
    assert abs(est.mean() - 0.25) < 4 * se
    assert abs(est.var(ddof=1) / (5.0 / 432.0) - 1.0) < 0.05
    assert abs(cost.mean() / 1.5 - 1.0) < 0.02
    assert not tr.any()


def test_recip_divergent_bound_truncates(oracle):
    """proj/tests/test_recip.cpp:165-182: B = 1.9 is supercritical and trips the guard."""
    est, cost, tr = oracle.recip_twopoint(300, 1.9, cap=10000, seed=8)
    assert tr.sum() > 15
    assert (cost <= 10001).all()


# ---------------------------------------------------------------- host scene mirror
MINI = """{
  "materials": [{"name": "w", "base_color": [0.7, 0.7, 0.7], "roughness": 1.0},
                {"name": "lamp", "base_color": [0, 0, 0]}],
  "primitives": [
    {"shape": "rectangle", "material": "w", "origin": [-1, 0, -1], "edge_u": [2, 0, 0], "edge_v": [0, 0, 2]},
    {"shape": "sphere", "material": "w", "center": [0, 1, 0], "radius": 0.5},
    {"shape": "triangle", "material": "w", "p0": [-1, 0, 1], "p1": [1, 0, 1], "p2": [0, 2, 1]},
    {"shape": "rectangle", "material": "lamp", "origin": [-0.25, 1.99, -0.25], "edge_u": [0.5, 0, 0], "edge_v": [0, 0, 0.5]}],
  "emitters": [{"primitive": 3, "radiance": [10, 10, 10]}],
  "camera": {"position": [0, 1, 4], "look_at": [0, 1, 0], "fov_y": 40, "resolution": [16, 8]},
  "settings": {"max_depth": 6, "spp": 4}
}"""


@pytest.mark.parametrize("needle,repl,fragment", [
    ('"radius": 0.5', '"radius": -1', "radius"),
    ('"emitters": [{"primitive": 3, "radiance": [10, 10, 10]}]', '"emitters": []', "at least one emitter"),
    ('"material": "lamp"', '"material": "nope"', "unknown material"),
    ('"fov_y": 40', '"fov_y": 200', "fov_y"),
    ('"edge_u": [0.5, 0, 0]', '"edge_u": [0, 0, 0]', "degenerate"),
    ('"roughness": 1.0}', '"roughness": 1.5}', "must lie in [0,1]"),
    ('"spp": 4', '"spp": 0', "spp must be at least 1"),
])
def test_scene_validation_mirrors_reference(oracle, needle, repl, fragment):
    body = MINI.replace(needle, repl, 1)
    assert body != MINI
    with pytest.raises(SceneError) as e:
        load_scene_from_string(body)
    assert fragment in str(e.value)
    with pytest.raises(RuntimeError) as e2:
        oracle.OracleScene(body)
    assert fragment in str(e2.value)


def test_scene_loader_roundtrip(oracle):
    sc = load_scene_from_string(MINI)
    assert sc.n_prims == 4 and sc.camera.width == 16 and sc.camera.height == 8
    o = oracle.OracleScene(sc.to_json())
    assert (o.width, o.height, o.n_prims, o.max_depth) == (16, 8, 4, 6)
    assert o.total_emitter_area == 0.25


def test_config_generators(oracle):
    c1 = scenes.cornell_c1(8)
    assert c1.n_prims == 10 + 2 + 5120
    c2 = scenes.cornell_c2(8)
    assert c2.n_prims == 10 + 2 + 5120 + 20480
    o = oracle.OracleScene(c1.to_json())
    assert o.n_prims == c1.n_prims
    assert abs(o.total_emitter_area - 0.0625) < 1e-15
    c3 = scenes.lens_room_c3(8)
    assert c3.n_prims == 6 + 2 * 19998 + 256 * 256 and len(c3.emitter_prim) == 256 * 256
    lit = c3.emitter_radiance[:, 0]
    assert set(np.unique(lit).tolist()) == {0.0, 20.0} and 0.48 < np.mean(lit > 0) < 0.52
    o3 = oracle.OracleScene(c3.to_json())
    assert o3.n_prims == c3.n_prims and abs(o3.total_emitter_area - 0.2) < 1e-9
    c4 = scenes.procedural_c4(8, 8, instances=40)
    assert len(c4.emitter_prim) == 4 and len(c4.materials) == 41
    full = scenes.procedural_c4(8, 8)
    assert 0.95e6 < full.n_prims < 1.1e6
    assert np.array_equal(full.a, scenes.procedural_c4(8, 8).a)  # seeded, deterministic


def test_scene_npz_cache_roundtrip(tmp_path):
    from paper_2503_23412_b200.scene import load_npz, save_npz
    for sc in (scenes.sphere_room(8), scenes.lens_room_c3(8, cells=16, rings=4, segs=8)):
        p = str(tmp_path / "s.npz")
        save_npz(sc, p)
        back = load_npz(p)
        assert json.loads(back.to_json()) == json.loads(sc.to_json())  # 0 == 0.0: same values


@pytest.mark.parametrize("name", ["c1", "caustic_box", "glass_slab"])
def test_replay_evaluator_reproduces_restated_loop(oracle, name):
    """The replay evaluator (orc_replay_bdpt: weighted_bdpt_value over given vertex rows) on the
    reference's own pass-0 sub-paths equals the restated loop's per-pixel standard-strategy value
    bitwise (proxy off: empty statistics, the balance heuristic) — the harness the GPU replay
    test (tests/test_replay.py) rescores device vertices with."""
    from paper_2503_23412_b200 import scenes
    sc = {"c1": lambda: scenes.cornell_c1(16, max_depth=8), "caustic_box": lambda: scenes.caustic_box(12),
          "glass_slab": lambda: scenes.glass_slab(12)}[name]()
    o = oracle.OracleScene(sc.to_json())
    pd = {"enabled": 0}
    _, run = o.render(1, 5, params=pd, threads=4, trace=True)
    eye, ne, light, nl = o.trace_subpaths(5, sc.n_px, threads=4)
    assert (ne >= 1).all()
    bd = o.replay_bdpt(eye, ne, light, nl, np.zeros((oracle.N_BUCKETS, 3)), threads=4)
    assert np.array_equal(bd, run.pass_bdpt[0])
    assert np.count_nonzero(bd) > 0
