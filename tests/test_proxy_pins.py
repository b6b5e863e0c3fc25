"""Device-level pins of the proxy pieces on caller-built vertices, the analogue of the
reference's own closed-form tests (proj/tests/test_proxy.cpp:480-618: support density closed
forms on an occluder bench; the support mixture integrates to one over surfaces and escapes).

pxg_proxy_probe runs dropout, support_pdf, target_density and support_sample on the device for
hand-built vertices; orc_proxy_probe runs the reference's functions on the same vertices.

* CPU (not gpu): the reference functions against closed forms written out here (pins the
  checker and the fixture);
* GPU: the device against the same closed forms, against the reference on hand-built and on
  traced sub-paths (1e-12 relative), support_sample draws bitwise (same Philox streams), and
  the mixture's surface mass (device quadrature) + escape mass (device draws) = 1.

Fixtures are this repository's own geometry (scenes._Builder), not the reference's strings.
"""
import numpy as np
import pytest

from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import VERTEX_DTYPE, ProxyParams, ProxyRenderer
from paper_2503_23412_b200.scenes import Camera, Material, Settings, _Builder

K_LIGHT, K_DIFFUSE, K_SPECULAR, K_CAMERA = 0, 1, 2, 3
TOL = 1e-12


def blocker_bench(resolution: int = 8):
    """Mirror floor, a wide downward lamp (area 3) at y = 2 and a matte shelf at y = 1 over
    x < 1.5: from the floor point (1, 0, 2) lamp points with x < 2 are hidden, x > 2 visible."""
    bld = _Builder()
    matte = bld.material(Material("matte", (0.5, 0.5, 0.5), 0.0, 0.9))
    mirror = bld.material(Material("mirror", (0.9, 0.9, 0.9), 1.0, 0.01))
    shell = bld.material(Material("shell", (0.05, 0.05, 0.05), 0.0, 0.9))
    bld.rect(mirror, (0, 0, 0), (0, 0, 4), (4, 0, 0))        # prim 0, normal +y
    bld.rect(matte, (0, 1, 0), (1.5, 0, 0), (0, 0, 4))       # prim 1, the shelf
    lamp = bld.rect(shell, (0.5, 2, 1.5), (3, 0, 0), (0, 0, 1))  # prim 2, normal -y, area 3
    bld.rect(matte, (0, 0, 0), (4, 0, 0), (0, 3, 0))         # prim 3, back wall z = 0, normal +z
    bld.emitter(lamp, (10.0, 10.0, 10.0))
    cam = Camera((2.0, 1.0, 3.8), (2.0, 0.5, 0.5), (0, 1, 0), 60.0, resolution, resolution)
    return bld.build(cam, Settings(6, 1, 0)), dict(matte=matte, mirror=mirror, shell=shell, lamp=lamp)


def vertex(p, n, mat, prim, flag, emitter=-1, wi=(0, 0, 0), pdf_fwd=1.0):
    v = np.zeros((), VERTEX_DTYPE)
    v["p"], v["n"], v["wi"] = p, n, wi
    v["throughput"] = (1.0, 1.0, 1.0)
    v["pdf_fwd"] = pdf_fwd
    v["material"], v["primitive"], v["emitter"], v["flag"] = mat, prim, emitter, flag
    return v


def stack(*vs):
    return np.stack(vs).astype(VERTEX_DTYPE)


def unit(a):
    a = np.asarray(a, float)
    return a / np.linalg.norm(a)


def areal(pdf_w, a, b, nb):
    d = np.asarray(b, float) - np.asarray(a, float)
    d2 = d @ d
    return pdf_w * abs(np.asarray(nb, float) @ d) / np.sqrt(d2) / d2


def sphere_cos_pdf(n, d):
    return abs(np.asarray(n, float) @ d) / (2 * np.pi)


def emit_dir_pdf(n, d):
    c = np.asarray(n, float) @ d
    return c / np.pi if c > 0 else 0.0


def bench_fixture():
    sc, ids = blocker_bench()
    y = vertex((1.0, 0.0, 2.0), (0, 1, 0), ids["mirror"], 0, K_SPECULAR, wi=unit((0.3, 1, 0.1)))
    lamp0 = vertex((3.0, 2.0, 2.0), (0, -1, 0), ids["shell"], ids["lamp"], K_LIGHT, emitter=0, pdf_fwd=1 / 3)
    walk_l = stack(lamp0, y)  # dropped light start: no control vertex
    mid = vertex((3.2, 1.4, 0.0), (0, 0, 1), ids["matte"], 3, K_DIFFUSE, wi=unit((-0.2, 0.6, 2.0)), pdf_fwd=0.3)
    walk_c = stack(lamp0, mid, y)  # dropped interior vertex: the lamp start is the control
    return sc, ids, y, walk_l, walk_c


def closed_forms(ids, y):
    """(candidate, expected support pdf under walk_l, expected target density under walk_l)"""
    yp, yn = y["p"], y["n"]
    out = []
    # hidden lamp point: only the light-surface strand, half of 1 / area; target hidden -> 0
    g = vertex((1.2, 2.0, 2.0), (0, -1, 0), ids["shell"], ids["lamp"], K_LIGHT, emitter=0)
    out.append((g, 0.5 * (1 / 3), 0.0))
    # visible lamp point: light-surface strand + the endpoint's two-sided cosine strand
    for gp in ((3.0, 2.0, 2.2), (2.6, 2.0, 1.7), (3.4, 2.0, 2.4)):
        g = vertex(gp, (0, -1, 0), ids["shell"], ids["lamp"], K_LIGHT, emitter=0)
        d = unit(np.asarray(gp) - yp)
        q = 0.5 * (1 / 3 + areal(sphere_cos_pdf(yn, d), yp, gp, (0, -1, 0)))
        f = (1 / 3) * areal(emit_dir_pdf((0, -1, 0), -d), gp, yp, yn)
        out.append((g, q, f))
    # visible wall point (not an emitter): only the endpoint strand; outside the target class
    gp = (2.5, 0.8, 0.0)
    g = vertex(gp, (0, 0, 1), ids["matte"], 3, K_DIFFUSE)
    d = unit(np.asarray(gp) - yp)
    out.append((g, 0.5 * areal(sphere_cos_pdf(yn, d), yp, gp, (0, 0, 1)), 0.0))
    return out


def check_closed_forms(probe, ids, y, walk_l, walk_c):
    cf = closed_forms(ids, y)
    cand = stack(*[c[0] for c in cf]).reshape(-1, 1)
    r = probe(walk_l, cand)
    assert r["info"][0] == 1 and r["info"][1] == 1 and r["info"][2] == 0 and r["info"][3] == 0  # u = 1, no prefix
    assert r["prefix_pdf"] == 1.0
    for k, (_, q, f) in enumerate(cf):
        assert r["q"][k] == pytest.approx(q, rel=1e-9), k
        assert r["f"][k] == pytest.approx(f, rel=1e-9, abs=0.0), k
    assert r["q"][0] == pytest.approx(1 / 6, rel=1e-12)  # exactly half the area density
    # control configuration: prefix = [lamp start], no control direction yet (terminal == 1)
    rc = probe(walk_c, cand)
    assert rc["info"][0] == 1 and rc["info"][1] == 1 and rc["info"][2] == 1 and rc["info"][3] == 0
    assert rc["prefix_pdf"] == pytest.approx(1 / 3, rel=1e-15)
    hc = walk_c[0]
    for k, (g, _, _) in enumerate(cf):
        dc = unit(g["p"] - hc["p"])
        de = unit(g["p"] - y["p"])
        vis_c = k != 0  # the shelf does not block lamp -> wall / lamp (coplanar lamp points: cosine 0)
        q_ctrl = areal(emit_dir_pdf(hc["n"], dc), hc["p"], g["p"], g["n"]) if vis_c else 0.0
        vis_e = k != 0
        q_end = areal(sphere_cos_pdf(y["n"], de), y["p"], g["p"], g["n"]) if vis_e else 0.0
        assert rc["q"][k] == pytest.approx(0.5 * (q_ctrl + q_end), rel=1e-9, abs=1e-300), k
    return r, rc


def test_reference_densities_match_closed_forms(oracle):
    sc, ids, y, walk_l, walk_c = bench_fixture()
    o = oracle.OracleScene(sc.to_json())
    check_closed_forms(o.proxy_probe, ids, y, walk_l, walk_c)
    # a walk that does not end on a specular vertex is not eligible
    assert o.proxy_probe(walk_c[:2])["info"][0] == 0


@pytest.mark.gpu
def test_device_densities_match_closed_forms_and_reference(pxg, oracle, parity_report):
    sc, ids, y, walk_l, walk_c = bench_fixture()
    o = oracle.OracleScene(sc.to_json())
    with ProxyRenderer(sc, 1, ProxyParams(pretrace_paths=500, light_walks=100)) as r:
        dl, dc = check_closed_forms(r.proxy_probe, ids, y, walk_l, walk_c)
        assert r.proxy_probe(walk_c[:2])["info"][0] == 0
        worst = 0.0
        for walk, dev in ((walk_l, dl), (walk_c, dc)):
            cf = closed_forms(ids, y)
            cand = stack(*[c[0] for c in cf]).reshape(-1, 1)
            ref = o.proxy_probe(walk, cand)
            assert np.array_equal(ref["info"], dev["info"])
            assert ref["prefix_pdf"] == dev["prefix_pdf"]
            for key in ("q", "f"):
                err = np.abs(ref[key] - dev[key]) / np.maximum(np.abs(ref[key]), 1e-300)
                worst = max(worst, float(err.max()))
        parity_report("proxy_pins", {"case": "blocker_bench closed forms", "max_rel_vs_reference": worst})
        assert worst <= TOL


def _light_block_candidates(light, nl, u, rng, count):
    """Candidate blocks of u consecutive real surface vertices (nearest-first order reversed
    like the retraced block: g[0] is the later vertex of the walk)."""
    blocks = []
    idx = np.flatnonzero(nl >= u + 1)
    for i in rng.choice(idx, size=min(count, len(idx)), replace=False):
        k = rng.integers(1, nl[i] - u + 1)  # vertices k .. k+u-1 (skip the light start)
        blocks.append(light[i, k:k + u][::-1])
    return np.stack(blocks) if blocks else np.zeros((0, u), VERTEX_DTYPE)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["caustic_box", "glass_slab", "c2_small"])
def test_device_densities_match_reference_on_traced_walks(pxg, oracle, parity_report, name):
    """Every dropout-eligible prefix of traced light sub-paths (the reference's own tracer),
    with candidate blocks cut from other traced sub-paths: the device's dropout labels,
    support_pdf and target_density against the reference's on identical vertices."""
    make = {"caustic_box": lambda: scenes.caustic_box(16), "glass_slab": lambda: scenes.glass_slab(16),
            "c2_small": lambda: scenes.cornell_c2(24, max_depth=10)}[name]
    sc = make()
    o = oracle.OracleScene(sc.to_json())
    n = min(o.n_px, 400)
    eye, ne, light, nl = o.trace_subpaths(5, n)
    rng = np.random.default_rng(3)
    rec = {"case": name, "walks": 0, "eligible": 0, "candidates": 0, "nonzero_q": 0, "nonzero_f": 0,
           "max_rel_q": 0.0, "max_rel_f": 0.0, "info_mismatch": 0, "by_u": {}}
    with ProxyRenderer(sc, 1, ProxyParams(pretrace_paths=500, light_walks=100)) as r:
        for i in range(n):
            for m in range(2, int(nl[i]) + 1):
                if light[i, m - 1]["flag"] != K_SPECULAR:
                    continue
                walk = light[i, :m]
                rec["walks"] += 1
                ref = o.proxy_probe(walk)
                dev = r.proxy_probe(walk)
                if not np.array_equal(ref["info"], dev["info"]) or ref["prefix_pdf"] != dev["prefix_pdf"]:
                    rec["info_mismatch"] += 1
                if not ref["info"][0]:
                    continue
                u = int(ref["info"][1])
                rec["eligible"] += 1
                rec["by_u"][str(u)] = rec["by_u"].get(str(u), 0) + 1
                cand = _light_block_candidates(light, nl, u, rng, 24)
                # plus the walk's own dropped block: a candidate with non-zero target density
                own = walk[m - 1 - u:m - 1][::-1][None]
                cand = np.concatenate([own, cand]) if len(cand) else own
                ref = o.proxy_probe(walk, cand)
                dev = r.proxy_probe(walk, cand)
                rec["candidates"] += len(cand)
                for key in ("q", "f"):
                    err = np.abs(ref[key] - dev[key]) / np.maximum(np.abs(ref[key]), 1e-300)
                    rec["max_rel_" + key] = max(rec["max_rel_" + key], float(err.max()))
                    rec["nonzero_" + key] += int(np.count_nonzero(ref[key]))
    parity_report("proxy_pins", rec)
    print(rec)
    assert rec["info_mismatch"] == 0
    assert rec["eligible"] > 0 and rec["nonzero_q"] > 0 and rec["nonzero_f"] > 0
    assert rec["max_rel_q"] <= TOL and rec["max_rel_f"] <= TOL


@pytest.mark.gpu
def test_device_support_samples_equal_reference_draws(pxg, oracle, parity_report):
    """support_sample on the device and in the reference on the same Philox streams: the same
    escapes, the same candidate vertices (positions bitwise) and densities."""
    rec = {"case": "support_sample", "draws": 0, "escape_mismatch": 0, "position_mismatch": 0, "max_rel_q": 0.0}
    sc, ids, y, walk_l, walk_c = bench_fixture()
    cases = [(sc, walk_l), (sc, walk_c)]
    cb = scenes.caustic_box(8)
    ocb = oracle.OracleScene(cb.to_json())
    _, _, light, nl = ocb.trace_subpaths(9, 64)
    for i in range(64):
        for m in range(2, int(nl[i]) + 1):
            if light[i, m - 1]["flag"] == K_SPECULAR and ocb.proxy_probe(light[i, :m])["info"][0]:
                cases.append((cb, light[i, :m].copy()))
    cases = cases[:12]
    for scn, walk in cases:
        o = oracle.OracleScene(scn.to_json())
        with ProxyRenderer(scn, 1, ProxyParams(pretrace_paths=500, light_walks=100)) as r:
            dev = r.proxy_probe(walk, None, n_draws=4000, seed=77)
        ref = o.proxy_probe(walk, None, n_draws=4000, seed=77)
        rec["draws"] += 4000
        rec["escape_mismatch"] += int(np.count_nonzero(dev["draw_escaped"] != ref["draw_escaped"]))
        live = ~ref["draw_escaped"] & ~dev["draw_escaped"]
        rec["position_mismatch"] += int(np.count_nonzero(
            (dev["draw_cand"]["p"][live] != ref["draw_cand"]["p"][live]).any(axis=(1, 2))))
        err = np.abs(dev["draw_q"] - ref["draw_q"]) / np.maximum(np.abs(ref["draw_q"]), 1e-300)
        rec["max_rel_q"] = max(rec["max_rel_q"], float(err.max()))
    parity_report("proxy_pins", rec)
    print(rec)
    assert rec["escape_mismatch"] == 0 and rec["position_mismatch"] == 0
    assert rec["max_rel_q"] <= TOL


@pytest.mark.gpu
def test_device_support_mixture_integrates_to_one(pxg, parity_report):
    """Surface mass of the device's support_pdf (midpoint quadrature over every face of the
    closed caustic box that can carry support) + escape mass of the device's support_sample
    draws = 1 (the reference's own check at proj/tests/test_proxy.cpp:551-618, 2.5%)."""
    sc = scenes.caustic_box(8)
    plaster, mirror, shell = 0, 1, 2
    y = vertex((1.3, 0.0, 1.1), (0, 1, 0), mirror, 0, K_SPECULAR, wi=unit((-0.3, 0.42, -0.1)))
    lamp0 = vertex((1.0, 0.42, 1.0), (0, -1, 0), shell, 6, K_LIGHT, emitter=0, pdf_fwd=1 / 0.28 ** 2)
    walk = stack(lamp0, y)
    # (origin, eu, ev, normal, material, prim, emitter, resolution): the five plaster faces and the lamp
    patches = [((0, 2, 0), (2, 0, 0), (0, 0, 2), (0, -1, 0), plaster, 1, -1, 200),
               ((0, 0, 0), (2, 0, 0), (0, 2, 0), (0, 0, 1), plaster, 2, -1, 200),
               ((0, 0, 2), (0, 2, 0), (2, 0, 0), (0, 0, -1), plaster, 3, -1, 200),
               ((0, 0, 0), (0, 2, 0), (0, 0, 2), (1, 0, 0), plaster, 4, -1, 200),
               ((2, 0, 0), (0, 0, 2), (0, 2, 0), (-1, 0, 0), plaster, 5, -1, 200),
               ((0.86, 0.42, 0.86), (0.28, 0, 0), (0, 0, 0.28), (0, -1, 0), shell, 6, 0, 64)]
    with ProxyRenderer(sc, 1, ProxyParams(pretrace_paths=500, light_walks=100)) as r:
        surface = 0.0
        for org, eu, ev, nrm, mat, prim, emit, res in patches:
            fu = (np.arange(res) + 0.5) / res
            P = (np.asarray(org, float)[None, None] + fu[:, None, None] * np.asarray(eu, float)[None, None]
                 + fu[None, :, None] * np.asarray(ev, float)[None, None]).reshape(-1, 3)
            cand = np.zeros((len(P), 1), VERTEX_DTYPE)
            cand["p"][:, 0] = P
            cand["n"][:, 0] = nrm
            cand["throughput"][:, 0] = 1.0
            cand["material"], cand["primitive"], cand["emitter"] = mat, prim, emit
            cand["flag"] = K_LIGHT if emit >= 0 else K_DIFFUSE
            q = r.proxy_probe(walk, cand)["q"]
            cell = np.linalg.norm(np.cross(eu, ev)) / res ** 2
            surface += float(q.sum()) * cell
        d = r.proxy_probe(walk, None, n_draws=200000, seed=5)
        escape = float(d["draw_escaped"].mean())
        assert np.all(d["draw_q"][d["draw_escaped"]] == 1.0)  # sentinel density of the extended space
        assert np.all(d["draw_q"][~d["draw_escaped"]] > 0.0)
    rec = {"case": "mixture mass", "surface_mass": surface, "escape_mass": escape, "total": surface + escape}
    parity_report("proxy_pins", rec)
    print(rec)
    assert 0.1 < escape < 0.4
    assert surface + escape == pytest.approx(1.0, rel=0.025)


@pytest.mark.gpu
def test_device_reciprocal_estimates_invert_the_density_integral(pxg, parity_report):
    """The production reciprocal machinery (global node wavefront + warp DFS) on a hand-built
    incomplete sub-path: the mean of 2,000 runs equals 1 / integral(target_density), the
    integral taken by midpoint quadrature of the device's target_density over the lamp (the
    dropped vertex is a light start, so the integrand lives there). The reference's own check
    (proj/tests/test_proxy.cpp:620-673: 4 standard errors + 0.5%), untruncated at the default
    recursion budget."""
    sc = scenes.caustic_box(8)
    mirror, shell = 1, 2
    y = vertex((1.3, 0.0, 1.1), (0, 1, 0), mirror, 0, K_SPECULAR, wi=unit((-0.3, 0.42, -0.1)))
    lamp0 = vertex((1.0, 0.42, 1.0), (0, -1, 0), shell, 6, K_LIGHT, emitter=0, pdf_fwd=1 / 0.28 ** 2)
    walk = stack(lamp0, y)
    res = 600
    fu = (np.arange(res) + 0.5) / res
    P = np.stack(np.meshgrid(0.86 + 0.28 * fu, [0.42], 0.86 + 0.28 * fu, indexing="ij"), axis=-1).reshape(-1, 3)
    cand = np.zeros((len(P), 1), VERTEX_DTYPE)
    cand["p"][:, 0] = P
    cand["n"][:, 0] = (0, -1, 0)
    cand["throughput"][:, 0] = 1.0
    cand["material"], cand["primitive"], cand["emitter"], cand["flag"] = shell, 6, 0, K_LIGHT
    with ProxyRenderer(sc, 1, ProxyParams(pretrace_paths=500, light_walks=100)) as r:
        pr = r.proxy_probe(walk, cand)
        f, q = pr["f"], pr["q"]
        total = float(f.sum()) * 0.28 ** 2 / res ** 2
        assert total > 0.0
        # the bound the estimator needs: f <= B q on the support (proxy.cpp:389-395 seeds it from
        # probes; here from the quadrature points, with the reference's 2x slack)
        bound = 2.0 * float(np.max(f[q > 0] / q[q > 0]))
        est, cost, tr = r.proxy_recip(walk, bound, 2000)
    se = est.std(ddof=1) / np.sqrt(est.size)
    want = 1.0 / total
    rec = {"case": "reciprocal vs quadrature", "want": want, "mean": float(est.mean()), "se": float(se),
           "mean_cost": float(cost.mean()), "truncated": int(tr.sum()), "bound": bound}
    parity_report("proxy_pins", rec)
    print(rec)
    assert tr.sum() <= est.size // 100
    assert abs(est.mean() - want) <= 4.0 * se + 0.005 * want
    assert cost.min() >= 1
