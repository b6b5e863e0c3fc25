"""Converged-image checks (BASELINE.json north star: converged images match a high-spp
reference render within relMSE 1e-3, with no bias trend as spp grows).

The converged reference is render_pt on the device (per pixel equal to the unmodified
reference render_pt on the same Philox streams,
tests/test_gpu_parity.py::test_pt_matches_reference_per_pixel) at 262,144 spp.

Only scenes where the reference's proxy-BDPT has a usable variance can pass a relMSE bar at
a test-sized spp: on caustic_box (mirror floor under a small lamp) the reference estimator
is heavy-tailed -- typical 1K-4K spp renders of both the reference and this library sit
~33% below PT and single rare samples later move the mean by more than that;
that scene is checked per path against the oracle instead (test_gpu_parity.py).

relMSE = mean over pixels and channels of (x - r)^2 / (r^2 + 1e-2).
"""
import numpy as np
import pytest

from paper_2503_23412_b200 import scenes
from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer, render_pt

pytestmark = pytest.mark.gpu


def relmse(x, r, eps=1e-2):
    return float(np.mean((x - r) ** 2 / (r ** 2 + eps)))


def test_c1_converges_to_pt_reference_without_bias_trend(pxg):
    sc = scenes.cornell_c1(32, max_depth=8)
    ref = render_pt(sc, 1024, 101, chunks=256)  # 262,144 spp
    ref2 = render_pt(sc, 1024, 202, chunks=256)
    assert relmse(ref2, ref) < 1e-4  # the reference's own noise floor
    errs = {}
    with ProxyRenderer(sc, 7, ProxyParams()) as r:
        done = 0
        for spp in (256, 1024, 4096):
            r.render_passes(spp - done)
            done = spp
            img = r.mean()
            errs[spp] = (relmse(img, ref), (img.mean() - ref.mean()) / ref.mean())
    for spp, (e, b) in errs.items():
        print(f"C1 32x32 proxy-BDPT {spp:5d} spp: relMSE {e:.3e} (x spp = {e * spp:.2f}), mean rel diff {b:+.2e}")
    assert errs[4096][0] <= 1e-3
    # no bias trend: the error falls like 1/spp (a bias would flatten relMSE * spp upwards)
    assert errs[4096][0] * 4096 <= 2.0 * errs[256][0] * 256
    assert abs(errs[4096][1]) <= 5e-3
