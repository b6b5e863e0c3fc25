"""Film IO and metrics: the Python film module against the reference's
own write_pfm / write_png / compare_images (proj/src/image.cpp, proj/src/metrics.cpp),
compiled into oracle/_ref/film_ref. CPU only."""
import numpy as np

from paper_2503_23412_b200 import film


def _images(seed=3, h=17, w=23):
    rng = np.random.default_rng(seed)
    img = rng.gamma(0.6, 0.7, size=(h, w, 3))
    img[0, 0] = 0.0
    img[1, 1] = [2.0, -0.5, 1.0]  # clamps
    img[2, 2] = (np.array([100, 128, 200]) / 255.0) ** 2.2  # near the rounding boundaries
    return img, img * rng.uniform(0.8, 1.2, size=img.shape)


def test_film_equals_reference(oracle, tmp_path):
    for seed in (3, 5, 7):
        est, ref = _images(seed)
        m = oracle.film_ref(est, ref, str(tmp_path / "r.pfm"), str(tmp_path / "r.png"))
        film.write_pfm(est, str(tmp_path / "a.pfm"))
        film.write_png(est, str(tmp_path / "a.png"))
        assert (tmp_path / "a.pfm").read_bytes() == (tmp_path / "r.pfm").read_bytes()
        assert (tmp_path / "a.png").read_bytes() == (tmp_path / "r.png").read_bytes()
        rep = film.compare_images(est, ref)
        assert (rep.mape, rep.smape, rep.mse, rep.epsilon) == m
        back = film.read_pfm(str(tmp_path / "r.pfm"))
        assert np.array_equal(back, est.astype(np.float32).astype(np.float64))
    assert film.compare_images(ref, ref).mape == 0.0


def test_relmse():
    _, ref = _images(9)
    assert film.relmse(ref, ref) == 0.0
    assert abs(film.relmse(ref * 1.01, ref) - np.mean((0.01 * ref) ** 2 / (ref ** 2 + 1e-2))) < 1e-18
