"""bench.py contract on CPU: the reference arm (`--impl reference`, the unmodified reference
compiled by oracle/Makefile) prints one JSON line with the fields the driver reads, and the
config table covers every BASELINE.json config."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line(oracle):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "Msamples/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("C1: BASELINE.json configs[0]")


def test_config_table_covers_baseline():
    sys.path.insert(0, REPO)
    import bench
    with open(os.path.join(REPO, "BASELINE.json")) as f:
        n = len(json.load(f)["configs"])
    assert sorted(v[0] for v in bench.CONFIGS.values()) == list(range(n))


def test_reference_fit_path(oracle):
    """The two-resolution fit of the reference arm (C3-C5): steady pass times at W/8 and W/4,
    linear in the pixel count, extrapolated to the full size."""
    sys.path.insert(0, REPO)
    import bench
    from paper_2503_23412_b200 import scenes
    sc = scenes.caustic_box(160)
    value, sample, wall = bench.reference_rate("C3", sc, sc.n_px, 2)
    assert value > 0 and "20x20" in sample and "40x40" in sample and "160x160" in sample
