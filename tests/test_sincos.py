"""sin / cos of the samplers' angles (include/pxg_sincos.h): the device returns glibc's
results bit for bit on phi = 2*pi*(k * 2^-32), the only angles the reference's samplers
produce (proj/src/bsdf.cpp:63-65, 226-227, proj/src/scene.cpp:199-201).

CPU: the table + correctly rounded evaluation (the same C code the device runs) equals this
host's glibc on bounded k ranges. GPU: the device equals the host glibc on every table entry
and 2^24 random draws, and the table is verified exhaustively on the GPU box's own libm.
"""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GEN = os.path.join(REPO, "paper_2503_23412_b200", "_build", "pxg_sincos_gen")
TABLE = os.path.join(REPO, "paper_2503_23412_b200", "pxg_sincos_glibc.bin")


def _verify(k0, k1):
    r = subprocess.run([GEN, "--verify", TABLE, str(k0), str(k1)], capture_output=True, text=True)
    assert r.stdout, r.stderr
    return json.loads(r.stdout), r.returncode


def _table_ks():
    """Every k listed in the table (glibc is not correctly rounded there)."""
    b = open(TABLE, "rb").read()
    n = int(np.frombuffer(b[4:8], np.uint32)[0])
    off = np.frombuffer(b[8 + 1024: 8 + 1024 + 4 * ((1 << 20) + 1)], np.uint32).astype(np.int64)
    ent = np.frombuffer(b[8 + 1024 + 4 * ((1 << 20) + 1):], np.uint16)
    assert ent.size == n == off[-1]
    bucket = np.repeat(np.arange(1 << 20, dtype=np.int64), np.diff(off))
    return ((bucket << 12) | (ent & 0xFFF)).astype(np.uint32), ent


def test_table_matches_glibc_on_sampled_ranges():
    # the start (small angles, glibc's least accurate range), a quadrant boundary and the end
    for k0 in (0, (1 << 30) - (1 << 21), (1 << 32) - (1 << 22)):
        out, rc = _verify(k0, k0 + (1 << 22))
        assert rc == 0 and out["differ"] == 0, out
        assert out["table_searches"] > 0


def test_table_lists_glibc_misroundings():
    ks, ent = _table_ks()
    assert ks.size > 1_000_000  # ~0.14% of the 2^32 angles per function
    assert np.all((ent >> 12) & 3)  # every entry flags sin or cos
    # entries are sorted within buckets and unique
    assert np.unique(ks).size == ks.size and np.all(np.diff(ks.astype(np.int64)) > 0)


def _host_glibc(ks):
    with tempfile.TemporaryDirectory() as d:
        kp, op = os.path.join(d, "k.u32"), os.path.join(d, "o.f64")
        ks.astype(np.uint32).tofile(kp)
        subprocess.run([GEN, "--eval", kp, op], check=True)
        o = np.fromfile(op, np.float64).reshape(-1, 2)
    return o[:, 0], o[:, 1]


@pytest.mark.gpu
def test_device_sincos_equals_host_glibc(pxg):
    from paper_2503_23412_b200.render import sincos_2pi
    ks, _ = _table_ks()
    rng = np.random.default_rng(5)
    ks = np.concatenate([ks, rng.integers(0, 1 << 32, size=1 << 24, dtype=np.uint64).astype(np.uint32),
                         np.array([0, 1, 0x40000000, 0x80000000, 0xC0000000, 0xFFFFFFFF], np.uint32)])
    s, c = sincos_2pi(ks)
    gs, gc = _host_glibc(ks)
    ds = np.count_nonzero(s.view(np.uint64) != gs.view(np.uint64))
    dc = np.count_nonzero(c.view(np.uint64) != gc.view(np.uint64))
    print(f"device vs host glibc: {ks.size} draws, sin differ {ds}, cos differ {dc}")
    assert ds == 0 and dc == 0


@pytest.mark.gpu
def test_table_exhaustive_on_this_host():
    """All 2^32 angles against the libm of the machine the reference runs on (the GPU box's
    host, where the oracle of the parity tests runs)."""
    out, rc = _verify(0, 1 << 32)
    print(json.dumps(out))
    assert rc == 0 and out["differ"] == 0
