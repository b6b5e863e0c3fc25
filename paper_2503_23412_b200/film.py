"""Film IO and image metrics around the render loop.

Host-side mirror of the reference's image output and comparison, byte for byte:
  write_pfm / read_pfm   proj/src/image.cpp:16-50   (PF, little-endian scale -1.0, rows
                                                      written bottom-up, fp32 RGB)
  write_png              proj/src/image.cpp:71-108  (8-bit RGB, gamma 1/2.2, clamp [0,1],
                                                      round half away from zero, filter 0,
                                                      zlib level 6)
  compare_images         proj/src/metrics.cpp:11-36 (MAPE / SMAPE / MSE over luminance with
                                                      the floor 1e-2 * mean reference
                                                      luminance)
plus relmse, the converged-image metric of the north star (not in the reference).

Images are numpy arrays [h][w][3] (fp64), y = 0 the top row, as render_proxy_bdpt returns.
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass

import numpy as np


def luminance(rgb: np.ndarray) -> np.ndarray:
    """proj/include/proxima/vec.hpp:50 (same fp64 operation order)."""
    return 0.2126 * rgb[..., 0] + 0.7152 * rgb[..., 1] + 0.0722 * rgb[..., 2]


def write_pfm(img: np.ndarray, path: str) -> None:
    h, w, _ = img.shape
    with open(path, "wb") as f:
        f.write(f"PF\n{w} {h}\n-1.0\n".encode())
        f.write(np.ascontiguousarray(img[::-1].astype("<f4")).tobytes())


def read_pfm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    toks, pos = [], 0
    while len(toks) < 4:  # magic, w, h, scale separated by whitespace (operator>> semantics)
        while data[pos:pos + 1].isspace():
            pos += 1
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        toks.append(data[start:pos].decode())
    magic, w, h, scale = toks[0], int(toks[1]), int(toks[2]), float(toks[3])
    if magic != "PF" or w <= 0 or h <= 0:
        raise RuntimeError(f"not a color PFM: {path}")
    if scale >= 0.0:
        raise RuntimeError(f"big-endian PFM unsupported: {path}")
    pos += 1  # single whitespace after the header
    need = w * h * 3 * 4
    if len(data) - pos < need:
        raise RuntimeError(f"truncated PFM: {path}")
    px = np.frombuffer(data, "<f4", w * h * 3, pos).reshape(h, w, 3)
    return px[::-1].astype(np.float64)


def _to_srgb8(v: np.ndarray) -> np.ndarray:
    g = np.power(np.clip(v, 0.0, 1.0), 1.0 / 2.2)
    x = g * 255.0
    r = np.floor(x)
    return (r + (x - r >= 0.5)).astype(np.uint8)  # std::lround (half away from zero), x >= 0


def _chunk(tag: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + tag + data + struct.pack(">I", zlib.crc32(tag + data) & 0xFFFFFFFF)


def write_png(img: np.ndarray, path: str) -> None:
    h, w, _ = img.shape
    rows = np.concatenate([np.zeros((h, 1), np.uint8), _to_srgb8(img).reshape(h, 3 * w)], axis=1)
    z = zlib.compress(rows.tobytes(), 6)
    ihdr = struct.pack(">II", w, h) + b"\x08\x02\x00\x00\x00"
    png = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", z) + _chunk(b"IEND", b"")
    with open(path, "wb") as f:
        f.write(png)


@dataclass
class MetricReport:
    """proj/include/proxima/image.hpp:33-38"""
    mape: float = 0.0
    smape: float = 0.0
    mse: float = 0.0
    epsilon: float = 0.0


def compare_images(estimate: np.ndarray, reference: np.ndarray) -> MetricReport:
    if estimate.shape != reference.shape:
        raise RuntimeError("compare: image dimensions differ")
    n = reference.shape[0] * reference.shape[1]
    if n == 0:
        raise RuntimeError("compare: empty image")
    lb = luminance(reference).ravel()
    la = luminance(estimate).ravel()
    ref_mean = 0.0
    for v in lb.tolist():  # the reference's sequential sum
        ref_mean += v
    ref_mean /= n
    eps = 1e-2 * ref_mean
    diff = np.abs(la - lb)
    rep = MetricReport(epsilon=eps)
    mape_t = diff / np.maximum(lb, eps)
    smape_t = 2.0 * diff / np.maximum(la + lb, eps)
    mse_t = (la - lb) * (la - lb)
    for a, b, c in zip(mape_t.tolist(), smape_t.tolist(), mse_t.tolist()):
        rep.mape += a
        rep.smape += b
        rep.mse += c
    rep.mape /= n
    rep.smape /= n
    rep.mse /= n
    return rep


def relmse(estimate: np.ndarray, reference: np.ndarray, eps: float = 1e-2) -> float:
    """Relative MSE over pixels and channels: mean((x - r)^2 / (r^2 + eps))."""
    return float(np.mean((estimate - reference) ** 2 / (reference ** 2 + eps)))
