"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes front-end of oracle/_ref/liboracle*.so.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl reference)
may import this module. It is the checker, never the thing measured or shipped.

liboracle.so is the unmodified reference library (proj/src/*.cpp) compiled with the Philox
shadow rng.hpp, plus oracle/src/oracle_driver.cpp (the restated render loop).
liboracle_pcg.so is the reference as shipped (PCG32) and only exposes the unmodified
renderers; bench.py times it as the reference CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
N_BUCKETS = 4000


# OrcVertex / OrcProxyIn / OrcProxyOut of oracle_driver.cpp (replay parity); OrcVertex has the
# byte layout of the device's pxg_vertex (include/pxg.h)
VERTEX_DTYPE = np.dtype([("p", "<f8", 3), ("n", "<f8", 3), ("wi", "<f8", 3), ("throughput", "<f8", 3),
                         ("pdf_fwd", "<f8"), ("material", "<i4"), ("primitive", "<i4"), ("emitter", "<i4"),
                         ("flag", "<i4"), ("reserved", "<f8")])
REPLAY_IN_DTYPE = np.dtype([("tp", "<i4"), ("u", "<i4"), ("n_prefix", "<i4"), ("has_cdir", "<i4"),
                            ("cdir", "<f8", 3), ("prefix_pdf", "<f8"), ("inverse_p", "<f8")])
REPLAY_OUT_DTYPE = np.dtype([("prefix_pdf", "<f8"), ("retrace_density", "<f8"), ("weight", "<f8"),
                             ("c", "<f8", 3), ("s_label", "<i4"), ("c_label", "<i4"), ("pad", "<i4", 2)])


class OracleUnavailable(RuntimeError):
    pass


class OrcParams(C.Structure):
    _fields_ = [
        ("enabled", C.c_int),
        ("pool_budget", C.c_int),
        ("recip_repeats", C.c_int),
        ("freeze_iteration", C.c_int),
        ("recursion_cap", C.c_longlong),
        ("pretrace_paths", C.c_int),
        ("light_walks", C.c_int),
        ("gate_high", C.c_double),
        ("gate_low", C.c_double),
        ("gate_threshold", C.c_double),
    ]


_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int)
_LP = C.POINTER(C.c_longlong)


class OrcTrace(C.Structure):
    _fields_ = [
        ("n_passes_cap", C.c_int),
        ("pass_val", _DP),
        ("pass_bdpt", _DP),
        ("pass_c", _DP),
        ("pass_flags", _IP),
        ("trace_pass", C.c_int),
        ("eye_prims", _IP),
        ("light_prims", _IP),
        ("pool_cap", C.c_int),
        ("pool_raw", _LP),
        ("pool_n", _IP),
        ("pool_walk", _IP),
        ("pool_end", _IP),
        ("pool_key", _IP),
        ("pool_inv_p", _DP),
        ("pool_inv_p_m2", _DP),
        ("pool_bound", _DP),
        ("pretrace_max", _DP),
        ("pretrace_cnt", _LP),
        ("stats_out", _DP),
        ("stats_cnt", _LP),
        ("gamma_rows", _DP),
        ("diag", _LP),
        ("diag_pool", _LP),
    ]


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


_libs: dict = {}


def lib(variant: str = "philox"):
    name = "liboracle.so" if variant == "philox" else "liboracle_pcg.so"
    if name in _libs:
        return _libs[name]
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        raise OracleUnavailable(f"{path} missing: run `make -C oracle` where /root/reference exists")
    L = C.CDLL(path, mode=C.RTLD_LOCAL)
    L.orc_last_error.restype = C.c_char_p
    L.orc_scene_load.restype = C.c_void_p
    L.orc_scene_load.argtypes = [C.c_char_p]
    L.orc_scene_free.argtypes = [C.c_void_p]
    L.orc_scene_info.argtypes = [C.c_void_p, _IP, _DP]
    L.orc_intersect.argtypes = [C.c_void_p, C.c_int, _DP, _DP, _IP, _DP, C.c_int]
    L.orc_occluded.argtypes = [C.c_void_p, C.c_int, _DP, _IP, C.c_int]
    L.orc_render_bdpt.argtypes = [C.c_void_p, C.c_int, C.c_ulonglong, _DP]
    L.orc_render_pt.argtypes = [C.c_void_p, C.c_int, C.c_ulonglong, _DP]
    L.orc_render_proxy_ref.argtypes = [C.c_void_p, C.c_int, C.c_ulonglong, C.POINTER(OrcParams), _DP, _LP]
    L.orc_render_proxy_ref_mt.argtypes = [C.c_void_p, C.c_int, C.c_ulonglong, C.POINTER(OrcParams), C.c_int, _DP,
                                          _DP]
    L.orc_render_proxy_ref_timed.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_ulonglong, C.POINTER(OrcParams),
                                             C.c_int, _DP]
    L.orc_scene_with_resolution.restype = C.c_void_p
    L.orc_scene_with_resolution.argtypes = [C.c_void_p, C.c_int, C.c_int]
    if variant == "philox":
        L.orc_render.argtypes = [C.c_void_p, C.c_int, C.c_ulonglong, C.POINTER(OrcParams), C.c_int, _DP,
                                 C.POINTER(OrcTrace)]
        L.orc_recip_twopoint.argtypes = [C.c_int, C.c_double, C.c_longlong, C.c_ulonglong, _DP, _LP, _IP]
        L.orc_replay_bdpt.argtypes = [C.c_void_p, C.c_int, C.c_void_p, _IP, C.c_int, C.c_void_p, _IP, C.c_int, _DP,
                                      C.c_int, _DP]
        L.orc_trace_subpaths.argtypes = [C.c_void_p, C.c_ulonglong, C.c_int, C.c_void_p, _IP, C.c_int, C.c_void_p,
                                         _IP, C.c_int, C.c_int]
        L.orc_replay_proxy.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                       _DP, C.c_int, C.c_void_p]
        L.orc_proxy_probe.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_ulonglong,
                                      _IP, _DP, _DP, _DP, C.c_void_p, _DP, _IP]
        L.orc_rng_draws.argtypes = [C.c_ulonglong, C.c_uint, C.c_uint, C.c_ulonglong, C.c_int,
                                    C.POINTER(C.c_uint)]
    _libs[name] = L
    return L


def film_ref(est: np.ndarray, ref: np.ndarray, pfm_path: str, png_path: str):
    """The reference's write_pfm / write_png of `est` and compare_images(est, ref)
    (proj/src/image.cpp, proj/src/metrics.cpp) via oracle/_ref/film_ref; returns
    (mape, smape, mse, epsilon)."""
    import subprocess
    import tempfile
    exe = os.path.join(REF_DIR, "film_ref")
    if not os.path.exists(exe):
        raise OracleUnavailable(f"{exe} missing: run `make -C oracle`")
    h, w = est.shape[:2]
    with tempfile.TemporaryDirectory() as d:
        pe, pr = os.path.join(d, "e.f64"), os.path.join(d, "r.f64")
        np.ascontiguousarray(est, np.float64).tofile(pe)
        np.ascontiguousarray(ref, np.float64).tofile(pr)
        out = subprocess.run([exe, str(w), str(h), pe, pr, pfm_path, png_path], capture_output=True, text=True,
                             check=True).stdout.split()
    return tuple(float(x) for x in out)


def _check(L, rc):
    if rc != 0:
        raise RuntimeError(L.orc_last_error().decode())


def make_params(p=None) -> OrcParams:
    """ProxyParams defaults of proj/include/proxima/proxy.hpp:162-173."""
    d = dict(enabled=1, pool_budget=400, recip_repeats=5, freeze_iteration=40, recursion_cap=10000,
             pretrace_paths=20000, light_walks=0, gate_high=1.0, gate_low=0.2, gate_threshold=0.05)
    if p is not None:
        for k in d:
            if hasattr(p, k):
                d[k] = getattr(p, k)
            elif isinstance(p, dict) and k in p:
                d[k] = p[k]
    d["enabled"] = int(bool(d["enabled"]))
    return OrcParams(**d)


class OracleScene:
    def __init__(self, json_text: str, variant: str = "philox"):
        self.L = lib(variant)
        h = self.L.orc_scene_load(json_text.encode())
        if not h:
            raise RuntimeError(self.L.orc_last_error().decode())
        self.h = C.c_void_p(h)
        ints = np.zeros(6, np.int32)
        dbl = np.zeros(7, np.float64)
        self.L.orc_scene_info(self.h, _ptr(ints, C.c_int), _ptr(dbl, C.c_double))
        self.width, self.height, self.max_depth, self.n_prims, self.n_emitters, self.spp = map(int, ints)
        self.total_emitter_area = float(dbl[0])
        self.bbox_min = dbl[1:4].copy()
        self.bbox_max = dbl[4:7].copy()

    def __del__(self):
        try:
            self.L.orc_scene_free(self.h)
        except Exception:
            pass

    @property
    def n_px(self):
        return self.width * self.height

    def intersect(self, rays: np.ndarray, tmax=None, threads: int = 8):
        rays = np.ascontiguousarray(rays, np.float64)
        n = rays.shape[0]
        prim = np.zeros(n, np.int32)
        t = np.zeros(n, np.float64)
        tm = None if tmax is None else np.ascontiguousarray(np.broadcast_to(tmax, (n,)), np.float64)
        _check(self.L, self.L.orc_intersect(self.h, n, _ptr(rays, C.c_double), _ptr(tm, C.c_double),
                                            _ptr(prim, C.c_int), _ptr(t, C.c_double), threads))
        return prim, t

    def occluded(self, segs: np.ndarray, threads: int = 8):
        segs = np.ascontiguousarray(segs, np.float64)
        occ = np.zeros(segs.shape[0], np.int32)
        _check(self.L, self.L.orc_occluded(self.h, segs.shape[0], _ptr(segs, C.c_double), _ptr(occ, C.c_int),
                                           threads))
        return occ.astype(bool)

    # -- replay parity (SURVEY §8c mode ii): device vertices rescored by the reference
    def replay_bdpt(self, eye, n_eye, light, n_light, stats3, threads: int = 8) -> np.ndarray:
        """weighted_bdpt_value (proj/src/proxy.cpp:621-643) of given sub-paths: eye [n, De] and
        light [n, Dl] vertex rows (pxg_vertex layout), stats3 [4000, 3] the pass's snapshot."""
        eye = np.ascontiguousarray(eye)
        light = np.ascontiguousarray(light)
        ne = np.ascontiguousarray(n_eye, np.int32)
        nl = np.ascontiguousarray(n_light, np.int32)
        s3 = np.ascontiguousarray(stats3, np.float64)
        n = eye.shape[0]
        out = np.zeros((n, 3))
        _check(self.L, self.L.orc_replay_bdpt(self.h, n, eye.ctypes.data, _ptr(ne, C.c_int), eye.shape[1],
                                              light.ctypes.data, _ptr(nl, C.c_int), light.shape[1],
                                              _ptr(s3, C.c_double), threads, _ptr(out, C.c_double)))
        return out

    def trace_subpaths(self, seed: int, n: int, threads: int = 8):
        """Pass 0's eye / light sub-paths of pixels [0, n) as the render loop traces them
        (proj/src/proxy.cpp:742-744), in the replay vertex layout."""
        eye = np.zeros((n, self.max_depth + 1), VERTEX_DTYPE)
        light = np.zeros((n, max(self.max_depth - 1, 1)), VERTEX_DTYPE)
        ne = np.zeros(n, np.int32)
        nl = np.zeros(n, np.int32)
        _check(self.L, self.L.orc_trace_subpaths(self.h, seed, n, eye.ctypes.data, _ptr(ne, C.c_int), eye.shape[1],
                                                 light.ctypes.data, _ptr(nl, C.c_int), light.shape[1], threads))
        return eye, ne, light, nl

    def proxy_probe(self, walk, cand=None, n_draws: int = 0, seed: int = 0):
        """The reference's dropout / support_pdf / target_density / support_sample
        (proj/src/proxy.cpp:59-269) on caller-built vertices: the checker of pxg_proxy_probe."""
        walk = np.ascontiguousarray(walk, VERTEX_DTYPE)
        info = np.zeros(8, np.int32)
        pp = np.zeros(1)
        nc = 0 if cand is None else cand.shape[0]
        cflat = None if cand is None else np.ascontiguousarray(cand, VERTEX_DTYPE)
        q, f = np.zeros(max(nc, 1)), np.zeros(max(nc, 1))
        dc = np.zeros((max(n_draws, 1), 4), VERTEX_DTYPE)
        dq = np.zeros(max(n_draws, 1))
        de = np.zeros(max(n_draws, 1), np.int32)
        _check(self.L, self.L.orc_proxy_probe(self.h, len(walk), walk.ctypes.data, nc,
                                              cflat.ctypes.data if nc else None, n_draws, seed, _ptr(info, C.c_int),
                                              _ptr(pp, C.c_double), _ptr(q, C.c_double), _ptr(f, C.c_double),
                                              dc.ctypes.data, _ptr(dq, C.c_double), _ptr(de, C.c_int)))
        u = int(info[1]) if info[0] else 0
        draws = dc.reshape(-1)[:n_draws * u].reshape(n_draws, u) if u else dc[:0]
        return {"info": info, "prefix_pdf": float(pp[0]), "q": q[:nc], "f": f[:nc], "draw_cand": draws,
                "draw_q": dq[:n_draws], "draw_escaped": de[:n_draws].astype(bool)}

    def replay_proxy(self, eye, tp, proxy, u, n_prefix, cdir, has_cdir, prefix_pdf, inverse_p, stats3,
                     threads: int = 8) -> np.ndarray:
        """proxy_pdf_components (proj/src/proxy.cpp:321-378), dropout labels and the
        proxy_connect value (proxy.cpp:562-602) of given proxy paths; returns REPLAY_OUT_DTYPE."""
        n = len(tp)
        inp = np.zeros(n, REPLAY_IN_DTYPE)
        inp["tp"], inp["u"], inp["n_prefix"], inp["has_cdir"] = tp, u, n_prefix, has_cdir
        inp["cdir"], inp["prefix_pdf"], inp["inverse_p"] = cdir, prefix_pdf, inverse_p
        out = np.zeros(n, REPLAY_OUT_DTYPE)
        eye = np.ascontiguousarray(eye)
        proxy = np.ascontiguousarray(proxy)
        s3 = np.ascontiguousarray(stats3, np.float64)
        _check(self.L, self.L.orc_replay_proxy(self.h, n, eye.ctypes.data, eye.shape[1], proxy.ctypes.data,
                                               proxy.shape[1], inp.ctypes.data, _ptr(s3, C.c_double), threads,
                                               out.ctypes.data))
        return out

    def render_bdpt(self, spp: int, seed: int) -> np.ndarray:
        out = np.zeros((self.height, self.width, 3))
        _check(self.L, self.L.orc_render_bdpt(self.h, spp, seed, _ptr(out, C.c_double)))
        return out

    def render_pt(self, spp: int, seed: int) -> np.ndarray:
        out = np.zeros((self.height, self.width, 3))
        _check(self.L, self.L.orc_render_pt(self.h, spp, seed, _ptr(out, C.c_double)))
        return out

    def render_proxy_ref(self, spp: int, seed: int, params=None):
        out = np.zeros((self.height, self.width, 3))
        rk = np.zeros(2, np.int64)
        op = make_params(params)
        _check(self.L, self.L.orc_render_proxy_ref(self.h, spp, seed, C.byref(op), _ptr(out, C.c_double),
                                                   _ptr(rk, C.c_longlong)))
        return out, int(rk[0]), int(rk[1])

    def render_proxy_ref_mt(self, spp: int, seed: int, copies: int, params=None, all_images: bool = False):
        """`copies` independent unmodified render_proxy_bdpt calls (seeds seed + i) on `copies`
        threads; returns copy 0's image, or all of them [copies, H, W, 3]."""
        out = np.zeros((self.height, self.width, 3))
        allimg = np.zeros((copies, self.height, self.width, 3)) if all_images else None
        op = make_params(params)
        _check(self.L, self.L.orc_render_proxy_ref_mt(self.h, spp, seed, C.byref(op), copies,
                                                      _ptr(out, C.c_double), _ptr(allimg, C.c_double)))
        return allimg if all_images else out

    def with_resolution(self, width: int, height: int) -> "OracleScene":
        """The same loaded scene rendered at another resolution (no reload)."""
        o = OracleScene.__new__(OracleScene)
        o.L = self.L
        h = self.L.orc_scene_with_resolution(self.h, width, height)
        if not h:
            raise RuntimeError(self.L.orc_last_error().decode())
        o.h = C.c_void_p(h)
        o.width, o.height = width, height
        o.max_depth, o.n_prims, o.n_emitters, o.spp = self.max_depth, self.n_prims, self.n_emitters, self.spp
        o.total_emitter_area, o.bbox_min, o.bbox_max = self.total_emitter_area, self.bbox_min, self.bbox_max
        return o

    def render_proxy_ref_timed(self, spp: int, seed: int, copies: int, params=None, scenes=None) -> np.ndarray:
        """`copies` concurrent unmodified render_proxy_bdpt calls of `spp` passes (copy i on
        scenes[i], default this scene); returns the pass end times [copies, spp] in seconds
        (pass_done callback timestamps from the common start)."""
        scenes = scenes or [self] * copies
        hs = (C.c_void_p * copies)(*[s.h.value for s in scenes])
        t = np.zeros((copies, spp))
        op = make_params(params)
        _check(self.L, self.L.orc_render_proxy_ref_timed(hs, spp, seed, C.byref(op), copies, _ptr(t, C.c_double)))
        return t

    def render(self, spp: int, seed: int, params=None, threads: int = 8, trace: bool = False,
               trace_pass: int = -1, pool_cap: int = 400):
        """Restated render loop (oracle_driver.cpp). Returns (image, OracleRun or None)."""
        out = np.zeros((self.height, self.width, 3))
        op = make_params(params)
        tr = None
        run = None
        if trace:
            P, N = spp, self.n_px
            run = OracleRun(
                pass_val=np.zeros((P, N, 3)), pass_bdpt=np.zeros((P, N, 3)), pass_c=np.zeros((P, N, 3)),
                pass_flags=np.zeros((P, N), np.int32),
                eye_prims=np.full((N, self.max_depth + 1), -3, np.int32),
                light_prims=np.full((N, max(self.max_depth - 1, 1)), -3, np.int32),
                pool_raw=np.zeros(P, np.int64), pool_n=np.zeros(P, np.int32),
                pool_walk=np.zeros((P, pool_cap), np.int32), pool_end=np.zeros((P, pool_cap), np.int32),
                pool_key=np.zeros((P, pool_cap), np.int32), pool_inv_p=np.zeros((P, pool_cap)),
                pool_inv_p_m2=np.zeros((P, pool_cap)), pool_bound=np.zeros((P, pool_cap)),
                pretrace_max=np.zeros(N_BUCKETS), pretrace_cnt=np.zeros(N_BUCKETS, np.int64),
                stats=np.zeros((N_BUCKETS, 3)), stats_cnt=np.zeros((N_BUCKETS, 2), np.int64),
                gamma_rows=np.zeros((32, 100)), diag=np.zeros((N_BUCKETS, 5), np.int64),
                diag_pool=np.zeros(2, np.int64))
            tr = OrcTrace(
                n_passes_cap=P, pass_val=_ptr(run.pass_val, C.c_double), pass_bdpt=_ptr(run.pass_bdpt, C.c_double),
                pass_c=_ptr(run.pass_c, C.c_double), pass_flags=_ptr(run.pass_flags, C.c_int),
                trace_pass=trace_pass, eye_prims=_ptr(run.eye_prims, C.c_int),
                light_prims=_ptr(run.light_prims, C.c_int), pool_cap=pool_cap,
                pool_raw=_ptr(run.pool_raw, C.c_longlong), pool_n=_ptr(run.pool_n, C.c_int),
                pool_walk=_ptr(run.pool_walk, C.c_int), pool_end=_ptr(run.pool_end, C.c_int),
                pool_key=_ptr(run.pool_key, C.c_int), pool_inv_p=_ptr(run.pool_inv_p, C.c_double),
                pool_inv_p_m2=_ptr(run.pool_inv_p_m2, C.c_double), pool_bound=_ptr(run.pool_bound, C.c_double),
                pretrace_max=_ptr(run.pretrace_max, C.c_double), pretrace_cnt=_ptr(run.pretrace_cnt, C.c_longlong),
                stats_out=_ptr(run.stats, C.c_double), stats_cnt=_ptr(run.stats_cnt, C.c_longlong),
                gamma_rows=_ptr(run.gamma_rows, C.c_double), diag=_ptr(run.diag, C.c_longlong),
                diag_pool=_ptr(run.diag_pool, C.c_longlong))
        _check(self.L, self.L.orc_render(self.h, spp, seed, C.byref(op), threads, _ptr(out, C.c_double),
                                         C.byref(tr) if tr is not None else None))
        return out, run


@dataclass
class OracleRun:
    pass_val: np.ndarray
    pass_bdpt: np.ndarray
    pass_c: np.ndarray
    pass_flags: np.ndarray
    eye_prims: np.ndarray
    light_prims: np.ndarray
    pool_raw: np.ndarray
    pool_n: np.ndarray
    pool_walk: np.ndarray
    pool_end: np.ndarray
    pool_key: np.ndarray
    pool_inv_p: np.ndarray
    pool_inv_p_m2: np.ndarray
    pool_bound: np.ndarray
    pretrace_max: np.ndarray
    pretrace_cnt: np.ndarray
    stats: np.ndarray
    stats_cnt: np.ndarray
    gamma_rows: np.ndarray
    diag: np.ndarray
    diag_pool: np.ndarray


def recip_twopoint(n: int, bound: float, cap: int = 10000, seed: int = 1):
    L = lib("philox")
    est = np.zeros(n)
    cost = np.zeros(n, np.int64)
    trunc = np.zeros(n, np.int32)
    _check(L, L.orc_recip_twopoint(n, bound, cap, seed, _ptr(est, C.c_double), _ptr(cost, C.c_longlong),
                                   _ptr(trunc, C.c_int)))
    return est, cost, trunc.astype(bool)


def rng_draws(seed: int, kind: int, sub: int, stream: int, n: int) -> np.ndarray:
    L = lib("philox")
    out = np.zeros(n, np.uint32)
    L.orc_rng_draws(seed, kind, sub, stream, n, out.ctypes.data_as(C.POINTER(C.c_uint)))
    return out
