"""Python mirror of the reference's render API for the hot path, backed by libpxg.

`render_proxy_bdpt(scene, spp, seed, params, diagnostics, pass_done)` has the argument
meaning and error behaviour of proxima::render_proxy_bdpt
(proj/include/proxima/proxy.hpp:197-200, proj/src/proxy.cpp:647-834): spp <= 0 uses the
scene's settings; one pass is one sample for every pixel; `pass_done(done, mean_image)`
runs after each pass and returning False stops early (the result then equals a shorter
render); `diagnostics` (a ProxyDiagnostics) is filled in place. `render_bdpt` is the same
call with proxy sampling disabled (proj/tests/test_proxy.cpp:1053-1079).

Images are numpy float64 arrays of shape (height, width, 3), row 0 at the top, like the
reference's `Image` (proj/include/proxima/image.hpp:13-23).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib
from .scene import Scene

N_BUCKETS = 4000
MAX_LIGHT = 16  # PXG_MAX_LIGHT

# pxg_vertex / pxg_path_record (include/pxg.h): the device PathVertex and the replay record.
VERTEX_DTYPE = np.dtype([("p", "<f8", 3), ("n", "<f8", 3), ("wi", "<f8", 3), ("throughput", "<f8", 3),
                         ("pdf_fwd", "<f8"), ("material", "<i4"), ("primitive", "<i4"), ("emitter", "<i4"),
                         ("flag", "<i4"), ("reserved", "<f8")])
PATH_RECORD_DTYPE = np.dtype([("n_eye", "<i4"), ("n_light", "<i4"), ("tp", "<i4"), ("flags", "<i4"),
                              ("entry", "<i4"), ("u", "<i4"), ("n_prefix", "<i4"), ("has_cdir", "<i4"),
                              ("c_label", "<i4"), ("s_label", "<i4"), ("key", "<i4"), ("reserved", "<i4"),
                              ("cdir", "<f8", 3), ("prefix_pdf", "<f8"), ("inverse_p", "<f8"),
                              ("inverse_p_m2", "<f8"), ("retrace_density", "<f8"), ("q_sel", "<f8"),
                              ("bdpt", "<f8", 3), ("c", "<f8", 3), ("val", "<f8", 3)])
assert VERTEX_DTYPE.itemsize == 128 and PATH_RECORD_DTYPE.itemsize == 48 + 24 + 40 + 72


@dataclass
class ProxyParams:
    """proxima::ProxyParams (proj/include/proxima/proxy.hpp:162-173)."""
    enabled: bool = True
    pool_budget: int = 400
    recip_repeats: int = 5
    freeze_iteration: int = 40
    recursion_cap: int = 10000
    pretrace_paths: int = 20000
    light_walks: int = 0
    gate_high: float = 1.0
    gate_low: float = 0.2
    gate_threshold: float = 0.05

    def to_c(self) -> _lib.Params:
        p = _lib.Params()
        for f in fields(self):
            v = getattr(self, f.name)
            setattr(p, f.name, int(v) if f.name == "enabled" else v)
        return p


@dataclass
class ProxyDiagRow:
    """proxima::ProxyDiagRow (proj/include/proxima/proxy.hpp:175-181)."""
    retrace_attempts: int = 0
    retrace_accepts: int = 0
    recip_runs: int = 0
    recip_truncated: int = 0
    estimates_failed: int = 0


def key_of(index: int):
    """Dense bucket index -> StatsKey (u, c, s)."""
    return (index // 1000 + 1, (index // 100) % 10, index % 100)


def index_of(u: int, c: int, s: int) -> int:
    return ((u - 1) * 10 + c) * 100 + s


@dataclass
class ProxyDiagnostics:
    """proxima::ProxyDiagnostics (proj/include/proxima/proxy.hpp:183-188)."""
    rows: dict = field(default_factory=dict)
    pool_raw: int = 0
    pool_kept: int = 0

    def write_csv(self, f) -> None:
        """ProxyDiagnostics::write_csv (proj/src/proxy.cpp:605-614)."""
        f.write("u,c,s,retrace_attempts,retrace_accepts,recip_runs,recip_truncated,estimates_failed\n")
        for (u, c, s) in sorted(self.rows):
            r = self.rows[(u, c, s)]
            f.write(f"{u},{c},{s},{r.retrace_attempts},{r.retrace_accepts},{r.recip_runs},"
                    f"{r.recip_truncated},{r.estimates_failed}\n")
        f.write(f"# pool_raw={self.pool_raw} pool_kept={self.pool_kept}\n")


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _lp(a):
    return a.ctypes.data_as(C.POINTER(C.c_longlong))


_FINALIZE_ENV = ("PXG_NODEQ", "PXG_LEAF", "PXG_SAH_BINS")  # host BVH build knobs (A/B experiments)


class FinalizedScene:
    """A pxg_scene handle: the scene validated, with emitter tables and BVH (include/pxg.h)."""

    def __init__(self, scene: Scene):
        import os
        L = _lib.lib()
        self.key = _finalize_key(scene)
        keep = dict(
            shape=np.ascontiguousarray(scene.shape, np.int32), mat=np.ascontiguousarray(scene.mat, np.int32),
            a=np.ascontiguousarray(scene.a, np.float64), b=np.ascontiguousarray(scene.b, np.float64),
            c=np.ascontiguousarray(scene.c, np.float64), r=np.ascontiguousarray(scene.radius, np.float64),
            m=np.ascontiguousarray(scene.material_table()[:, :7], np.float64),
            ep=np.ascontiguousarray(scene.emitter_prim, np.int32),
            er=np.ascontiguousarray(scene.emitter_radiance, np.float64))
        d = _lib.SceneDesc()
        d.n_prims = scene.n_prims
        d.shape, d.material = _ip(keep["shape"]), _ip(keep["mat"])
        d.a, d.b, d.c, d.radius = _dp(keep["a"]), _dp(keep["b"]), _dp(keep["c"]), _dp(keep["r"])
        d.n_materials = len(scene.materials)
        d.materials = _dp(keep["m"])
        d.n_emitters = int(keep["ep"].shape[0])
        d.emitter_prim, d.emitter_radiance = _ip(keep["ep"]), _dp(keep["er"])
        d.cam_position[:] = scene.camera.position
        d.cam_look_at[:] = scene.camera.look_at
        d.cam_up[:] = scene.camera.up
        d.fov_y = scene.camera.fov_y
        d.width, d.height = scene.camera.width, scene.camera.height
        d.max_depth = scene.settings.max_depth
        h = C.c_void_p()
        _lib.check(L.pxg_scene_create(C.byref(d), C.byref(h)), None)
        self._h = h
        self._L = L

    @property
    def handle(self):
        return self._h

    def device_bytes(self) -> int:
        """Bytes a context uploads from this scene (pxg_scene_device_bytes)."""
        return int(self._L.pxg_scene_device_bytes(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._L.pxg_scene_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _finalize_key(scene: Scene):
    import os
    cam = scene.camera
    return (tuple(os.environ.get(k) for k in _FINALIZE_ENV), tuple(cam.position), tuple(cam.look_at), tuple(cam.up),
            cam.fov_y, cam.width, cam.height, scene.settings.max_depth, scene.n_prims, len(scene.materials),
            id(scene.a), id(scene.shape), id(scene.emitter_prim))


def finalized_scene(scene: Scene) -> FinalizedScene:
    """The scene's pxg_scene, built on first use and kept on the Scene object (the reference
    keeps its BVH in the Scene after finalize)."""
    f = getattr(scene, "_pxg_finalized", None)
    if f is None or f.key != _finalize_key(scene):
        f = FinalizedScene(scene)
        scene._pxg_finalized = f
    return f


class ProxyRenderer:
    """One libpxg context: the scene resident in HBM, the per-pass state, the film."""

    def __init__(self, scene: Scene, seed: int, params: ProxyParams | None = None, device: int = 0,
                 rows: tuple | None = None, walks: tuple | None = None):
        L = _lib.lib()
        self.scene = scene
        self.params = params or ProxyParams()
        W, H = scene.camera.width, scene.camera.height
        self.width, self.height, self.max_depth = W, H, scene.settings.max_depth
        fin = finalized_scene(scene)
        cp = self.params.to_c()
        shard = None
        light_walks = self.params.light_walks if self.params.light_walks > 0 else W * H
        if rows is not None or walks is not None:
            r0, r1 = rows if rows is not None else (0, H)
            w0, w1 = walks if walks is not None else (0, light_walks)
            shard = _lib.Shard(r0, r1, w0, w1)
        self.row0, self.row1 = (rows if rows is not None else (0, H))
        ctx = C.c_void_p()
        rc = L.pxg_create_from_scene(fin.handle, C.byref(cp), C.c_uint64(seed), device,
                                     C.byref(shard) if shard is not None else None, C.byref(ctx))
        _lib.check(rc, None)
        self._fin = fin  # the context was built from it; keep it alive with the renderer
        self._ctx = ctx
        self._L = L

    # -- lifecycle
    def close(self):
        if getattr(self, "_ctx", None):
            self._L.pxg_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def n(self):
        return (self.row1 - self.row0) * self.width

    def _check(self, rc):
        _lib.check(rc, self._ctx)

    # -- passes
    def render_passes(self, n: int = 1):
        self._check(self._L.pxg_render_passes(self._ctx, n))

    def render_passes_async(self, n: int = 1):
        """Enqueue n passes without waiting for them (see snapshot / read_snapshot)."""
        self._check(self._L.pxg_render_passes_async(self._ctx, n))

    def snapshot(self, slot: int):
        self._check(self._L.pxg_snapshot_mean(self._ctx, slot))

    def read_snapshot(self, slot: int) -> np.ndarray:
        out = np.zeros((self.row1 - self.row0, self.width, 3))
        done = C.c_int()
        self._check(self._L.pxg_read_snapshot(self._ctx, slot, _dp(out), C.byref(done)))
        return out

    def synchronize(self):
        """Waits for every pass enqueued on the context (pxg_synchronize)."""
        self._check(self._L.pxg_synchronize(self._ctx))

    def set_pass_limit(self, limit: int):
        """No look-ahead Stage 1 for passes >= limit (the render's spp)."""
        self._check(self._L.pxg_set_pass_limit(self._ctx, int(limit)))

    def node_bytes(self) -> int:
        """Bytes per BVH node visit of this context's persistent traversal (pxg_node_bytes)."""
        return int(self._L.pxg_node_bytes(self._ctx))

    def measure_traversal(self, n: int = 1) -> dict:
        """Render n passes with every traversal launch timed by CUDA events and its work
        counted by an instrumented copy on the same rays (roofline numerator)."""
        out = np.zeros(10)
        self._check(self._L.pxg_measure_traversal(self._ctx, n, _dp(out)))
        keys = ["ms", "launches", "rays", "nodes", "prims"]
        return {"closest": dict(zip(keys, out[:5].tolist())), "anyhit": dict(zip(keys, out[5:].tolist()))}

    def render_pass_traced(self):
        """One pass that also records the sub-path primitive ids (dump_prims)."""
        self._check(self._L.pxg_render_pass_traced(self._ctx))

    def mean(self) -> np.ndarray:
        out = np.zeros((self.row1 - self.row0, self.width, 3))
        done = C.c_int()
        self._check(self._L.pxg_read_mean(self._ctx, _dp(out), C.byref(done)))
        return out

    def passes_done(self) -> int:
        done = C.c_int()
        tmp = np.zeros((self.row1 - self.row0, self.width, 3))
        self._check(self._L.pxg_read_accum(self._ctx, _dp(tmp), C.byref(done)))
        return done.value

    def accum(self):
        out = np.zeros((self.row1 - self.row0, self.width, 3))
        done = C.c_int()
        self._check(self._L.pxg_read_accum(self._ctx, _dp(out), C.byref(done)))
        return out, done.value

    def accum_to_device(self, ptr: int, stream: int | None = None) -> int:
        """Copy the fp64 accumulator (H_shard x W x 3) into device memory at `ptr`, ordered
        after the work on CUDA stream `stream` (a cudaStream_t handle, e.g.
        torch.cuda.current_stream().cuda_stream) and before the work enqueued on it next.
        stream=None: the legacy default stream, and the call waits for the copy."""
        done = C.c_int()
        if stream is None:
            self._check(self._L.pxg_accum_to_device(self._ctx, C.c_void_p(ptr), C.byref(done)))
        else:
            self._check(self._L.pxg_accum_to_device_async(self._ctx, C.c_void_p(ptr), C.c_void_p(stream),
                                                          C.byref(done)))
        return done.value

    def timing(self):
        t = np.zeros(8)
        cnt = np.zeros(2, np.int64)
        self._check(self._L.pxg_read_timing(self._ctx, _dp(t), _lp(cnt)))
        return t, cnt

    def recip_counts(self):
        """Reciprocal tree nodes evaluated ahead of the DFS, nodes the runs consumed, runs
        (pxg_read_recip_counts): the waste of the round schedule is evaluated / consumed."""
        out = np.zeros(3, np.int64)
        self._check(self._L.pxg_read_recip_counts(self._ctx, _lp(out)))
        return {"evaluated": int(out[0]), "consumed": int(out[1]), "runs": int(out[2])}

    def diagnostics(self) -> ProxyDiagnostics:
        rows = np.zeros((N_BUCKETS, 5), np.int64)
        touched = np.zeros(N_BUCKETS, np.int32)
        pool = np.zeros(2, np.int64)
        self._check(self._L.pxg_read_diag(self._ctx, _lp(rows), _ip(touched), _lp(pool)))
        d = ProxyDiagnostics(pool_raw=int(pool[0]), pool_kept=int(pool[1]))
        for k in np.nonzero(touched)[0]:
            d.rows[key_of(int(k))] = ProxyDiagRow(*[int(v) for v in rows[k]])
        return d

    def stats(self):
        s3 = np.zeros((N_BUCKETS, 3))
        c2 = np.zeros((N_BUCKETS, 2), np.int64)
        g = np.zeros((32, 100))
        self._check(self._L.pxg_read_stats(self._ctx, _dp(s3), _lp(c2), _dp(g)))
        return s3, c2, g

    def dump_pass(self):
        n = self.n
        val, bd, c = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3))
        fl = np.zeros(n, np.int32)
        self._check(self._L.pxg_dump_pass(self._ctx, _dp(val), _dp(bd), _dp(c), _ip(fl)))
        return val, bd, c, fl

    def dump_prims(self):
        n = self.n
        eye = np.zeros((n, self.max_depth + 1), np.int32)
        light = np.zeros((n, max(self.max_depth - 1, 1)), np.int32)
        self._check(self._L.pxg_dump_prims(self._ctx, _ip(eye), _ip(light)))
        return eye, light

    def dump_pool(self, cap: int = 4096):
        n = C.c_int()
        raw = C.c_longlong()
        walk, end, key = (np.zeros(cap, np.int32) for _ in range(3))
        ip, m2, bd = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        self._check(self._L.pxg_dump_pool(self._ctx, cap, C.byref(n), C.byref(raw), _ip(walk), _ip(end), _ip(key),
                                          _dp(ip), _dp(m2), _dp(bd)))
        k = min(n.value, cap)
        return dict(n=n.value, raw=raw.value, walk=walk[:k], end=end[:k], key=key[:k], inv_p=ip[:k],
                    inv_p_m2=m2[:k], bound=bd[:k])

    def dump_paths(self, px_begin: int = 0, px_end: int | None = None):
        """Replay dump of the last pass (pxg_dump_paths): per-pixel records (PATH_RECORD_DTYPE),
        eye [m, max_depth+1] / light [m, max_depth-1] / proxy [m, PXG_MAX_LIGHT] vertices
        (VERTEX_DTYPE) and the pass's statistics snapshot [4000, 3] (sum_est, sum_est_sq,
        est_count)."""
        px_end = self.n if px_end is None else px_end
        m = max(px_end - px_begin, 0)
        rec = np.zeros(m, PATH_RECORD_DTYPE)
        eye = np.zeros((m, self.max_depth + 1), VERTEX_DTYPE)
        light = np.zeros((m, max(self.max_depth - 1, 1)), VERTEX_DTYPE)
        proxy = np.zeros((m, MAX_LIGHT), VERTEX_DTYPE)
        stats = np.zeros((N_BUCKETS, 3))
        self._check(self._L.pxg_dump_paths(self._ctx, px_begin, px_end, rec.ctypes.data, eye.ctypes.data,
                                           light.ctypes.data, proxy.ctypes.data, _dp(stats)))
        return rec, eye, light, proxy, stats

    # -- traversal parity entry points (Scene::intersect / Scene::occluded)
    def intersect(self, rays: np.ndarray, tmax=None):
        rays = np.ascontiguousarray(rays, np.float64)
        n = rays.shape[0]
        prim = np.zeros(n, np.int32)
        t = np.zeros(n)
        tm = None if tmax is None else np.ascontiguousarray(np.broadcast_to(tmax, (n,)), np.float64)
        self._check(self._L.pxg_intersect(self._ctx, n, _dp(rays), _dp(tm) if tm is not None else None, _ip(prim),
                                          _dp(t)))
        return prim, t

    def render_pt(self, spp: int, seed: int, chunks: int = 1) -> np.ndarray:
        """proxima::render_pt (proj/src/transport.cpp:376-381) on the device for this
        context's pixels; `chunks` > 1 averages independent renders (see include/pxg.h)."""
        if spp <= 0:
            spp = self.scene.settings.spp
        out = np.zeros((self.n, 3))
        self._check(self._L.pxg_render_pt(self._ctx, spp, seed & (2**64 - 1), chunks, _dp(out)))
        return out.reshape(-1, self.scene.camera.width, 3)

    def occluded(self, segs: np.ndarray):
        segs = np.ascontiguousarray(segs, np.float64)
        occ = np.zeros(segs.shape[0], np.int32)
        self._check(self._L.pxg_occluded(self._ctx, segs.shape[0], _dp(segs), _ip(occ)))
        return occ.astype(bool)

    def trace_rays(self, kernel: int, rays: np.ndarray, tmax=None, any_hit: bool = False):
        """The same rays through a chosen traversal kernel (include/pxg.h pxg_trace_rays):
        0 single-ray paths, 1 the production persistent kernels, 2 the reciprocal
        wavefront's inlined step loops. Returns (prim, t) or the occlusion booleans."""
        rays = np.ascontiguousarray(rays, np.float64)
        n = rays.shape[0]
        prim = np.zeros(n, np.int32)
        t = np.zeros(n)
        tm = None if (tmax is None or any_hit) else np.ascontiguousarray(np.broadcast_to(tmax, (n,)), np.float64)
        self._check(self._L.pxg_trace_rays(self._ctx, kernel, int(any_hit), n, _dp(rays),
                                           _dp(tm) if tm is not None else None, _ip(prim), _dp(t)))
        return prim.astype(bool) if any_hit else (prim, t)


    def proxy_probe(self, walk: np.ndarray, cand: np.ndarray | None = None, n_draws: int = 0, seed: int = 0):
        """dropout, support_pdf, target_density and support_sample on the device for a
        caller-built light walk (pxg_proxy_probe; VERTEX_DTYPE records). Returns a dict:
        info (valid, u, n_prefix, has_cdir, c_label, s_label, key, dropped flag), prefix_pdf,
        q / f per candidate block cand[i, :u], and n_draws support samples (cand, q, escaped)."""
        walk = np.ascontiguousarray(walk, VERTEX_DTYPE)
        info = np.zeros(8, np.int32)
        pp = np.zeros(1)
        nc = 0 if cand is None else cand.shape[0]
        cflat = None if cand is None else np.ascontiguousarray(cand, VERTEX_DTYPE)
        q, f = np.zeros(max(nc, 1)), np.zeros(max(nc, 1))
        dc = np.zeros((max(n_draws, 1), 4), VERTEX_DTYPE)
        dq = np.zeros(max(n_draws, 1))
        de = np.zeros(max(n_draws, 1), np.int32)
        # the draw buffer is sized for u = 4 and re-read at the walk's u below
        self._check(self._L.pxg_proxy_probe(self._ctx, len(walk), walk.ctypes.data, nc,
                                            cflat.ctypes.data if nc else None, n_draws, seed, _ip(info), _dp(pp),
                                            _dp(q), _dp(f), dc.ctypes.data, _dp(dq), _ip(de)))
        u = int(info[1]) if info[0] else 0
        draws = dc.reshape(-1)[:n_draws * u].reshape(n_draws, u) if u else dc[:0]
        return {"info": info, "prefix_pdf": float(pp[0]), "q": q[:nc], "f": f[:nc], "draw_cand": draws,
                "draw_q": dq[:n_draws], "draw_escaped": de[:n_draws].astype(bool)}


    def proxy_recip(self, walk: np.ndarray, bound: float, n_runs: int):
        """n_runs reciprocal runs for the incomplete sub-path of `walk` at a fixed bound, through
        the production node wavefront and DFS (pxg_proxy_recip). Returns (est, cost, truncated)."""
        walk = np.ascontiguousarray(walk, VERTEX_DTYPE)
        est = np.zeros(n_runs)
        cost = np.zeros(n_runs, np.int64)
        tr = np.zeros(n_runs, np.int32)
        self._check(self._L.pxg_proxy_recip(self._ctx, len(walk), walk.ctypes.data, float(bound), n_runs, _dp(est),
                                            _lp(cost), _ip(tr)))
        return est, cost, tr.astype(bool)


SNAPSHOT_SLOTS = 4   # PXG_SNAPSHOT_SLOTS (include/pxg.h)
PIPELINE_AHEAD = 3   # passes in flight in the pipelined pass_done loop (< SNAPSHOT_SLOTS)


def render_proxy_bdpt(scene: Scene, spp: int, seed: int, params: ProxyParams | None = None,
                      diagnostics: ProxyDiagnostics | None = None, pass_done=None, device: int = 0) -> np.ndarray:
    """proxima::render_proxy_bdpt on the GPU (proj/src/proxy.cpp:647-834)."""
    if spp <= 0:
        spp = scene.settings.spp
    with ProxyRenderer(scene, seed, params, device=device) as r:
        r.set_pass_limit(spp)
        if pass_done is None:
            r.render_passes(spp)
            img = r.mean()
        elif diagnostics is None:
            # pipelined: passes k+1 .. k+AHEAD-1 are already enqueued while pass_done sees the
            # mean after k, so the GPU never drains while the host reads back and runs the
            # callback; an early stop returns that snapshot (bitwise the k-pass image) and
            # discards the passes rendered beyond it
            ahead = min(PIPELINE_AHEAD, spp)
            for j in range(ahead):
                r.render_passes_async(1)
                r.snapshot(j % SNAPSHOT_SLOTS)
            img = None
            for k in range(1, spp + 1):
                j = k + ahead - 1  # next pass index to enqueue (0-based)
                if j < spp:
                    r.render_passes_async(1)
                    r.snapshot(j % SNAPSHOT_SLOTS)
                img = r.read_snapshot((k - 1) % SNAPSHOT_SLOTS)
                if not pass_done(k, img):
                    break
        else:
            # diagnostics must not include a pass beyond an early stop: one pass at a time
            for _ in range(spp):
                r.render_passes(1)
                if not pass_done(r.passes_done(), r.mean()):
                    break
            img = r.mean()
        if diagnostics is not None:
            d = r.diagnostics()
            diagnostics.rows = d.rows
            diagnostics.pool_raw = d.pool_raw
            diagnostics.pool_kept = d.pool_kept
    return img


def render_bdpt(scene: Scene, spp: int, seed: int, device: int = 0) -> np.ndarray:
    """proxima::render_bdpt (proj/src/transport.cpp:380-386): the proxy renderer with proxy off."""
    return render_proxy_bdpt(scene, spp, seed, ProxyParams(enabled=False), device=device)


def render_pt(scene: Scene, spp: int, seed: int, chunks: int = 1, device: int = 0) -> np.ndarray:
    """proxima::render_pt(scene, spp, seed) (proj/include/proxima/transport.hpp:88) on the GPU."""
    with ProxyRenderer(scene, seed, ProxyParams(enabled=False), device=device) as r:
        return r.render_pt(spp, seed, chunks)


def recip_twopoint(n: int, bound: float, cap: int = 10000, seed: int = 1):
    """The device reciprocal estimator on the reference's two-point fixture."""
    L = _lib.lib()
    est = np.zeros(n)
    cost = np.zeros(n, np.int64)
    tr = np.zeros(n, np.int32)
    _lib.check(L.pxg_recip_twopoint(n, bound, cap, seed, _dp(est), _lp(cost), _ip(tr)))
    return est, cost, tr.astype(bool)


def rng_draws(seed: int, kind: int, sub: int, stream: int, n: int) -> np.ndarray:
    L = _lib.lib()
    out = np.zeros(n, np.uint32)
    _lib.check(L.pxg_rng_draws(seed, kind, sub, stream, n, out.ctypes.data_as(C.POINTER(C.c_uint))))
    return out


def sincos_2pi(k: np.ndarray, device: int = 0):
    """sin / cos of phi = 2*pi*(k * 2^-32) on the device, with the samplers' code path
    (bitwise the host glibc's, include/pxg_sincos.h)."""
    L = _lib.lib()
    k = np.ascontiguousarray(k, dtype=np.uint32)
    s = np.zeros(k.size)
    c = np.zeros(k.size)
    _lib.check(L.pxg_sincos_2pi(device, k.size, k.ctypes.data_as(C.POINTER(C.c_uint)), _dp(s), _dp(c)))
    return s, c
