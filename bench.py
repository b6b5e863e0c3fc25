"""Benchmark of the proxy-BDPT hot path (BASELINE.json metric: Msamples/s of full proxy-BDPT
pixel samples, with the fraction of the HBM traversal roofline).

One step = one progressive pass = one sample for every pixel of the workload: Stage 1 (pool
walks, priority selection, reciprocal estimates) + Stage 2 (eye/light sub-paths, all
standard strategies with reciprocal-aware MIS, the gated proxy connection, film, gamma).

Workload (N=1): BASELINE.json configs[3] ("C4"), the north star's 1M-triangle scene and the
largest single-GPU config: 1920x1080, max depth 12, 2,073,600 pool walks per pass (one per
pixel, the reference default), 2,000 seeded instances (1,011,340 triangles), 4 area lights,
Philox seed 0 -- a seeded synthetic scene (paper_2503_23412_b200/scenes.py) standing in for
the paper's proprietary scenes. L2: the per-pass working set (vertex pools, connection slots,
queues: tens of GB) is far larger than the 126 MB L2, and so is the ~200 MB scene.
The line also carries a C2 device measurement (configs[1]) as the extra key "C2".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C1..C5]

--impl reference times the reference's own CPU implementation (the unmodified
proxima::render_proxy_bdpt compiled from /root/reference by oracle/Makefile, PCG32 as
shipped) on the same config, one independent render per host core (see reference_rate).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Msamples/s (full proxy-BDPT px samples)"
PRIM_BYTES = 80  # PrimRec (csrc/pxg_scene.cuh); node bytes per context: pxg_node_bytes (64 or 128)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # default: passes 8..31 of the C4 render (BASELINE configs[3])
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="tuning sweeps: skip roofline, e2e and cpu_baseline")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra C2 device line of the C4 run")
    ap.add_argument("--e2e-spp", type=int, default=64,
                    help="spp of the end-to-end render call (capped at the config's spp)")
    return ap.parse_args()


CONFIGS = {
    # name: (BASELINE.json configs index, generator, kwargs, pool walks per pass; None = one
    # per pixel, the reference default n_px, proj/src/proxy.cpp:674)
    "C1": (0, "cornell_c1", dict(resolution=256, max_depth=8), 65536),
    "C2": (1, "cornell_c2", dict(resolution=512, max_depth=10), 262144),
    "C3": (2, "lens_room_c3", dict(resolution=1024, max_depth=12), None),
    "C4": (3, "procedural_c4", dict(width=1920, height=1080, max_depth=12), None),
    "C5": (4, "procedural_c5", dict(width=3840, height=2160, max_depth=16), 4 << 20),
}


def make_scene(cfg: str):
    from paper_2503_23412_b200 import scenes
    _, gen, kw, walks = CONFIGS[cfg]
    sc = getattr(scenes, gen)(**kw)
    return sc, (walks if walks is not None else sc.n_px)


def config_json(cfg, sc, walks):
    scene_mb = (sc.n_prims * 80 + 2 * sc.n_prims * 64) / 2**20  # primitive records + ~2 4-wide nodes/4 prims
    return {"workload": f"{cfg}: BASELINE.json configs[{CONFIGS[cfg][0]}], {sc.camera.width}x{sc.camera.height}, "
                        f"max_depth {sc.settings.max_depth}, {walks} pool walks/pass, {sc.n_prims} prims, proxy on",
            "step": "1 progressive pass (1 sample per pixel)",
            "spp": sc.settings.spp,
            "window": "warm-up passes 0..W-1 (W rounded up to the 8-pass Stage-1 batch), timed passes W..W+K-1 "
                      "of the config's render",
            "l2": ("inputs larger than L2: per-pass vertex pools/queues ~1 GB >> 126 MB L2 (scene itself "
                   "L2-resident)" if scene_mb < 60 else
                   f"inputs larger than L2: per-pass vertex pools/queues >> 126 MB L2; scene ~{scene_mb:.0f} MB "
                   "of BVH + primitive records, not L2-resident")}


def measured_peak_gbs():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def measure_l2_gbs():
    """L2-resident copy bandwidth on this GPU (GB/s, read + write): the denominator of
    roofline.l2 (the traversal's node and primitive loads are served from L1/L2, not HBM)."""
    import torch
    n = 32 << 20
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    a.zero_()
    for _ in range(5):
        b.copy_(a)
    best = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        e0.record()
        for _ in range(10):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 10 * 2.0 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return round(best, 1)


def ncu_traffic(cfg: str, kernel: str):
    """DRAM bytes per launch of `kernel` on config `cfg` from the committed ncu --set full
    summary (profiles/ncu_traffic.json), if any."""
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            v = json.load(f).get(cfg, {}).get(kernel)
            return v.get("dram_bytes") if isinstance(v, dict) else v
    except (OSError, ValueError, AttributeError):
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int = 0):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda x: x.replace(".", "", 1).isdigit()
        sm = [float(s[0]) for s in self.samples if num(s[0])]
        mx = [float(s[1]) for s in self.samples if num(s[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------ reference CPU path
# Scenes whose full-size reference pass takes minutes per core (C3-C5: the reference's fixed
# Stage-1 cost is ~34 s per pass on C4, its per-pixel cost ~0.43 ms) are timed at two reduced
# resolutions (W/8 x H/8 and W/4 x H/4, same geometry, camera, depth and walks per pixel) and
# the steady-state full-size pass time is the linear fit T(N) = F + c N at the full pixel count.
FIT_CONFIGS = {"C3", "C4", "C5"}


def reference_rate(cfg: str, sc, walks: int, cores: int, seed: int = 0):
    """Steady-state throughput of the unmodified reference (proxima::render_proxy_bdpt, PCG32
    as shipped) on this host: `cores` concurrent single-threaded renders of 2 passes each; the
    time of pass 1 comes from the pass_done callback's timestamps (pass 0 also holds the
    render's one-time pretrace and first-pass gate). Returns (Msamples/s, sample description,
    wall seconds)."""
    from oracle import oracle as orc
    t_start = time.perf_counter()
    o = orc.OracleScene(sc.to_json(), variant="pcg")
    W, H, N = sc.camera.width, sc.camera.height, sc.n_px
    if cfg not in FIT_CONFIGS:
        te = o.render_proxy_ref_timed(2, seed, cores, {"light_walks": walks})
        t1 = float(np.mean(te[:, 1] - te[:, 0]))
        value = cores * N / t1 / 1e6
        sample = (f"{cores} concurrent unmodified proxima::render_proxy_bdpt renders (PCG32) of {cfg} at full size "
                  f"({W}x{H}, {walks} pool walks), 2 passes each; steady pass time {t1:.2f} s (pass 1, pass_done "
                  f"timestamps)")
        return value, sample, time.perf_counter() - t_start
    sizes = [(max(10, W // 8), max(10, H // 8)), (max(10, W // 4), max(10, H // 4))]
    per = max(1, cores // 2)
    scs = [o.with_resolution(w, h) for (w, h) in sizes]
    n_s = [w * h for (w, h) in sizes]
    walks_s = [max(1, round(walks * n / N)) for n in n_s]
    # the reference's light_walks is one per pixel by default (0): keep the walks per pixel
    params = {"light_walks": 0} if walks == N else None
    if params is None and walks_s[0] != walks_s[1]:
        raise RuntimeError("reference fit needs walks per pixel equal across sizes")
    te = o.render_proxy_ref_timed(2, seed, 2 * per, params or {"light_walks": walks_s[0]},
                                  scenes=[scs[0]] * per + [scs[1]] * per)
    t1 = te[:, 1] - te[:, 0]
    T = [float(np.mean(t1[:per])), float(np.mean(t1[per:]))]
    c = (T[1] - T[0]) / (n_s[1] - n_s[0])
    F = T[0] - c * n_s[0]
    t_full = F + c * N
    value = cores * N / t_full / 1e6
    sample = (f"{2 * per} concurrent unmodified proxima::render_proxy_bdpt renders (PCG32) of the {cfg} scene, "
              f"{per} at {sizes[0][0]}x{sizes[0][1]} and {per} at {sizes[1][0]}x{sizes[1][1]} (same geometry, camera, "
              f"depth, one pool walk per pixel), 2 passes each; steady pass times {T[0]:.1f} s / {T[1]:.1f} s (pass 1, "
              f"pass_done timestamps) -> T(N) = {F:.1f} s + {c * 1e3:.4f} ms x N px; full size {W}x{H}: "
              f"{t_full:.0f} s per pass per core, x {cores} cores")
    return value, sample, time.perf_counter() - t_start


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc, walks = make_scene(args.config)
    cores = host_cores()
    try:
        value, sample, wall = reference_rate(args.config, sc, walks, cores, seed=0)
    except Exception as e:  # the reference library is test infrastructure; report, do not crash
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"[:300]}), flush=True)
        return
    # one timed step = one steady-state pass on every core (pass 0 is the warm-up)
    ms = 1e3 * cores * sc.n_px / (value * 1e6)
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Msamples/s",
           "n_gpus": args.gpus, "steps": 1, "warmup": 1, "ms_per_step": round(ms, 1), "wall_s": round(wall, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded scene generator)", "config": config_json(args.config, sc, walks),
           "cpu_baseline": {"value": round(value, 6), "unit": "Msamples/s", "cores": cores, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": round(value, 6), "unit": "Msamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ our arm
def measure_device(sc, params, seed, steps, warmup, world, local, quick, cfg):
    """Device-resident throughput of `steps` passes after the warm-up (CUDA events on the
    pass stream), then the traversal roofline over one more batch cycle."""
    import torch
    import torch.distributed as dist

    from paper_2503_23412_b200.render import ProxyRenderer
    W, H = sc.camera.width, sc.camera.height
    r = ProxyRenderer(sc, seed, params, device=local)
    acc = torch.zeros((H, W, 3), dtype=torch.float64, device="cuda") if world > 1 else None
    # Stage 1 runs one batch (8 passes) ahead of Stage 2. Steady-state accounting: warm-up is
    # rounded up to a batch multiple and ends with exactly one batch pre-computed; the timed
    # call's look-ahead is capped so it computes Stage 1 for exactly K passes. The timed
    # window therefore holds K passes of Stage 2 and K passes of Stage 1, like the pipeline
    # in steady state.
    BATCH = 8
    warm = -(-max(warmup, 3) // BATCH) * BATCH
    r.set_pass_limit(warm + BATCH)
    ts = torch.cuda.current_stream()

    def one_pass():
        if world > 1:  # pass -> stream-ordered accumulator copy -> NCCL all-reduce, no host wait
            r.render_passes_async(1)
            r.accum_to_device(acc.data_ptr(), stream=ts.cuda_stream)
            dist.all_reduce(acc)
        else:
            r.render_passes(1)

    for _ in range(warm):
        one_pass()
    r.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    r.set_pass_limit(warm + BATCH + steps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world == 1:
        r.render_passes(steps)
        torch.cuda.synchronize()
    else:
        ev0.record(ts)
        for _ in range(steps):
            one_pass()
        ev1.record(ts)
        torch.cuda.synchronize()
    stage_ms, counts = r.timing()
    recip = r.recip_counts()
    if world == 1:
        dev_ms = float(stage_ms[6])  # first pass start -> last pass end on the device, host gaps included
    else:
        dev_ms = float(ev0.elapsed_time(ev1))
    t = torch.tensor([dev_ms], device="cuda")
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    value = W * H * steps * world / (dev_ms / 1e3) / 1e6
    free, total = torch.cuda.mem_get_info()
    hbm_gb_used = round((total - free) / 1e9, 1)

    # ---- roofline: every traversal launch of one batch cycle (8 more passes of Stage 2 and the
    # one 8-pass Stage-1 batch they launch) timed + work-counted, so the launch mix is the
    # steady-state one
    r.set_pass_limit(-1)
    tr = r.measure_traversal(BATCH) if not quick else {"closest": {"launches": 0}, "anyhit": {"launches": 0}}
    nb = r.node_bytes()
    # bytes the kernels actually load per node visit: the whole 64 B quantised node; of a 128 B
    # node the six plane vectors and the child codes (3 x 32 B + 16 B; 16 B of padding unread)
    nb = 112 if nb == 128 else nb
    r.close()
    peak, peak_src = measured_peak_gbs()
    l2_peak = None if quick else measure_l2_gbs()
    roof = {}
    for kind, kname in (("closest", "k_trav_persistent<0>"), ("anyhit", "k_trav_persistent<1>")):
        m = tr[kind]
        if m["launches"] <= 0 or m["ms"] <= 0:
            continue
        bytes_total = m["nodes"] * nb + m["prims"] * PRIM_BYTES
        roof[kind] = {"kernel": kname, "launches": int(m["launches"]), "rays": int(m["rays"]),
                      "bytes_per_ray": round(bytes_total / max(m["rays"], 1), 1),
                      "nodes_per_ray": round(m["nodes"] / max(m["rays"], 1), 2),
                      "prims_per_ray": round(m["prims"] / max(m["rays"], 1), 2),
                      "bytes_per_launch": bytes_total / m["launches"], "ms_per_launch": m["ms"] / m["launches"],
                      "achieved_gbs": bytes_total / (m["ms"] / 1e3) / 1e9, "ms_total": m["ms"]}
    dom = max(roof, key=lambda k: roof[k]["ms_total"]) if roof else None
    roofline = None
    if dom:
        d = roof[dom]
        roofline = {"bound": "hbm", "achieved": round(d["achieved_gbs"], 1), "peak": peak, "unit": "GB/s",
                    "frac": round(d["achieved_gbs"] / peak, 4), "traffic": ncu_traffic(cfg, d["kernel"]),
                    "kernel": d["kernel"], "peak_source": peak_src,
                    "algorithmic_bytes": f"{nb} B fetched per BVH node visit + {PRIM_BYTES} B per primitive test, "
                                         "counted by an instrumented copy on the same rays",
                    # the same bytes against the L2: ncu shows these loads served by L1/L2 (DRAM
                    # traffic = `traffic`, a few % of them), so this is the fraction that bounds it
                    "l2": {"peak": l2_peak, "unit": "GB/s", "frac": round(d["achieved_gbs"] / l2_peak, 4)
                           if l2_peak else None,
                           "peak_source": "measured here: device-to-device copy of a 32 MB buffer (L2-resident, "
                                          "read + write bytes, 10 copies per timing, best of 20, CUDA events)"},
                    "per_kernel": roof}
    return {"value": value, "dev_ms": dev_ms, "warm": warm, "counts": counts, "stage_ms": stage_ms,
            "roofline": roofline, "hbm_gb_used": hbm_gb_used, "recip": recip}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer, render_proxy_bdpt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    sc, walks = make_scene(args.config)
    # Scene::finalize (validation, emitter tables, BVH) happens once when the scene is loaded,
    # as in the reference (load_scene -> finalize); every render call and context reuses it
    from paper_2503_23412_b200.render import finalized_scene
    t_fin = time.perf_counter()
    scene_dev_bytes = finalized_scene(sc).device_bytes()
    t_fin = time.perf_counter() - t_fin
    W, H = sc.camera.width, sc.camera.height
    params = ProxyParams(light_walks=walks)
    if os.environ.get("PXG_TUNE_PARAMS") and args.quick:  # tuning sweeps only (--quick lines are never bench values)
        for k, v in json.loads(os.environ["PXG_TUNE_PARAMS"]).items():
            setattr(params, k, v)

    # ---- device-resident throughput: K passes after W warm-up passes (CUDA events)
    # N > 1: sample sharding (paper_2503_23412_b200/distributed.py): every rank renders K
    # passes of its own Philox key and the fp64 accumulators are summed with one NCCL
    # all-reduce per pass; N = 1 is the plain single-GPU render.
    from paper_2503_23412_b200.distributed import rank_seed
    seed = rank_seed(0, rank)
    with ClockSampler(local) as clk:
        dev = measure_device(sc, params, seed, args.steps, args.warmup, world, local, args.quick, args.config)
    value, dev_ms, warm, counts, stage_ms, roofline = (dev[k] for k in ("value", "dev_ms", "warm", "counts",
                                                                        "stage_ms", "roofline"))
    # Extra key: BASELINE.json configs[1] (C2, the L2-resident Cornell box) measured the same way.
    extra = None
    if args.config == "C4" and world == 1 and not args.quick and not args.no_extra:
        sc2, walks2 = make_scene("C2")
        d2 = measure_device(sc2, ProxyParams(light_walks=walks2), seed, 56, 8, 1, local, False, "C2")
        extra = {"config": config_json("C2", sc2, walks2)["workload"], "value": round(d2["value"], 4),
                 "unit": "Msamples/s", "steps": 56, "warmup": d2["warm"], "ms_per_step": round(d2["dev_ms"] / 56, 4),
                 "roofline": d2["roofline"], "hbm_gb_used": d2["hbm_gb_used"]}
        del sc2

    # ---- end to end through the public API: render_proxy_bdpt(scene arrays on the host, spp=K)
    # with the pass_done callback reading the running mean image back every pass
    # (N > 1: render_proxy_bdpt_distributed, K passes per rank, NCCL all-reduce per round)
    e2e = None
    reads = [0]
    spp_e2e = min(sc.settings.spp, args.e2e_spp)  # one render call (C2: the config's full 64 spp)

    def cb(done, img):
        reads[0] += img.nbytes
        return True

    if args.quick:
        pass
    elif world == 1:
        render_proxy_bdpt(sc, 1, seed + 1000, params, pass_done=cb, device=local)  # warm the path
        torch.cuda.synchronize()
        reads[0] = 0
        t0 = time.perf_counter()
        img = render_proxy_bdpt(sc, spp_e2e, seed + 2000, params, pass_done=cb, device=local)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
    else:
        from paper_2503_23412_b200.distributed import render_proxy_bdpt_distributed
        render_proxy_bdpt_distributed(sc, world, 1000, params, pass_done=cb, local_rank=local)
        torch.cuda.synchronize()
        dist.barrier()
        reads[0] = 0
        t0 = time.perf_counter()
        img = render_proxy_bdpt_distributed(sc, spp_e2e * world, 2000, params, pass_done=cb, local_rank=local)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    if not args.quick:
        d2h = (reads[0] + img.nbytes) / spp_e2e
        e2e = {"value": round(W * H * spp_e2e * world / e2e_s / 1e6, 4), "unit": "Msamples/s",
               "h2d_bytes_per_step": int(scene_dev_bytes / spp_e2e), "d2h_bytes_per_step": int(d2h),
               "spp": spp_e2e,
               "includes": f"one full render call render_proxy_bdpt(scene, spp={spp_e2e}) per rank on a finalised "
                           "scene (host arrays): context creation (upload of the scene's BVH nodes and primitive "
                           "records from host memory, per-pass state, pretrace) + every pass + the running-mean "
                           "read-back after every pass (the reference's pass_done callback) + the final image",
               "excludes": f"Scene::finalize (validation, emitter tables, host BVH build: {t_fin:.2f} s), done once "
                           "when the scene is loaded, as the reference's load_scene does before any render call"}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        try:
            cores = host_cores()
            v, sample, wall = reference_rate(args.config, sc, walks, cores, seed=0)
            cpu_baseline = {"value": round(v, 6), "unit": "Msamples/s", "cores": cores, "kind": "reference",
                            "sample": sample, "wall_s": round(wall, 1)}
        except Exception as e:
            cpu_baseline = {"value": None, "unit": "Msamples/s", "cores": 0, "kind": "reference",
                            "sample": f"unavailable: {type(e).__name__}: {e}"[:200]}

    out = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "Msamples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": warm,
        "ms_per_step": round(dev_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded scene generator, paper_2503_23412_b200/scenes.py)",
        "parallelism": ("single GPU" if world == 1 else
                        f"sample-sharded x{world}: per-rank Philox keys, NCCL all-reduce of fp64 film every pass"),
        "config": config_json(args.config, sc, walks),
        "clocks": clk.summary(),
        "gpu_launches": int(counts[0]),
        "roofline": roofline,
        "hbm_gb_used": dev["hbm_gb_used"],
        "C2": extra,
        "cpu_baseline": cpu_baseline,
        "e2e": e2e,
        "stage_ms": {"stage1_batches_total": round(float(stage_ms[0]), 3),
                     "recip_rounds_total": round(float(stage_ms[1]), 3)},
        # reciprocal tree nodes evaluated ahead of the DFS vs consumed by it (whole run so far)
        "recip_nodes": dict(dev["recip"], evaluated_per_consumed=round(dev["recip"]["evaluated"] /
                                                                      max(dev["recip"]["consumed"], 1), 3)),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
