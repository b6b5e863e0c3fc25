"""Benchmark of the proxy-BDPT hot path (BASELINE.json metric: Msamples/s of full proxy-BDPT
pixel samples). One step = one progressive pass = 1 sample for every pixel of the workload
(Stage 1 pool + reciprocal estimates, Stage 2 strategies + proxy connection, film).

Workload (N=1): BASELINE.json configs[1] ("C2"): 512x512, max depth 10, 256K pool walks per
pass, Cornell box + mirror icosphere (5,120 tris) + dielectric icosphere (20,480 tris) + GGX
floor; seeded synthetic scene (paper_2503_23412_b200/scenes.py). Inputs larger than L2?
no — the scene (~3.3 MB of BVH + primitives) is L2-resident by design; the per-pixel vertex
pools (~670 MB) are far larger than L2 and are rewritten every pass.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2]
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--resolution", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


CONFIGS = {
    # name: (generator kwargs, light_walks, spp of the config)
    "C1": (dict(resolution=256, max_depth=8), 65536, 16),
    "C2": (dict(resolution=512, max_depth=10), 262144, 64),
}


def make_scene(cfg: str, resolution: int = 0):
    from paper_2503_23412_b200 import scenes
    kw, walks, spp = CONFIGS[cfg]
    kw = dict(kw)
    if resolution:
        walks = walks * resolution * resolution // (kw["resolution"] ** 2)
        kw["resolution"] = resolution
    gen = scenes.cornell_c1 if cfg == "C1" else scenes.cornell_c2
    return gen(**kw), walks, spp


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
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    sc, walks, spp_cfg = make_scene(args.config, args.resolution)
    W, H = sc.camera.width, sc.camera.height
    params = ProxyParams(light_walks=walks)
    # weak scaling: every rank renders the full workload on its own replica stream set
    r = ProxyRenderer(sc, 7 + rank, params, device=local)
    for _ in range(args.warmup):
        r.render_passes(1)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        r.render_passes(args.steps)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    stage_ms, counts = r.timing()
    dev_ms = float(stage_ms[6])  # whole call on the device timeline, host gaps included
    t = torch.tensor([dev_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    samples = W * H * args.steps * world
    value = samples / (dev_ms / 1e3) / 1e6
    out = {
        "metric": "Msamples/s (full proxy-BDPT px samples)",
        "value": round(value, 4),
        "unit": "Msamples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded scene generator, paper_2503_23412_b200/scenes.py)",
        "config": {"workload": f"{args.config}: {W}x{H}, max_depth {sc.settings.max_depth}, {walks} pool walks/pass, "
                               f"{sc.n_prims} prims, proxy on", "passes_per_step": 1,
                   "l2": "scene L2-resident; per-pixel vertex pools >> L2 rewritten each pass"},
        "clocks": clk.summary(),
        "wall_ms_per_step": round(wall * 1e3 / args.steps, 4),
        "stage_ms_per_step": {k: round(v / args.steps, 4) for k, v in
                              zip(["stage1_pool", "recip", "trace", "connect", "proxy", "gate_film"], stage_ms[:6])},
        "gpu_launches": int(counts[0]),
    }
    r.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    print(json.dumps({"impl": "reference", "unavailable": "not yet wired"}), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
