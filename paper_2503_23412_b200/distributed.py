"""Multi-GPU proxy-BDPT: one process per GPU, torch.distributed for the plumbing.

Sample sharding (BASELINE.json north star): every rank runs its own progressive render of
the whole image on disjoint Philox streams (its own key, so its own light-path pool,
subspace statistics, gamma and gate grid), global passes are assigned round-robin
(rank r renders global passes r, r + N, r + 2N, ...), and after every round the fp64
accumulators are summed across ranks with one all-reduce (NCCL over NVLink on GPUs, gloo on
CPU). The sum over ranks of independent unbiased progressive estimators is unbiased; with
N = 1 this is exactly render_proxy_bdpt. Early stopping through pass_done is decided on
rank 0 and broadcast, so every rank leaves the loop after the same round.

The renderer is pluggable (`make_renderer(seed) -> object with render_passes(n),
accum_into(tensor) and close()`), which lets the CPU tests drive this exact orchestration
with gloo and a CPU renderer.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

_GOLDEN = 0x9E3779B97F4A7C15
_MASK = (1 << 64) - 1


def rank_seed(seed: int, rank: int) -> int:
    """Philox key of rank `rank`: rank 0 keeps the caller's seed (N = 1 == single GPU)."""
    return seed if rank == 0 else (seed ^ ((_GOLDEN * (rank + 1)) & _MASK)) & _MASK


def passes_of_rank(spp: int, rank: int, world: int) -> int:
    return len(range(rank, spp, world))


def passes_done_after_round(spp: int, world: int, k: int) -> int:
    """Global passes completed after round k (0-based) of the round-robin assignment."""
    return min(spp, (k + 1) * world)


class GpuRenderer:
    """ProxyRenderer adapter. Passes are enqueued without waiting for them; the accumulator is
    copied device-to-device into a CUDA tensor, stream-ordered on torch's current stream
    (after the previous round's reduce of that tensor, before the next one), so the host
    never blocks inside the loop unless a pass_done callback needs the image."""

    def __init__(self, scene, seed, params, device: int, spp_local: int):
        from .render import ProxyRenderer
        self.device = device
        self.r = ProxyRenderer(scene, seed, params, device=device)
        self.r.set_pass_limit(spp_local)

    def render_passes(self, n: int):
        self.r.render_passes_async(n)

    def accum_into(self, t: torch.Tensor) -> int:
        stream = torch.cuda.current_stream(t.device).cuda_stream
        return self.r.accum_to_device(t.data_ptr(), stream=stream)

    def close(self):
        self.r.close()


def render_sample_sharded(make_renderer, shape, spp: int, seed: int, pass_done=None, device=None):
    """Runs the round-robin sharded render. Returns (mean image as numpy on every rank,
    global passes done).

    Round k: every rank with a pass left has it enqueued; its accumulator is copied into the
    reduction buffer and summed across ranks (in place); the next round's pass is enqueued
    before the host looks at round k's image, so with a pass_done callback the GPUs keep
    rendering while rank 0 runs it. Without a callback the loop never waits on the devices."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    dev = device if device is not None else torch.device("cpu")
    mine = passes_of_rank(spp, rank, world)
    rounds = math.ceil(spp / world) if spp > 0 else 0
    r = make_renderer(rank_seed(seed, rank), mine)
    acc = torch.zeros(shape, dtype=torch.float64, device=dev)
    done = 0
    try:
        if mine > 0:
            r.render_passes(1)
        for k in range(rounds):
            r.accum_into(acc)  # this rank's passes of rounds 0..k
            if world > 1:
                dist.all_reduce(acc, op=dist.ReduceOp.SUM)
            if k + 1 < mine:
                r.render_passes(1)  # round k+1 runs while round k is reduced / shown
            done = passes_done_after_round(spp, world, k)
            if pass_done is not None:
                stop = torch.zeros(1, dtype=torch.int32, device=dev)
                if rank == 0:
                    mean = (acc * (1.0 / done)).cpu().numpy()
                    if not pass_done(done, mean):
                        stop[0] = 1
                if world > 1:
                    dist.broadcast(stop, src=0)
                if int(stop.item()):
                    break
        mean = (acc * (1.0 / max(done, 1))).cpu().numpy()
    finally:
        r.close()
    return mean, done


def render_proxy_bdpt_distributed(scene, spp: int, seed: int, params=None, pass_done=None, local_rank=None):
    """render_proxy_bdpt over all ranks of the default process group (one GPU each)."""
    from .render import ProxyParams
    if spp <= 0:
        spp = scene.settings.spp
    params = params or ProxyParams()
    dev_index = local_rank if local_rank is not None else torch.cuda.current_device()
    shape = (scene.camera.height, scene.camera.width, 3)
    make = lambda s, n: GpuRenderer(scene, s, params, dev_index, n)  # noqa: E731
    img, _ = render_sample_sharded(make, shape, spp, seed, pass_done, device=torch.device("cuda", dev_index))
    return img


def merge_means(means, passes):
    """Reference combination of per-rank means (weights = passes), for tests."""
    tot = sum(passes)
    return sum(m * p for m, p in zip(means, passes)) / tot if tot else np.zeros_like(means[0])
