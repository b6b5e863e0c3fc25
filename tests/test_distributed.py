"""Multi-process (world size 2, gloo, CPU) tests of the sample-sharded multi-GPU driver
(paper_2503_23412_b200/distributed.py). The per-rank renderer is the oracle's restated
render loop on CPU, so the exact orchestration used on GPUs (round-robin passes, disjoint
per-rank Philox keys, per-round all-reduce of fp64 accumulators, rank-0 early stop) is
exercised end to end and compared with a single-process combination of the same renders."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_23412_b200 import distributed as D
from paper_2503_23412_b200 import scenes

PARAMS = {"pretrace_paths": 1000, "light_walks": 600}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleRenderer:
    def __init__(self, json_text, seed, n_passes):
        from oracle import oracle as orc
        o = orc.OracleScene(json_text)
        self.shape = (o.height, o.width, 3)
        self.vals = []
        if n_passes > 0:
            _, run = o.render(n_passes, seed, params=PARAMS, threads=2, trace=True)
            self.vals = [run.pass_val[p].reshape(self.shape) for p in range(n_passes)]
        self.done = 0

    def render_passes(self, n):
        self.done += n

    def accum_into(self, t):
        acc = np.zeros(self.shape)
        for p in range(self.done):
            acc += self.vals[p]
        t.copy_(torch.from_numpy(acc))
        return self.done

    def close(self):
        pass


def _worker(rank, world, port, json_text, spp, seed, stop_after, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = None

        def make(s, n):
            r = OracleRenderer(json_text, s, n)
            return r

        from oracle import oracle as orc
        o = orc.OracleScene(json_text)
        shape = (o.height, o.width, 3)
        seen = []

        def cb(done, img):
            seen.append(done)
            return stop_after is None or done < stop_after

        img, done = D.render_sample_sharded(make, shape, spp, seed, pass_done=cb)
        np.save(os.path.join(out_dir, f"img{rank}.npy"), img)
        np.save(os.path.join(out_dir, f"meta{rank}.npy"), np.array([done] + seen))
    finally:
        dist.destroy_process_group()


def _run(tmp_path, spp, seed, stop_after=None):
    sc = scenes.caustic_box(8)
    port = free_port()
    mp.spawn(_worker, args=(2, port, sc.to_json(), spp, seed, stop_after, str(tmp_path)), nprocs=2, join=True)
    return sc, [np.load(tmp_path / f"img{r}.npy") for r in range(2)], [np.load(tmp_path / f"meta{r}.npy")
                                                                        for r in range(2)]


def test_rank_seeds_and_pass_partition():
    assert D.rank_seed(7, 0) == 7
    seeds = {D.rank_seed(7, r) for r in range(8)}
    assert len(seeds) == 8
    for spp in (1, 5, 16, 17):
        parts = [D.passes_of_rank(spp, r, 4) for r in range(4)]
        assert sum(parts) == spp and max(parts) - min(parts) <= 1


def test_two_ranks_equal_the_combined_single_process_renders(oracle, tmp_path):
    spp, seed = 5, 3
    sc, imgs, metas = _run(tmp_path, spp, seed)
    assert np.array_equal(imgs[0], imgs[1])          # every rank holds the reduced image
    assert int(metas[0][0]) == spp
    # single-process combination of the two ranks' independent renders
    o = oracle.OracleScene(sc.to_json())
    means, passes = [], []
    for r in range(2):
        n = D.passes_of_rank(spp, r, 2)
        img, _ = o.render(n, D.rank_seed(seed, r), params=PARAMS, threads=2)
        means.append(img)
        passes.append(n)
    ref = D.merge_means(means, passes)
    assert np.allclose(imgs[0], ref, rtol=1e-12, atol=1e-15)


def test_early_stop_is_collective(oracle, tmp_path):
    spp, seed = 6, 4
    sc, imgs, metas = _run(tmp_path, spp, seed, stop_after=2)
    for m in metas:
        assert int(m[0]) == 2                       # both ranks stopped after round 0 (2 passes)
    assert list(metas[0][1:]) == [2]                # rank 0 saw one callback
    o = oracle.OracleScene(sc.to_json())
    a, _ = o.render(1, D.rank_seed(seed, 0), params=PARAMS, threads=2)
    b, _ = o.render(1, D.rank_seed(seed, 1), params=PARAMS, threads=2)
    assert np.allclose(imgs[0], (a + b) / 2, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- real GPU contexts (cuda:0)
def _gpu_worker(rank, world, port, spp, seed, stop_after, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_23412_b200.render import ProxyParams
        sc = scenes.caustic_box(24)
        params = ProxyParams(pretrace_paths=2000, light_walks=2000)
        seen = []

        def cb(done, img):
            seen.append(done)
            return stop_after is None or done < stop_after

        make = lambda s, n: D.GpuRenderer(sc, s, params, 0, n)  # noqa: E731
        img, done = D.render_sample_sharded(make, (sc.camera.height, sc.camera.width, 3), spp, seed,
                                            pass_done=cb if stop_after is not None else None,
                                            device=torch.device("cuda", 0))
        np.save(os.path.join(out_dir, f"gimg{rank}.npy"), img)
        np.save(os.path.join(out_dir, f"gmeta{rank}.npy"), np.array([done] + seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("stop_after", [None, 2])
def test_two_gpu_contexts_gloo_equal_single_process(pxg, tmp_path, stop_after):
    """Two ranks (gloo, both on cuda:0, no rank waits on another's kernels) running the real
    GpuRenderer: the reduced image equals the two contexts rendered in one process, bitwise
    (the fp64 sum of two accumulators is order-independent), with and without an early stop."""
    from paper_2503_23412_b200.render import ProxyParams, ProxyRenderer
    spp, seed = 5, 3
    port = free_port()
    mp.spawn(_gpu_worker, args=(2, port, spp, seed, stop_after, str(tmp_path)), nprocs=2, join=True)
    imgs = [np.load(tmp_path / f"gimg{r}.npy") for r in range(2)]
    metas = [np.load(tmp_path / f"gmeta{r}.npy") for r in range(2)]
    assert np.array_equal(imgs[0], imgs[1])
    done = int(metas[0][0])
    assert done == (spp if stop_after is None else stop_after)
    sc = scenes.caustic_box(24)
    params = ProxyParams(pretrace_paths=2000, light_walks=2000)
    acc = 0.0
    rounds = -(-done // 2)
    for r in range(2):
        n = min(D.passes_of_rank(spp, r, 2), rounds)
        with ProxyRenderer(sc, D.rank_seed(seed, r), params) as pr:
            pr.set_pass_limit(n)
            pr.render_passes(n)
            a, _ = pr.accum()
        acc = acc + a
    assert np.array_equal(imgs[0], acc * (1.0 / done))
