"""Builds libpxg.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

  python -m paper_2503_23412_b200.build [--force]

Device code is compiled with --fmad=false: the path math must keep the reference's fp64
operation order (no fused multiply-add), see csrc/pxg_math.cuh.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpxg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["pxg_main.cu"]
CPP_SOURCES = ["pxg_host.cpp"]
SINCOS_TABLE = os.path.join(HERE, "pxg_sincos_glibc.bin")
SINCOS_GEN = os.path.join(HERE, "_build", "pxg_sincos_gen")
HEADERS = ["pxg_pt.cuh", "pxg_stage_kernels.cuh", "pxg_proxy_wave.cuh", "pxg_wave.cuh", "pxg_math.cuh", "pxg_bsdf.cuh", "pxg_scene.cuh", "pxg_path.cuh", "pxg_proxy.cuh", "pxg_host.h"]


def _inputs():
    files = [os.path.join(CSRC, f) for f in CU_SOURCES + CPP_SOURCES + HEADERS]
    files += [os.path.join(REPO, "include", "pxg.h"), os.path.join(REPO, "include", "pxg_philox.h"),
              os.path.join(REPO, "include", "pxg_sincos.h")]
    return files


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build_sincos_table(force: bool = False, verbose: bool = False) -> str:
    """The glibc agreement table of the device sin / cos (include/pxg_sincos.h): every one of
    the 2^32 sampler angles evaluated with this host's libm (~2 min on 8 cores), written next
    to libpxg.so. Rebuilt only when the generator or the header changes."""
    gen_src = os.path.join(CSRC, "pxg_sincos_gen.cpp")
    hdr = os.path.join(REPO, "include", "pxg_sincos.h")
    os.makedirs(os.path.dirname(SINCOS_GEN), exist_ok=True)
    if force or not os.path.exists(SINCOS_GEN) or any(os.path.getmtime(f) > os.path.getmtime(SINCOS_GEN)
                                                       for f in (gen_src, hdr)):
        _run(["g++", "-std=c++20", "-O2", "-pthread", "-ffp-contract=off", "-I", os.path.join(REPO, "include"),
              gen_src, "-o", SINCOS_GEN], verbose)
    if force or not os.path.exists(SINCOS_TABLE) or os.path.getmtime(SINCOS_GEN) > os.path.getmtime(SINCOS_TABLE):
        _run([SINCOS_GEN, SINCOS_TABLE], verbose)
    return SINCOS_TABLE


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    """`out` / `defines` (-DNAME=V for the device code): A/B variants of the same sources for
    tuning runs (loaded through PXG_LIBRARY); the shipped library is the default build."""
    build_sincos_table(force=False, verbose=verbose)
    if out == OUT and not defines and not force and up_to_date():
        return OUT
    bdir = os.path.join(HERE, "_build" if out == OUT else "_build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(bdir, exist_ok=True)
    inc = ["-I", os.path.join(REPO, "include"), "-I", CSRC]
    objs = []
    for src in CPP_SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = ["g++", "-std=c++20", "-O3", "-pthread", "-fPIC", "-ffp-contract=off", *inc, "-c", os.path.join(CSRC, src),
               "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    for src in CU_SOURCES:
        obj = os.path.join(bdir, src + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "--expt-relaxed-constexpr",
               "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3", *defines, *inc, "-c", os.path.join(CSRC, src),
               "-o", obj]
        _run(cmd, verbose)
        objs.append(obj)
    tmp = out + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lpthread"], verbose)
    os.replace(tmp, out)
    return out


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (exit {r.returncode})")


if __name__ == "__main__":
    # python -m paper_2503_23412_b200.build [--force] [-v] [--out PATH -DNAME=V ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else OUT
    defs = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, out=os.path.abspath(out), defines=defs))
