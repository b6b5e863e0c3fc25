"""CPU checks of the drop-in boundary: the C ABI library loads, exports every symbol that
include/pxg.h declares, the headers compile, and the product path refuses to run without a
GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(REPO, "include", "pxg.h")
LIB = os.path.join(REPO, "paper_2503_23412_b200", "libpxg.so")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"\b(pxg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2503_23412_b200 import _lib
    _lib.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pxg_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared in pxg.h but not exported: {missing}"
    assert set(_lib.EXPORTED_SYMBOLS) <= exported


def test_c_header_is_plain_c():
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-fsyntax-only", "-x", "c", "-I",
                        os.path.join(REPO, "include"), "-"], input='#include "pxg.h"\n#include "pxg_philox.h"\n'
                       'int main(void){pxg_params p; pxg_default_params(&p); return p.pool_budget != 400;}\n',
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_cpp_dropin_wrapper_compiles_against_reference_headers():
    json_inc = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-I", os.path.join(REPO, "include"),
                        "-I", "/root/reference/proj/include", "-I", json_inc, "-"],
                       input='#include "pxg_proxima.hpp"\nint main(){return 0;}\n', capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_default_params_match_reference_defaults():
    from paper_2503_23412_b200 import _lib
    from paper_2503_23412_b200.render import ProxyParams
    p = _lib.Params()
    _lib.lib().pxg_default_params(C.byref(p))
    d = ProxyParams()
    for f, _ in _lib.Params._fields_:
        assert getattr(p, f) == getattr(d, f), f


def test_no_cpu_fallback_without_device():
    """On a machine without a GPU, creating a context fails with PXG_E_NODEVICE."""
    from paper_2503_23412_b200 import _lib, scenes
    from paper_2503_23412_b200.render import ProxyRenderer
    if _lib.lib().pxg_device_count() > 0:
        pytest.skip("a CUDA device is visible")
    with pytest.raises(_lib.PxgError) as e:
        ProxyRenderer(scenes.caustic_box(4), 0)
    assert e.value.code == -4
