"""B200-native (sm_100a) proxy-sampling BDPT: the hot path `render_proxy_bdpt` of
arXiv 2503.23412's reference (proxima), as hand-written CUDA behind a C ABI (include/pxg.h).

Public surface (mirrors the reference's names and argument meaning):
  load_scene, load_scene_from_string, Scene          scene schema (proj/src/scene.cpp:317-436)
  ProxyParams, ProxyDiagnostics, ProxyDiagRow        proj/include/proxima/proxy.hpp:162-188
  render_proxy_bdpt, render_bdpt                     proj/src/proxy.cpp:647, transport.cpp:380
  ProxyRenderer                                      one GPU context (pass-by-pass control)
"""
from .scene import Scene, SceneError, Material, Camera, Settings, load_scene, load_scene_from_string, is_specular
from .render import (ProxyParams, ProxyDiagnostics, ProxyDiagRow, ProxyRenderer, render_proxy_bdpt, render_bdpt,
                     recip_twopoint, rng_draws)
from . import scenes

__all__ = ["Scene", "SceneError", "Material", "Camera", "Settings", "load_scene", "load_scene_from_string",
           "is_specular", "ProxyParams", "ProxyDiagnostics", "ProxyDiagRow", "ProxyRenderer", "render_proxy_bdpt",
           "render_bdpt", "recip_twopoint", "rng_draws", "scenes"]
