"""Host-side scene description: the reference's JSON scene schema as flat numpy arrays.

Mirrors `proxima::load_scene_from_string` (proj/src/scene.cpp:317-428): same keys, same
defaults, same validation order and messages (errors are `SceneError`, a RuntimeError,
like the reference's std::runtime_error("scene: ...")). Derived quantities
(`Scene::finalize`, proj/src/scene.cpp:234-252: emitter areas, emitter prefix sums,
bbox) and the BVH are built in C++ inside libpxg (`pxg_create`), so this module only
parses and validates.

Primitive arrays (n = number of primitives), in the reference's own field meaning
(proj/include/proxima/scene.hpp:20-31):
  shape  int32   0 sphere, 1 triangle, 2 rectangle (Primitive::Shape order)
  mat    int32   material index
  a,b,c  f64[n,3] sphere: a = center; triangle: vertices; rectangle: a = origin, b,c = edges
  radius f64[n]
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

SPHERE, TRIANGLE, RECTANGLE = 0, 1, 2


class SceneError(RuntimeError):
    """Mirror of the reference's scene validation error (proj/src/scene.cpp:299)."""

    def __init__(self, msg: str):
        super().__init__("scene: " + msg)


@dataclass
class Material:
    """proj/include/proxima/bsdf.hpp:13-20"""
    name: str
    base_color: tuple = (0.8, 0.8, 0.8)
    metallic: float = 0.0
    roughness: float = 0.5
    transmission: float = 0.0
    ior: float = 1.5


def is_specular(m: Material) -> bool:
    """proj/include/proxima/bsdf.hpp:26-28"""
    return (m.metallic >= 0.5 or m.transmission >= 0.5) and m.roughness < 0.2


@dataclass
class Camera:
    """proj/include/proxima/scene.hpp:38-48"""
    position: tuple = (0.0, 0.0, 0.0)
    look_at: tuple = (0.0, 0.0, -1.0)
    up: tuple = (0.0, 1.0, 0.0)
    fov_y: float = 45.0
    width: int = 64
    height: int = 64


@dataclass
class Settings:
    """proj/include/proxima/scene.hpp:50-54"""
    max_depth: int = 8
    spp: int = 16
    seed: int = 0


@dataclass
class Scene:
    materials: list
    shape: np.ndarray
    mat: np.ndarray
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    radius: np.ndarray
    emitter_prim: np.ndarray          # int32 [n_emitters]
    emitter_radiance: np.ndarray      # f64 [n_emitters, 3]
    camera: Camera = field(default_factory=Camera)
    settings: Settings = field(default_factory=Settings)

    @property
    def n_prims(self) -> int:
        return int(self.shape.shape[0])

    @property
    def n_px(self) -> int:
        return self.camera.width * self.camera.height

    def has_specular(self) -> bool:
        return any(is_specular(m) for m in self.materials)

    def finalize(self) -> "Scene":
        """Scene::finalize (proj/src/scene.cpp:234-252): validation, emitter tables and the
        BVH, built once on the host by libpxg (pxg_scene_create) and reused by every render
        call and context, as the reference's render functions receive a finalised Scene. Like
        the reference's, the scene is immutable afterwards (rendering calls this lazily)."""
        from .render import finalized_scene
        finalized_scene(self)
        return self

    def material_table(self) -> np.ndarray:
        """f64 [n_mat, 8]: base_color xyz, metallic, roughness, transmission, ior, 0."""
        t = np.zeros((len(self.materials), 8))
        for i, m in enumerate(self.materials):
            t[i, 0:3] = m.base_color
            t[i, 3] = m.metallic
            t[i, 4] = m.roughness
            t[i, 5] = m.transmission
            t[i, 6] = m.ior
        return t

    def to_json(self) -> str:
        """Serialise in the reference schema; floats use repr so values round-trip exactly."""
        prims = []
        names = [m.name for m in self.materials]
        A, B, C, Rr = self.a.tolist(), self.b.tolist(), self.c.tolist(), self.radius.tolist()
        for s, mi, a, b, c, r in zip(self.shape.tolist(), self.mat.tolist(), A, B, C, Rr):
            m = names[mi]
            if s == SPHERE:
                prims.append({"shape": "sphere", "material": m, "center": a, "radius": r})
            elif s == TRIANGLE:
                prims.append({"shape": "triangle", "material": m, "p0": a, "p1": b, "p2": c})
            else:
                prims.append({"shape": "rectangle", "material": m, "origin": a, "edge_u": b, "edge_v": c})
        doc = {
            "materials": [{"name": m.name, "base_color": list(m.base_color), "metallic": m.metallic,
                           "roughness": m.roughness, "transmission": m.transmission, "ior": m.ior}
                          for m in self.materials],
            "primitives": prims,
            "emitters": [{"primitive": int(p), "radiance": r.tolist()}
                         for p, r in zip(self.emitter_prim, self.emitter_radiance)],
            "camera": {"position": list(self.camera.position), "look_at": list(self.camera.look_at),
                       "up": list(self.camera.up), "fov_y": self.camera.fov_y,
                       "resolution": [self.camera.width, self.camera.height]},
            "settings": {"max_depth": self.settings.max_depth, "spp": self.settings.spp,
                         "seed": self.settings.seed},
        }
        return json.dumps(doc, separators=(",", ":"))


def save_npz(scene: Scene, path: str) -> None:
    """Binary scene cache for large scenes: a 1M-triangle scene is
    ~220 MB of reference JSON (~20 s through a JSON parser); the same arrays load from .npz in
    well under a second and describe exactly the same Scene."""
    mats = json.dumps([m.__dict__ for m in scene.materials])
    cam, st = scene.camera, scene.settings
    np.savez(path, shape=scene.shape, mat=scene.mat, a=scene.a, b=scene.b, c=scene.c, radius=scene.radius,
             emitter_prim=scene.emitter_prim, emitter_radiance=scene.emitter_radiance,
             materials=np.frombuffer(mats.encode(), np.uint8),
             camera=np.array([*cam.position, *cam.look_at, *cam.up, cam.fov_y, cam.width, cam.height], np.float64),
             settings=np.array([st.max_depth, st.spp, st.seed], np.int64))


def load_npz(path: str) -> Scene:
    z = np.load(path)
    mats = [Material(**m) for m in json.loads(bytes(z["materials"]).decode())]
    for m in mats:
        m.base_color = tuple(m.base_color)
    c = z["camera"].tolist()
    cam = Camera(tuple(c[0:3]), tuple(c[3:6]), tuple(c[6:9]), c[9], int(c[10]), int(c[11]))
    st = z["settings"].tolist()
    return Scene(materials=mats, shape=z["shape"], mat=z["mat"], a=z["a"], b=z["b"], c=z["c"], radius=z["radius"],
                 emitter_prim=z["emitter_prim"], emitter_radiance=z["emitter_radiance"], camera=cam,
                 settings=Settings(int(st[0]), int(st[1]), int(st[2])))


def _cross(u, v):
    return (u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0])


def _length(v):
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


def _sub(u, v):
    return (u[0] - v[0], u[1] - v[1], u[2] - v[2])


def primitive_area(shape: int, a, b, c, radius: float) -> float:
    """Primitive::area (proj/src/scene.cpp:107-114), same op order."""
    if shape == SPHERE:
        return 4.0 * math.pi * radius * radius
    if shape == TRIANGLE:
        return 0.5 * _length(_cross(_sub(b, a), _sub(c, a)))
    return _length(_cross(b, c))


def _vec3(j: dict, key: str):
    v = j.get(key)
    if not isinstance(v, list) or len(v) != 3:
        raise SceneError(f"expected 3-vector for '{key}'")
    return tuple(float(x) for x in v)


def _unit(j: dict, key: str, fallback: float) -> float:
    v = float(j.get(key, fallback))
    if v < 0.0 or v > 1.0:
        raise SceneError(f"'{key}' must lie in [0,1]")
    return v


def load_scene_from_string(text: str) -> Scene:
    """Mirror of proxima::load_scene_from_string (proj/src/scene.cpp:317-428)."""
    try:
        root = json.loads(text)
    except json.JSONDecodeError as e:
        raise SceneError(f"invalid JSON: {e}") from None

    mats = root.get("materials")
    if not mats:
        raise SceneError("no materials defined")
    materials = []
    for jm in mats:
        name = jm.get("name", "")
        if not name:
            raise SceneError("material without a name")
        m = Material(name=name)
        if "base_color" in jm:
            m.base_color = _vec3(jm, "base_color")
        m.metallic = _unit(jm, "metallic", 0.0)
        m.roughness = _unit(jm, "roughness", 0.5)
        m.transmission = _unit(jm, "transmission", 0.0)
        m.ior = float(jm.get("ior", 1.5))
        if m.transmission > 0.0 and m.ior <= 1.0:
            raise SceneError("ior must exceed 1")
        materials.append(m)
    names = [m.name for m in materials]

    def material_index(name):
        for i, n in enumerate(names):
            if n == name:
                return i
        raise SceneError(f"unknown material '{name}'")

    jprims = root.get("primitives")
    if not jprims:
        raise SceneError("no primitives defined")
    n = len(jprims)
    shape = np.zeros(n, np.int32)
    mat = np.zeros(n, np.int32)
    A = np.zeros((n, 3))
    B = np.zeros((n, 3))
    Cc = np.zeros((n, 3))
    R = np.ones(n)
    for i, jp in enumerate(jprims):
        s = jp.get("shape", "")
        mat[i] = material_index(jp.get("material", ""))
        if s == "sphere":
            shape[i] = SPHERE
            A[i] = _vec3(jp, "center")
            R[i] = float(jp.get("radius", 0.0))
            if R[i] <= 0.0:
                raise SceneError("sphere radius must be positive")
        elif s == "triangle":
            shape[i] = TRIANGLE
            A[i], B[i], Cc[i] = _vec3(jp, "p0"), _vec3(jp, "p1"), _vec3(jp, "p2")
            if primitive_area(TRIANGLE, A[i], B[i], Cc[i], 0.0) <= 0.0:
                raise SceneError("degenerate triangle")
        elif s == "rectangle":
            shape[i] = RECTANGLE
            A[i], B[i], Cc[i] = _vec3(jp, "origin"), _vec3(jp, "edge_u"), _vec3(jp, "edge_v")
            if primitive_area(RECTANGLE, A[i], B[i], Cc[i], 0.0) <= 0.0:
                raise SceneError("degenerate rectangle")
        else:
            raise SceneError(f"unknown shape '{s}'")

    jem = root.get("emitters")
    if not jem:
        raise SceneError("scene must contain at least one emitter")
    eprim, erad = [], []
    for je in jem:
        p = int(je.get("primitive", -1))
        if p < 0 or p >= n:
            raise SceneError("emitter references unknown primitive")
        r = _vec3(je, "radiance")
        if r[0] < 0.0 or r[1] < 0.0 or r[2] < 0.0:
            raise SceneError("emitter radiance must be non-negative")
        eprim.append(p)
        erad.append(r)

    if "camera" not in root:
        raise SceneError("no camera defined")
    jc = root["camera"]
    for key in jc:
        if key not in ("position", "look_at", "up", "fov_y", "resolution"):
            raise SceneError(f"unknown camera key '{key}'")
    cam = Camera()
    cam.position = _vec3(jc, "position")
    cam.look_at = _vec3(jc, "look_at")
    if "up" in jc:
        cam.up = _vec3(jc, "up")
    cam.fov_y = float(jc.get("fov_y", 45.0))
    if cam.fov_y <= 0.0 or cam.fov_y >= 180.0:
        raise SceneError("fov_y must lie in (0,180)")
    if "resolution" in jc:
        cam.width = int(jc["resolution"][0])
        cam.height = int(jc["resolution"][1])
    if cam.width <= 0 or cam.height <= 0:
        raise SceneError("resolution must be positive")
    if _length(_sub(cam.look_at, cam.position)) < 1e-12:
        raise SceneError("camera look_at coincides with position")

    st = Settings()
    if "settings" in root:
        js = root["settings"]
        for key in js:
            if key not in ("max_depth", "spp", "seed"):
                raise SceneError(f"unknown settings key '{key}'")
        st.max_depth = int(js.get("max_depth", 8))
        st.spp = int(js.get("spp", 16))
        st.seed = int(js.get("seed", 0))
        if st.max_depth < 1:
            raise SceneError("max_depth must be at least 1")
        if st.spp < 1:
            raise SceneError("spp must be at least 1")

    return Scene(materials=materials, shape=shape, mat=mat, a=A, b=B, c=Cc, radius=R,
                 emitter_prim=np.asarray(eprim, np.int32), emitter_radiance=np.asarray(erad, np.float64),
                 camera=cam, settings=st)


def load_scene(path: str) -> Scene:
    """Mirror of proxima::load_scene (proj/src/scene.cpp:430-436)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise SceneError("cannot open " + path) from None
    return load_scene_from_string(text)
