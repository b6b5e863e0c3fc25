"""Seeded synthetic scenes for the BASELINE.json configs (they stand in for the paper's
proprietary scenes, which are not available). Every generator is
deterministic and emits a `Scene` in the reference schema, so the same scene loads in
the reference (via `Scene.to_json()`) and in libpxg.

C1  Cornell box, 10 Lambertian triangles + 2-triangle 0.25x0.25 ceiling lamp (L = 15) +
    subdiv-4 mirror icosphere (5,120 tris) at (0.5, 0.3, 0.5), r = 0.2.
C2  C1 + subdiv-5 dielectric icosphere (20,480 tris, IOR 1.5) + GGX floor (roughness 0.1).
C3/C4 generators follow the same pattern.

Fixed choices not given by BASELINE.json (recorded here once): box = unit cube open at
z = 1; lamp at y = 0.998 facing down; camera at (0.5, 0.5, 2.2) looking at (0.5, 0.5, 0),
fov_y 40; glass sphere centre (0.25, 0.205, 0.81); mirror/glass roughness 0.01 (the
reference has no delta BSDF); mirror base colour 0.95.
"""
from __future__ import annotations

import numpy as np

from .scene import RECTANGLE, SPHERE, TRIANGLE, Camera, Material, Scene, Settings


def icosphere(subdiv: int):
    """Unit icosphere with outward winding; shared edges share exact vertex values."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
             (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.asarray(v, np.float64) / np.linalg.norm(v) for v in verts]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
             (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache = {}

        def mid(i, j):
            key = (min(i, j), max(i, j))
            if key not in cache:
                m = verts[i] + verts[j]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    V = np.stack(verts)
    F = np.asarray(faces, np.int64)
    return V, F


class _Builder:
    def __init__(self):
        self.materials = []
        self.shape, self.mat, self.a, self.b, self.c, self.r = [], [], [], [], [], []
        self.eprim, erad = [], []
        self.erad = erad

    def material(self, m: Material) -> int:
        self.materials.append(m)
        return len(self.materials) - 1

    def tri(self, m, p0, p1, p2):
        self.shape.append(TRIANGLE); self.mat.append(m)
        self.a.append(p0); self.b.append(p1); self.c.append(p2); self.r.append(1.0)
        return len(self.shape) - 1

    def rect(self, m, origin, eu, ev):
        self.shape.append(RECTANGLE); self.mat.append(m)
        self.a.append(origin); self.b.append(eu); self.c.append(ev); self.r.append(1.0)
        return len(self.shape) - 1

    def sphere(self, m, center, radius):
        self.shape.append(SPHERE); self.mat.append(m)
        self.a.append(center); self.b.append((0.0, 0.0, 0.0)); self.c.append((0.0, 0.0, 0.0)); self.r.append(radius)
        return len(self.shape) - 1

    def quad_tris(self, m, p0, p1, p2, p3):
        """Two triangles (p0,p1,p2), (p0,p2,p3)."""
        self.tri(m, p0, p1, p2)
        self.tri(m, p0, p2, p3)

    def mesh(self, m, V, F, center, radius):
        P = V * radius + np.asarray(center, np.float64)
        A, B, C = P[F[:, 0]], P[F[:, 1]], P[F[:, 2]]
        n0 = len(self.shape)
        self.shape += [TRIANGLE] * len(F)
        self.mat += [m] * len(F)
        self.a += list(A); self.b += list(B); self.c += list(C); self.r += [1.0] * len(F)
        return n0

    def emitter(self, prim, radiance):
        self.eprim.append(prim)
        self.erad.append(radiance)

    def build(self, camera: Camera, settings: Settings) -> Scene:
        f = lambda L: np.asarray(L, np.float64).reshape(-1, 3)
        return Scene(materials=self.materials, shape=np.asarray(self.shape, np.int32),
                     mat=np.asarray(self.mat, np.int32), a=f(self.a), b=f(self.b), c=f(self.c),
                     radius=np.asarray(self.r, np.float64), emitter_prim=np.asarray(self.eprim, np.int32),
                     emitter_radiance=f(self.erad), camera=camera, settings=settings)


def _cornell(bld: _Builder, floor_mat: int, white: int, red: int, green: int, lamp: int, radiance: float):
    o = 0.0
    bld.quad_tris(floor_mat, (o, o, o), (o, o, 1.0), (1.0, o, 1.0), (1.0, o, o))          # floor y=0
    bld.quad_tris(white, (o, 1.0, o), (1.0, 1.0, o), (1.0, 1.0, 1.0), (o, 1.0, 1.0))      # ceiling y=1
    bld.quad_tris(white, (o, o, o), (1.0, o, o), (1.0, 1.0, o), (o, 1.0, o))              # back z=0
    bld.quad_tris(red, (o, o, o), (o, 1.0, o), (o, 1.0, 1.0), (o, o, 1.0))                # left x=0
    bld.quad_tris(green, (1.0, o, o), (1.0, o, 1.0), (1.0, 1.0, 1.0), (1.0, 1.0, o))      # right x=1
    h, lo, hi = 0.998, 0.375, 0.625
    l0 = bld.tri(lamp, (lo, h, lo), (hi, h, lo), (hi, h, hi))                             # normals face -y
    l1 = bld.tri(lamp, (lo, h, lo), (hi, h, hi), (lo, h, hi))
    bld.emitter(l0, (radiance, radiance, radiance))
    bld.emitter(l1, (radiance, radiance, radiance))


def cornell_c1(resolution: int = 256, spp: int = 16, max_depth: int = 8, seed: int = 0,
               subdiv: int = 4) -> Scene:
    """BASELINE.json configs[0]."""
    bld = _Builder()
    white = bld.material(Material("white", (0.7, 0.7, 0.7), 0.0, 1.0, 0.0, 1.5))
    red = bld.material(Material("red", (0.7, 0.1, 0.1), 0.0, 1.0, 0.0, 1.5))
    green = bld.material(Material("green", (0.1, 0.7, 0.1), 0.0, 1.0, 0.0, 1.5))
    lamp = bld.material(Material("lamp", (0.04, 0.04, 0.04), 0.0, 1.0, 0.0, 1.5))
    mirror = bld.material(Material("mirror", (0.95, 0.95, 0.95), 1.0, 0.01, 0.0, 1.5))
    _cornell(bld, white, white, red, green, lamp, 15.0)
    V, F = icosphere(subdiv)
    bld.mesh(mirror, V, F, (0.5, 0.3, 0.5), 0.2)
    cam = Camera((0.5, 0.5, 2.2), (0.5, 0.5, 0.0), (0.0, 1.0, 0.0), 40.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, spp, seed))


def cornell_c2(resolution: int = 512, spp: int = 64, max_depth: int = 10, seed: int = 0,
               mirror_subdiv: int = 4, glass_subdiv: int = 5) -> Scene:
    """BASELINE.json configs[1]: adds a dielectric icosphere and a GGX (roughness 0.1) floor."""
    bld = _Builder()
    white = bld.material(Material("white", (0.7, 0.7, 0.7), 0.0, 1.0, 0.0, 1.5))
    red = bld.material(Material("red", (0.7, 0.1, 0.1), 0.0, 1.0, 0.0, 1.5))
    green = bld.material(Material("green", (0.1, 0.7, 0.1), 0.0, 1.0, 0.0, 1.5))
    lamp = bld.material(Material("lamp", (0.04, 0.04, 0.04), 0.0, 1.0, 0.0, 1.5))
    mirror = bld.material(Material("mirror", (0.95, 0.95, 0.95), 1.0, 0.01, 0.0, 1.5))
    glass = bld.material(Material("glass", (1.0, 1.0, 1.0), 0.0, 0.01, 1.0, 1.5))
    floor = bld.material(Material("glossy_floor", (0.8, 0.8, 0.8), 1.0, 0.1, 0.0, 1.5))
    _cornell(bld, floor, white, red, green, lamp, 15.0)
    V, F = icosphere(mirror_subdiv)
    bld.mesh(mirror, V, F, (0.5, 0.3, 0.5), 0.2)
    V, F = icosphere(glass_subdiv)
    bld.mesh(glass, V, F, (0.25, 0.205, 0.81), 0.2)
    cam = Camera((0.5, 0.5, 2.2), (0.5, 0.5, 0.0), (0.0, 1.0, 0.0), 40.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, spp, seed))


# ---------------------------------------------------------------- small test scenes
def caustic_box(resolution: int = 8, max_depth: int = 6) -> Scene:
    """Closed box, mirrored floor, small downward lamp: every proxy stage is reachable
    (same role as the reference's caustic-box fixture, own geometry)."""
    bld = _Builder()
    plaster = bld.material(Material("plaster", (0.45, 0.45, 0.45), 0.0, 0.9))
    mirror = bld.material(Material("mirror", (0.9, 0.9, 0.9), 1.0, 0.01))
    shell = bld.material(Material("shell", (0.05, 0.05, 0.05), 0.0, 0.9))
    bld.rect(mirror, (0, 0, 0), (0, 0, 2), (2, 0, 0))
    bld.rect(plaster, (0, 2, 0), (2, 0, 0), (0, 0, 2))
    bld.rect(plaster, (0, 0, 0), (2, 0, 0), (0, 2, 0))
    bld.rect(plaster, (0, 0, 2), (0, 2, 0), (2, 0, 0))
    bld.rect(plaster, (0, 0, 0), (0, 2, 0), (0, 0, 2))
    bld.rect(plaster, (2, 0, 0), (0, 0, 2), (0, 2, 0))
    lamp = bld.rect(shell, (0.86, 0.42, 0.86), (0.28, 0, 0), (0, 0, 0.28))
    bld.emitter(lamp, (100.0, 100.0, 100.0))
    cam = Camera((1.0, 0.35, 1.8), (1.0, 1.9, 0.9), (0, 1, 0), 60.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, 4, 0))


def diffuse_box(resolution: int = 8, max_depth: int = 6) -> Scene:
    """No specular material: the proxy machinery can never activate."""
    bld = _Builder()
    wall = bld.material(Material("wall", (0.65, 0.65, 0.65), 0.0, 1.0))
    glow = bld.material(Material("glow", (0.0, 0.0, 0.0), 0.0, 1.0))
    bld.rect(wall, (0, 0, 0), (0, 0, 2), (2, 0, 0))
    bld.rect(wall, (0, 2, 0), (2, 0, 0), (0, 0, 2))
    bld.rect(wall, (0, 0, 0), (2, 0, 0), (0, 2, 0))
    bld.rect(wall, (0, 0, 2), (0, 2, 0), (2, 0, 0))
    bld.rect(wall, (0, 0, 0), (0, 2, 0), (0, 0, 2))
    bld.rect(wall, (2, 0, 0), (0, 0, 2), (0, 2, 0))
    lamp = bld.rect(glow, (0.65, 1.97, 0.65), (0.7, 0, 0), (0, 0, 0.7))
    bld.emitter(lamp, (6.0, 6.0, 6.0))
    cam = Camera((1, 1, 1.8), (1, 1, 0), (0, 1, 0), 60.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, 4, 0))


def glass_slab(resolution: int = 8, max_depth: int = 6) -> Scene:
    """Two parallel glass faces under a small lamp: dropped blocks of two vertices (u = 2)."""
    bld = _Builder()
    felt = bld.material(Material("felt", (0.25, 0.25, 0.25), 0.0, 0.9))
    glass = bld.material(Material("glass", (1, 1, 1), 0.0, 0.01, 1.0, 1.5))
    shell = bld.material(Material("shell", (0.05, 0.05, 0.05), 0.0, 0.9))
    bld.rect(felt, (0, 0, 0), (0, 0, 2), (2, 0, 0))
    bld.rect(glass, (0.25, 1.15, 0.25), (0, 0, 1.5), (1.5, 0, 0))
    bld.rect(glass, (0.25, 1.05, 0.25), (1.5, 0, 0), (0, 0, 1.5))
    lamp = bld.rect(shell, (0.85, 1.75, 0.85), (0.3, 0, 0), (0, 0, 0.3))
    bld.emitter(lamp, (35.0, 35.0, 35.0))
    cam = Camera((1.0, 0.45, 1.9), (1.0, 1.1, 0.5), (0, 1, 0), 60.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, 1, 0))


def sphere_room(resolution: int = 16, max_depth: int = 6) -> Scene:
    """Analytic spheres (mirror, glass, diffuse, an emissive sphere) in an open room:
    covers the sphere intersection, sphere light sampling and both sphere roots."""
    bld = _Builder()
    wall = bld.material(Material("wall", (0.6, 0.55, 0.5), 0.0, 1.0))
    mirror = bld.material(Material("mirror", (0.9, 0.9, 0.9), 1.0, 0.01))
    glass = bld.material(Material("glass", (1, 1, 1), 0.0, 0.01, 1.0, 1.5))
    rough = bld.material(Material("rough_metal", (0.8, 0.6, 0.4), 1.0, 0.35))
    glow = bld.material(Material("glow", (0, 0, 0), 0.0, 1.0))
    bld.rect(wall, (-2, 0, -2), (0, 0, 4), (4, 0, 0))
    bld.rect(wall, (-2, 0, -2), (4, 0, 0), (0, 3, 0))
    bld.sphere(mirror, (-0.7, 0.5, -0.3), 0.5)
    bld.sphere(glass, (0.6, 0.45, 0.2), 0.45)
    bld.sphere(rough, (0.1, 0.3, -1.0), 0.3)
    s = bld.sphere(glow, (0.0, 2.2, 0.0), 0.25)
    bld.emitter(s, (12.0, 12.0, 12.0))
    cam = Camera((0, 1.0, 3.5), (0, 0.6, 0), (0, 1, 0), 45.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, 4, 0))


CONFIGS = {"C1": cornell_c1, "C2": cornell_c2}
