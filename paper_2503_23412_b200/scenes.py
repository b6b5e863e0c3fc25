"""Seeded synthetic scenes for the BASELINE.json configs (they stand in for the paper's
proprietary scenes, which are not available). Every generator is
deterministic and emits a `Scene` in the reference schema, so the same scene loads in
the reference (via `Scene.to_json()`) and in libpxg.

C1  Cornell box, 10 Lambertian triangles + 2-triangle 0.25x0.25 ceiling lamp (L = 15) +
    subdiv-4 mirror icosphere (5,120 tris) at (0.5, 0.3, 0.5), r = 0.2.
C2  C1 + subdiv-5 dielectric icosphere (20,480 tris, IOR 1.5) + GGX floor (roughness 0.1).
C3  Lens-caustic room: 6 Lambertian rectangles (albedo U(0.3, 0.8) per channel), a 0.2 m^2
    area light of 256x256 rectangle cells with a seeded Bernoulli(0.5) radiance pattern
    {0, 20} (the reference has no textures: one emitter per texel, zero-radiance texels
    included, so area-uniform light sampling sees the same texture a textured light would),
    behind a biconvex dielectric lens (IOR 1.5, aperture radius 0.15, 2 x 19,998 tris)
    that images the light onto the diffuse back wall 3 m away. 105,538 prims.
C4  Procedural scene: 2,000 instances (icosphere subdiv 3 = 1,280 tris, torus 16x8 = 256
    tris, box = 12 tris; type uniform) flattened into ~1.03M triangles, positions U in a
    20 m cube, scale U(0.1, 1), uniform random rotation; per-instance material 60% Lambert
    albedo U(0.2, 0.8), 25% GGX metal roughness U(0.02, 0.2), 15% dielectric IOR 1.5;
    4 rectangular area lights with radiance U(5, 30). 1920x1080, max depth 12.
C5  The C4 scene at 3840x2160, max depth 16 (its 4M-walk pool is a ProxyParams setting).

Fixed choices not given by BASELINE.json (recorded here once): box = unit cube open at
z = 1; lamp at y = 0.998 facing down; camera at (0.5, 0.5, 2.2) looking at (0.5, 0.5, 0),
fov_y 40; glass sphere centre (0.25, 0.205, 0.81); mirror/glass roughness 0.01 (the
reference has no delta BSDF); mirror base colour 0.95.
C3: room x in [-2, 2], y in [0, 3], z in [0, 4.5]; back wall z = 0; lens centre
(0, 1.5, 3), axis -z, surface radius 0.75 (thin-lens focal length 0.75 m), so the light
square centred at (0, 1.5, 4), facing -z, is imaged 3 m away onto the back wall; camera
(1.7, 2.2, 3.6) looking at (-0.3, 1.4, 0), fov_y 55; generator seed 3.
C4: cube [-10, 10]^3; lights 3 x 3 m at y = 9.5 facing down, centres (+-5, 9.5, +-5);
torus radii 1 / 0.3; box half-extent 0.7; dielectric roughness 0.01; camera (0, 2, 14)
looking at the origin, fov_y 55; generator seed 7 (BASELINE.json's seed).
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
    """Accumulates primitives in chunks (numpy blocks), so the 1M-triangle configs build fast."""

    def __init__(self):
        self.materials = []
        self._shape, self._mat, self._a, self._b, self._c, self._r = [], [], [], [], [], []
        self.n = 0
        self.eprim, self.erad = [], []

    def material(self, m: Material) -> int:
        self.materials.append(m)
        return len(self.materials) - 1

    def _add(self, shape, mat, a, b, c, r):
        k = len(a)
        self._shape.append(np.full(k, shape, np.int32) if np.isscalar(shape) else np.asarray(shape, np.int32))
        self._mat.append(np.full(k, mat, np.int32) if np.isscalar(mat) else np.asarray(mat, np.int32))
        for dst, x in ((self._a, a), (self._b, b), (self._c, c)):
            dst.append(np.asarray(x, np.float64).reshape(k, 3))
        self._r.append(np.full(k, r, np.float64) if np.isscalar(r) else np.asarray(r, np.float64))
        self.n += k
        return self.n - k

    def tri(self, m, p0, p1, p2):
        return self._add(TRIANGLE, m, [p0], [p1], [p2], 1.0)

    def rect(self, m, origin, eu, ev):
        return self._add(RECTANGLE, m, [origin], [eu], [ev], 1.0)

    def rects(self, m, origins, eu, ev):
        """Many rectangles sharing edges eu, ev; m scalar or per-rectangle."""
        k = len(origins)
        return self._add(RECTANGLE, m, origins, np.tile(np.asarray(eu, np.float64), (k, 1)),
                         np.tile(np.asarray(ev, np.float64), (k, 1)), 1.0)

    def sphere(self, m, center, radius):
        return self._add(SPHERE, m, [center], [(0.0, 0.0, 0.0)], [(0.0, 0.0, 0.0)], radius)

    def quad_tris(self, m, p0, p1, p2, p3):
        """Two triangles (p0,p1,p2), (p0,p2,p3)."""
        self.tri(m, p0, p1, p2)
        self.tri(m, p0, p2, p3)

    def mesh(self, m, V, F, center, radius):
        P = V * radius + np.asarray(center, np.float64)
        return self.tris(m, P[F[:, 0]], P[F[:, 1]], P[F[:, 2]])

    def tris(self, m, A, B, C):
        """Triangles (A[i], B[i], C[i]); m scalar or per-triangle."""
        return self._add(TRIANGLE, m, A, B, C, 1.0)

    def emitter(self, prim, radiance):
        self.eprim.append(prim)
        self.erad.append(radiance)

    def build(self, camera: Camera, settings: Settings) -> Scene:
        cat = lambda L, shape: np.concatenate(L) if L else np.zeros(shape)
        return Scene(materials=self.materials, shape=cat(self._shape, (0,)).astype(np.int32),
                     mat=cat(self._mat, (0,)).astype(np.int32), a=cat(self._a, (0, 3)), b=cat(self._b, (0, 3)),
                     c=cat(self._c, (0, 3)), radius=cat(self._r, (0,)),
                     emitter_prim=np.asarray(self.eprim, np.int32).reshape(-1),
                     emitter_radiance=np.asarray(self.erad, np.float64).reshape(-1, 3), camera=camera,
                     settings=settings)


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


def _orient_outward(A, B, C, centers):
    """Swap B and C where the geometric normal cross(B-A, C-A) points towards `centers`."""
    n = np.cross(B - A, C - A)
    flip = np.einsum("ij,ij->i", n, (A + B + C) / 3.0 - centers) < 0.0
    B2, C2 = B.copy(), C.copy()
    B2[flip], C2[flip] = C[flip], B[flip]
    return A, B2, C2


def _lens_cap(R: float, aperture: float, rings: int, segs: int, z0: float, sign: float):
    """Spherical cap of a biconvex lens as triangles: z = z0 + sign*(sqrt(R^2-r^2) -
    sqrt(R^2-a^2)) on a polar grid (rings x segs). Rim vertices sit exactly at z = z0, so
    the two caps meet without cracks."""
    r = aperture * np.arange(rings + 1) / rings
    phi = 2.0 * np.pi * np.arange(segs) / segs
    zr = z0 + sign * (np.sqrt(R * R - r * r) - np.sqrt(R * R - aperture * aperture))
    zr[-1] = z0
    P = np.stack([np.outer(r, np.cos(phi)), np.outer(r, np.sin(phi)), np.repeat(zr[:, None], segs, 1)], -1)
    A, B, C = [], [], []
    j = np.arange(segs)
    jn = (j + 1) % segs
    A.append(P[0, j]); B.append(P[1, j]); C.append(P[1, jn])  # centre fan (ring 0 is one point)
    for i in range(1, rings):
        A.append(P[i, j]); B.append(P[i + 1, j]); C.append(P[i + 1, jn])
        A.append(P[i, j]); B.append(P[i + 1, jn]); C.append(P[i, jn])
    return np.concatenate(A), np.concatenate(B), np.concatenate(C)


def lens_room_c3(resolution: int = 1024, spp: int = 256, max_depth: int = 12, seed: int = 0,
                 cells: int = 256, rings: int = 50, segs: int = 202) -> Scene:
    """BASELINE.json configs[2]."""
    rng = np.random.default_rng(3)
    bld = _Builder()
    walls = [bld.material(Material(f"wall{i}", tuple(rng.uniform(0.3, 0.8, 3)), 0.0, 1.0)) for i in range(6)]
    glass = bld.material(Material("lens", (1.0, 1.0, 1.0), 0.0, 0.01, 1.0, 1.5))
    housing = bld.material(Material("light_cell", (0.04, 0.04, 0.04), 0.0, 1.0))
    X0, X1, Y1, Z1 = -2.0, 2.0, 3.0, 4.5
    bld.rect(walls[0], (X0, 0, 0), (0, 0, Z1), (X1 - X0, 0, 0))       # floor, normal +y
    bld.rect(walls[1], (X0, Y1, 0), (X1 - X0, 0, 0), (0, 0, Z1))      # ceiling, normal -y
    bld.rect(walls[2], (X0, 0, 0), (X1 - X0, 0, 0), (0, Y1, 0))       # back wall z = 0, normal +z
    bld.rect(walls[3], (X0, 0, Z1), (0, Y1, 0), (X1 - X0, 0, 0))      # front wall, normal -z
    bld.rect(walls[4], (X0, 0, 0), (0, Y1, 0), (0, 0, Z1))            # left, normal +x
    bld.rect(walls[5], (X1, 0, 0), (0, 0, Z1), (0, Y1, 0))            # right, normal -x
    R, ap, zc = 0.75, 0.15, 3.0
    for sign in (1.0, -1.0):
        A, B, C = _lens_cap(R, ap, rings, segs, 0.0, sign)
        off = np.array([0.0, 1.5, zc])
        A, B, C = _orient_outward(A + off, B + off, C + off, np.tile(off, (len(A), 1)))
        bld.tris(glass, A, B, C)
    side = 0.2 ** 0.5
    d = side / cells
    pattern = rng.random((cells, cells)) < 0.5
    iy, ix = np.meshgrid(np.arange(cells), np.arange(cells), indexing="ij")
    org = np.stack([-side / 2 + ix.ravel() * d, 1.5 - side / 2 + iy.ravel() * d, np.full(cells * cells, 4.0)], -1)
    first = bld.rects(housing, org, (0.0, d, 0.0), (d, 0.0, 0.0))    # cross(eu, ev) = -z: faces the lens
    for k, on in enumerate(pattern.ravel()):
        L = 20.0 if on else 0.0
        bld.emitter(first + k, (L, L, L))
    cam = Camera((1.7, 2.2, 3.6), (-0.3, 1.4, 0.0), (0.0, 1.0, 0.0), 55.0, resolution, resolution)
    return bld.build(cam, Settings(max_depth, spp, seed))


def _torus(R: float, r: float, nu: int, nv: int):
    u = 2.0 * np.pi * np.arange(nu) / nu
    v = 2.0 * np.pi * np.arange(nv) / nv
    U, Vv = np.meshgrid(u, v, indexing="ij")
    P = np.stack([(R + r * np.cos(Vv)) * np.cos(U), (R + r * np.cos(Vv)) * np.sin(U), r * np.sin(Vv)], -1)
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    i, j = i.ravel(), j.ravel()
    i1, j1 = (i + 1) % nu, (j + 1) % nv
    A = np.concatenate([P[i, j], P[i, j]])
    B = np.concatenate([P[i1, j], P[i1, j1]])
    C = np.concatenate([P[i1, j1], P[i, j1]])
    ring = lambda Q: np.stack([R * np.cos(np.arctan2(Q[:, 1], Q[:, 0])), R * np.sin(np.arctan2(Q[:, 1], Q[:, 0])),
                               np.zeros(len(Q))], -1)
    return _orient_outward(A, B, C, ring((A + B + C) / 3.0))


def _box(h: float):
    c = np.array([[x, y, z] for x in (-h, h) for y in (-h, h) for z in (-h, h)])
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    A = np.array([c[q[0]] for q in quads] * 2)
    B = np.array([c[q[1]] for q in quads] + [c[q[2]] for q in quads])
    C = np.array([c[q[2]] for q in quads] + [c[q[3]] for q in quads])
    return _orient_outward(A, B, C, np.zeros_like(A))


def _rotations(rng, n: int):
    """Uniform random rotation matrices (Shoemake's quaternion method)."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    q = np.stack([np.sqrt(1 - u1) * np.sin(2 * np.pi * u2), np.sqrt(1 - u1) * np.cos(2 * np.pi * u2),
                  np.sqrt(u1) * np.sin(2 * np.pi * u3), np.sqrt(u1) * np.cos(2 * np.pi * u3)], -1)
    x, y, z, w = q.T
    return np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
                     np.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
                     np.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1)], 1)


def procedural_c4(width: int = 1920, height: int = 1080, spp: int = 1024, max_depth: int = 12, seed: int = 0,
                  instances: int = 2000, gen_seed: int = 7) -> Scene:
    """BASELINE.json configs[3] (configs[4] is the same scene at 3840x2160, depth 16)."""
    rng = np.random.default_rng(gen_seed)
    Vi, Fi = icosphere(3)
    shapes = [(Vi[Fi[:, 0]], Vi[Fi[:, 1]], Vi[Fi[:, 2]]), _torus(1.0, 0.3, 16, 8), _box(0.7)]
    bld = _Builder()
    kind = rng.integers(0, 3, instances)
    pos = rng.uniform(-10.0, 10.0, (instances, 3))
    scale = rng.uniform(0.1, 1.0, instances)
    rot = _rotations(rng, instances)
    mkind = rng.random(instances)
    for i in range(instances):
        if mkind[i] < 0.60:
            m = Material(f"m{i:04d}", tuple(rng.uniform(0.2, 0.8, 3)), 0.0, 1.0)
        elif mkind[i] < 0.85:
            m = Material(f"m{i:04d}", tuple(rng.uniform(0.6, 0.95, 3)), 1.0, float(rng.uniform(0.02, 0.2)))
        else:
            m = Material(f"m{i:04d}", (1.0, 1.0, 1.0), 0.0, 0.01, 1.0, 1.5)
        mi = bld.material(m)
        A, B, C = shapes[kind[i]]
        M = rot[i] * scale[i]
        bld.tris(mi, A @ M.T + pos[i], B @ M.T + pos[i], C @ M.T + pos[i])
    lamp = bld.material(Material("lamp", (0.04, 0.04, 0.04), 0.0, 1.0))
    for (x, z) in ((-5.0, -5.0), (5.0, -5.0), (-5.0, 5.0), (5.0, 5.0)):
        L = float(rng.uniform(5.0, 30.0))
        k = bld.rect(lamp, (x - 1.5, 9.5, z - 1.5), (3.0, 0.0, 0.0), (0.0, 0.0, 3.0))  # cross = -y: faces down
        bld.emitter(k, (L, L, L))
    cam = Camera((0.0, 2.0, 14.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 55.0, width, height)
    return bld.build(cam, Settings(max_depth, spp, seed))


def procedural_c5(width: int = 3840, height: int = 2160, spp: int = 4096, max_depth: int = 16,
                  seed: int = 0, instances: int = 2000) -> Scene:
    """BASELINE.json configs[4]: the C4 scene at 4K, depth 16 (pool of 4M walks per pass is
    ProxyParams.light_walks = 4 << 20)."""
    return procedural_c4(width, height, spp, max_depth, seed, instances)


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


CONFIGS = {"C1": cornell_c1, "C2": cornell_c2, "C3": lens_room_c3, "C4": procedural_c4, "C5": procedural_c5}
