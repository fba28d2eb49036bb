"""Seeded synthetic inputs shaped like the paper's workloads (numpy only).

This module is the ONE piece shared by the CUDA path's tests/bench and the
oracle's tests: it draws Gaussians, lights, query positions and test atlases.
It holds none of the method's arithmetic (no beta, no octahedral map, no
footprints, no erf): only scene geometry and random numbers.

Workload recipe.  World axes are
z-up, metres.  Counts / atlas sizes / light counts come from BASELINE.json
``configs``; the distributions are our proposal, modelled on trained 3DGS
content (the paper gives no Gaussian statistics):

* rotations: surface Gaussians align their thin axis (local z) with the surface
  normal with a random in-plane spin; volumetric ones are uniform (Shoemake);
* scene scales: log-normal per axis (indoor median 1.5 cm, sigma_ln 0.7;
  outdoor 4 cm, 0.9), thin axis x U(0.05, 0.5), clipped to [0.5 mm, 0.5 m];
* avatar scales: median 6 mm, sigma_ln 0.4, clipped to [1 mm, 3 cm];
* opacity: alpha = sigmoid(z), z ~ 0.7 N(4, 1.5^2) + 0.3 N(-1.5, 1.5^2);
* every Gaussian keeps >= 0.3 m + 3 sigma_max from every light;
* t_max = max distance from the light to the scene AABB corners + 0.5 m;
* seed: ``np.random.Generator(PCG64(260101660 + cfg))``.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional

import numpy as np

SEED_BASE = 260101660


@dataclasses.dataclass
class Scene:
    name: str
    gaussians: Dict[str, np.ndarray]  # occluders: means[n,3] scales[n,3] rotations[n,4] opacities[n]
    lights: Dict[str, np.ndarray]     # position[L,3], t_max[L]
    res: int
    K: int
    queries: np.ndarray               # receiver centres [m,3] float32
    note: str = ""

    @property
    def n(self) -> int:
        return int(self.gaussians["means"].shape[0])

    @property
    def L(self) -> int:
        return int(self.lights["position"].shape[0])


def rng_for(cfg: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + cfg + 1000 * salt))


# ---------------------------------------------------------------- rotations
def random_quaternions(rng, n):
    """Uniform random unit quaternions (Shoemake), (w, x, y, z)."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    q = np.stack([a * np.sin(2 * np.pi * u2), a * np.cos(2 * np.pi * u2),
                  b * np.sin(2 * np.pi * u3), b * np.cos(2 * np.pi * u3)], axis=1)
    return q


def matrix_to_quaternion(R):
    """Rotation matrices [n,3,3] -> unit quaternions [n,4] (w,x,y,z), the
    inverse of the standard (3DGS) quaternion->matrix convention."""
    R = np.asarray(R, dtype=np.float64)
    n = R.shape[0]
    q = np.zeros((n, 4))
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    c0 = tr > 0
    s = np.sqrt(np.maximum(tr[c0] + 1.0, 1e-300)) * 2
    q[c0, 0] = 0.25 * s
    q[c0, 1] = (R[c0, 2, 1] - R[c0, 1, 2]) / s
    q[c0, 2] = (R[c0, 0, 2] - R[c0, 2, 0]) / s
    q[c0, 3] = (R[c0, 1, 0] - R[c0, 0, 1]) / s
    rest = ~c0
    i1 = rest & (R[:, 0, 0] >= R[:, 1, 1]) & (R[:, 0, 0] >= R[:, 2, 2])
    s = np.sqrt(np.maximum(1.0 + R[i1, 0, 0] - R[i1, 1, 1] - R[i1, 2, 2], 1e-300)) * 2
    q[i1, 0] = (R[i1, 2, 1] - R[i1, 1, 2]) / s
    q[i1, 1] = 0.25 * s
    q[i1, 2] = (R[i1, 0, 1] + R[i1, 1, 0]) / s
    q[i1, 3] = (R[i1, 0, 2] + R[i1, 2, 0]) / s
    i2 = rest & ~i1 & (R[:, 1, 1] >= R[:, 2, 2])
    s = np.sqrt(np.maximum(1.0 + R[i2, 1, 1] - R[i2, 0, 0] - R[i2, 2, 2], 1e-300)) * 2
    q[i2, 0] = (R[i2, 0, 2] - R[i2, 2, 0]) / s
    q[i2, 1] = (R[i2, 0, 1] + R[i2, 1, 0]) / s
    q[i2, 2] = 0.25 * s
    q[i2, 3] = (R[i2, 1, 2] + R[i2, 2, 1]) / s
    i3 = rest & ~i1 & ~i2
    s = np.sqrt(np.maximum(1.0 + R[i3, 2, 2] - R[i3, 0, 0] - R[i3, 1, 1], 1e-300)) * 2
    q[i3, 0] = (R[i3, 1, 0] - R[i3, 0, 1]) / s
    q[i3, 1] = (R[i3, 0, 2] + R[i3, 2, 0]) / s
    q[i3, 2] = (R[i3, 1, 2] + R[i3, 2, 1]) / s
    q[i3, 3] = 0.25 * s
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def quaternion_to_matrix(q):
    """Standard (3DGS) convention, (w,x,y,z) -> [n,3,3]; used only to move
    scenes around (rotating test scenes), never by the method."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((q.shape[0], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z); R[:, 0, 1] = 2 * (x * y - w * z); R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z); R[:, 1, 1] = 1 - 2 * (x * x + z * z); R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y); R[:, 2, 1] = 2 * (y * z + w * x); R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def surface_quaternions(rng, normals):
    """Rotation whose local z axis is the surface normal, random spin about it."""
    n = normals / np.linalg.norm(normals, axis=1, keepdims=True)
    a = np.where(np.abs(n[:, :1]) < 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 1.0, 0]]))
    t1 = np.cross(n, a)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(n, t1)
    phi = rng.random(n.shape[0]) * 2 * np.pi
    c, s = np.cos(phi)[:, None], np.sin(phi)[:, None]
    e1, e2 = c * t1 + s * t2, -s * t1 + c * t2
    R = np.stack([e1, e2, n], axis=2)  # columns: local x, y, z
    return matrix_to_quaternion(R)


# ------------------------------------------------------------------ scales
def lognormal_scales(rng, n, median, sigma_ln, lo, hi, thin=True):
    s = median * np.exp(sigma_ln * rng.standard_normal((n, 3)))
    if thin:
        s[:, 2] *= rng.uniform(0.05, 0.5, n)
    return np.clip(s, lo, hi)


def opacities_3dgs(rng, n):
    z = np.where(rng.random(n) < 0.7, rng.normal(4.0, 1.5, n), rng.normal(-1.5, 1.5, n))
    return 1.0 / (1.0 + np.exp(-z))


# -------------------------------------------------------- surface samplers
def sample_rect(rng, n, origin, e1, e2, normal, jitter=0.002):
    a, b = rng.random(n), rng.random(n)
    p = origin[None] + a[:, None] * e1[None] + b[:, None] * e2[None]
    p += normal[None] * rng.normal(0, jitter, n)[:, None]
    return p, np.repeat(normal[None], n, axis=0)


def sample_box(rng, n, lo, hi, bottom=False):
    """Points on the faces of an axis-aligned box (area-weighted)."""
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    ext = hi - lo
    faces = [  # origin, e1, e2, normal
        (np.array([lo[0], lo[1], hi[2]]), np.array([ext[0], 0, 0]), np.array([0, ext[1], 0]), np.array([0, 0, 1.0])),
        (np.array([lo[0], lo[1], lo[2]]), np.array([ext[0], 0, 0]), np.array([0, 0, ext[2]]), np.array([0, -1.0, 0])),
        (np.array([lo[0], hi[1], lo[2]]), np.array([ext[0], 0, 0]), np.array([0, 0, ext[2]]), np.array([0, 1.0, 0])),
        (np.array([lo[0], lo[1], lo[2]]), np.array([0, ext[1], 0]), np.array([0, 0, ext[2]]), np.array([-1.0, 0, 0])),
        (np.array([hi[0], lo[1], lo[2]]), np.array([0, ext[1], 0]), np.array([0, 0, ext[2]]), np.array([1.0, 0, 0])),
    ]
    if bottom:
        faces.append((np.array([lo[0], lo[1], lo[2]]), np.array([ext[0], 0, 0]), np.array([0, ext[1], 0]), np.array([0, 0, -1.0])))
    areas = np.array([np.linalg.norm(np.cross(f[1], f[2])) for f in faces])
    counts = rng.multinomial(n, areas / areas.sum())
    P, N = [], []
    for f, c in zip(faces, counts):
        if c:
            p, nn = sample_rect(rng, c, *f)
            P.append(p); N.append(nn)
    return np.concatenate(P), np.concatenate(N)


def sample_capsules(rng, n, caps):
    """Points on the surfaces of capsules [(p0, p1, radius)], area-weighted."""
    areas = np.array([2 * np.pi * r * np.linalg.norm(np.subtract(p1, p0)) + 4 * np.pi * r * r
                      for p0, p1, r in caps])
    counts = rng.multinomial(n, areas / areas.sum())
    P, N = [], []
    for (p0, p1, r), c in zip(caps, counts):
        if c == 0:
            continue
        p0, p1 = np.asarray(p0, float), np.asarray(p1, float)
        axis = p1 - p0
        Lc = np.linalg.norm(axis)
        ax = axis / Lc
        a = np.array([1.0, 0, 0]) if abs(ax[0]) < 0.9 else np.array([0, 1.0, 0])
        t1 = np.cross(ax, a); t1 /= np.linalg.norm(t1)
        t2 = np.cross(ax, t1)
        # position along the capsule's "unrolled" length: cylinder then caps
        side = rng.random(c) < (2 * np.pi * r * Lc) / (2 * np.pi * r * Lc + 4 * np.pi * r * r)
        phi = rng.random(c) * 2 * np.pi
        radial = np.cos(phi)[:, None] * t1 + np.sin(phi)[:, None] * t2
        h = rng.random(c) * Lc
        pts = np.where(side[:, None], p0 + h[:, None] * ax + r * radial, 0)
        nrm = np.where(side[:, None], radial, 0)
        # caps: uniform on sphere, assigned to the nearer end
        v = rng.standard_normal((c, 3)); v /= np.linalg.norm(v, axis=1, keepdims=True)
        end = np.where((v @ ax)[:, None] > 0, p1, p0)
        pts = np.where(side[:, None], pts, end + r * v)
        nrm = np.where(side[:, None], nrm, v)
        P.append(pts); N.append(nrm)
    return np.concatenate(P), np.concatenate(N)


def human_capsules(root, height=1.75, phase=0.0, heading=0.0):
    """Ten-capsule human proxy standing at `root` (x, y, 0); limbs swing by
    +/-30 deg * sin(phase)."""
    s = height / 1.75
    sw = np.deg2rad(30.0) * np.sin(phase)
    ch, sh = np.cos(heading), np.sin(heading)

    def P(x, y, z):  # body frame -> world (heading about z)
        return np.array([root[0] + ch * x - sh * y, root[1] + sh * x + ch * y, z])

    def limb(top, length, angle, lateral):
        # swing in the body's x-z plane
        bot = (top[0] + length * np.sin(angle), top[1], top[2] - length * np.cos(angle))
        return P(top[0], top[1] + lateral, top[2] * 1.0), P(bot[0], bot[1] + lateral, bot[2])

    caps = []
    caps.append((P(0, 0, 1.00 * s), P(0, 0, 1.40 * s), 0.15 * s))          # torso
    caps.append((P(0, 0, 1.55 * s), P(0, 0, 1.65 * s), 0.10 * s))          # head
    for side, sgn in ((0.20 * s, 1.0), (-0.20 * s, -1.0)):
        a0, a1 = limb((0, 0, 1.42 * s), 0.30 * s, sgn * sw, side)
        caps.append((a0, a1, 0.05 * s))                                     # upper arm
        b1 = a1 + (a1 - a0) * 0.9
        caps.append((a1, b1, 0.04 * s))                                     # forearm
        l0, l1 = limb((0, 0, 0.95 * s), 0.45 * s, -sgn * sw, side * 0.5)
        caps.append((l0, l1, 0.07 * s))                                     # thigh
        f1 = l1 + np.array([0, 0, -0.43 * s]) + (l1 - l0) * np.array([0.3, 0.3, 0.0])
        f1[2] = max(f1[2], 0.06 * s)
        caps.append((l1, f1, 0.055 * s))                                    # shin
    return caps


# ------------------------------------------------------------- assembling
def _gaussians(means, scales, quats, alphas):
    return dict(means=np.ascontiguousarray(means, np.float32),
                scales=np.ascontiguousarray(scales, np.float32),
                rotations=np.ascontiguousarray(quats, np.float32),
                opacities=np.ascontiguousarray(alphas, np.float32))


def concat_gaussians(*gs):
    return {k: np.ascontiguousarray(np.concatenate([g[k] for g in gs]), dtype=np.float32)
            for k in ("means", "scales", "rotations", "opacities")}


def keep_clear_of_lights(g, light_pos, margin=0.3):
    """Drop Gaussians whose 3-sigma ellipsoid comes within `margin` of a light."""
    mu, smax = g["means"].astype(np.float64), g["scales"].max(axis=1).astype(np.float64)
    keep = np.ones(mu.shape[0], bool)
    for o in np.asarray(light_pos, np.float64).reshape(-1, 3):
        keep &= np.linalg.norm(mu - o[None], axis=1) > margin + 3.0 * smax
    return {k: v[keep] for k, v in g.items()}


def t_max_for(light_pos, lo, hi):
    """Q2: t_max = max distance from the light to the AABB corners + 0.5 m."""
    corners = np.array([[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])])
    lp = np.asarray(light_pos, np.float64).reshape(-1, 3)
    return (np.linalg.norm(corners[None] - lp[:, None], axis=2).max(axis=1) + 0.5).astype(np.float32)


def _fill(rng, n, make, light_pos, margin=0.3):
    """Draw with `make(rng, m)` until exactly n Gaussians survive the light clearance."""
    parts, have = [], 0
    while have < n:
        g = keep_clear_of_lights(make(rng, int((n - have) * 1.05) + 16), light_pos, margin)
        parts.append(g); have += g["means"].shape[0]
    g = concat_gaussians(*parts)
    return {k: v[:n] for k, v in g.items()}


def surface_set(rng, pts, nrm, median, sigma_ln, lo=5e-4, hi=0.5):
    n = pts.shape[0]
    return _gaussians(pts, lognormal_scales(rng, n, median, sigma_ln, lo, hi, True),
                      surface_quaternions(rng, nrm), opacities_3dgs(rng, n))


def avatar_set(rng, n, caps):
    pts, nrm = sample_capsules(rng, n, caps)
    return _gaussians(pts, lognormal_scales(rng, n, 0.006, 0.4, 1e-3, 3e-2, True),
                      surface_quaternions(rng, nrm), opacities_3dgs(rng, n))


def room_scene(rng, n, size, furniture=6, median=0.015, sigma_ln=0.7):
    """Floor 40 %, walls 35 %, ceiling 10 %, furniture boxes 15 %."""
    X, Y, Z = size
    nf, nw, nc = int(0.40 * n), int(0.35 * n), int(0.10 * n)
    nb = n - nf - nw - nc
    P, N = [], []
    p, q = sample_rect(rng, nf, np.array([0, 0, 0.0]), np.array([X, 0, 0.0]), np.array([0, Y, 0.0]), np.array([0, 0, 1.0]))
    P.append(p); N.append(q)
    p, q = sample_rect(rng, nc, np.array([0, 0, Z]), np.array([X, 0, 0.0]), np.array([0, Y, 0.0]), np.array([0, 0, -1.0]))
    P.append(p); N.append(q)
    walls = [(np.array([0, 0, 0.0]), np.array([X, 0, 0.0]), np.array([0, 0, Z]), np.array([0, 1.0, 0])),
             (np.array([0, Y, 0.0]), np.array([X, 0, 0.0]), np.array([0, 0, Z]), np.array([0, -1.0, 0])),
             (np.array([0, 0, 0.0]), np.array([0, Y, 0.0]), np.array([0, 0, Z]), np.array([1.0, 0, 0])),
             (np.array([X, 0, 0.0]), np.array([0, Y, 0.0]), np.array([0, 0, Z]), np.array([-1.0, 0, 0]))]
    wa = np.array([np.linalg.norm(np.cross(w[1], w[2])) for w in walls])
    for w, c in zip(walls, rng.multinomial(nw, wa / wa.sum())):
        p, q = sample_rect(rng, c, *w)
        P.append(p); N.append(q)
    boxes = []
    for _ in range(furniture):
        w, d, h = rng.uniform(0.4, 1.6), rng.uniform(0.4, 1.0), rng.uniform(0.4, 1.2)
        # furniture along the walls, leaving the room centre free for the avatar
        if rng.random() < 0.5:
            x0 = rng.uniform(0.1, X - w - 0.1); y0 = rng.choice([0.05, Y - d - 0.05])
        else:
            y0 = rng.uniform(0.1, Y - d - 0.1); x0 = rng.choice([0.05, X - w - 0.05])
        boxes.append(([x0, y0, 0.0], [x0 + w, y0 + d, h]))
    ba = np.array([np.prod(np.subtract(b[1], b[0])[:2]) + 2 * (np.subtract(b[1], b[0])[0] + np.subtract(b[1], b[0])[1]) * (b[1][2]) for b in boxes])
    for b, c in zip(boxes, rng.multinomial(nb, ba / ba.sum())):
        if c:
            p, q = sample_box(rng, c, *b)
            P.append(p); N.append(q)
    return surface_set(rng, np.concatenate(P), np.concatenate(N), median, sigma_ln)


# ------------------------------------------------------------------ configs
def config1(seed_salt: int = 0, n: int = 1000) -> Scene:
    """cfg1: 1 light at the origin, 1000 random anisotropic Gaussians in
    [-1.5,1.5]^2 x [1.5,4.5], scales log-uniform [3 cm, 30 cm], alpha ~ U(0.05,
    0.95); 64x64 x 16 shells, t_max = 6 m; query at all centres."""
    rng = rng_for(1, seed_salt)
    mu = np.stack([rng.uniform(-1.5, 1.5, n), rng.uniform(-1.5, 1.5, n), rng.uniform(1.5, 4.5, n)], 1)
    s = np.exp(rng.uniform(np.log(0.03), np.log(0.30), (n, 3)))
    g = _gaussians(mu, s, random_quaternions(rng, n), rng.uniform(0.05, 0.95, n))
    lights = dict(position=np.zeros((1, 3), np.float32), t_max=np.array([6.0], np.float32))
    return Scene("cfg1", g, lights, 64, 16, g["means"].copy(),
                 "1 light, 1000 Gaussians, 64x64x16 (oracle in seconds)")


def rotate_scene(scene: Scene, R: np.ndarray, name: Optional[str] = None) -> Scene:
    """Rotate Gaussians, lights and queries about the origin by R (3x3)."""
    R = np.asarray(R, np.float64)
    g = scene.gaussians
    Rg = quaternion_to_matrix(g["rotations"])
    q = matrix_to_quaternion(R[None] @ Rg)
    g2 = _gaussians(g["means"].astype(np.float64) @ R.T, g["scales"], q, g["opacities"])
    lights = dict(position=(scene.lights["position"].astype(np.float64) @ R.T).astype(np.float32),
                  t_max=scene.lights["t_max"].copy())
    return Scene(name or scene.name + "-rot", g2, lights, scene.res, scene.K,
                 (scene.queries.astype(np.float64) @ R.T).astype(np.float32), scene.note)


def axis_rotation(src, dst):
    """Rotation taking unit vector src to dst (Rodrigues)."""
    a = np.asarray(src, float) / np.linalg.norm(src)
    b = np.asarray(dst, float) / np.linalg.norm(dst)
    v, c = np.cross(a, b), float(a @ b)
    if np.linalg.norm(v) < 1e-12:
        if c > 0:
            return np.eye(3)
        p = np.array([1.0, 0, 0]) if abs(a[0]) < 0.9 else np.array([0, 1.0, 0])
        v = np.cross(a, p); v /= np.linalg.norm(v)
        return 2 * np.outer(v, v) - np.eye(3)
    vx = np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])
    return np.eye(3) + vx + vx @ vx / (1 + c)


SEAM_DIRECTIONS = {"-z": (0, 0, -1.0), "+x": (1.0, 0, 0), "corner": (1.0, 1.0, -1.0)}


def config1_seam(direction: str) -> Scene:
    """cfg1 rotated to face -z, +x or a corner direction (atlas borders)."""
    base = config1()
    return rotate_scene(base, axis_rotation((0, 0, 1.0), SEAM_DIRECTIONS[direction]),
                        f"cfg1-seam{direction}")


def config2(scale: float = 1.0, res: int = 512, K: int = 64) -> Scene:
    """cfg2 (ScanNet++-scale room): 6x5x3 m room with 1.0 M scene Gaussians and
    a 100 k avatar at the centre; 1 light at avatar xy + (0.4, -0.3), z = 2.6;
    512^2 x 64; query all 1.0 M scene centres.  `scale` shrinks the counts
    (parity tests at oracle-sized cases)."""
    rng = rng_for(2)
    size = (6.0, 5.0, 3.0)
    root = (3.0, 2.5, 0.0)
    lp = np.array([[root[0] + 0.4, root[1] - 0.3, 2.6]])
    n_scene, n_av = int(round(1_000_000 * scale)), int(round(100_000 * scale))
    scene = _fill(rng, n_scene, lambda r, m: room_scene(r, m, size), lp)
    avatar = _fill(rng, n_av, lambda r, m: avatar_set(r, m, human_capsules(root)), lp)
    g = concat_gaussians(scene, avatar)
    lights = dict(position=lp.astype(np.float32), t_max=t_max_for(lp, (0, 0, 0), size))
    return Scene("cfg2", g, lights, res, K, scene["means"].copy(),
                 f"room 6x5x3 m, {n_scene} scene + {n_av} avatar Gaussians, 1 light, {res}^2 x {K}")


def terrain_scene(rng, n, extent=80.0):
    """80x80 m height field (70 %), 20 boxes up to 15 m (15 %), tree clusters (15 %)."""
    nt, nb = int(0.70 * n), int(0.15 * n)
    nr = n - nt - nb
    x, y = rng.uniform(0, extent, nt), rng.uniform(0, extent, nt)
    k1, k2 = 2 * np.pi / 37.0, 2 * np.pi / 23.0
    h = 1.5 * np.sin(k1 * x) * np.cos(k2 * y) + 0.7 * np.sin(k2 * x + 1.0)
    dhx = 1.5 * k1 * np.cos(k1 * x) * np.cos(k2 * y) + 0.7 * k2 * np.cos(k2 * x + 1.0)
    dhy = -1.5 * k2 * np.sin(k1 * x) * np.sin(k2 * y)
    pts = np.stack([x, y, h], 1)
    nrm = np.stack([-dhx, -dhy, np.ones_like(x)], 1)
    parts = [surface_set(rng, pts, nrm, 0.04, 0.9)]
    boxes = []
    for _ in range(20):
        w, d, hh = rng.uniform(3, 10), rng.uniform(3, 10), rng.uniform(3, 15)
        x0, y0 = rng.uniform(2, extent - w - 2), rng.uniform(2, extent - d - 2)
        boxes.append(([x0, y0, -1.0], [x0 + w, y0 + d, hh]))
    ba = np.array([(b[1][0] - b[0][0]) * (b[1][1] - b[0][1]) + 2 * ((b[1][0] - b[0][0]) + (b[1][1] - b[0][1])) * (b[1][2] - b[0][2]) for b in boxes])
    P, N = [], []
    for b, c in zip(boxes, rng.multinomial(nb, ba / ba.sum())):
        if c:
            p, q = sample_box(rng, c, *b)
            P.append(p); N.append(q)
    parts.append(surface_set(rng, np.concatenate(P), np.concatenate(N), 0.04, 0.9))
    # trees: trunks are not modelled; crowns are isotropic-ish volumetric blobs
    n_trees = 60
    centers = np.stack([rng.uniform(2, extent - 2, n_trees), rng.uniform(2, extent - 2, n_trees), rng.uniform(4, 8, n_trees)], 1)
    which = rng.integers(0, n_trees, nr)
    v = rng.standard_normal((nr, 3))
    v *= (rng.random(nr) ** (1 / 3) * rng.uniform(1.5, 3.0, nr))[:, None] / np.linalg.norm(v, axis=1, keepdims=True)
    tp = centers[which] + v
    ts = lognormal_scales(rng, nr, 0.04, 0.9, 5e-4, 0.5, False)
    parts.append(_gaussians(tp, ts, random_quaternions(rng, nr), opacities_3dgs(rng, nr)))
    return concat_gaussians(*parts)


def config3(scale: float = 1.0, res: int = 1024, K: int = 64) -> Scene:
    """cfg3 (DL3DV/SuperSplat-scale outdoor): 3 M Gaussians, 4 lights on a 2x2
    grid at z = 10-15 m, 1024^2 x 64, query all 3 M."""
    rng = rng_for(3)
    n = int(round(3_000_000 * scale))
    lp = np.array([[25.0, 25.0, 12.0], [55.0, 25.0, 10.0], [25.0, 55.0, 15.0], [55.0, 55.0, 13.0]])
    g = _fill(rng, n, lambda r, m: terrain_scene(r, m), lp)
    lights = dict(position=lp.astype(np.float32), t_max=t_max_for(lp, (0, 0, -3.0), (80.0, 80.0, 16.0)))
    return Scene("cfg3", g, lights, res, K, g["means"].copy(),
                 f"outdoor 80x80 m, {n} Gaussians, 4 lights, {res}^2 x {K}")


def _config4_light():
    size = (10.0, 8.0, 3.5)
    lp = np.array([[5.5, 3.5, 3.1]])
    return size, lp, dict(position=lp.astype(np.float32), t_max=t_max_for(lp, (0, 0, 0), size))


def _config4_prop(scale: float = 1.0):
    """cfg4's 50 k prop (its own seed: frames can be generated without the room)."""
    _, lp, _ = _config4_light()
    return _fill(rng_for(4, 3), int(round(50_000 * scale)),
                 lambda r, m: surface_set(r, *sample_box(r, m, (6.2, 4.6, 0.0), (6.7, 5.1, 0.9)), 0.01, 0.5), lp)


def _config4_static(scale: float = 1.0, room: bool = True):
    """cfg4's static part: the 2.0 M room (the receivers), the 50 k prop, the light."""
    size, lp, lights = _config4_light()
    n_room, n_av = (int(round(x * scale)) for x in (2_000_000, 150_000))
    room_g = _fill(rng_for(4), n_room, lambda r, m: room_scene(r, m, size, furniture=8), lp) if room else None
    return room_g, _config4_prop(scale), lights, n_av


def config4_avatar(frame: int, n_av: int, light_pos) -> Dict[str, np.ndarray]:
    """The walking avatar of cfg4 at `frame` (30 fps): root +3.33 cm/frame along x,
    limbs swinging at 1 Hz; its Gaussians keep their body-relative sampling
    (the same seed every frame)."""
    arng = rng_for(4, 7)
    caps = human_capsules(config4_root(frame), phase=2 * np.pi * frame / 30.0)
    return keep_clear_of_lights(avatar_set(arng, n_av, caps), light_pos)


def config4_root(frame: int):
    return (3.0 + 0.0333 * frame, 4.0, 0.0)


def config4(frame: int = 0, scale: float = 1.0, occluders: str = "avatar+prop",
            res: int = 512, K: int = 64) -> Scene:
    """cfg4 (animated avatar): 2.0 M-Gaussian 10x8x3.5 m room, a 150 k avatar
    walking 4 m over 120 frames (root +3.33 cm/frame, limbs +/-30 deg at 1 Hz,
    30 fps) and a 50 k prop (0.5x0.5x0.9 m box); 1 light at 512^2 x 64.
    Occluders are avatar + prop (the paper's setting) or 'all'; the query
    runs over the 2.0 M scene centres."""
    room, prop, lights, n_av = _config4_static(scale)
    avatar = config4_avatar(frame, n_av, lights["position"])
    occ = concat_gaussians(avatar, prop) if occluders != "all" else concat_gaussians(room, avatar, prop)
    return Scene(f"cfg4-f{frame}", occ, lights, res, K, room["means"].copy(),
                 f"room + walking avatar frame {frame}, occluders={occluders}, {res}^2 x {K}")


class Config4Sequence:
    """cfg4 as BASELINE defines it: 120 frames of the walking avatar + the prop
    (the occluders of the paper's setting) over the static 2 M room
    (the receivers).  frame(f) = the occluders of frame f (== config4(f).gaussians)."""

    def __init__(self, n_frames: int = 120, scale: float = 1.0, res: int = 512, K: int = 64, room: bool = True):
        self.room, self.prop, self.lights, self.n_av = _config4_static(scale, room)
        self.n_frames, self.res, self.K = n_frames, res, K
        self.queries = self.room["means"].copy() if room else None

    def frame(self, f: int) -> Dict[str, np.ndarray]:
        return concat_gaussians(config4_avatar(f, self.n_av, self.lights["position"]), self.prop)

    _static = None

    @classmethod
    def frame_static(cls, f: int) -> Dict[str, np.ndarray]:
        """frame(f) of the full-scale sequence, the static part built once per
        process (for generating frames in worker processes)."""
        if cls._static is None:
            cls._static = cls(room=False)
        return cls._static.frame(f)

    def roi(self, f: int):
        """ROI B of P:L156-158 around the avatar: centre = its root at mid-height
        (the paper's alpha-weighted avatar centroid, here from the synthetic rig),
        R = 2 m (the paper's example), z in [-0.1, 2.5] m."""
        x, y, _ = config4_root(f)
        return (x, y, 0.9, 2.0, -0.1, 2.5)


def config5(scale: float = 1.0, res: int = 2048, K: int = 128) -> Scene:
    """cfg5 (multi-avatar stress): 30x20x6 m hall, 5.4 M scene + 4 x 150 k
    avatars = 6 M; 8 lights on a 4x2 ceiling grid at z = 5.5; 2048^2 x 128."""
    rng = rng_for(5)
    size = (30.0, 20.0, 6.0)
    lp = np.array([[x, y, 5.5] for x in (4.0, 11.0, 19.0, 26.0) for y in (6.0, 14.0)])
    n_scene, n_av = int(round(5_400_000 * scale)), int(round(150_000 * scale))
    scene = _fill(rng, n_scene, lambda r, m: room_scene(r, m, size, furniture=30), lp)
    roots = [(8.0, 8.0, 0.0), (13.0, 12.0, 0.0), (18.0, 9.0, 0.0), (23.0, 12.5, 0.0)]
    avs = [_fill(rng, n_av, lambda r, m, rt=rt: avatar_set(r, m, human_capsules(rt)), lp) for rt in roots]
    g = concat_gaussians(scene, *avs)
    lights = dict(position=lp.astype(np.float32), t_max=t_max_for(lp, (0, 0, 0), size))
    return Scene("cfg5", g, lights, res, K, scene["means"].copy(),
                 f"hall 30x20x6 m, {n_scene}+4x{n_av} Gaussians, 8 lights, {res}^2 x {K}")


def make_config(cfg: int, **kw) -> Scene:
    return {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[cfg](**kw)


# --------------------------------------------------------- small test inputs
def random_scene(seed: int, n: int, res: int = 32, K: int = 8, L: int = 1,
                 dist=(1.0, 4.0), scale=(0.02, 0.4), m_queries: int = 256,
                 everywhere: bool = True) -> Scene:
    """Tiny random scenes for parity: Gaussians in a shell around the lights
    in all directions (everywhere=True exercises every atlas border/seam)."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 7919 * (seed + 1)))
    lp = rng.uniform(-0.5, 0.5, (L, 3))
    if everywhere:
        v = rng.standard_normal((n, 3)); v /= np.linalg.norm(v, axis=1, keepdims=True)
    else:
        v = np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n), np.ones(n)], 1)
        v /= np.linalg.norm(v, axis=1, keepdims=True)
    mu = lp[rng.integers(0, L, n)] + v * rng.uniform(*dist, n)[:, None]
    s = np.exp(rng.uniform(np.log(scale[0]), np.log(scale[1]), (n, 3)))
    g = _gaussians(mu, s, random_quaternions(rng, n), rng.uniform(0.02, 0.98, n))
    g = keep_clear_of_lights(g, lp, 0.05)
    vq = rng.standard_normal((m_queries, 3)); vq /= np.linalg.norm(vq, axis=1, keepdims=True)
    q = lp[rng.integers(0, L, m_queries)] + vq * rng.uniform(0.2, dist[1] * 1.3, m_queries)[:, None]
    tmax = np.full(L, dist[1] + 1.0, np.float32)
    return Scene(f"random{seed}", g, dict(position=lp.astype(np.float32), t_max=tmax), res, K,
                 q.astype(np.float32))


def random_atlas(seed: int, L: int, K: int, res: int, smooth: bool = False) -> np.ndarray:
    """Seeded [L][K][res][res] float32 table in [0, 1] for query parity."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 104729 * (seed + 1)))
    a = rng.random((L, K, res, res))
    if smooth:
        a = np.sort(a, axis=1)[:, ::-1]  # non-increasing in k, like a transmittance
    return np.ascontiguousarray(a, dtype=np.float32)


def random_queries(seed: int, lights, m: int, r_max: float) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 15485863 * (seed + 1)))
    lp = np.asarray(lights["position"], np.float64).reshape(-1, 3)
    v = rng.standard_normal((m, 3)); v /= np.linalg.norm(v, axis=1, keepdims=True)
    x = lp[rng.integers(0, lp.shape[0], m)] + v * rng.uniform(0.0, r_max, m)[:, None]
    return x.astype(np.float32)


def mc_offsets(n: int, seed: int = 0) -> np.ndarray:
    """Monte Carlo footprint offsets z_i ~ N(0, I_3) (the paper's default receiver
    footprint sampling), seeded; the same draws feed both the CUDA query
    and the oracle.  Weights are 1/n."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 31337 * (seed + 1)))
    return rng.standard_normal((n, 3)).astype(np.float32)
