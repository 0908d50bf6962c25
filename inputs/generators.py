"""Seeded synthetic inputs: the config-4 bump-channel mesh and the dual-solve stress state.

Random draws and geometry only.  Nothing here evaluates the IPM method
(no basis, quadrature, closure or flux); each side (oracle, CUDA path) derives
its own dual variables, normals, areas and neighbour tables from these arrays.
"""
from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------
# cfg 4: seeded jittered Delaunay mesh of the bump channel (reading 18)
# ----------------------------------------------------------------------------

BUMP_X0, BUMP_X1, BUMP_R, BUMP_YC = 1.0, 2.0, 1.3, -1.2


def bump_height(x):
    """Circular-arc bump of height 0.1 on x in [1, 2]: y_b = sqrt(1.3^2 - (x-1.5)^2) - 1.2."""
    x = np.asarray(x, dtype=np.float64)
    yb = np.sqrt(np.maximum(BUMP_R**2 - (x - 1.5) ** 2, 0.0)) + BUMP_YC
    return np.where((x > BUMP_X0) & (x < BUMP_X1), np.maximum(yb, 0.0), 0.0)


def bump_channel_mesh(nx_pts: int = 548, ny_pts: int = 183, seed: int = 9238):
    """Vertices [V,2], CCW triangles [T,3] int32, edge tags [T,3] int32.

    Points of an nx_pts x ny_pts grid on (x,t) in [0,3]x[0,1] are jittered by
    +-0.25 h (boundary points slide only along their boundary), Delaunay
    triangulated, and mapped to y = y_b(x) + t (1 - y_b(x)).
    Edge e of triangle t joins vertices (e, e+1 mod 3); tag 0 bottom wall,
    1 outlet x=3, 2 top wall, 3 inlet x=0, -1 interior.
    """
    from scipy.spatial import Delaunay

    rng = np.random.default_rng(seed)
    hx, ht = 3.0 / (nx_pts - 1), 1.0 / (ny_pts - 1)
    X, T = np.meshgrid(np.linspace(0.0, 3.0, nx_pts), np.linspace(0.0, 1.0, ny_pts), indexing="xy")
    X, T = X.ravel().copy(), T.ravel().copy()
    jx = rng.uniform(-0.25, 0.25, X.shape) * hx
    jt = rng.uniform(-0.25, 0.25, T.shape) * ht
    on_l, on_r = np.isclose(X, 0.0), np.isclose(X, 3.0)
    on_b, on_t = np.isclose(T, 0.0), np.isclose(T, 1.0)
    X = X + np.where(on_l | on_r, 0.0, jx)
    T = T + np.where(on_b | on_t, 0.0, jt)
    pts = np.stack([X, T], axis=1)
    tri = Delaunay(pts).simplices.astype(np.int64)
    a, b, c = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]
    area2 = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1])
    neg = area2 < 0
    tri[neg] = tri[neg][:, [0, 2, 1]]
    side = np.stack([on_b, on_r, on_t, on_l], axis=1)  # [V,4]
    tags = np.full(tri.shape, -1, dtype=np.int32)
    for e in range(3):
        va, vb = tri[:, e], tri[:, (e + 1) % 3]
        common = side[va] & side[vb]
        for s in range(4):
            tags[common[:, s], e] = s
    yb = bump_height(X)
    Y = yb + T * (1.0 - yb)
    vert = np.stack([X, Y], axis=1)
    return vert.astype(np.float64), tri.astype(np.int32), tags


# ----------------------------------------------------------------------------
# Dual-solve stress state (SURVEY §8d "Dual-solve stress input")
# ----------------------------------------------------------------------------

def _smooth_fields(rng, xy: np.ndarray, count: int) -> np.ndarray:
    """count smooth fields in [-1,1] over cell centres xy [C,2] (random low-frequency modes)."""
    out = np.empty((count, xy.shape[0]))
    for i in range(count):
        fx, fy = rng.integers(1, 3, size=2)
        px, py = rng.uniform(0.0, 1.0, size=2)
        out[i] = np.sin(2 * np.pi * (fx * xy[:, 0] + px)) * np.cos(2 * np.pi * (fy * xy[:, 1] + py))
    return out


def stress_state(kind: str, xy: np.ndarray, N: int, m: int, seed: int, gamma: float = 1.4):
    """Base conserved state per cell [C,m] (smooth in space, inside the config's IC ranges)
    and standard-normal draws z [C,N,m] for the higher dual modes (clipped to +-3).

    kind: "burgers" | "euler1d" | "euler2d" | "bump".  Conserved variables are
    (rho, rho v, E = p/(gamma-1) + rho|v|^2/2) — the definition of total energy.
    """
    rng = np.random.default_rng(seed)
    C = xy.shape[0]
    if kind == "burgers":
        s = _smooth_fields(rng, xy, 1)
        base = (7.5 + 3.5 * s[0])[:, None]
    elif kind == "euler1d":
        s = _smooth_fields(rng, xy, 3)
        rho, v, p = 0.55 + 0.4 * s[0], 0.25 + 0.6 * s[1], 0.55 + 0.4 * s[2]
        base = np.stack([rho, rho * v, p / (gamma - 1) + 0.5 * rho * v * v], axis=1)
    elif kind == "euler2d":
        s = _smooth_fields(rng, xy, 4)
        rho, vx, vy, p = 0.82 + 0.6 * s[0], 0.6 + 0.5 * s[1], 0.6 + 0.5 * s[2], 0.75 + 0.6 * s[3]
        base = np.stack([rho, rho * vx, rho * vy, p / (gamma - 1) + 0.5 * rho * (vx * vx + vy * vy)], axis=1)
    elif kind == "bump":
        s = _smooth_fields(rng, xy, 3)
        rho, mach, th = 1.0 + 0.2 * s[0], 0.5 + 0.2 * s[1], 0.05 * s[2]
        p = 1.0 / gamma
        cs = np.sqrt(gamma * p / rho)
        vx, vy = mach * cs * np.cos(th), mach * cs * np.sin(th)
        base = np.stack([rho, rho * vx, rho * vy, p / (gamma - 1) + 0.5 * rho * (vx * vx + vy * vy)], axis=1)
    else:
        raise KeyError(kind)
    z = np.clip(rng.standard_normal((C, N, m)), -3.0, 3.0)
    return base.astype(np.float64), z.astype(np.float64)


# stress amplitudes: lambda_{i,a} = (rel |lambda_{0,a}| + abs) 2^{-|i|} z_{i,a}
STRESS_AMP = {"burgers": (0.0, 0.5), "euler1d": (0.05, 0.0), "euler2d": (0.05, 0.0), "bump": (0.05, 0.0)}


def cell_centres(mesh: dict, vert=None, tri=None) -> np.ndarray:
    """Cell centres [C,2] of a config mesh (1D: y=0)."""
    if mesh["kind"] == "1d":
        dx = (mesh["x1"] - mesh["x0"]) / mesh["nx"]
        x = mesh["x0"] + (np.arange(mesh["nx"]) + 0.5) * dx
        return np.stack([x, np.zeros_like(x)], axis=1)
    if mesh["kind"] == "cart2d":
        dx = (mesh["x1"] - mesh["x0"]) / mesh["nx"]
        dy = (mesh["y1"] - mesh["y0"]) / mesh["ny"]
        X, Y = np.meshgrid(mesh["x0"] + (np.arange(mesh["nx"]) + 0.5) * dx,
                           mesh["y0"] + (np.arange(mesh["ny"]) + 0.5) * dy, indexing="xy")
        return np.stack([X.ravel(), Y.ravel()], axis=1)
    return vert[tri].mean(axis=1)
