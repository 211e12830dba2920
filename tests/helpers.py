"""Tiny hand-built scenes and motions for pins and parity edge cases (no method arithmetic)."""
import numpy as np

from paper_2604_23960_b200 import gen


def ball(r, offset=(0.0, 0.0, 0.0)):
    """An SE(3) body carrying one sphere of radius r at ``offset``."""
    return gen.Robot(kind=gen.SE3, dof=7, sphere_link=np.zeros(1, np.int32),
                     sphere=np.array([[offset[0], offset[1], offset[2], r]], np.float32))


def pose(p, q=(1.0, 0.0, 0.0, 0.0)):
    return list(p) + list(q)


def scene(robots, obs_spheres=None, boxes=None):
    return gen.Scene(list(robots),
                     np.asarray(obs_spheres if obs_spheres is not None else np.zeros((0, 4)), np.float32).reshape(-1, 4),
                     np.asarray(boxes if boxes is not None else np.zeros((0, 6)), np.float32).reshape(-1, 6))


def motions(wp, T):
    """wp: [M][n][K][S] nested lists; T: int (fixed) or list per motion."""
    wp = np.asarray(wp, np.float32)
    if np.isscalar(T):
        return gen.Motions(wp, None, int(T))
    return gen.Motions(wp, np.asarray(T, np.int32), 0)


def knots_motion(positions, S=7):
    """One motion whose robot r sits at positions[r][k] at knot k (identity orientation)."""
    wp = [[pose(p) for p in rob] for rob in positions]
    return np.asarray(wp, np.float32)[None]


def rand_tiny_case(rng, max_robots=4, max_T=20, max_spheres=3, env=True):
    """Tiny random scene + one motion (SE3 bodies with up to 3 spheres, random K)."""
    n = int(rng.integers(1, max_robots + 1))
    robots = []
    for _ in range(n):
        ns = int(rng.integers(1, max_spheres + 1))
        sph = np.concatenate([rng.uniform(-0.3, 0.3, (ns, 3)), rng.uniform(0.1, 0.4, (ns, 1))], axis=1)
        robots.append(gen.Robot(kind=gen.SE3, dof=7, sphere_link=np.zeros(ns, np.int32), sphere=sph.astype(np.float32)))
    osph = np.concatenate([rng.uniform(0, 3, (2, 3)), rng.uniform(0.1, 0.4, (2, 1))], axis=1) if env else np.zeros((0, 4))
    c = rng.uniform(0, 3, (2, 3))
    h = rng.uniform(0.05, 0.3, (2, 3))
    boxes = np.concatenate([c - h, c + h], axis=1) if env else np.zeros((0, 6))
    K = int(rng.integers(1, 4))
    T = int(rng.integers(1, max_T + 1))
    pos = rng.uniform(0, 3, (n, K, 3))
    q = rng.normal(size=(n, K, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    for k in range(1, K):
        q[:, k] *= np.sign(np.sum(q[:, k] * q[:, k - 1], axis=-1, keepdims=True) + 1e-30)
    wp = np.concatenate([pos, q], axis=-1)[None].astype(np.float32)
    return scene(robots, osph, boxes), gen.Motions(wp, None, T)
