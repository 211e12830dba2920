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


def general_chain(rng, dof, base_xyz):
    """A chain with arbitrary joint origins (random rotations, not DH form), mixed
    revolute / prismatic joints and a rotated base -- the general FK path."""
    from scipy.spatial.transform import Rotation
    origins, sph, link, jt = [], [], [], []
    for j in range(dof):
        R = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
        origins.append(gen._affine(R, rng.uniform(-0.15, 0.15, 3)))
        jt.append(1 if rng.uniform() < 0.3 else 0)
        for _ in range(int(rng.integers(1, 6))):
            sph.append(list(rng.uniform(-0.1, 0.1, 3)) + [float(rng.uniform(0.03, 0.08))])
            link.append(j)
    Rb = Rotation.random(random_state=int(rng.integers(1 << 30))).as_matrix()
    return gen.Robot(kind=gen.CHAIN, dof=dof, sphere_link=np.asarray(link, np.int32), sphere=gen._f32(sph),
                     joint_origin=gen._f32(origins), joint_type=np.asarray(jt, np.int32),
                     base=gen._f32(gen._affine(Rb, np.asarray(base_xyz, float))))


def random_scene(rng):
    """A random scene mixing every robot kind the ABI has: DH-form arms (fast path), general
    chains (rotated joint origins, prismatic joints, self-collision pairs), SE(2) and SE(3)
    bodies; links carrying 1..40 spheres (groups split at 32, mixed group sizes); 0..10
    sphere and 0..10 box obstacles."""
    robots = []
    for _ in range(int(rng.integers(2, 7))):
        kind = rng.choice(["dh", "general", "se2", "se3"])
        if kind == "dh":
            dof = int(rng.integers(2, 8))
            origins, sph, link = [], [], []
            for j in range(dof):
                a = rng.uniform(0.05, 0.25)
                s = rng.choice([-1.0, 1.0])
                ca, sa = (0.0, s) if rng.uniform() < 0.7 else (np.cos(0.4), np.sin(0.4))
                rx = np.array([[1.0, 0.0, 0.0], [0.0, ca, -sa], [0.0, sa, ca]])
                origins.append(gen._affine(np.eye(3), np.zeros(3)) if j == 0 else gen._affine(rx, np.array([a, 0.0, rng.uniform(0.0, 0.1)])))
                ns = int(rng.integers(1, 12))
                for k in range(ns):
                    sph.append([(k + 0.5) / ns * a, rng.uniform(-0.02, 0.02), 0.0, rng.uniform(0.02, 0.07)])
                    link.append(j)
            base = gen._affine(np.eye(3), np.concatenate([rng.uniform(-2.0, 2.0, 2), [0.0]]))
            pairs = np.array([(i, j) for i in range(dof) for j in range(i + 3, dof)], np.int32).reshape(-1, 2)
            robots.append(gen.Robot(kind=gen.CHAIN, dof=dof, sphere_link=np.asarray(link, np.int32),
                                    sphere=gen._f32(sph), joint_origin=gen._f32(origins),
                                    joint_type=np.zeros(dof, np.int32), base=gen._f32(base),
                                    self_pairs=pairs if len(pairs) else None))
        elif kind == "general":
            r = general_chain(rng, int(rng.integers(1, 7)), rng.uniform(-2.0, 2.0, 3))
            if r.dof >= 3:
                r.self_pairs = np.array([(0, r.dof - 1)], np.int32)
            robots.append(r)
        elif kind == "se2":
            ns = int(rng.integers(1, 6))
            sph = np.concatenate([rng.uniform(-0.2, 0.2, (ns, 2)), np.zeros((ns, 1)), rng.uniform(0.05, 0.15, (ns, 1))], 1)
            robots.append(gen.Robot(kind=gen.SE2, dof=3, sphere_link=np.zeros(ns, np.int32), sphere=gen._f32(sph)))
        else:
            ns = int(rng.integers(1, 41))
            sph = np.concatenate([rng.uniform(-0.3, 0.3, (ns, 3)), rng.uniform(0.03, 0.12, (ns, 1))], 1)
            robots.append(gen.Robot(kind=gen.SE3, dof=7, sphere_link=np.zeros(ns, np.int32), sphere=gen._f32(sph)))
    no = int(rng.integers(0, 11))
    osph = np.concatenate([rng.uniform(-2.5, 2.5, (no, 3)), rng.uniform(0.05, 0.3, (no, 1))], 1)
    nb = int(rng.integers(0, 11))
    c = rng.uniform(-2.5, 2.5, (nb, 3))
    h = rng.uniform(0.03, 0.25, (nb, 3))
    return scene(robots, osph, np.concatenate([c - h, c + h], 1))


def random_motions(rng, sc, M):
    K = int(rng.integers(1, 6))
    T = int(rng.integers(1, 70))
    S = max(r.dof for r in sc.robots)
    wp = np.zeros((M, sc.n_robots, K, S), np.float32)
    for i, r in enumerate(sc.robots):
        if r.kind == gen.CHAIN:
            wp[:, i, :, :r.dof] = rng.uniform(-3.5, 3.5, (M, K, r.dof))   # beyond +-pi: the wrapped sincos path
        elif r.kind == gen.SE2:
            wp[:, i, :, :2] = rng.uniform(-2.5, 2.5, (M, K, 2))
            th = rng.uniform(-np.pi, np.pi, (M, K))
            for k in range(1, K):
                d = th[:, k] - th[:, k - 1]
                th[:, k] -= 2 * np.pi * np.round(d / (2 * np.pi))
            wp[:, i, :, 2] = th
        else:
            wp[:, i, :, :3] = rng.uniform(-2.5, 2.5, (M, K, 3))
            q = rng.normal(size=(M, K, 4))
            q /= np.linalg.norm(q, axis=-1, keepdims=True)
            for k in range(1, K):
                q[:, k] *= np.sign(np.sum(q[:, k] * q[:, k - 1], axis=-1, keepdims=True) + 1e-30)
            wp[:, i, :, 3:7] = q
    return motions(wp, T)


def random_dh_team(rng, n, dof, first_link_dh=False, rotated_bases=False):
    """n DH-form arms with the same dof (the fused / spread-packing path) on bases within
    ~2 m of each other, 1..11 spheres per link, plus 0..12 sphere and box obstacles
    around them.  first_link_dh: link 0's origin is a DH step Tz(d) Tx(a) Rx(alpha) too
    (the kernels fold it into the base); rotated_bases: bases turned about z."""
    robots = []
    for _ in range(n):
        origins, sph, link = [], [], []
        for j in range(dof):
            a = rng.uniform(0.1, 0.3)
            sgn = rng.choice([-1.0, 1.0])
            ca, sa = (0.0, sgn) if rng.uniform() < 0.7 else (np.cos(0.4), np.sin(0.4))
            rx = np.array([[1.0, 0.0, 0.0], [0.0, ca, -sa], [0.0, sa, ca]])
            if j == 0 and not first_link_dh:
                origins.append(gen._affine(np.eye(3), np.zeros(3)))
            else:
                origins.append(gen._affine(rx, np.array([a, 0.0, rng.uniform(0.0, 0.3 if j == 0 else 0.1)])))
            ns = int(rng.integers(1, 12))
            for k in range(ns):
                sph.append([(k + 0.5) / ns * a, rng.uniform(-0.02, 0.02), 0.0, rng.uniform(0.03, 0.08)])
                link.append(j)
        th = rng.uniform(-np.pi, np.pi) if rotated_bases else 0.0
        rz = np.array([[np.cos(th), -np.sin(th), 0.0], [np.sin(th), np.cos(th), 0.0], [0.0, 0.0, 1.0]])
        base = gen._affine(rz, np.concatenate([rng.uniform(-1.0, 1.0, 2), [rng.uniform(0.0, 0.2) if rotated_bases
                                                                            else 0.0]]))
        robots.append(gen.Robot(kind=gen.CHAIN, dof=dof, sphere_link=np.asarray(link, np.int32),
                                sphere=gen._f32(sph), joint_origin=gen._f32(origins),
                                joint_type=np.zeros(dof, np.int32), base=gen._f32(base)))
    no, nb = int(rng.integers(0, 13)), int(rng.integers(0, 13))
    osph = np.concatenate([rng.uniform(-1.5, 1.5, (no, 3)), rng.uniform(0.05, 0.2, (no, 1))], 1)
    c = rng.uniform(-1.5, 1.5, (nb, 3))
    h = rng.uniform(0.03, 0.2, (nb, 3))
    return scene(robots, osph, np.concatenate([c - h, c + h], 1))
