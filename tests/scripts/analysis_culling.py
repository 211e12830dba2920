"""Culling statistics behind DESIGN.md §5 (capsule prefilter) and §10 (interval culling,
supergroup partitions), computed with the fp64 oracle's sphere centres on cfg5 motions.
Analysis only (not a test; lives under tests/ because it calls oracle/).

  python tests/scripts/analysis_culling.py [motions]

Prints, per evaluated state before a motion's first conflict:
  * group-pair survivors of the group-bound test, of the capsule test, and sphere-hit pairs;
  * supergroup-level survivors for several partitions of a 7-link arm;
  * the fraction of B-state intervals that still need per-state tests when every sphere
    is inflated by a Lipschitz bound on its motion over the interval (B = 2, 4, 8).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from paper_2604_23960_b200 import gen  # noqa: E402

NM = int(sys.argv[1]) if len(sys.argv) > 1 else 150
sc, mo = gen.make("cfg5", NM)
os_, om = oracle.OScene(sc), oracle.OMotions(mo)
rob = sc.robots
n = len(rob)
off = np.cumsum([0] + [r.n_spheres for r in rob])
R = np.concatenate([r.sphere[:, 3] for r in rob]).astype(np.float64)
pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
T = mo.fixed_timesteps
wp = mo.waypoints.astype(np.float64)


def ritter(balls):
    C = None
    for c, r in balls:
        if C is None:
            C, Rr = c.copy(), r
            continue
        d = np.linalg.norm(c - C)
        if Rr + d <= r:
            C, Rr = c.copy(), r
        elif d + r > Rr:
            nr = 0.5 * (Rr + d + r)
            C = C + (nr - Rr) / d * (c - C)
            Rr = nr
    return C, Rr


def segdist(p0, p1, q0, q1):
    d1, d2, r = p1 - p0, q1 - q0, p0 - q0
    a, e, f, c, b = d1 @ d1, d2 @ d2, d2 @ r, d1 @ r, d1 @ d2
    den = a * e - b * b
    s = np.clip((b * f - c * e) / den, 0, 1) if den > 1e-12 else 0.0
    t = (b * s + f) / e
    if t < 0:
        t, s = 0.0, np.clip(-c / a, 0, 1)
    elif t > 1:
        t, s = 1.0, np.clip((b - c) / a, 0, 1)
    return np.linalg.norm(p0 + d1 * s - (q0 + d2 * t))


def groups(C):
    G = []
    for r in range(n):
        gs = []
        for g in range(7):
            idx = off[r] + np.arange(8 * g, 8 * g + 8)
            c = C[idx].mean(0)
            gs.append((c, np.max(np.linalg.norm(C[idx] - c, axis=1) + R[idx]), idx))
        G.append(gs)
    return G


parts = {"3+3+1 (kernel)": [(0, 3), (3, 6), (6, 7)], "2+3+2": [(0, 2), (2, 5), (5, 7)], "4+3": [(0, 4), (4, 7)]}
stat = {"states": 0, "l2": 0, "cap": 0, "hit": 0}
sg = {k: [0, 0] for k in parts}
for m in range(NM):
    _, _, ph, _ = oracle.state_tables(sc, mo, m, check_env=False)
    hit = np.nonzero(ph.any(1))[0]
    tc = hit[0] if len(hit) else T
    for t in range(0, min(tc + 1, T), 2):
        C = oracle.centres_at(sc, mo, m, t, os_, om)
        G = groups(C)
        stat["states"] += 1
        for (i, j) in pairs:
            for a in G[i]:
                for b in G[j]:
                    if np.linalg.norm(a[0] - b[0]) <= a[1] + b[1]:
                        stat["l2"] += 1
                        if segdist(C[a[2][0]], C[a[2][-1]], C[b[2][0]], C[b[2][-1]]) <= R[a[2]].max() + R[b[2]].max():
                            stat["cap"] += 1
                            d = np.linalg.norm(C[a[2]][:, None] - C[b[2]][None], axis=2) - R[a[2]][:, None] - R[b[2]][None]
                            stat["hit"] += d.min() < 0
        for name, pt in parts.items():
            S = [[ritter([(G[r][g][0], G[r][g][1]) for g in range(a, b)]) for a, b in pt] for r in range(n)]
            for (i, j) in pairs:
                for A in S[i]:
                    for B in S[j]:
                        sg[name][0] += 1
                        sg[name][1] += np.linalg.norm(A[0] - B[0]) <= A[1] + B[1]
N = stat["states"]
print(f"states sampled: {N}")
print(f"group pairs per state: bound-test survivors {stat['l2'] / N:.2f}, capsule survivors {stat['cap'] / N:.3f}, "
      f"sphere-hit pairs {stat['hit'] / N:.3f}")
for name, (t, s) in sg.items():
    print(f"supergroups {name}: {t / N:.0f} level-1 tests, {s / N:.2f} survivors per state")

# interval culling: inflate every sphere by sum_j |dq_j| * lever_j over the interval
levs = []
for r in rob:
    tl = np.array([np.linalg.norm(np.asarray(r.joint_origin[j]).reshape(3, 4)[:, 3]) for j in range(r.dof)])
    L = np.zeros((r.n_spheres, r.dof))
    for s_ in range(r.n_spheres):
        k = r.sphere_link[s_]
        cn = np.linalg.norm(r.sphere[s_, :3])
        for j in range(k + 1):
            L[s_, j] = tl[j + 1:k + 1].sum() + cn
    levs.append(L)


def q_at(m, t):
    u = t / (T - 1)
    return wp[m, :, 0] + u * (wp[m, :, 1] - wp[m, :, 0])


for B in (2, 4, 8):
    tot = hot = 0
    for m in range(NM):
        _, _, ph, _ = oracle.state_tables(sc, mo, m, check_env=False)
        hit = np.nonzero(ph.any(1))[0]
        tc = hit[0] if len(hit) else T
        for b0 in range(0, tc, B):
            t1 = min(b0 + B, T) - 1
            tm = (b0 + t1) // 2
            dq = np.maximum(np.abs(q_at(m, b0) - q_at(m, tm)), np.abs(q_at(m, t1) - q_at(m, tm)))
            e = np.concatenate([levs[r] @ dq[r] for r in range(n)])
            C = oracle.centres_at(sc, mo, m, tm, os_, om)
            h = False
            for (i, j) in pairs:
                A, Bc = C[off[i]:off[i + 1]], C[off[j]:off[j + 1]]
                d = (np.linalg.norm(A[:, None] - Bc[None], axis=2) - R[off[i]:off[i + 1], None]
                     - R[None, off[j]:off[j + 1]] - e[off[i]:off[i + 1], None] - e[None, off[j]:off[j + 1]])
                if d.min() <= 0:
                    h = True
                    break
            tot += 1
            hot += h
    print(f"{B}-state intervals needing per-state tests (sphere-level Lipschitz inflation): {hot / max(tot, 1):.2f}")
