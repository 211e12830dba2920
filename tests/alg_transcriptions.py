"""Test-only transcriptions of the paper's Alg. 1 (MotVal) and Alg. 2 (FFC), line by
line, over per-state strict-hit tables.  They exist to pin
the readings c.12-c.14 / c.18: packing and ordering change effort, never results.

Tables: env_hit[t][i] = CC(S_i, E) at timestep t (robot i's spheres vs obstacles);
pair_hit[t][p] = CC(S_i, S_j) at t for the p-th pair (i<j, lexicographic).
"""
import math


def pack_rake(b, t_max, W):
    """PackCfgBatch(p, b, rake): timesteps b, b+nb, ..., b+nb(W-1), nb = ceil(t_max/W)
    (PAPER.md:246-248); lanes >= t_max are inactive."""
    nb = math.ceil(t_max / W)
    return [b + k * nb for k in range(W) if b + k * nb < t_max]


def pack_linear(b, t_max, W):
    """PackCfgBatch(p, b, linear): b*W ... b*W+W-1."""
    return [b * W + k for k in range(W) if b * W + k < t_max]


def pair_index(n):
    idx, p = {}, 0
    for i in range(n):
        for j in range(i + 1, n):
            idx[(i, j)] = p
            p += 1
    return idx


def motval_alg1(env_hit, pair_hit, n, W, hierarchical, check_env, packing="rake"):
    """Alg. 1.  Returns (result, cc_calls)."""
    t_max = len(env_hit)
    num_batches = math.ceil(t_max / W)                                 # line 2
    pack = pack_rake if packing == "rake" else pack_linear
    pidx = pair_index(n)
    calls = 0
    if hierarchical and check_env:                                     # line 3
        for b in range(num_batches):                                   # line 4
            for i in range(n):                                         # line 5
                B = pack(b, t_max, W)                                  # line 6 (+7 SpheresFK)
                calls += 1
                if any(env_hit[t][i] for t in B):                      # line 8
                    return False, calls                                # line 9
    for b in range(num_batches):                                       # line 13
        if not hierarchical and check_env:                             # line 14
            for i in range(n):
                B = pack(b, t_max, W)
                calls += 1
                if any(env_hit[t][i] for t in B):
                    return False, calls
        for i in range(n - 1):                                         # line 22 (1-based i < n)
            Bi = pack(b, t_max, W)
            for j in range(i + 1, n):                                  # line 24
                Bj = pack(b, t_max, W)
                assert Bi == Bj
                calls += 1
                if any(pair_hit[t][pidx[(i, j)]] for t in Bi):         # line 27
                    return False, calls                                # line 28
    return True, calls                                                 # line 33


def ffc_alg2(pair_hit, n, W):
    """Alg. 2.  Returns ((t, i, j) or None, batches evaluated)."""
    t_max = len(pair_hit)
    num_batches = math.ceil(t_max / W)
    pidx = pair_index(n)
    C = None
    for b in range(num_batches):
        # t_batch_start = b * batch_size; PackCfgBatch(p, t_batch_start, linear) read as
        # "linear batch b" (reading c.13)
        B = pack_linear(b, t_max, W)
        for i in range(n - 1):
            for j in range(i + 1, n):
                t_conflict = next((t for t in B if pair_hit[t][pidx[(i, j)]]), None)
                if t_conflict is not None:
                    if C is None or C[0] > t_conflict:                 # strict replacement
                        C = (t_conflict, i, j)
        if C is not None:
            return C, b + 1
    return None, num_batches
