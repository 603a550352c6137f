"""Model of the sorted-greedy region insert (csrc/staged.cu k_st_insert_sg).

1. Deferral rates of the window-0 placement in arbitrary vs window-start order (one region
   of R = 2^13 slots filled from empty at the bench's load).
2. Check of the parallel formulation (prefix maximum over window-start groups, clusters,
   exact warp-style fix-up of the clusters with a violation) against the sequential greedy,
   with pre-occupied slots.
usage: python tools/sim_sorted_greedy.py [trials]
"""
import sys

import numpy as np

R, W = 8192, 32


def first_free_factory(occ):
    nxt = np.arange(len(occ) + 1)
    for i in range(len(occ) - 1, -1, -1):
        if occ[i]:
            nxt[i] = nxt[i + 1]

    def find(x):
        r = x
        while nxt[r] != r:
            r = nxt[r]
        while nxt[x] != r:
            nxt[x], x = r, nxt[x]
        return r
    return nxt, find


def sequential(lo_sorted, occ):
    """Reference: each key (window-start order) takes the first free slot of its window."""
    nxt, find = first_free_factory(occ)
    out = []
    for l in lo_sorted:
        p = find(l)
        if p >= l + W:
            out.append(-1)
        else:
            out.append(p)
            nxt[p] = p + 1
    return out


def parallel(lo_sorted, occ):
    free = ~occ
    fpre = np.concatenate([[0], np.cumsum(free)])  # free slots before s
    slots_free = np.nonzero(free)[0]
    cnt = np.bincount(lo_sorted, minlength=R)
    a = fpre[np.arange(R)]
    b = fpre[np.minimum(np.arange(R) + W, len(occ))]
    part = (cnt > 0) & (a < b)
    c = np.where(part, cnt, 0)
    # no-deferral prefix maximum with clusters
    first = np.zeros(R, int)
    cstart = np.zeros(R, bool)
    cmark = np.zeros(R, bool)
    run, cm, ca = 0, -10**9, 0
    for l in range(R):
        if c[l]:
            x = a[l] - run
            if x > cm:
                cm, ca = x, l
                cstart[l] = True
            fi = run + cm
            if fi + c[l] - 1 >= b[l]:
                cmark[ca] = True
            first[l] = fi
        run += c[l]
    placed = c.copy()
    starts = np.nonzero(cstart)[0]
    for cs in np.nonzero(cmark)[0]:
        nxts = starts[starts > cs]
        ce = nxts[0] if len(nxts) else R
        L = a[cs] - 1
        base = cs
        while base < ce:  # 32 lanes per step, restart after each violation (as the warp does)
            lanes = np.arange(base, min(base + 32, ce))
            s = 0
            while True:
                cc = np.where(np.arange(len(lanes)) >= s, c[lanes], 0)
                cx = np.cumsum(cc)
                mx = np.where(cc > 0, a[lanes] - 1 - (cx - cc), -10**9)
                mx = np.maximum.accumulate(mx)
                end = cx + np.maximum(L, mx)
                viol = (cc > 0) & (end >= b[lanes])
                v = int(np.argmax(viol)) if viol.any() else len(lanes)
                for j in range(s, v):
                    if cc[j]:
                        first[lanes[j]] = end[j] - cc[j] + 1
                if v == len(lanes):
                    L = end[-1] if len(lanes) else L
                    break
                prev = end[v - 1] if v > s else L
                fv = max(end[v] - cc[v] + 1, prev + 1)
                pl = max(b[lanes[v]] - fv, 0)
                first[lanes[v]] = fv
                placed[lanes[v]] = pl
                L = fv + pl - 1 if pl else prev
                s = v + 1
                if s >= len(lanes):
                    break
            base += 32
    out = []
    seen = {}
    for l in lo_sorted:
        r = seen.get(l, 0)
        seen[l] = r + 1
        if not part[l] or r >= placed[l]:
            out.append(-1)
        else:
            out.append(int(slots_free[first[l] + r]))
    return out


INF = 1 << 30


def compose(h1, h2):
    """h2 after h1 for clamp maps h(x) = min(max(x + P, Q), R)."""
    p1, q1, r1 = h1
    p2, q2, r2 = h2
    return (p1 + p2, max(q1 + p2, q2), min(max(r1 + p2, q2), r2))


def apply(h, x):
    p, q, r = h
    return min(max(x + p, q), r)


def clamp_scan(lo_sorted, occ):
    """The kernel's form: the lag of the greedy chain behind each window start,
    lam_{j+1} = min(max(lam_j, 0) + c_j, w_j) - d_j (c_j > 0) or lam_j - d_j, is a clamped
    addition, so one prefix composition over the window starts gives the exact greedy."""
    free = ~occ
    fpre = np.concatenate([[0], np.cumsum(free)])
    slots_free = np.nonzero(free)[0]
    cnt = np.bincount(lo_sorted, minlength=R)
    a = fpre[np.arange(R)]
    b = fpre[np.minimum(np.arange(R) + W, len(occ))]
    w = b - a
    c = np.where((cnt > 0) & (w > 0), cnt, 0)
    d = free[:R].astype(int)
    # exclusive prefix compositions in chunks of 11 (threads), as the block scan does
    lam = np.zeros(R, int)
    H = (0, -INF, INF)
    for j in range(R):
        lam[j] = apply(H, 0)
        hj = (c[j] - d[j], c[j] - d[j], w[j] - d[j]) if c[j] else (-d[j], -INF, INF)
        H = compose(H, hj)
    first = a + np.maximum(lam, 0)
    placed = np.minimum(c, w - np.maximum(lam, 0))
    out = []
    seen = {}
    for l in lo_sorted:
        r = seen.get(l, 0)
        seen[l] = r + 1
        if c[l] == 0 or r >= placed[l]:
            out.append(-1)
        else:
            out.append(int(slots_free[first[l] + r]))
    return out


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(5)
    for load in (0.8, 0.9, 0.95):
        m = int(R * load)
        d_rand = d_sort = 0
        for _ in range(5):
            lo = rng.integers(0, R - W + 1, size=m)
            occ = np.zeros(R, bool)
            d_rand += sequential(lo, occ).count(-1)
            d_sort += sequential(np.sort(lo), occ).count(-1)
        print(f"load {load}: deferred {d_rand / 5 / m * 100:.2f}% arbitrary order, {d_sort / 5 / m * 100:.3f}% by window start")
    bad = 0
    for tr in range(trials):
        load = rng.uniform(0.5, 1.05)
        pre = rng.uniform(0, 0.5)
        occ = rng.random(R) < pre
        m = int(R * load * (1 - pre))
        lo = np.sort(rng.integers(0, R - W + 1, size=m))
        ps, pp, pc = sequential(lo, occ), parallel(lo, occ), clamp_scan(lo, occ)
        if sorted(ps) != sorted(pp) or ps.count(-1) != pp.count(-1) or ps != pc:
            bad += 1
    print(f"cluster and clamp-scan formulations vs sequential greedy: {trials - bad}/{trials} identical")
    assert bad == 0


if __name__ == "__main__":
    main()
