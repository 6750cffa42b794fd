"""Partition maps restated from SPEC.md:550-623 (the reference has no partition code).

Oracle / test infrastructure only.  Written with plain loops, independently of
paper_2605_16082_b200/partition.py, to pin its integer maps bit-exactly.
"""


def owners(weights, P):
    """Greedy prefix split: column i goes to the part whose share its prefix
    weight has not yet exceeded; boundary k is the first prefix reaching k W / P."""
    n = len(weights)
    W = sum(int(w) for w in weights)
    own = [0] * n
    part, acc = 0, 0
    bounds = [0]
    for k in range(1, P):
        acc, b = 0, 0
        for i in range(n):
            acc += int(weights[i])
            if acc * P >= k * W:
                b = i + 1
                break
        b = max(b, bounds[-1] + 1)
        b = min(b, n - (P - k))
        bounds.append(b)
    bounds.append(n)
    for r in range(P):
        for i in range(bounds[r], bounds[r + 1]):
            own[i] = r
    return own, bounds


def maps(nbr, weights, P):
    """(bounds, ghosts[r], send[s][r], recv[r][s]) with local indices as in the product."""
    own, bounds = owners(weights, P)
    ghosts, send, recv = [], [dict() for _ in range(P)], [dict() for _ in range(P)]
    for r in range(P):
        lo, hi = bounds[r], bounds[r + 1]
        gs = set()
        for c in range(lo, hi):
            for e in nbr[c]:
                if e >= 0 and not (lo <= e < hi):
                    gs.add(int(e))
        ghosts.append(sorted(gs))
    for r in range(P):
        n_own = bounds[r + 1] - bounds[r]
        for pos, g in enumerate(ghosts[r]):
            s = own[g]
            recv[r].setdefault(s, []).append(n_own + pos)
            send[s].setdefault(r, []).append(g - bounds[s])
    return bounds, ghosts, send, recv


def deep_maps(nbr, weights, P, depth):
    """Ghost rings by breadth-first layers (ring k+1 = edge neighbours of ring k not yet local),
    all ghosts ascending; recv/send over all rings and restricted to ring 1 (plain loops)."""
    own, bounds = owners(weights, P)
    ghosts, rings = [], []
    for r in range(P):
        lo, hi = bounds[r], bounds[r + 1]
        local = set(range(lo, hi))
        front = list(range(lo, hi))
        ring_of = {}
        for k in range(1, depth + 1):
            nxt = set()
            for c in front:
                for e in nbr[c]:
                    if e >= 0 and e not in local:
                        nxt.add(int(e))
            for e in nxt:
                ring_of[e] = k
            local |= nxt
            front = sorted(nxt)
        gs = sorted(ring_of)
        ghosts.append(gs)
        rings.append([ring_of[g] for g in gs])
    send, recv = [dict() for _ in range(P)], [dict() for _ in range(P)]
    send1, recv1 = [dict() for _ in range(P)], [dict() for _ in range(P)]
    for r in range(P):
        n_own = bounds[r + 1] - bounds[r]
        for pos, g in enumerate(ghosts[r]):
            s = own[g]
            recv[r].setdefault(s, []).append(n_own + pos)
            send[s].setdefault(r, []).append(g - bounds[s])
            if rings[r][pos] == 1:
                recv1[r].setdefault(s, []).append(n_own + pos)
                send1[s].setdefault(r, []).append(g - bounds[s])
    return bounds, ghosts, rings, send, recv, send1, recv1
