"""Decentralized static schedules (TEST INFRASTRUCTURE ONLY; see oracle/__init__).

PAPER.md §4.2 "Decentralized Static Scheduler": a periodic,
conflict-free schedule, "groups in the same row are expected to execute
concurrently", computed by a local rule function S, so
every worker gets the same groups without contacting the GG.

Worker numbering (reading R6): w = node*m + r, r = local rank on its node
(P:879 names W0, W4, W8, W12 as "local worker 0" of 4 nodes).

Each function returns the list of synchronizing groups for step t (each a
sorted list of >= 2 workers); workers in no group skip synchronization that
step (the "-" cells) and apply SGD alone.
"""


def paper4(nodes, m, t):
    """fig:scheduler, the paper's 4-phase rule, phase = t mod 4.

    Printed for m = 4 (L.W. 0-3); generalized as SURVEY §8(c) c.1 step 2 (reading R4):
      phase 1, 3: one whole-node group per node ("Sync L.W. 0-3").
      phase 0: all nodes' rank 0 form one group ("Sync with L.W. 0s on ALL NODES");
               local ranks 1..m-1, dropping rank 1 if that count is odd, pair
               consecutively (m=4: {2,3}; rank 1 "No sync", reading R5).
      phase 2: rank 1 pairs with rank 1 on node a + nodes//2 for a < nodes//2
               ("on the opposite node on the ring"; odd node count: the last
               node's rank 1 skips); locally (0, m-1) pair when m >= 3, then
               ranks 2..m-2 pair consecutively, the odd one out skipping
               (m=4: {0,3}; rank 2 "No sync", reading R5).
    Groups of fewer than 2 workers are skips.
    """
    if nodes < 1 or m < 1:
        raise ValueError("paper4 needs nodes >= 1 and m >= 1")
    phase = t % 4
    groups = []
    W = lambda a, r: a * m + r  # noqa: E731
    if phase in (1, 3):
        for a in range(nodes):
            groups.append([W(a, r) for r in range(m)])
    elif phase == 0:
        groups.append([W(a, 0) for a in range(nodes)])
        local = list(range(1, m))
        if len(local) % 2 == 1:
            local = local[1:]  # drop rank 1
        for a in range(nodes):
            for p in range(0, len(local) - 1, 2):
                groups.append([W(a, local[p]), W(a, local[p + 1])])
    else:  # phase == 2
        half = nodes // 2
        if m >= 2:
            for a in range(half):
                groups.append([W(a, 1), W(a + half, 1)])
        for a in range(nodes):
            if m >= 3:
                groups.append([W(a, 0), W(a, m - 1)])
            rest = list(range(2, m - 1))
            for p in range(0, len(rest) - 1, 2):
                groups.append([W(a, rest[p]), W(a, rest[p + 1])])
    return [sorted(g) for g in groups if len(g) >= 2]


def shift_k(n, k, t):
    """SHIFT_K(n, k): phase p = t mod k; group of w = ((w + p) mod n) // k (reading R4).

    Not printed in the paper, whose rule has no group-size parameter; it is the
    cyclic form of the commented-out S(n, i) = d_{i mod k} and is
    used for fixed group size k (cfg 1: SHIFT_K(4,2); cfg 3: (8,3); cfg 4: (16,3)).
    Groups of fewer than 2 workers are skips.
    """
    if n < 1 or k < 1:
        raise ValueError("shift_k needs n >= 1 and k >= 1")
    p = t % k
    buckets = {}
    for w in range(n):
        buckets.setdefault(((w + p) % n) // k, []).append(w)
    return [sorted(buckets[b]) for b in sorted(buckets) if len(buckets[b]) >= 2]


def groups_for(rule, t, *, n=None, k=None, nodes=None, m=None):
    if rule == "paper4":
        return paper4(nodes, m, t)
    if rule == "shift_k":
        return shift_k(n, k, t)
    raise ValueError(f"unknown rule {rule!r}")
