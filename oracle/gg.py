"""Group Generator with Group Buffer, Global Division and the slowdown filter.

TEST INFRASTRUCTURE ONLY (see oracle/__init__).

PAPER.md passages followed, in the paper's order of operations:
  * request: "When a worker needs to perform a synchronization, it just needs to
    contact GG"; the GG "generates groups in a serial manner"
  * request counter c_w: "records how many times the worker requires a group"
    (P:1184-1185); incremented at request time (reading R10)
  * Group Buffer: "the ordered list of groups that include the corresponding
    worker"; a non-empty GB serves its first group
  * Global Division: "divides all current workers with empty GBs into several
    non-conflicting groups", called "only when the initiator's GB is empty"
    
  * slowdown filter: a GD admits w only if c_i - c_w < C_thres
  * lock vector: "a bit vector indicating whether each worker is currently
    performing a P-Reduce"; set on grant, released by the ack after P-Reduce
    

Readings (= SURVEY §8(c) c.2): candidates are workers with empty GB,
passing the filter, not retired (R7, R19); the random partition is splitmix64
+ Fisher-Yates, the initiator's group first, chunks of k, the last one possibly
shorter, no candidates -> singleton (R8); C_thres <= 0 disables the filter (R9).
"""
from dataclasses import dataclass, field

_MASK = (1 << 64) - 1


def _mix(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _MASK
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _MASK
    z ^= z >> 31
    return z


class ProtocolError(Exception):
    pass


class ConflictError(Exception):
    pass


@dataclass
class GGState:
    n: int
    k: int
    c_thres: int
    rng: int                       # splitmix64 state (seed_gd)
    seq: int = 0                   # next group sequence number
    gb: list = field(default_factory=list)        # per worker: list of seq (FIFO)
    counters: list = field(default_factory=list)  # c_w
    lock: int = 0                  # bit w set while w holds a granted, unfinished group
    retired: int = 0               # bit w set once w finished its final step
    retiring: int = 0              # bit w set: retire w when its held group completes
    handed: list = field(default_factory=list)    # per worker: seq handed out by req, or -1
    groups: dict = field(default_factory=dict)    # seq -> tuple(members)

    def key(self):
        return (self.rng, self.seq, tuple(tuple(b) for b in self.gb), tuple(self.counters),
                self.lock, self.retired, self.retiring, tuple(self.handed),
                tuple(sorted((s, m) for s, m in self.groups.items())))


class GroupGenerator:
    """The GG of §5 with GB + GD + filter; one instance = one serial decision loop."""

    def __init__(self, n, k, c_thres=4, seed_gd=3, nodes=0):
        """nodes > 0: Inter-Intra Synchronization (§5.2) over nodes of n // nodes workers."""
        if not (1 <= k <= n):
            raise ValueError("need 1 <= k <= n")
        if nodes and n % nodes:
            raise ValueError("n must be a multiple of nodes")
        self.s = GGState(n=n, k=k, c_thres=c_thres, rng=seed_gd & _MASK,
                         gb=[[] for _ in range(n)], counters=[0] * n, handed=[-1] * n)
        self.trace = []
        self.gd_calls = 0
        self.nodes = nodes
        self.head_rot = [0] * max(nodes, 1)

    # -- RNG: splitmix64 (next = MIX(state += golden)) -------------------------
    def _next(self):
        self.s.rng = (self.s.rng + 0x9E3779B97F4A7C15) & _MASK
        return _mix(self.s.rng)

    def _idle(self, i):
        """Workers a division may assign: empty GB, slowdown filter, not retired (R7)."""
        s = self.s
        cand = []
        for v in range(s.n):
            if v == i or s.gb[v] or (s.retired >> v) & 1:
                continue
            if s.c_thres > 0 and not (s.counters[i] - s.counters[v] < s.c_thres):
                continue  # slowdown filter
            cand.append(v)
        return cand

    def _shuffle(self, cand):
        for q in range(len(cand) - 1, 0, -1):  # Fisher-Yates
            j = self._next() % (q + 1)
            cand[q], cand[j] = cand[j], cand[q]
        return cand

    def _push(self, chunks):
        """Create the groups in order and append them to their members' GBs. Lock bit w is
        held while GB[w] is non-empty; a division may only use workers without one."""
        s = self.s
        before = s.lock
        for ch in chunks:
            members = tuple(sorted(ch))
            bits = 0
            for m in members:
                bits |= 1 << m
            if before & bits:  # overlapping groups must be serialized
                raise ConflictError(f"division produced a group overlapping a held lock: {members}")
            s.lock |= bits
            s.groups[s.seq] = members
            for m in members:
                s.gb[m].append(s.seq)
            s.seq += 1

    def _global_division(self, i):
        """partition the idle workers (empty GB), initiator's group first."""
        s = self.s
        self.gd_calls += 1
        if self.nodes:
            return self._inter_intra_division(i)
        cand = self._shuffle(self._idle(i))
        chunks = [[i] + cand[:s.k - 1]]
        rest = cand[s.k - 1:]
        chunks += [rest[p:p + s.k] for p in range(0, len(rest), s.k)]
        self._push(chunks)

    def _inter_intra_division(self, i):
        """§5.2 Inter-Intra Synchronization realized as two divisions.

        Inter phase: one Head Worker per node "randomly divided into several groups"
        across nodes; the other workers "randomly assigned to groups with only local workers".
        Intra phase: "a P-Reduce among all the workers in the same node". Both groups go to
        every worker's GB, Inter first. Readings (R23): over the idle
        set of the division; heads rotate per node (round-robin over the node's idle workers
        in ascending order); groups of k, the last one of a list shorter.
        """
        s = self.s
        m = s.n // self.nodes
        idle = sorted(self._idle(i) + [i])
        per_node = [[v for v in idle if v // m == a] for a in range(self.nodes)]
        heads = []
        for a, ws in enumerate(per_node):
            if ws:
                heads.append(ws[self.head_rot[a] % len(ws)])
                self.head_rot[a] += 1
        chunks = []
        hs = self._shuffle(list(heads))
        chunks += [hs[p:p + s.k] for p in range(0, len(hs), s.k)]
        for ws in per_node:
            loc = self._shuffle([v for v in ws if v not in heads])
            chunks += [loc[p:p + s.k] for p in range(0, len(loc), s.k)]
        inter = chunks
        intra = [ws for ws in per_node if ws]
        self._push(inter + intra)

    def req(self, i):
        """Synchronization request of worker i. Returns (seq, members)."""
        s = self.s
        if not (0 <= i < s.n) or (s.retired >> i) & 1:
            raise ProtocolError(f"request from invalid or retired worker {i}")
        if s.handed[i] != -1:
            raise ProtocolError(f"worker {i} requested again before its group {s.handed[i]} completed")
        s.counters[i] += 1
        if not s.gb[i]:
            self._global_division(i)
        seq = s.gb[i][0]
        s.handed[i] = seq
        self.trace.append(("req", i, seq, s.groups[seq]))
        return seq, s.groups[seq]

    def done(self, seq):
        """Completion (ack) of group seq: pop GBs, release lock bits."""
        s = self.s
        members = s.groups.pop(seq)
        for m in members:
            if not s.gb[m] or s.gb[m][0] != seq:
                raise ProtocolError(f"group {seq} is not at the head of worker {m}'s GB")
            if s.handed[m] != seq:
                raise ProtocolError(f"group {seq} completed before member {m} requested it")
            s.gb[m].pop(0)
            s.handed[m] = -1
            if not s.gb[m]:
                s.lock &= ~(1 << m)
        self.trace.append(("done", seq))
        for m in members:  # retire atomically with the completion (reading R19)
            if (s.retiring >> m) & 1:
                s.retiring &= ~(1 << m)
                s.retired |= 1 << m
                self.trace.append(("retire", m))
        return members

    def retire(self, w):
        """Worker w will not request again; GD must never assign it again (reading R19).

        If w holds a group, it retires when that group completes (same decision
        step), so no GD can pick it between its last completion and retirement.
        """
        s = self.s
        if s.handed[w] != -1:
            s.retiring |= 1 << w
        else:
            s.retired |= 1 << w
            self.trace.append(("retire", w))

    def gb_depth(self):
        return max(len(b) for b in self.s.gb)


class RandomGroupGenerator:
    """The basic GG of §4.1: random groups, lock vector, pending group queue.

    TEST INFRASTRUCTURE ONLY. Steps, in the paper's protocol order:
      * a worker's request: if the GG already notified it of a granted group
        (its inbox, the per-worker queue of P:705 "notifies the workers"), serve that;
      * otherwise "randomly generates a group" containing the initiator:
        the initiator plus k-1 distinct others drawn uniformly (splitmix64 Fisher-Yates over
        the non-retired workers, first k-1; reading R8);
      * "sets the corresponding bits in the lock vector" if none is set and notifies the
        members; a group overlapping a held lock is "blocked ... in a pending
        group queue" and the initiator waits;
      * on the ack after P-Reduce the bits are released and the pending queue is rescanned
        in FIFO order; newly unblocked groups are granted.
    Readings (R21-R22): a waiting initiator's repeated request is a retry (its
    counter is not incremented again) and is served any group it was notified of first; a
    pending group that contains a retired worker is cancelled and its initiator draws again.
    AD-PSGD is the k = 2 special case.
    """

    def __init__(self, n, k, seed_gd=3):
        if not (1 <= k <= n):
            raise ValueError("need 1 <= k <= n")
        self.n, self.k = n, k
        self.rng = seed_gd & _MASK
        self.seq = 0
        self.lock = 0
        self.retired = 0
        self.retiring = 0
        self.inbox = [[] for _ in range(n)]
        self.pending = []                 # FIFO of seq
        self.pending_of = [-1] * n        # pending group initiated by w
        self.waiting = [False] * n
        self.handed = [-1] * n
        self.groups = {}                  # seq -> members (granted or pending)
        self.initiator = {}
        self.counters = [0] * n
        self.trace = []
        self.n_pending = 0
        self.n_granted = 0

    def _next(self):
        self.rng = (self.rng + 0x9E3779B97F4A7C15) & _MASK
        return _mix(self.rng)

    def _bits(self, members):
        b = 0
        for m in members:
            b |= 1 << m
        return b

    def _grant(self, seq):
        members = self.groups[seq]
        self.lock |= self._bits(members)
        for m in members:
            self.inbox[m].append(seq)
        self.n_granted += 1

    def req(self, i, members=None):
        """Returns ("ok", seq, members) or ("pending", seq, members). `members` (tests only)
        replaces the random draw, to replay the paper's walk-through."""
        if not (0 <= i < self.n) or (self.retired >> i) & 1:
            raise ProtocolError(f"request from invalid or retired worker {i}")
        if self.handed[i] != -1:
            raise ProtocolError(f"worker {i} requested again before its group {self.handed[i]} completed")
        if not self.waiting[i]:
            self.counters[i] += 1
        if self.inbox[i]:
            seq = self.inbox[i][0]
            self.handed[i] = seq
            self.waiting[i] = False
            self.trace.append(("req", i, "ok", seq))
            return "ok", seq, self.groups[seq]
        if self.pending_of[i] != -1:
            self.waiting[i] = True
            self.trace.append(("req", i, "pending", self.pending_of[i]))
            return "pending", self.pending_of[i], self.groups[self.pending_of[i]]
        if members is None:
            cand = [v for v in range(self.n) if v != i and not (self.retired >> v) & 1]
            for q in range(len(cand) - 1, 0, -1):  # Fisher-Yates, as in GD
                j = self._next() % (q + 1)
                cand[q], cand[j] = cand[j], cand[q]
            members = [i] + cand[:self.k - 1]
        members = tuple(sorted(members))
        seq = self.seq
        self.seq += 1
        self.groups[seq] = members
        self.initiator[seq] = i
        if self.lock & self._bits(members):      # conflict: serialize
            self.pending.append(seq)
            self.pending_of[i] = seq
            self.waiting[i] = True
            self.n_pending += 1
            self.trace.append(("req", i, "pending", seq))
            return "pending", seq, members
        self._grant(seq)
        self.handed[i] = seq
        self.waiting[i] = False
        self.trace.append(("req", i, "ok", seq))
        return "ok", seq, members

    def _rescan(self):
        for seq in list(self.pending):
            members = self.groups[seq]
            ini = self.initiator[seq]
            if self.retired & self._bits(members):          # reading R22: cancel
                self.pending.remove(seq)
                self.pending_of[ini] = -1
                del self.groups[seq]
                continue
            if not (self.lock & self._bits(members)):
                self.pending.remove(seq)
                self.pending_of[ini] = -1
                self._grant(seq)

    def done(self, seq):
        members = self.groups[seq]
        for m in members:
            if not self.inbox[m] or self.inbox[m][0] != seq or self.handed[m] != seq:
                raise ProtocolError(f"group {seq} completed out of protocol at worker {m}")
        for m in members:
            self.inbox[m].pop(0)
            self.handed[m] = -1
            self.lock &= ~(1 << m)
            if (self.retiring >> m) & 1:
                self.retiring &= ~(1 << m)
                self.retired |= 1 << m
        del self.groups[seq]
        self.trace.append(("done", seq))
        self._rescan()
        return members

    def retire(self, w):
        if self.handed[w] != -1:
            self.retiring |= 1 << w
        else:
            self.retired |= 1 << w
            self._rescan()
