"""Sequential simulator of n workers running alg1 (TEST INFRASTRUCTURE ONLY).

alg1, per worker i and iteration t:
  Step 1-2  y_i = x_i - eta * grad_i^t
  Step 3    a group G containing i
  Step 4    x_g <- (1/|G|) sum_{g in G} y_g for g in G
Disjoint groups commute exactly (F^G's of non-overlapping G), so a
step's groups can be applied in any order; the simulator applies them in a
fixed order. Workers that skip synchronization apply Step 2 only.

Two drivers:
  * run_lockstep: every worker does step t before any does t+1 (cfg 1-4).
    Groups come from a static rule or the GG with requests in
    ascending worker order and every group completed at the end of the step.
  * replay_trace: an asynchronous run (cfg 5) is replayed from the engine's
    JSONL decision trace (req / done / retire in GG order): the oracle GG must
    reproduce every grant, then parameters are updated per completed group in
    trace order, each member using its own step count t (reading R18).
Gradients are xi(SEED_G, w, t, j) from rp_inputs (x-independent, reading R14).
"""
import numpy as np

from rp_inputs import gen as xi_mod
from . import schedule as sched_mod
from .gg import GroupGenerator, ProtocolError, RandomGroupGenerator
from .update import bf16_round, fused_group_update, fused_group_update_bf16

F32 = np.float32


def init_replicas(n, n_params, lo=0, hi=None):
    return {w: xi_mod.x0(w, n_params, lo, hi) for w in range(n)}


def run_lockstep(n, n_params, steps, *, mode, lr=0.1, workers_per_gpu=None,
                 rule=None, k=None, nodes=None, m=None, c_thres=4, seed_gd=3,
                 lo=0, hi=None, X=None, first_step=1, gg=None, log=None, ii_nodes=0,
                 section_length=1, momentum=None, V=None, dtype="f32", grad_step=None):
    """Simulate `steps` lockstep steps; returns (X, log).

    mode: "static" (rule "paper4" or "shift_k") or "gd" (GB + GD + filter; ii_nodes > 0
    makes every division Inter-Intra, §5.2).
    section_length L ("# of iterations between two synchronizations"): only steps
    t with t % L == 0 synchronize; the others are SGD only (no group requested).
    momentum = (mu, wd): alg1 step 2 with momentum + weight decay; per-worker
    momentum buffers V (zero-initialized) stay local.
    [lo, hi) restricts the simulated element range (elementwise method, so a
    slice is computed exactly as in the full run).
    log: list receiving (t, [groups]) per step, groups as sorted tuples.
    dtype "bf16": bf16 replicas and gradients (the generator's fp32 values rounded to bf16),
    fp32 arithmetic, bf16 result (reading R26, fused_group_update_bf16).
    grad_step: None draws g_w^t = xi(2, w, t) every step; an integer T keeps g_w^T for every
    step (the resident-gradient harness of the bench and of rp_lockstep_run).
    """
    hi = n_params if hi is None else hi
    X = init_replicas(n, n_params, lo, hi) if X is None else X
    if dtype == "bf16":
        X = {w: bf16_round(X[w]) for w in range(n)}
        if momentum is not None:
            raise ValueError("bf16 replicas: plain SGD only (reading R26)")
    elif dtype != "f32":
        raise ValueError(dtype)
    wpg = workers_per_gpu or n
    log = [] if log is None else log
    if mode == "gd" and gg is None:
        gg = GroupGenerator(n, k, c_thres=c_thres, seed_gd=seed_gd, nodes=ii_nodes)
    if momentum is not None and V is None:
        V = {w: np.zeros(hi - lo, F32) for w in range(n)}
    mu, wd = momentum if momentum is not None else (0.0, 0.0)
    for t in range(first_step, first_step + steps):
        if section_length > 1 and t % section_length != 0:
            groups = []
        elif mode == "static":
            groups = [tuple(g) for g in sched_mod.groups_for(rule, t, n=n, k=k, nodes=nodes, m=m)]
        elif mode == "gd":
            seen = {}
            for w in range(n):              # requests in ascending worker order
                seq, members = gg.req(w)
                seen[seq] = members
            groups = [seen[s] for s in sorted(seen)]
            for s in sorted(seen):          # all groups complete at the end of the step
                gg.done(s)
        else:
            raise ValueError(mode)
        in_group = set(w for g in groups for w in g)
        singles = [(w,) for w in range(n) if w not in in_group]   # skip: SGD only
        for g in [tuple(g) for g in groups] + singles:
            G = {w: xi_mod.grad(w, t if grad_step is None else grad_step, n_params, lo, hi) for w in g}
            if dtype == "bf16":
                fused_group_update_bf16(X, {w: bf16_round(G[w]) for w in g}, g, lr, wpg)
            else:
                fused_group_update(X, G, g, lr, wpg, V=V, mu=mu, wd=wd)
        log.append((t, [tuple(g) for g in groups] + [(w,) for w in range(n) if w not in in_group]))
    return X, log


def replay_trace(events, n, n_params, *, k, c_thres, seed_gd, lr=0.1,
                 workers_per_gpu=None, lo=0, hi=None, policy="gd", ii_nodes=0):
    """Replay an async decision trace; returns (X, steps_per_worker).

    events: iterable of dicts {"ev": "req", "w", "seq", "members"} |
            {"ev": "done", "seq"} | {"ev": "retire", "w"} in GG order; with the random GG
            (policy "random") a blocked request is {"ev": "req", "w", "pending": seq}.
    Raises ProtocolError if a recorded grant differs from the oracle GG's.
    """
    hi = n_params if hi is None else hi
    X = init_replicas(n, n_params, lo, hi)
    wpg = workers_per_gpu or n
    gg = (GroupGenerator(n, k, c_thres=c_thres, seed_gd=seed_gd, nodes=ii_nodes) if policy == "gd"
          else RandomGroupGenerator(n, k, seed_gd=seed_gd))
    t_of = [0] * n
    for e in events:
        if e["ev"] == "req" and policy == "random":
            status, seq, members = gg.req(e["w"])
            want = ("pending", e["pending"]) if "pending" in e else ("ok", e["seq"])
            if (status, seq) != want or ("members" in e and tuple(members) != tuple(e["members"])):
                raise ProtocolError(f"decision mismatch at req w={e['w']}: oracle {status} {seq}:{members} "
                                    f"vs trace {e}")
        elif e["ev"] == "req":
            seq, members = gg.req(e["w"])
            if seq != e["seq"] or tuple(members) != tuple(e["members"]):
                raise ProtocolError(f"grant mismatch at req w={e['w']}: oracle {seq}:{members} "
                                    f"vs trace {e['seq']}:{e['members']}")
        elif e["ev"] == "done":
            members = gg.done(e["seq"])
            members = tuple(members)
            G = {}
            for w in members:
                t_of[w] += 1
                G[w] = xi_mod.grad(w, t_of[w], n_params, lo, hi)
            fused_group_update(X, G, members, lr, wpg)
        elif e["ev"] == "retire":
            gg.retire(e["w"])
        else:
            raise ValueError(e)
    return X, t_of
