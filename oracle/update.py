"""Local SGD step fused with P-Reduce, pinned fp32 order (TEST INFRASTRUCTURE ONLY).

Follows alg1 in the paper's order:
  Step 2  x_i <- x_i - eta * grad
  Step 4  xbar_G = (1/|G|) * sum_{g in G} x_g ;  x_g <- xbar_G for all g in G
applied to the members of one group G; non-members are untouched (F^G_uu = 1).

Precision: the paper trains "32-bit floating-point weights", so the
oracle computes in fp32. The summation order is not fixed by the paper (it
used an NCCL ring); this build pins it (reading R1 = SURVEY
§8(c) A1):
  * y_m = fl(x_m - fl(eta * g_m))            two roundings, no fused multiply-add
  * per GPU in ascending GPU id: partial = left fold (+) of that GPU's members
    in ascending worker id; s = left fold of the partials in ascending GPU id
    (GPU(w) = w // workers_per_gpu, reading R6)
  * xbar = fl(s / float32(|G|))              IEEE divide, never multiply by fl(1/|G|)
With one GPU (or one worker per GPU) this is the plain ascending left fold.

NumPy float32 array operations are IEEE-754 binary32 round-to-nearest-even and
NumPy never contracts a*b+c into an FMA, so each line below is one rounding.

``*_fp64`` variants are the fp64 shadow used by the invariant pins.

bf16 replicas with fp32 reduction (reading R26): replicas and
gradients are stored as bfloat16; every value is widened exactly to fp32, step 2 and the
fold / divide run in fp32 exactly as above, and the mean is rounded ONCE to bf16
(IEEE round-to-nearest-even) when it is written to the members.
"""
import numpy as np

F32 = np.float32


def sgd_fp32(x, g, lr):
    """alg1 step 2: y = fl(x - fl(lr*g)). g=None means no staged step: y = x."""
    x = np.asarray(x, dtype=F32)
    if g is None:
        return x.copy()
    prod = F32(lr) * np.asarray(g, dtype=F32)   # one rounding
    return x - prod                             # one rounding


def momentum_sgd_fp32(x, g, v, lr, mu, wd):
    """alg1 step 2 with the paper's ResNet-50 optimizer ("Momentum optimizer is used with
    momentum=0.9 and weight_decay=1e-4"; TF MomentumOptimizer with an L2 term, reading R24):
        g' = fl(g + fl(wd*x));  v <- fl(fl(mu*v) + g');  y = fl(x - fl(lr*v)).
    Returns (y, v_new); each line is one fp32 rounding."""
    x = np.asarray(x, dtype=F32)
    gp = np.asarray(g, dtype=F32) + F32(wd) * x
    v_new = F32(mu) * np.asarray(v, dtype=F32) + gp
    return x - F32(lr) * v_new, v_new


def bf16_round(x):
    """fp32 -> bfloat16, IEEE round-to-nearest-even on the 16 dropped mantissa bits; returned
    as float32 holding the bf16 value (overflow rounds to inf as IEEE does; a NaN stays a NaN).
    bf16 = the upper 16 bits of a binary32: add 0x7FFF plus the lowest kept bit, truncate."""
    b = np.ascontiguousarray(x, dtype=F32).view(np.uint32).astype(np.uint64)
    keep_lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = ((b + np.uint64(0x7FFF) + keep_lsb) >> np.uint64(16)) << np.uint64(16)
    # NaN stays NaN (reading R26): the carry above could turn a NaN into +-0 or +-inf; keep
    # its top 16 bits and set the quiet bit instead (IEEE 754 conversion of a NaN is a NaN)
    nan = (b & np.uint64(0x7FFFFFFF)) > np.uint64(0x7F800000)
    r = np.where(nan, ((b >> np.uint64(16)) | np.uint64(0x40)) << np.uint64(16), r)
    return r.astype(np.uint32).view(F32)


def _fold_order(members, workers_per_gpu):
    """Members grouped by GPU in ascending GPU id, each list ascending (reading R1/R6)."""
    by_gpu = {}
    for m in sorted(members):
        by_gpu.setdefault(m // workers_per_gpu, []).append(m)
    return [by_gpu[gid] for gid in sorted(by_gpu)]


def preduce_fp32(ys, members, workers_per_gpu=None):
    """alg1 step 4: xbar = (1/|G|) sum y_m in the pinned fp32 order.

    ys: dict member -> fp32 vector (the SGD-updated replicas y_m).
    """
    members = sorted(members)
    wpg = workers_per_gpu or (max(members) + 1)
    s = None
    for gpu_members in _fold_order(members, wpg):
        partial = ys[gpu_members[0]].astype(F32, copy=True)
        for m in gpu_members[1:]:
            partial = partial + ys[m]
        s = partial if s is None else s + partial
    return s / F32(len(members))


def fused_group_update(X, G, members, lr, workers_per_gpu=None, V=None, mu=0.0, wd=0.0):
    """Apply alg1 steps 2+4 for one group in place on X (dict or list of fp32 vectors).

    G: dict member -> gradient vector or None (no staged step).
    V: optional dict member -> momentum buffer (updated in place) for momentum_sgd_fp32.
    Returns the mean written to every member ("x_g <- xbar_G").
    """
    members = sorted(members)
    ys = {}
    for m in members:
        if V is not None and m in V and G.get(m) is not None:
            ys[m], V[m] = momentum_sgd_fp32(X[m], G[m], V[m], lr, mu, wd)
        else:
            ys[m] = sgd_fp32(X[m], G.get(m), lr)
    if len(members) == 1:
        # |G| = 1: fl(y / 1) = y exactly; F^G is the identity (SURVEY c.3 "singleton = SGD only").
        X[members[0]] = ys[members[0]]
        return X[members[0]]
    xbar = preduce_fp32(ys, members, workers_per_gpu)
    for m in members:
        X[m] = xbar.copy()
    return xbar


def fused_group_update_bf16(X, G, members, lr, workers_per_gpu=None):
    """fused_group_update for bf16 replicas (reading R26): X[m], G[m] hold bf16 values (as
    float32 arrays, widening is exact); step 2 and step 4 in the pinned fp32 order; every
    member receives bf16_round(xbar). Returns the bf16 mean."""
    members = sorted(members)
    ys = {m: sgd_fp32(X[m], G.get(m), lr) for m in members}
    xbar = ys[members[0]] if len(members) == 1 else preduce_fp32(ys, members, workers_per_gpu)
    out = bf16_round(xbar)
    for m in members:
        X[m] = out.copy()
    return out


def preduce_fp64(vectors):
    """fp64 shadow of step 4: mean of the member vectors."""
    acc = np.zeros_like(np.asarray(vectors[0], dtype=np.float64))
    for v in vectors:
        acc = acc + np.asarray(v, dtype=np.float64)
    return acc / len(vectors)
