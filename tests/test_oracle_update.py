"""Pins for oracle.update (alg1 steps 2+4) against closed forms and invariants."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import algebra as A
from oracle import update as U

F32 = np.float32
LR = F32(0.1)


def _vecs(rng, n, N, scale=1.0):
    return {w: (rng.standard_normal(N) * scale).astype(F32) for w in range(n)}


@pytest.mark.parametrize("n,G", [(5, [0, 3, 4]), (8, [1, 2, 6]), (16, list(range(0, 16, 2))), (4, [0, 1, 2, 3])])
def test_preduce_equals_matrix_closed_form(n, G):
    # P:566-569 + P:595: X' = Y F^G, with Y the SGD-updated replicas (fp64 library matmul)
    rng = np.random.default_rng(len(G))
    N = 4096
    X = _vecs(rng, n, N)
    grads = _vecs(rng, n, N)
    Y = {w: U.sgd_fp32(X[w], grads[w] if w in G else None, LR) for w in range(n)}
    Xn = dict(X)
    U.fused_group_update(Xn, {w: grads[w] for w in G}, G, LR)
    # non-members untouched bitwise (F^G_uu = 1); they did not step here
    for w in range(n):
        if w not in G:
            assert np.array_equal(Xn[w], X[w])
    Ymat = np.stack([Y[w].astype(np.float64) for w in range(n)], axis=1)   # N x n
    ref = A.apply(Ymat, A.group_matrix(n, G))
    for w in G:
        # fp32 fold of |G| terms + one divide: error <= (|G|+1) u sum|y|/|G| per element
        bound = (len(G) + 1) * 2.0**-24 * np.abs(Ymat[:, G]).sum(axis=1) / len(G) + 1e-30
        assert np.all(np.abs(Xn[w].astype(np.float64) - ref[:, w]) <= bound)


def test_members_identical_after():
    rng = np.random.default_rng(1)
    X = _vecs(rng, 6, 1000)
    U.fused_group_update(X, {}, [1, 4, 5], LR)
    assert np.array_equal(X[1], X[4]) and np.array_equal(X[4], X[5])


def test_k2_is_exact_halving_of_rounded_sum():
    # |G| = 2: s/2 is exact, so the result equals round_fp32((y_a + y_b)/2) computed in fp64
    rng = np.random.default_rng(2)
    X = _vecs(rng, 2, 1 << 16)
    Y = {w: X[w].copy() for w in X}
    U.fused_group_update(X, {}, [0, 1], LR)
    ref = ((Y[0].astype(np.float64) + Y[1].astype(np.float64)) / 2).astype(F32)
    assert np.array_equal(X[0], ref)


def test_singleton_is_sgd_within_two_roundings():
    # |G| = 1: F^G = I, only step 2: x - lr*g, exact value vs two fp32 roundings:
    # |y - exact| <= ulp(lr*g)/2 + ulp(y)/2
    rng = np.random.default_rng(3)
    X = _vecs(rng, 1, 1 << 16)
    g = rng.standard_normal(1 << 16).astype(F32)
    x0 = X[0].copy()
    U.fused_group_update(X, {0: g}, [0], LR)
    prod = np.float64(LR) * g.astype(np.float64)
    exact = x0.astype(np.float64) - prod
    bound = 0.5 * np.spacing(np.abs(prod).astype(F32)).astype(np.float64) \
        + 0.5 * np.spacing(np.abs(X[0])).astype(np.float64)
    assert np.all(np.abs(X[0].astype(np.float64) - exact) <= bound)
    # and a worked SPEC example: x=(1,2), g=(10,-10), lr=0.1 -> (0,3) up to rounding
    Z = {0: np.array([1, 2], F32)}
    U.fused_group_update(Z, {0: np.array([10, -10], F32)}, [0], LR)
    assert np.allclose(Z[0], [0, 3], atol=2e-7)


def test_no_staged_step_means_y_equals_x():
    rng = np.random.default_rng(4)
    X = _vecs(rng, 3, 512)
    x = {w: X[w].copy() for w in X}
    U.fused_group_update(X, {}, [0, 1, 2], LR)
    ref = ((x[0] + x[1]) + x[2]) / F32(3)
    assert np.array_equal(X[0], ref)


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_mass_conservation(k):
    # doubly stochastic: sum of members after = sum of y before, up to fp32 rounding
    rng = np.random.default_rng(10 + k)
    N = 1 << 16
    X = _vecs(rng, k, N)
    ysum = sum(X[w].astype(np.float64) for w in range(k))
    yabs = sum(np.abs(X[w].astype(np.float64)) for w in range(k))
    U.fused_group_update(X, {}, range(k), F32(0))
    after = sum(X[w].astype(np.float64) for w in range(k))
    assert np.all(np.abs(after - ysum) <= k * 2.0**-24 * yabs * 2 + 1e-30)


@pytest.mark.parametrize("k,exact", [(2, True), (3, True), (4, True), (8, False)])
def test_idempotence(k, exact):
    # (F^G)^T F^G = F^G: applying P-Reduce twice (eta = 0) changes nothing.
    # Bitwise for k = 2 (provable), observed bitwise for 3, 4. For larger k the second
    # fold of k equal values is within the recursive-summation bound (k-1)u*k|v|, i.e.
    # after the divide <= (k - 1/2) ulp(v).
    rng = np.random.default_rng(20 + k)
    X = _vecs(rng, k, 1 << 18)
    U.fused_group_update(X, {}, range(k), F32(0))
    once = X[0].copy()
    U.fused_group_update(X, {}, range(k), F32(0))
    if exact:
        assert np.array_equal(X[0], once)
    else:
        ulp = np.spacing(np.abs(once)).astype(np.float64)
        assert np.all(np.abs(X[0].astype(np.float64) - once) <= (k - 0.5) * ulp)
        assert np.any(X[0] != once)   # genuinely not bitwise for k = 8


def test_global_group_is_allreduce_mean():
    # P-Reduce with G = all workers is All-Reduce
    rng = np.random.default_rng(5)
    X = _vecs(rng, 16, 4096)
    ref = U.preduce_fp64([X[w] for w in range(16)])
    U.fused_group_update(X, {}, range(16), F32(0))
    assert np.max(np.abs(X[7] - ref)) <= 17 * 2.0**-24 * max(np.abs(ref).max(), 1)


def test_pinned_fold_with_gpu_partials():
    # reading R1: members {0, 2, 3} with 2 workers per GPU -> y0 + (y2 + y3), not (y0 + y2) + y3
    ys = {0: np.array([1.0], F32), 2: np.array([2.0**-24], F32), 3: np.array([2.0**-24], F32)}
    got = U.preduce_fp32(ys, [0, 2, 3], workers_per_gpu=2)
    assert got[0] == F32((1.0 + 2.0**-23) / 3)
    plain = U.preduce_fp32(ys, [0, 2, 3], workers_per_gpu=4)      # one GPU: plain left fold
    assert plain[0] == F32(F32(1.0) / F32(3))                      # 1 + 2^-24 rounds to 1 twice


def test_exact_small_case_against_rationals():
    # dyadic data and lr = 1/2: steps 2 and 4 are checked in exact rational arithmetic
    x = {0: [Fraction(3), Fraction(-1)], 1: [Fraction(5), Fraction(2)], 2: [Fraction(1, 2), Fraction(7)]}
    g = {0: [Fraction(2), Fraction(0)], 1: [Fraction(-4), Fraction(6)], 2: [Fraction(1), Fraction(1)]}
    lr = Fraction(1, 2)
    y = {w: [x[w][j] - lr * g[w][j] for j in range(2)] for w in x}
    mean = [sum(y[w][j] for w in y) / 3 for j in range(2)]
    X = {w: np.array([float(v) for v in x[w]], F32) for w in x}
    Gd = {w: np.array([float(v) for v in g[w]], F32) for w in g}
    U.fused_group_update(X, Gd, [0, 1, 2], F32(0.5))
    for w in x:
        for j in range(2):
            assert X[w][j] == F32(float(mean[j]))   # sum exact, one rounding in the divide


def test_momentum_reduces_to_sgd():
    # mu = 0, wd = 0: the momentum form is plain SGD bit for bit
    rng = np.random.default_rng(7)
    x, g = (rng.standard_normal(4096).astype(F32) for _ in range(2))
    v = rng.standard_normal(4096).astype(F32)
    y, v2 = U.momentum_sgd_fp32(x, g, v, LR, 0.0, 0.0)
    assert np.array_equal(y, U.sgd_fp32(x, g, LR)) and np.array_equal(v2, g)


def test_momentum_constant_gradient_closed_form():
    # constant g, wd = 0, v0 = 0: v_t = g (1 - mu^t) / (1 - mu) (geometric series) and
    # x_t = x0 - lr * sum_s v_s; checked against the closed form in fp64
    mu, lr, T = 0.9, 0.1, 60
    x0 = np.linspace(-1, 1, 1001).astype(F32)
    g = np.full(1001, 0.25, F32)
    x, v = x0.copy(), np.zeros(1001, F32)
    for _ in range(T):
        x, v = U.momentum_sgd_fp32(x, g, v, lr, mu, 0.0)
    t = np.arange(1, T + 1)
    vs = 0.25 * (1 - np.float64(np.float32(mu)) ** t) / (1 - np.float64(np.float32(mu)))
    assert np.allclose(v, vs[-1], rtol=2e-6)
    assert np.allclose(x, x0.astype(np.float64) - np.float64(np.float32(lr)) * vs.sum(), atol=2e-5)


def test_weight_decay_shrinks_toward_zero():
    # g = 0, mu = 0: x <- x - lr*wd*x = (1 - lr*wd) x, per step
    x = np.linspace(-3, 3, 101).astype(F32)
    y, _ = U.momentum_sgd_fp32(x, np.zeros_like(x), np.zeros_like(x), 0.5, 0.0, 0.1)
    assert np.allclose(y, x * (1 - 0.05), atol=1e-6)


def test_fused_update_with_momentum_buffers_stay_local():
    # only the weights are averaged; every member keeps its own momentum buffer
    rng = np.random.default_rng(8)
    X = {w: rng.standard_normal(512).astype(F32) for w in range(3)}
    G = {w: rng.standard_normal(512).astype(F32) for w in range(3)}
    V = {w: rng.standard_normal(512).astype(F32) for w in range(3)}
    V0 = {w: V[w].copy() for w in V}
    ys = {w: U.momentum_sgd_fp32(X[w], G[w], V0[w], LR, 0.9, 1e-4) for w in range(3)}
    U.fused_group_update(X, G, [0, 1, 2], LR, V=V, mu=0.9, wd=1e-4)
    assert np.array_equal(X[0], ((ys[0][0] + ys[1][0]) + ys[2][0]) / F32(3))
    for w in range(3):
        assert np.array_equal(V[w], ys[w][1])
