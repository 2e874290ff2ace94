"""Pins for the bf16-replica oracle (reading R26): bf16 storage,
fp32 arithmetic in the pinned order of alg1 steps 2 + 4, one final rounding."""
import os

import numpy as np
import pytest
import torch

from oracle import sim
from oracle import update as U

F32 = np.float32
LR = F32(0.1)
GOLD = os.path.join(os.path.dirname(__file__), "golden", "bf16_rne_ties.txt")


def _golden():
    rows = []
    for ln in open(GOLD):
        if ln.startswith("#") or not ln.strip():
            continue
        a, b = ln.split()[:2]
        rows.append((int(a, 16), int(b, 16)))
    return rows


def test_bf16_round_hand_derived_ties():
    for a, b in _golden():
        got = U.bf16_round(np.array([a], dtype=np.uint32).view(F32)).view(np.uint32)[0]
        assert got == b, (hex(a), hex(got), hex(b))


def test_bf16_round_matches_torch_conversion():
    # an independent implementation of IEEE RNE fp32 -> bf16 (torch CPU .to(bfloat16))
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**32, 200_000, dtype=np.uint64).astype(np.uint32)
    x = bits.view(F32)
    x = x[np.isfinite(x)]
    x = np.concatenate([x, (rng.standard_normal(50_000) * 10.0 ** rng.integers(-30, 30, 50_000)).astype(F32)])
    want = torch.from_numpy(x.copy()).to(torch.bfloat16).to(torch.float32).numpy()
    got = U.bf16_round(x)
    same = (got.view(np.uint32) == want.view(np.uint32))
    assert same.all(), x[~same][:5]


def test_bf16_round_non_finite():
    # reading R26: +-inf stay +-inf, every NaN (any payload, either sign) stays a NaN; before this
    # pin the carry of the rounding turned 0xffffffff into +0.0 (found by review, round 2).
    # torch's CPU conversion is the independent implementation for the class of each result.
    bits = np.array([0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x7FFFFFFF, 0xFFFFFFFF,
                     0x7F800001, 0xFF800001, 0x7FBFFFFF, 0x7F7FFFFF], dtype=np.uint32)
    x = bits.view(F32)
    got = U.bf16_round(x)
    want = torch.from_numpy(x.copy()).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(np.isnan(got), np.isnan(x))
    fin = ~np.isnan(x)
    assert np.array_equal(got[fin].view(np.uint32), want[fin].view(np.uint32))   # inf, FLT_MAX -> inf
    assert np.array_equal(np.signbit(got[~fin]), np.signbit(x[~fin]))
    assert np.all(got.view(np.uint32) & 0xFFFF == 0)                                 # a bf16 value


def _bf16_vecs(rng, n, N):
    return {w: U.bf16_round(rng.standard_normal(N).astype(F32)) for w in range(n)}


@pytest.mark.parametrize("members", [(0, 1), (0, 2, 3), (1, 2, 3, 4, 5, 6, 7, 8)])
def test_bf16_update_is_fp32_update_rounded_once(members):
    # R26: the bf16 variant = the (separately pinned) fp32 fused update, then ONE rounding
    rng = np.random.default_rng(len(members))
    X = _bf16_vecs(rng, 9, 3001)
    G = {w: v for w, v in _bf16_vecs(rng, 9, 3001).items() if w in members}
    X32 = {w: X[w].copy() for w in X}
    U.fused_group_update(X32, G, members, LR)
    out = U.fused_group_update_bf16(X, G, members, LR)
    assert np.array_equal(out.view(np.uint32), U.bf16_round(X32[members[0]]).view(np.uint32))
    for m in members:                                      # every member gets the mean
        assert np.array_equal(X[m].view(np.uint32), out.view(np.uint32))
    assert np.array_equal(out, U.bf16_round(out))         # representable in bf16


@pytest.mark.parametrize("k", [2, 3, 5])
def test_bf16_mean_within_half_ulp_plus_fp32_bound(k):
    # closed form: |out - mean_fp64(y)| <= 1/2 ulp_bf16(out) + (k + 1) 2^-24 max|y| (fp32 fold + divide)
    rng = np.random.default_rng(k)
    members = tuple(range(k))
    X = _bf16_vecs(rng, k, 20_000)
    G = _bf16_vecs(rng, k, 20_000)
    Y = [X[m].astype(np.float64) - np.float64(LR) * G[m].astype(np.float64) for m in members]
    mean = U.preduce_fp64(Y)
    out = U.fused_group_update_bf16(X, G, members, LR).astype(np.float64)
    ulp = np.ldexp(1.0, np.frexp(np.abs(out) + 1e-300)[1] - 8)          # bf16 spacing at |out|
    bound = 0.5 * ulp + (k + 2) * 2.0 ** -24 * np.max(np.abs(np.array(Y)), axis=0)
    assert np.all(np.abs(out - mean) <= bound)


def test_bf16_pair_without_step_is_identity():
    # k = 2, no staged step, equal members: x + x = 2x and 2x / 2 = x exactly, x already bf16
    rng = np.random.default_rng(5)
    x = U.bf16_round(rng.standard_normal(5000).astype(F32))
    X = {0: x.copy(), 1: x.copy()}
    out = U.fused_group_update_bf16(X, {}, (0, 1), LR)
    assert np.array_equal(out.view(np.uint32), x.view(np.uint32))


def test_bf16_singleton_is_rounded_sgd():
    rng = np.random.default_rng(6)
    X = _bf16_vecs(rng, 1, 7000)
    G = _bf16_vecs(rng, 1, 7000)
    y32 = X[0] - LR * G[0]                                   # numpy fp32: two roundings, no FMA
    want = torch.from_numpy(y32.copy()).to(torch.bfloat16).to(torch.float32).numpy()
    out = U.fused_group_update_bf16(X, G, (0,), LR)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))


def test_bf16_lockstep_invariants():
    # sim with bf16 replicas: members of each step's groups identical, values bf16, global
    # mean tracks the fp64 SGD mean (P-Reduce preserves the mean) within rounding
    n, N, T = 8, 2048, 6
    log = []
    X, _ = sim.run_lockstep(n, N, T, mode="gd", k=3, log=log, dtype="bf16")
    for w in range(n):
        assert np.array_equal(X[w], U.bf16_round(X[w]))
    last = log[-1][1]
    for g in last:
        for m in g[1:]:
            assert np.array_equal(X[m].view(np.uint32), X[g[0]].view(np.uint32))
    from rp_inputs import gen
    m = np.mean([U.bf16_round(sim.init_replicas(n, N, 0, N)[w]).astype(np.float64) for w in range(n)], axis=0)
    for t in range(1, T + 1):
        m -= float(LR) * np.mean([U.bf16_round(gen.grad(w, t, N, 0, N)).astype(np.float64) for w in range(n)], axis=0)
    scale = max(float(np.max(np.abs(X[w]))) for w in range(n))
    assert np.max(np.abs(np.mean([X[w].astype(np.float64) for w in range(n)], axis=0) - m)) <= T * 2.0 ** -8 * scale
    with pytest.raises(ValueError):
        sim.run_lockstep(n, N, 1, mode="gd", k=3, dtype="bf16", momentum=(0.9, 1e-4))
