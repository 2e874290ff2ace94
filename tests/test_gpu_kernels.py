"""GPU parity of the CUDA kernels against the oracle, element by element (needs a B200)."""
import numpy as np
import pytest
import torch

import paper_1909_08029_b200 as rp
from oracle import update as U
from rp_inputs import gen

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.mark.parametrize("n,seed,w,t,j0", [(1, 1, 0, 0, 0), (3, 2, 5, 7, 0), (4, 2, 1, 1, 0),
                                          (4099, 1, 63, 0, 17), ((1 << 20) + 3, 2, 15, 100, 0),
                                          (1000, 2, 7, 2**40, 2**33)])
def test_fill_xi_bit_exact(n, seed, w, t, j0):
    dst = torch.empty(n + 4, dtype=torch.float32, device="cuda")
    rp.fill_xi(dst, n, seed, w, t, j0, 0)
    torch.cuda.synchronize()
    want = gen.xi(seed, w, t, np.arange(j0, j0 + n, dtype=np.uint64))
    assert np.array_equal(dst[:n].cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_fill_xi_unaligned_destination():
    buf = torch.zeros(5000, dtype=torch.float32, device="cuda")
    rp.fill_xi(buf[1:], 4001, 2, 3, 4, 0, 0)           # 4-byte aligned, not 16-byte aligned
    torch.cuda.synchronize()
    want = gen.xi(2, 3, 4, np.arange(4001, dtype=np.uint64))
    assert np.array_equal(buf[1:4002].cpu().numpy(), want)
    assert buf[0].item() == 0 and buf[4002].item() == 0


def _setup(world, n):
    ctx = rp.Context(world, n, n_gpus=1, group_size=min(2, world))
    ld = (n + 63) // 64 * 64
    X = torch.empty((world, ld), dtype=torch.float32, device="cuda")
    G = torch.empty((world, ld), dtype=torch.float32, device="cuda")
    for w in range(world):
        rp.fill_xi(X[w, :n], n, 1, w, 0, 0, 0)
        rp.fill_xi(G[w, :n], n, 2, w, 1, 0, 0)
        ctx.bind_worker(w, X[w, :n], G[w, :n])
    torch.cuda.synchronize()
    return ctx, X, G


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 7, 8, 11, 16])
@pytest.mark.parametrize("n", [70001, 4, 3])
def test_single_group_bit_exact(k, n):
    world = min(k + 2, 64)
    ctx, X, G = _setup(world, n)
    members = list(range(1, k + 1))                   # 0 and k+1 are non-members
    staged = [m for m in members if m % 3 != 2]       # some members have no staged step
    Xh = {w: X[w, :n].cpu().numpy().copy() for w in range(world)}
    Gh = {w: G[w, :n].cpu().numpy().copy() for w in range(world)}
    grp = rp.rp_group.make(-1, members)
    for m in members:
        if m in staged:
            ctx.step(m, None, 0.1)
        ctx.preduce(m, grp)
    for m in members:
        ctx.barrier_free_wait(m, rp.RP_WAIT_DEVICE)
    torch.cuda.synchronize()
    U.fused_group_update(Xh, {m: Gh[m] for m in staged}, members, F32(0.1))
    for w in range(world):
        got = X[w, :n].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), Xh[w].view(np.uint32)), w   # members and non-members
    ctx.close()


def test_mixed_group_sizes_in_one_batch():
    world, n = 12, 3 * 2048 * 5 + 2                     # several tiles and a ragged tail
    ctx, X, G = _setup(world, n)
    groups = [[0, 1, 2], [3, 4, 5], [6, 7], [8], [9, 10, 11]]
    Xh = {w: X[w, :n].cpu().numpy().copy() for w in range(world)}
    Gh = {w: G[w, :n].cpu().numpy().copy() for w in range(world)}
    ctx.batch_begin()
    for i, g in enumerate(groups):
        grp = rp.rp_group.make(-(i + 1), g)
        for m in g:
            ctx.step(m, None, 0.1)
            ctx.preduce(m, grp)
    ctx.batch_end()
    for w in range(world):
        ctx.barrier_free_wait(w, rp.RP_WAIT_DEVICE)
    torch.cuda.synchronize()
    st = ctx.stats()
    assert st["kernel_launches"] == 1                   # all sizes (3, 3, 2, 1, 3) in one launch
    assert st["groups_launched"] == 5 and st["singleton_groups"] == 1
    assert st["bytes_hbm"] == 12 * world * n
    for g in groups:
        U.fused_group_update(Xh, {m: Gh[m] for m in g}, g, F32(0.1))
    for w in range(world):
        assert np.array_equal(X[w, :n].cpu().numpy().view(np.uint32), Xh[w].view(np.uint32))
    ctx.close()


def test_explicit_gradient_pointer_and_lr_per_member():
    world, n = 3, 10000
    ctx, X, G = _setup(world, n)
    other = torch.randn(n, device="cuda")
    Xh = {w: X[w, :n].cpu().numpy().copy() for w in range(world)}
    grp = rp.rp_group.make(-5, [0, 1, 2])
    ctx.step(0, other, 0.5)
    ctx.step(1, None, 0.25)
    for m in range(3):
        ctx.preduce(m, grp)
    for m in range(3):
        ctx.barrier_free_wait(m, 10_000_000)            # host wait
    ys = {0: U.sgd_fp32(Xh[0], other.cpu().numpy(), F32(0.5)),
          1: U.sgd_fp32(Xh[1], G[1, :n].cpu().numpy(), F32(0.25)),
          2: U.sgd_fp32(Xh[2], None, F32(0))}
    want = U.preduce_fp32(ys, [0, 1, 2])
    assert np.array_equal(X[2, :n].cpu().numpy(), want)
    ctx.close()


def test_more_groups_than_one_launch_holds():
    world, n = 40, 4099                                 # 20 pairs -> 16 + 4 groups, two launches
    ctx, X, G = _setup(world, n)
    Xh = {w: X[w, :n].cpu().numpy().copy() for w in range(world)}
    Gh = {w: G[w, :n].cpu().numpy().copy() for w in range(world)}
    ctx.batch_begin()
    for p in range(20):
        grp = rp.rp_group.make(-(p + 1), [2 * p, 2 * p + 1])
        for m in grp.member_list():
            ctx.step(m, None, 0.1)
            ctx.preduce(m, grp)
    ctx.batch_end()
    for w in range(world):
        ctx.barrier_free_wait(w, rp.RP_WAIT_DEVICE)
    torch.cuda.synchronize()
    assert ctx.stats()["kernel_launches"] == 2
    for p in range(20):
        U.fused_group_update(Xh, {m: Gh[m] for m in (2 * p, 2 * p + 1)}, [2 * p, 2 * p + 1], F32(0.1))
    for w in range(world):
        assert np.array_equal(X[w, :n].cpu().numpy(), Xh[w])
    ctx.close()
