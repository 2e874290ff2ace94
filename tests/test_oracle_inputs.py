"""Pins for the shared synthetic generator rp_inputs.xi."""
import numpy as np

from rp_inputs import gen as X
from conftest import golden_lines


def test_mix_matches_published_splitmix64():
    # splitmix64 from state 0: output_i = MIX(i * golden); published reference values.
    want = [int(v) for v in golden_lines("splitmix64_seed0.txt")]
    states = np.array([(i + 1) * 0x9E3779B97F4A7C15 % 2**64 for i in range(4)], dtype=np.uint64)
    assert [int(v) for v in X.mix64(states)] == want


def test_key_is_affine_mod_2_64():
    # KEY(s,w,t,j) = s*A + w*B + t*C + j mod 2^64, checked with Python big ints.
    A, B, C = 0x9E3779B97F4A7C15, 0xD1B54A32D192ED03, 0x8CB92BA72F3D8DD7
    for (s, w, t, j) in [(1, 0, 0, 0), (2, 15, 99, 2**20 - 1), (2, 7, 123456, 138357543)]:
        assert int(X.key64(s, w, t, j)) == (s * A + w * B + t * C + j) % 2**64


def test_xi_exact_grid_and_range():
    v = X.xi(2, 3, 5, np.arange(1 << 16, dtype=np.uint64))
    assert v.dtype == np.float32
    assert v.min() >= -1.0 and v.max() < 1.0
    # exactly representable as (m - 2^23) * 2^-23 with integer m in [0, 2^24)
    m = v.astype(np.float64) * 2.0**23 + 2.0**23
    assert np.all(m == np.round(m)) and m.min() >= 0 and m.max() < 2**24
    # the top 24 bits of MIX give m directly
    top = X.mix64(X.key64(2, 3, 5, np.arange(1 << 16, dtype=np.uint64))) >> np.uint64(40)
    assert np.array_equal(top.astype(np.float64), m)


def test_xi_uniform_moments():
    v = X.xi(1, 0, 0, np.arange(1 << 20, dtype=np.uint64)).astype(np.float64)
    assert abs(v.mean()) < 3e-3            # U[-1,1): mean 0, sd of mean ~ 0.00056
    assert abs(v.var() - 1.0 / 3.0) < 3e-3  # variance 1/3


def test_streams_differ_by_coordinate():
    j = np.arange(1024, dtype=np.uint64)
    a = X.xi(2, 0, 1, j)
    assert not np.array_equal(a, X.xi(2, 1, 1, j))
    assert not np.array_equal(a, X.xi(2, 0, 2, j))
    assert not np.array_equal(a, X.xi(1, 0, 1, j))
    assert np.array_equal(X.grad(0, 1, 4096, 1000, 2024), X.xi(2, 0, 1, np.arange(1000, 2024, dtype=np.uint64)))
