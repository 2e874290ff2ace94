"""Counter-based synthetic generator xi(s, w, t, j).

The paper trains on real data; this build has no dataset
and no model, so every per-worker vector is drawn from a stateless hash of its
coordinates. The generator is the splitmix64 finalizer applied to a key:

    KEY(s, w, t, j) = s*0x9E3779B97F4A7C15 + w*0xD1B54A32D192ED03
                      + t*0x8CB92BA72F3D8DD7 + j              (mod 2^64)
    MIX(z): z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
            z *= 0x94D049BB133111EB; z ^= z>>31              (mod 2^64)
    xi = float32(MIX(KEY) >> 40) * 2^-23 - 1.0

Every step of the float conversion is exact in fp32: the result is
(m - 2^23) * 2^-23 for a 24-bit integer m, i.e. uniform on
{-1 + m*2^-23 : 0 <= m < 2^24} in [-1, 1).

Uses:
  * initial replicas  x_w^0[j] = xi(SEED_X=1, w, 0, j)   (per-worker init, A14)
  * gradients         g_w^t[j] = xi(SEED_G=2, w, t, j)   for the worker's own step t >= 1

Gradients do not depend on x, so parity runs isolate the library's arithmetic.
"""
import numpy as np

SEED_X = 1
SEED_G = 2

_C_S = np.uint64(0x9E3779B97F4A7C15)
_C_W = np.uint64(0xD1B54A32D192ED03)
_C_T = np.uint64(0x8CB92BA72F3D8DD7)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """splitmix64 finalizer on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def key64(s, w, t, j):
    """KEY(s, w, t, j) mod 2^64; j may be an array."""
    j = np.asarray(j, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = (np.uint64(s) * _C_S + np.uint64(w) * _C_W + np.uint64(t) * _C_T)
        return base + j


def xi(s, w, t, j):
    """xi(s, w, t, j) as float32, exact (see module docstring)."""
    m = (mix64(key64(s, w, t, j)) >> np.uint64(40)).astype(np.float32)
    return m * np.float32(2.0 ** -23) - np.float32(1.0)


def x0(w, n_params, lo=0, hi=None):
    """Initial replica of worker w, elements [lo, hi)."""
    hi = n_params if hi is None else hi
    return xi(SEED_X, w, 0, np.arange(lo, hi, dtype=np.uint64))


def grad(w, t, n_params, lo=0, hi=None):
    """Synthetic gradient of worker w at its step t (t >= 1), elements [lo, hi)."""
    hi = n_params if hi is None else hi
    return xi(SEED_G, w, t, np.arange(lo, hi, dtype=np.uint64))
