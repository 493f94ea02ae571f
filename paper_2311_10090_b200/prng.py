"""Key helpers of the reference PRNG (prng.hpp:21-57) through the C-ABI.

Host-side key arithmetic only (deriving a handful of parent keys); every
per-env / per-step key of the hot path is derived on the device."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _k(key):
    return np.ascontiguousarray(np.asarray(key, dtype=np.uint32).reshape(4))


def key_from_seed(seed: int) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    N.lib().marl_prng_key_from_seed(int(seed), _p(out))
    return out


def split(key, n: int) -> np.ndarray:
    out = np.zeros((int(n), 4), np.uint32)
    N.lib().marl_prng_split(_p(_k(key)), int(n), _p(out))
    return out


def fold_in(key, data: int) -> np.ndarray:
    out = np.zeros(4, np.uint32)
    N.lib().marl_prng_fold_in(_p(_k(key)), int(data), _p(out))
    return out


def bits(key, index: int) -> int:
    return int(N.lib().marl_prng_bits(_p(_k(key)), int(index)))


def threefry2x32(k0: int, k1: int, x0: int, x1: int):
    out = np.zeros(2, np.uint32)
    N.lib().marl_threefry2x32(k0, k1, x0, x1, _p(out))
    return int(out[0]), int(out[1])
