"""Counter RNG restated from reference `hybridrt/rng.py:14-57`.

TEST INFRASTRUCTURE ONLY. h starts at the golden-ratio constant; for each
key k (int64 reinterpreted as uint64): h = fmix(h + G ^ (k*B + G)) where
fmix is the splitmix64 finalizer (shifts 30/27/31, multipliers A/B). The
uniform is (h >> 11) * 2^-53 as a double.
"""

from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MUL_A = np.uint64(0xBF58476D1CE4E5B9)
MUL_B = np.uint64(0x94D049BB133111EB)

# purpose tags (rng.py:22-30)
PIXEL_X, PIXEL_Y, BSDF_LOBE, BSDF_U, BSDF_V, LIGHT_PICK, LIGHT_U, LIGHT_V, GENERIC = range(9)


def _fmix(h):
    h = h ^ (h >> np.uint64(30))
    h = h * MUL_A
    h = h ^ (h >> np.uint64(27))
    h = h * MUL_B
    return h ^ (h >> np.uint64(31))


def key_hash(*keys) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = np.asarray(GOLDEN)
        for k in keys:
            k = np.asarray(k).astype(np.int64).view(np.uint64)
            h = _fmix((h + GOLDEN) ^ (k * MUL_B + GOLDEN))
    return h


def uniform(*keys) -> np.ndarray:
    return (key_hash(*keys) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
