"""Counter-RNG surface mirroring `hybridrt.rng` (reference rng.py:22-75).

Draws are computed on the GPU (`hrt_uniform`, csrc/common.cuh rng::uniform)
with the reference's splitmix64 key chain, so every stream matches the
reference bit-for-bit; `PathRng` is the same (seed, pixel, sample) record
`trace_path` takes.
"""

from __future__ import annotations

import numpy as np

PIXEL_X, PIXEL_Y, BSDF_LOBE, BSDF_U, BSDF_V, LIGHT_PICK, LIGHT_U, LIGHT_V, GENERIC = range(9)


class PathRng:
    def __init__(self, seed: int, pixel: int = 0, sample: int = 0):
        self.seed, self.pixel, self.sample = int(seed), int(pixel), int(sample)

    def draw(self, purpose: int, bounce: int = 0, lane: int = 0) -> float:
        return float(uniform(self.seed, self.pixel, self.sample, bounce, purpose, lane))


def uniform(*keys) -> np.ndarray:
    """uniform(seed, pixel, sample, bounce, purpose, lane) with numpy
    broadcasting of the six keys, evaluated on the current CUDA device."""
    import torch

    from .renderer import uniform_keys
    if len(keys) != 6:
        raise TypeError("uniform takes the six keys (seed, pixel, sample, bounce, purpose, lane)")
    cols = np.broadcast_arrays(*[np.asarray(k) for k in keys])
    for c in cols:
        if c.dtype.kind not in "ui":
            raise TypeError(f"rng keys must be integers, got {c.dtype}")
    shape = cols[0].shape
    table = np.stack([c.astype(np.int64).reshape(-1) for c in cols], axis=1)
    dev = torch.device("cuda", torch.cuda.current_device())
    out = uniform_keys(torch.from_numpy(np.ascontiguousarray(table)).to(dev)).cpu().numpy()
    return out.reshape(shape) if shape else out[0]
