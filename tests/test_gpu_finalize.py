"""K9 finalize on the GPU vs the reference's own PFM / PPM bytes
(tests/golden/images.npz from hybridrt.render.finalize, render.py:399-401,
images.py:37-64, core.py:51-64), and the gather-fused unpack + encode."""

import os

import numpy as np
import pytest
import torch

from paper_2309_04581_b200 import renderer
from paper_2309_04581_b200.images import HdrImage
from paper_2309_04581_b200.tiles import FrameGather, tile_pixels

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "images.npz")


@pytest.mark.parametrize("i", [0, 1, 2])
def test_finalize_bytes_equal_reference(i):
    g = np.load(GOLD)
    img = HdrImage(g[f"px{i}"])
    assert renderer.finalize(img, False) == g[f"ppm{i}"].tobytes()
    assert renderer.finalize(img, True) == g[f"pfm{i}"].tobytes()


def test_finalize_rejects_non_finite_ppm_only():
    px = np.full((2, 3, 3), 0.5)
    px[1, 2, 0] = np.nan
    with pytest.raises(AssertionError):
        renderer.finalize(HdrImage(px), False)
    b = renderer.finalize(HdrImage(px), True)            # PFM stores it (encode_pfm)
    assert len(b) == len(b"PF\n3 2\n-1.0\n") + 2 * 3 * 12


def test_tiled_rows_unpack_and_encode():
    """Rank buffers (16x16 tiles round-robin, padded) -> frame bytes in one pass."""
    w, h, world = 37, 21, 3
    rng = np.random.default_rng(3)
    frame = np.exp(rng.normal(-1.0, 1.5, (h, w, 3)))
    want_ppm = renderer.finalize(HdrImage(frame), False)
    want_pfm = renderer.finalize(HdrImage(frame), True)
    n_max = max(len(tile_pixels(w, h, q, world)) for q in range(world))
    rows = np.zeros((world, n_max, 3))
    pix = np.full((world, n_max), -1, np.int32)
    for q in range(world):
        ids = tile_pixels(w, h, q, world)
        rows[q, :len(ids)] = frame.reshape(-1, 3)[ids]
        pix[q, :len(ids)] = ids
    src = torch.as_tensor(rows.reshape(-1, 3), device="cuda")
    pt = torch.as_tensor(pix.reshape(-1), device="cuda")
    assert renderer.finalize_device(src, w, h, False, pixel=pt).cpu().numpy().tobytes() == want_ppm
    assert renderer.finalize_device(src, w, h, True, pixel=pt).cpu().numpy().tobytes() == want_pfm
    fg = FrameGather(w, h, 0, 1, torch.device("cuda"))
    ids = tile_pixels(w, h, 0, 1)
    fg.local[:len(ids)] = torch.as_tensor(frame.reshape(-1, 3)[ids], device="cuda")
    assert fg.finalize(False) == want_ppm
