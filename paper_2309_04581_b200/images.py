"""Render target and byte codecs mirroring `hybridrt.images`
(reference `pkg/src/hybridrt/images.py:17-116`).

PFM: `PF\\n<w> <h>\\n-1.0\\n` then little-endian float32 RGB, rows bottom-up.
PPM P6: tone-mapped, round-half-up 8-bit codes, rows top-down.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import tone_map


@dataclass
class HdrImage:
    """Linear radiance, (h, w, 3) float64, row 0 at the top (images.py:17-34)."""

    pixels: np.ndarray

    def __post_init__(self):
        self.pixels = np.asarray(self.pixels, dtype=np.float64)
        if self.pixels.ndim != 3 or self.pixels.shape[2] != 3:
            raise ValueError(f"HdrImage needs (h, w, 3) pixels, got {self.pixels.shape}")

    @property
    def w(self) -> int:
        return int(self.pixels.shape[1])

    @property
    def h(self) -> int:
        return int(self.pixels.shape[0])


def encode_pfm(img: HdrImage) -> bytes:
    head = b"PF\n%d %d\n-1.0\n" % (img.w, img.h)
    return head + np.ascontiguousarray(img.pixels[::-1]).astype("<f4").tobytes()


def decode_pfm(blob: bytes) -> HdrImage:
    fields = blob.split(b"\n", 3)
    if len(fields) < 4 or fields[0] != b"PF":
        raise ValueError("not an RGB PFM file")
    w, h = (int(v) for v in fields[1].split())
    order = "<f4" if float(fields[2]) < 0 else ">f4"
    raw = np.frombuffer(fields[3], dtype=order, count=w * h * 3).reshape(h, w, 3)
    return HdrImage(raw[::-1].astype(np.float64))


def quantize(img: HdrImage) -> np.ndarray:
    return np.floor(tone_map(img.pixels) * 255.0 + 0.5).astype(np.uint8)


def encode_ppm(img: HdrImage) -> bytes:
    return b"P6\n%d %d\n255\n" % (img.w, img.h) + quantize(img).tobytes()


def decode_ppm(blob: bytes) -> np.ndarray:
    fields = blob.split(b"\n", 3)
    if len(fields) < 4 or fields[0] != b"P6":
        raise ValueError("not a P6 PPM file")
    w, h = (int(v) for v in fields[1].split())
    return np.frombuffer(fields[3], dtype=np.uint8, count=w * h * 3).reshape(h, w, 3).copy()
