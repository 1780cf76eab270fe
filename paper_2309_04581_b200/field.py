"""Radiance-field plugins for the render path.

Two field types fill the reference's field seam (`scene.field`, used by
`render._march_field` at reference `render.py:142-172` and by
`field.march_arrays` at `field.py:223-255`):

* `RadianceGrid` - the reference's own dense trilinear sigma/RGB grid
  (`field.py:104-175`), kept so the reference's render tests run unchanged
  against the GPU renderer.
* `NeuralField` - the paper's mesh-aware NeRF: a multiresolution hash grid
  (Instant-NGP formulas restated), a 64-wide density
  MLP, degree-4 SH view encoding and a 64-wide colour MLP (P2/P3), plus a
  density-thresholded occupancy bitfield (P4). It does not exist in the
  reference; `oracle/field.py` is its CPU definition.

Both only hold parameters on the host; evaluation happens in the sm_100a
kernels (`csrc/field.cuh`).
"""

from __future__ import annotations

import math

import numpy as np

from .core import Transform, vec3

HASH_PRIMES = (1, 2654435761, 805459861)
DENSITY_WIDTH = 64
GEO_FEATURES = 16          # density head outputs: [log sigma, 15 geometry features]
COLOR_IN = 32              # 16 SH + 15 geometry features + 1 zero pad
COLOR_WIDTH = 64
SH_COEFFS = 16
ACT_SIGMOID = 0
ACT_SOFTPLUS = 1


def _bbox(lo, hi):
    lo, hi = vec3(lo), vec3(hi)
    if (hi <= lo).any():
        raise ValueError(f"grid bbox must have positive extent, got {lo} .. {hi}")
    return lo, hi


class RadianceGrid:
    """Dense trilinear sigma (nx,ny,nz) and RGB (nx,ny,nz,3) over a box
    (reference `field.py:104-175`). Vacuum outside the box."""

    kind = "dense"

    def __init__(self, bbox_lo, bbox_hi, sigma, radiance, world_from_field=None):
        self.bbox_lo, self.bbox_hi = _bbox(bbox_lo, bbox_hi)
        sigma = np.asarray(sigma, dtype=np.float64)
        radiance = np.asarray(radiance, dtype=np.float64)
        if sigma.ndim != 3 or min(sigma.shape) < 1:
            raise ValueError(f"grid resolution must be 3 positive ints, got {sigma.shape}")
        if radiance.shape != sigma.shape + (3,):
            raise ValueError(f"radiance shape {radiance.shape} does not match sigma {sigma.shape} + (3,)")
        if not np.isfinite(sigma).all() or (sigma < 0).any():
            raise ValueError("sigma must be finite and >= 0")
        if not np.isfinite(radiance).all() or (radiance < 0).any():
            raise ValueError("radiance must be finite and >= 0")
        self.sigma, self.radiance = sigma, radiance
        self.res = tuple(int(v) for v in sigma.shape)
        self.world_from_field = world_from_field or Transform.identity()

    @staticmethod
    def constant(bbox_lo, bbox_hi, sigma: float, radiance, res=(2, 2, 2)) -> "RadianceGrid":
        res = tuple(int(r) for r in res)
        return RadianceGrid(bbox_lo, bbox_hi, np.full(res, float(sigma)),
                            np.broadcast_to(vec3(radiance), res + (3,)).copy())


def level_resolutions(n_levels: int, n_min: int, n_max: int) -> np.ndarray:
    """N_l = floor(N_min * b^l), b = exp((ln N_max - ln N_min)/(L-1)), in
    float64 (so the L16/N_max=4096 top level lands on 4095)."""
    if n_levels == 1:
        return np.array([n_min], dtype=np.int64)
    b = math.exp((math.log(n_max) - math.log(n_min)) / (n_levels - 1))
    return np.array([math.floor(n_min * b ** lvl) for lvl in range(n_levels)], dtype=np.int64)


class NeuralField:
    """Hash-grid NeRF parameters.

    Table layout is [level][entry][feature] float32; a level is dense
    (index = x + r*y + r^2*z with r = N_l + 1) when r^3 <= T, otherwise
    hashed with (x ^ y*2654435761 ^ z*805459861) mod T in uint32.
    MLP weights are stored [in][out] in float16 (the MMA operand type):
    density enc->64 (ReLU)->16, colour 32->64 (ReLU)->64 (ReLU)->3. No biases.
    """

    kind = "neural"

    def __init__(self, bbox_lo, bbox_hi, n_levels, n_features, log2_table,
                 n_min, n_max, table, w_density1, w_density2, w_color1,
                 w_color2, w_color3, out_activation="sigmoid",
                 occupancy_res=32, occupancy_threshold=0.01,
                 world_from_field=None):
        self.bbox_lo, self.bbox_hi = _bbox(bbox_lo, bbox_hi)
        self.world_from_field = world_from_field or Transform.identity()
        self.n_levels, self.n_features = int(n_levels), int(n_features)
        self.log2_table = int(log2_table)
        self.n_min, self.n_max = int(n_min), int(n_max)
        if self.n_features not in (2, 4):
            raise ValueError("n_features must be 2 or 4")
        if self.enc_dim not in (16, 32, 64):
            raise ValueError(f"encoding width L*F={self.enc_dim} must be 16, 32 or 64")
        self.level_n = level_resolutions(self.n_levels, self.n_min, self.n_max)
        verts = self.level_n + 1
        t_size = 1 << self.log2_table
        self.level_dense = (verts ** 3 <= t_size)
        self.level_size = np.where(self.level_dense, verts ** 3, t_size).astype(np.int64)
        self.level_offset = np.concatenate([[0], np.cumsum(self.level_size)[:-1]]).astype(np.int64)
        self.n_entries = int(self.level_size.sum())
        table = np.asarray(table, dtype=np.float32)
        if table.shape != (self.n_entries, self.n_features):
            raise ValueError(f"table must be ({self.n_entries}, {self.n_features}), got {table.shape}")
        self.table = np.ascontiguousarray(table)
        shapes = {"w_density1": (self.enc_dim, DENSITY_WIDTH),
                  "w_density2": (DENSITY_WIDTH, GEO_FEATURES),
                  "w_color1": (COLOR_IN, COLOR_WIDTH),
                  "w_color2": (COLOR_WIDTH, COLOR_WIDTH),
                  "w_color3": (COLOR_WIDTH, 3)}
        given = dict(w_density1=w_density1, w_density2=w_density2, w_color1=w_color1,
                     w_color2=w_color2, w_color3=w_color3)
        for name, shape in shapes.items():
            w = np.asarray(given[name], dtype=np.float16)
            if w.shape != shape:
                raise ValueError(f"{name} must be {shape}, got {w.shape}")
            setattr(self, name, np.ascontiguousarray(w))
        if out_activation not in ("sigmoid", "softplus"):
            raise ValueError("out_activation must be 'sigmoid' or 'softplus'")
        self.out_activation = out_activation
        self.occupancy_res = int(occupancy_res)
        self.occupancy_threshold = float(occupancy_threshold)
        # Optional explicit occupancy bitfield (uint32 words, bit i = cell
        # x + G*(y + G*z)); None means "build from density on the device".
        self.occupancy_bits = None

    @property
    def enc_dim(self) -> int:
        return self.n_levels * self.n_features

    @property
    def act_code(self) -> int:
        return ACT_SIGMOID if self.out_activation == "sigmoid" else ACT_SOFTPLUS

    @staticmethod
    def random(seed: int, n_levels=8, n_features=2, log2_table=12, n_min=16, n_max=128,
               bbox_lo=(-1.5, -1.5, -1.5), bbox_hi=(1.5, 1.5, 1.5), param_std=0.1,
               out_activation="sigmoid", occupancy_res=32, occupancy_threshold=0.01):
        """Seeded init: table ~ N(0, std^2), then Xavier-uniform
        density and colour layers, all drawn in that order from
        `np.random.default_rng(seed)`."""
        rng = np.random.default_rng(seed)
        probe = NeuralField.__new__(NeuralField)
        probe.n_levels, probe.n_features, probe.log2_table = n_levels, n_features, log2_table
        levels = level_resolutions(n_levels, n_min, n_max)
        t_size = 1 << log2_table
        n_entries = int(np.where((levels + 1) ** 3 <= t_size, (levels + 1) ** 3, t_size).sum())
        table = rng.normal(0.0, param_std, size=(n_entries, n_features)).astype(np.float32)

        def xavier(fan_in, fan_out, rows=None):
            lim = math.sqrt(6.0 / (fan_in + fan_out))
            return rng.uniform(-lim, lim, size=(rows or fan_in, fan_out))

        enc = n_levels * n_features
        wd1 = xavier(enc, DENSITY_WIDTH)
        wd2 = xavier(DENSITY_WIDTH, GEO_FEATURES)
        wc1 = np.zeros((COLOR_IN, COLOR_WIDTH))
        wc1[:COLOR_IN - 1] = xavier(COLOR_IN - 1, COLOR_WIDTH)
        wc2 = xavier(COLOR_WIDTH, COLOR_WIDTH)
        wc3 = xavier(COLOR_WIDTH, 3)
        return NeuralField(bbox_lo, bbox_hi, n_levels, n_features, log2_table, n_min, n_max,
                           table, wd1, wd2, wc1, wc2, wc3, out_activation=out_activation,
                           occupancy_res=occupancy_res, occupancy_threshold=occupancy_threshold)

    def level_scales(self) -> np.ndarray:
        """float32 per-level, per-axis scale N_l / (hi - lo)."""
        ext = self.bbox_hi - self.bbox_lo
        return (self.level_n[:, None].astype(np.float64) / ext[None, :]).astype(np.float32)

    def occupancy_scale(self) -> np.ndarray:
        return (self.occupancy_res / (self.bbox_hi - self.bbox_lo)).astype(np.float32)

    def cell_centers(self) -> np.ndarray:
        """World-frame centres of the occupancy cells, index x + G*(y + G*z)."""
        g = self.occupancy_res
        ijk = np.stack(np.meshgrid(np.arange(g), np.arange(g), np.arange(g), indexing="ij"), -1)
        ijk = ijk.transpose(2, 1, 0, 3).reshape(-1, 3).astype(np.float64)   # x fastest
        cell = (self.bbox_hi - self.bbox_lo) / g
        pf = self.bbox_lo + (ijk + 0.5) * cell
        return pf if self.world_from_field.is_identity() else self.world_from_field.point(pf)
