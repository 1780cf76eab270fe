"""NeRF field files and scene loading through the reference's scene JSON.

The reference loads a scene from JSON (`scene.py:557-559` `load_scene` ->
`parse_scene` -> `build_scene`), whose `field.path` names a dense
`.rfgrid` file (`field.py:568-614`). Its parser rejects unknown keys
(`scene.py:35-54`), so the neural field's hyper-parameters live in the
field FILE: `save_nerf` / `load_nerf` write / read a
`.hrtnerf` file (magic, a JSON header with the hash-grid / MLP / occupancy
hyper-parameters and the field placement, then the raw little-endian
arrays). `load_scene(path)` reads a reference scene JSON with the
reference's own parser and builder and, when `field.path` is a `.hrtnerf`
file, attaches the `NeuralField` instead of a dense grid - the result is a
reference `Scene` that `paper_2309_04581_b200.render` draws.
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np

from .core import Transform
from .field import NeuralField

MAGIC = b"HRTNERF\x01"
ARRAYS = ("table", "w_density1", "w_density2", "w_color1", "w_color2", "w_color3")


def is_nerf_file(path) -> bool:
    try:
        with open(path, "rb") as f:
            return f.read(len(MAGIC)) == MAGIC
    except OSError:
        return False


def save_nerf(path, field: NeuralField) -> None:
    arrays = {name: np.ascontiguousarray(getattr(field, name)) for name in ARRAYS}
    header = {
        "n_levels": field.n_levels, "n_features": field.n_features, "log2_table": field.log2_table,
        "n_min": field.n_min, "n_max": field.n_max, "out_activation": field.out_activation,
        "occupancy_res": field.occupancy_res, "occupancy_threshold": field.occupancy_threshold,
        "bbox_lo": [float(v) for v in field.bbox_lo], "bbox_hi": [float(v) for v in field.bbox_hi],
        "world_from_field": np.asarray(field.world_from_field.m, np.float64).tolist(),
        "arrays": [],
    }
    off = 0
    for name, a in arrays.items():
        header["arrays"].append({"name": name, "dtype": a.dtype.newbyteorder("<").str, "shape": list(a.shape),
                                 "offset": off})
        off += a.nbytes
    blob = json.dumps(header).encode()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", len(blob)))
        f.write(blob)
        for a in arrays.values():
            f.write(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())


def load_nerf(path) -> NeuralField:
    with open(path, "rb") as f:
        if f.read(len(MAGIC)) != MAGIC:
            raise ValueError(f"{path}: not a .hrtnerf field file")
        (n,) = struct.unpack("<I", f.read(4))
        header = json.loads(f.read(n).decode())
        data = f.read()
    arrays = {}
    for spec in header["arrays"]:
        dt = np.dtype(spec["dtype"])
        count = int(np.prod(spec["shape"]))
        a = np.frombuffer(data, dtype=dt, count=count, offset=spec["offset"])
        if a.size != count:
            raise ValueError(f"{path}: truncated array {spec['name']}")
        arrays[spec["name"]] = a.reshape(spec["shape"]).astype(dt.newbyteorder("="))
    missing = [k for k in ARRAYS if k not in arrays]
    if missing:
        raise ValueError(f"{path}: missing arrays {missing}")
    m = np.asarray(header["world_from_field"], np.float64)
    return NeuralField(header["bbox_lo"], header["bbox_hi"], header["n_levels"], header["n_features"],
                       header["log2_table"], header["n_min"], header["n_max"], arrays["table"],
                       arrays["w_density1"], arrays["w_density2"], arrays["w_color1"], arrays["w_color2"],
                       arrays["w_color3"], out_activation=header["out_activation"],
                       occupancy_res=header["occupancy_res"],
                       occupancy_threshold=header["occupancy_threshold"],
                       world_from_field=Transform(m))


def load_scene(path):
    """The reference's `load_scene(path)` (`scene.py:557-559`, its own
    parser and builder, imported from the installed `hybridrt`), with a
    `.hrtnerf` field file loaded as a `NeuralField`. Returns the reference
    `Scene`; spawn_eps = 1e-4 x the scene diagonal over the NeRF box and the
    meshes, as `build_scene` computes it (`scene.py:552`)."""
    import dataclasses
    import importlib
    rs = importlib.import_module("hybridrt.scene")
    cfg = rs.load_scene_config(path)
    base_dir = os.path.dirname(os.path.abspath(path))
    if cfg.field is None or not is_nerf_file(os.path.join(base_dir, cfg.field.path)):
        return rs.build_scene(cfg, base_dir=base_dir)
    nerf = load_nerf(os.path.join(base_dir, cfg.field.path))
    if cfg.field.transform is not None:
        nerf.world_from_field = cfg.field.transform.build()
    scene = rs.build_scene(dataclasses.replace(cfg, field=None), base_dir=base_dir)
    scene.config = cfg
    scene.field = nerf
    scene.spawn_eps = 1e-4 * rs.scene_diagonal(nerf, scene.meshes)
    return scene
