"""N > 1 frame path on CPU: two gloo ranks each trace their round-robin
16x16 tiles (with the CPU oracle standing in for the per-rank renderer) and
all-gather to rank 0; the assembled frame must bit-equal one-process
rendering (paths are keyed by global pixel id, reference render.py:337)."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_04581_b200.tiles import FrameGather, tile_pixels


def _scene():
    from paper_2309_04581_b200 import assets
    from paper_2309_04581_b200.core import Transform
    from paper_2309_04581_b200.field import RadianceGrid
    from paper_2309_04581_b200.scene import Camera, make_scene
    from paper_2309_04581_b200.surface import Dielectric, TriangleMesh
    g = np.random.default_rng(3)
    field = RadianceGrid((-1.5,) * 3, (1.5,) * 3, g.uniform(0.5, 1.5, (4, 4, 4)),
                         g.uniform(0, 1, (4, 4, 4, 3)))
    v, f = assets.icosphere(0.4, 1)
    cam = Camera(Transform.look_at([0, 0, 3], [0, 0, 0]), math.radians(40), (40, 24))
    return make_scene(field=field, meshes=[TriangleMesh(v, f, Dielectric(1.5))], camera=cam,
                      spp=2, n_bounces=3, march_step=0.08)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import tracer
    from paper_2309_04581_b200.pack import pack_camera, pack_scene
    sc = _scene()
    w, h = sc.camera.resolution
    g = FrameGather(w, h, rank, world, torch.device("cpu"))
    pix = tile_pixels(w, h, rank, world)
    local = tracer.render(pack_scene(sc), pack_camera(sc.camera), 2, 0, pixels=pix.astype(np.int64))
    g.local[:len(pix)] = torch.from_numpy(local)
    frame = g.gather()
    if rank == 0:
        np.save(out, frame.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tile_partition_covers_frame_once():
    for w, h in [(800, 800), (1920, 1080), (37, 23), (16, 16)]:
        for world in (1, 2, 3, 8):
            allp = np.concatenate([tile_pixels(w, h, r, world) for r in range(world)])
            assert np.array_equal(np.sort(allp), np.arange(w * h))


@pytest.mark.parametrize("world", [2])
def test_gloo_gather_equals_single_process(tmp_path, world):
    from oracle import tracer
    from paper_2309_04581_b200.pack import pack_camera, pack_scene
    out = str(tmp_path / "frame.npy")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="fork")
    frame = np.load(out)
    sc = _scene()
    want = tracer.render(pack_scene(sc), pack_camera(sc.camera), 2, 0).reshape(-1, 3)
    assert np.array_equal(frame, want)
