"""Multi-rank frame assembly over peer memory (tiles.PeerFrame): two processes
share one GPU (CUDA IPC works within a device as across NVLink peers), each
renders its round-robin 16x16 tiles straight into rank 0's frame
(HRT_OUT_BY_PIXEL stores from k_accumulate); the assembled frame and its
encoded bytes must equal one-process rendering bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _scene():
    from paper_2309_04581_b200 import configs
    return configs.cfg0()


def _peer_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2309_04581_b200.renderer import Renderer
    from paper_2309_04581_b200.tiles import PeerFrame, tile_pixels
    sc = _scene()
    w, h = sc.camera.resolution
    r = Renderer(sc)
    pf = PeerFrame(w, h, rank, world)
    pix = torch.as_tensor(tile_pixels(w, h, rank, world), device="cuda")
    r.render_pixels(sc.camera, 1, 0, pixels=pix, frame_ptr=pf.ptr)
    pf.done()
    if rank == 0:
        np.save(os.path.join(out_dir, "frame.npy"), pf.frame().cpu().numpy())
        with open(os.path.join(out_dir, "frame.ppm"), "wb") as f:
            f.write(pf.finalize(False))
    pf.close()
    r.close()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_peer_frame_equals_single_process(tmp_path):
    from paper_2309_04581_b200.images import HdrImage, encode_ppm
    from paper_2309_04581_b200.renderer import Renderer
    mp.start_processes(_peer_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    frame = np.load(tmp_path / "frame.npy")
    sc = _scene()
    r = Renderer(sc)
    want = r.render_pixels(sc.camera, 1, 0).cpu().numpy()
    r.close()
    assert np.array_equal(frame, want)
    w, h = sc.camera.resolution
    assert (tmp_path / "frame.ppm").read_bytes() == encode_ppm(HdrImage(want.reshape(h, w, 3)))


def test_out_by_pixel_single_process(cuda):
    """frame_ptr stores a pixel subset at its raster positions, nothing else."""
    from paper_2309_04581_b200.renderer import Renderer
    sc = _scene()
    r = Renderer(sc)
    full = r.render_pixels(sc.camera, 1, 0)
    frame = torch.full_like(full, -1.0)
    pix = torch.arange(500, 900, dtype=torch.int32, device=cuda)
    r.render_pixels(sc.camera, 1, 0, pixels=pix, frame_ptr=frame.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(frame[500:900], full[500:900])
    assert bool((frame[:500] == -1).all()) and bool((frame[900:] == -1).all())
    r.close()


def _nccl_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda:0"))
    from paper_2309_04581_b200.renderer import Renderer
    from paper_2309_04581_b200.tiles import FrameGather, tile_pixels
    sc = _scene()
    w, h = sc.camera.resolution
    r = Renderer(sc)
    fg = FrameGather(w, h, rank, world, "cuda")
    pix = torch.as_tensor(tile_pixels(w, h, rank, world), device="cuda")
    r.render_pixels(sc.camera, 1, 0, pixels=pix, out=fg.local[:len(pix)])
    frame = fg.gather()
    ppm = fg.finalize(False)
    if rank == 0:
        np.save(os.path.join(out_dir, "frame.npy"), frame.cpu().numpy())
        with open(os.path.join(out_dir, "frame.ppm"), "wb") as f:
            f.write(ppm)
    r.close()
    dist.destroy_process_group()


def test_nccl_gather_one_rank(tmp_path):
    """The NCCL frame gather (bench.py --gather nccl) on the one-GPU box: a
    1-rank NCCL group runs the all-gather, the unpack by tile index and the
    fused finalize; the frame and its bytes equal one-process rendering."""
    from paper_2309_04581_b200.images import HdrImage, encode_ppm
    from paper_2309_04581_b200.renderer import Renderer
    mp.start_processes(_nccl_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True,
                       start_method="spawn")
    frame = np.load(tmp_path / "frame.npy")
    sc = _scene()
    r = Renderer(sc)
    want = r.render_pixels(sc.camera, 1, 0).cpu().numpy()
    r.close()
    assert np.array_equal(frame, want)
    w, h = sc.camera.resolution
    assert (tmp_path / "frame.ppm").read_bytes() == encode_ppm(HdrImage(want.reshape(h, w, 3)))
