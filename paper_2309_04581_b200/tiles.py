"""Multi-GPU frame partition: 16x16 pixel tiles dealt
round-robin to ranks, each rank renders its tiles with a replicated scene,
and the frame is gathered to rank 0 over the process group (NCCL on B200s,
gloo in the CPU tests). Every pixel's paths are keyed by the global pixel id
(reference render.py:337), so any partition is bit-identical to one GPU."""

from __future__ import annotations

import math

import numpy as np

TILE = 16


def tile_pixels(w: int, h: int, rank: int, world: int, tile: int = TILE) -> np.ndarray:
    """Global pixel ids (int32) of the tiles owned by `rank`, tile by tile,
    rows inside a tile."""
    tx, ty = math.ceil(w / tile), math.ceil(h / tile)
    parts = []
    for t in range(rank, tx * ty, world):
        x0, y0 = (t % tx) * tile, (t // tx) * tile
        ys, xs = np.meshgrid(np.arange(y0, min(y0 + tile, h)), np.arange(x0, min(x0 + tile, w)),
                             indexing="ij")
        parts.append((ys * w + xs).reshape(-1))
    return np.concatenate(parts).astype(np.int32) if parts else np.zeros(0, np.int32)


def max_pixels_per_rank(w: int, h: int, world: int, tile: int = TILE) -> int:
    return max(len(tile_pixels(w, h, r, world, tile)) for r in range(world))


class FrameGather:
    """All-gather of per-rank (n_r, 3) radiance into a (w*h, 3) frame on
    rank 0. Buffers are padded to the largest rank so one collective moves
    the frame (torch.distributed: NCCL over NVLink on the B200 box)."""

    def __init__(self, w, h, rank, world, device, dtype=None, group=None):
        import torch
        self.w, self.h, self.rank, self.world, self.group = w, h, rank, world, group
        self.n_max = max_pixels_per_rank(w, h, world)
        dtype = dtype or torch.float64
        self.local = torch.zeros((self.n_max, 3), dtype=dtype, device=device)
        self.parts = [torch.empty_like(self.local) for _ in range(world)]
        self.index = [torch.as_tensor(tile_pixels(w, h, q, world).astype(np.int64), device=device)
                      for q in range(world)]
        self.frame = torch.zeros((w * h, 3), dtype=dtype, device=device) if rank == 0 else None
        # global pixel id of every row of the concatenated rank buffers (-1 = padding)
        pad = np.full((world, self.n_max), -1, np.int32)
        for q in range(world):
            ids = tile_pixels(w, h, q, world)
            pad[q, :len(ids)] = ids
        self.row_pixel = torch.as_tensor(pad.reshape(-1), device=device)

    def _collective(self):
        # the all-gather runs whenever a process group exists (a 1-rank NCCL group
        # too, so the collective path is exercised on a one-GPU box); without one
        # (plain single process) the local buffer is the frame
        import torch.distributed as dist
        return self.world > 1 or (dist.is_available() and dist.is_initialized())

    def gather(self):
        import torch.distributed as dist
        if self._collective():
            dist.all_gather(self.parts, self.local, group=self.group)
            parts = self.parts
        else:
            parts = [self.local]
        if self.rank == 0:
            for q in range(self.world):
                n = len(self.index[q])
                self.frame.index_copy_(0, self.index[q], parts[q][:n])
        return self.frame

    def finalize(self, hdr_output):
        """All-gather, then unpack + encode (PFM / PPM, K9 hrt_finalize) in one
        device pass over the rank buffers on rank 0; returns the file bytes
        (rank 0) or None."""
        import torch
        import torch.distributed as dist
        if self._collective():
            dist.all_gather(self.parts, self.local, group=self.group)
            rows = torch.cat(self.parts)
        else:
            rows = self.local
        if self.rank != 0:
            return None
        from .renderer import finalize_device
        return finalize_device(rows, self.w, self.h, hdr_output, pixel=self.row_pixel).cpu().numpy().tobytes()


class _DeviceArray:
    """__cuda_array_interface__ view of a raw device buffer (zero-copy torch.as_tensor)."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape),
                                         "typestr": "<f8", "version": 3, "strides": None}


class PeerFrame:
    """Frame assembly over peer memory instead of a gather collective: rank 0
    owns the raster (w*h, 3) float64 frame, every other rank maps it with CUDA
    IPC (peer access over NVLink / NVSwitch), and each rank's accumulate kernel
    stores its pixels straight into it (Renderer.render_pixels(...,
    frame_ptr=pf.ptr)). `done()` (stream sync + barrier) makes rank 0's frame
    complete; `finalize()` encodes it there (hrt_finalize). The process group
    only carries the 64-byte handle and the barrier."""

    def __init__(self, w, h, rank, world, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib
        self.w, self.h, self.rank, self.world, self.group = w, h, rank, world, group
        self.lib = _lib.load()
        self._owner = rank == 0
        p = ctypes.c_void_p()
        self.ptr = None
        err = None
        blob = [None]
        if self._owner:
            try:
                _lib.check(self.lib.hrt_buffer_alloc(w * h * 3 * 8, ctypes.byref(p)), "hrt_buffer_alloc")
                self.ptr = p.value
                hd = (ctypes.c_uint8 * 64)()
                _lib.check(self.lib.hrt_ipc_handle(p, hd), "hrt_ipc_handle")
                blob = [bytes(hd)]
            except Exception as e:        # noqa: BLE001 - every rank must still reach the broadcast
                err = e
        if world > 1:
            dist.broadcast_object_list(blob, src=0, group=group)
        if not self._owner and blob[0] is not None:
            hd = (ctypes.c_uint8 * 64).from_buffer_copy(blob[0])
            _lib.check(self.lib.hrt_ipc_open(hd, ctypes.byref(p)), "hrt_ipc_open")
            self.ptr = p.value
        if blob[0] is None:
            if self._owner and self.ptr is not None:
                self.lib.hrt_buffer_free(self.ptr)
                self.ptr = None
            raise RuntimeError(f"rank 0 could not export its frame: {err}")

    def done(self):
        import torch
        import torch.distributed as dist
        torch.cuda.current_stream().synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)

    def frame(self):
        """Rank 0: the assembled (w*h, 3) frame as a zero-copy CUDA tensor."""
        import torch
        assert self._owner, "the frame lives on rank 0"
        return torch.as_tensor(_DeviceArray(self.ptr, (self.w * self.h, 3)), device="cuda")

    def finalize(self, hdr_output):
        if not self._owner:
            return None
        from .renderer import finalize_device
        return finalize_device(self.frame(), self.w, self.h, hdr_output).cpu().numpy().tobytes()

    def close(self, barrier=True):
        import torch.distributed as dist
        if self.ptr is None:
            return
        if self.world > 1 and barrier:
            dist.barrier(group=self.group)        # no rank still writes into rank 0's frame
        if self._owner:
            self.lib.hrt_buffer_free(self.ptr)
        else:
            self.lib.hrt_ipc_close(self.ptr)
        self.ptr = None
