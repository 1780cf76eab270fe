#!/usr/bin/env python
"""Benchmark: NeRF samples/s and Mrays/s per frame for the hybrid NeRF/mesh
render path (BASELINE.json metric), on BASELINE config 1 (glass icosphere in
an L16/T2^19 hash-grid NeRF, 800x800, 1 spp, 4 bounces, 100 cameras).

One step = one full 800x800 frame from camera (step mod 100), rendered by
the sm_100a kernels through the C ABI with scene and network resident in
HBM. With N GPUs (torchrun, one rank per GPU) the frame is split into 16x16
pixel tiles dealt round-robin to ranks; every rank's accumulate kernel stores
its pixels straight into rank 0's frame over peer memory (CUDA IPC, NVLink)
- `--gather nccl` uses an NCCL all-gather instead
(strong scaling: the frame is fixed). `--impl reference` times the CPU
oracle port of the reference path (oracle/, numpy) on the host cores instead.

Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NeRF samples/sec and Mrays/sec per frame at 1/2/4/8 B200 vs CPU ref"
TILE = 16
WORKLOAD = "cfg1: glass icosphere s5 (20480 tris, IOR 1.5) in L16 F2 T2^19 16->2048 hash-grid NeRF, 800x800, 1 spp, 4 bounces, 128^3 occupancy, 1024-sample cap, early-out 1e-4, 100 seeded cameras"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-tiles", type=int, default=0,
                    help="16x16 tiles per CPU-baseline sample (0 = 2 per worker process)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gather", choices=["peer", "nccl"], default="peer",
                    help="frame assembly: peer-memory stores from the render (default) or NCCL all-gather")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ------------------------------------------------------------ clocks ----

class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), \
            "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch DRAM bytes and L2->L1 requests / sectors per sample of the
    field engine from the committed ncu capture (profiles/r01e_field_traffic.json,
    made by tools/field_traffic.py)."""
    path = os.path.join(ROOT, "profiles", "r01e_field_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


# --------------------------------------------------- CPU baseline (oracle) -

_CPU_SCENE = None


def _cpu_scene():
    """Oracle scene for cfg1, built once in the parent (scene load, BVH and
    occupancy build are outside the timed sample, as for the GPU arm) and
    inherited by the forked workers."""
    global _CPU_SCENE
    if _CPU_SCENE is None:
        from oracle import tracer
        from oracle.field import occupancy_bits
        from paper_2309_04581_b200 import configs
        from paper_2309_04581_b200.pack import pack_scene
        _CPU_SCENE = tracer.OracleScene(pack_scene(configs.cfg1()))
        occupancy_bits(_CPU_SCENE.field)
    return _CPU_SCENE


def _cpu_tile(args):
    cam_index, pixels = args
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)                 # one BLAS thread per worker process
    from oracle import tracer
    from paper_2309_04581_b200 import configs
    from paper_2309_04581_b200.pack import pack_camera
    cam = pack_camera(configs.cfg1_cameras()[cam_index])
    st = {}
    tracer.render(_cpu_scene(), cam, 1, 0, pixels=pixels, stats=st)
    return st["nerf_samples"], st["paths"]


def cpu_pool(workers):
    """One forked worker per core, created once (scene inherited, imports
    warmed by a tiny job) so timed samples measure tracing, not start-up."""
    import multiprocessing as mp
    _cpu_scene()
    pool = mp.get_context("fork").Pool(workers)
    pool.map(_warm, range(workers))
    return pool


def _warm(_):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import tracer  # noqa: F401
    return 0


def cpu_sample(n_tiles, workers, cam_index=0, seed=0, pool=None):
    """Oracle (numpy port of the reference path) on `n_tiles` seeded 16x16
    tiles of the cfg1 frame, one process per core."""
    import numpy as np
    rng = np.random.default_rng(seed)
    all_t = (800 // TILE) * (800 // TILE)
    chosen = rng.choice(all_t, n_tiles, replace=False)
    jobs = []
    for t in chosen:
        x0, y0 = (t % (800 // TILE)) * TILE, (t // (800 // TILE)) * TILE
        ys, xs = np.meshgrid(np.arange(y0, y0 + TILE), np.arange(x0, x0 + TILE), indexing="ij")
        jobs.append((cam_index, (ys * 800 + xs).reshape(-1)))
    own = pool is None
    if own:
        pool = cpu_pool(workers)
    t0 = time.perf_counter()
    res = pool.map(_cpu_tile, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    if own:
        pool.close()
        pool.join()
    samples = sum(r[0] for r in res)
    paths = sum(r[1] for r in res)
    return samples, paths, dt


def cpu_workers():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline_block(n_tiles=0):
    workers = cpu_workers()
    n_tiles = n_tiles or max(16, 8 * workers)
    pool = cpu_pool(workers)             # forked + warmed before the timed sample
    samples, paths, dt = cpu_sample(n_tiles, workers, pool=pool)
    pool.close()
    pool.join()
    return {"value": samples / dt, "unit": "samples/s", "cores": workers, "kind": "port",
            "mrays_per_s": paths / dt / 1e6,
            "sample": f"{n_tiles} seeded 16x16 tiles ({paths} paths, {samples} NeRF samples) of the "
                      f"cfg1 camera-0 frame, oracle/ numpy port of the reference path, one process "
                      f"per core, {dt:.1f} s wall"}


# ------------------------------------------------------------ arms ------

def run_reference(args, rank, world):
    if rank != 0:
        return
    workers = cpu_workers()
    n_tiles = args.cpu_tiles or max(8, 4 * workers)
    pool = cpu_pool(workers)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(max(1, workers), workers, pool=pool)
    tot_s = tot_p = tot_t = 0.0
    for k in range(args.steps):
        s, p, dt = cpu_sample(n_tiles, workers, cam_index=k % 100, seed=k, pool=pool)
        tot_s, tot_p, tot_t = tot_s + s, tot_p + p, tot_t + dt
    pool.close()
    pool.join()
    value = tot_s / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "mrays_per_s": tot_p / tot_t / 1e6,
        "config": {"workload": WORKLOAD + f"; CPU sample per step = {n_tiles} seeded 16x16 tiles"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": workers, "kind": "port",
                         "sample": f"{n_tiles} seeded 16x16 tiles per step x {args.steps} steps, "
                                   f"oracle/ numpy port of the reference render loop + neural "
                                   f"field, one process per core (pool forked and warmed once)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def open_peer_frame(w, h, rank, world):
    """PeerFrame (rank 0's frame mapped into every rank with CUDA IPC), or None
    on every rank if any rank cannot map it (then the frame is assembled with
    the NCCL all-gather instead): the ranks agree before the first frame."""
    import torch
    import torch.distributed as dist

    from paper_2309_04581_b200.tiles import PeerFrame
    peer, ok = None, 1
    try:
        peer = PeerFrame(w, h, rank, world)
    except Exception as e:        # noqa: BLE001 - any IPC failure -> the NCCL path
        print(f"rank {rank}: peer-memory frame unavailable ({e}); using the NCCL all-gather",
              file=sys.stderr, flush=True)
        ok = 0
    if world > 1:
        flag = torch.tensor([ok], dtype=torch.int32, device=torch.cuda.current_device())
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = int(flag.item())
    if not ok and peer is not None:
        peer.close(barrier=False)         # (no frame was rendered into it)
        peer = None
    return peer


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2309_04581_b200 import configs
    from paper_2309_04581_b200.renderer import Renderer
    from paper_2309_04581_b200.tiles import FrameGather, PeerFrame, tile_pixels

    # one process per GPU; HRT_DIST_BACKEND=gloo lets several ranks share one GPU to test the
    # multi-rank flow where only one device exists (timings then mean nothing)
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    backend = os.environ.get("HRT_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    scene = configs.cfg1()
    cams = configs.cfg1_cameras()
    field = scene.field
    r = Renderer(scene)
    w, h = cams[0].resolution
    pix_host = tile_pixels(w, h, rank, world)
    pix = torch.as_tensor(pix_host, device=dev)
    n_local = len(pix_host)
    gather = FrameGather(w, h, rank, world, dev)
    out = gather.local
    peer = open_peer_frame(w, h, rank, world) if args.gather == "peer" else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step(k, timed):
        cam = cams[k % len(cams)]
        if timed:
            flush.fill_(float(k))          # evict L2 between timed steps (outside the events)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if peer is not None:               # pixels stored into rank 0's frame (peer memory)
            r.render_pixels(cam, 1, 0, pixels=pix, frame_ptr=peer.ptr)
            st = dict(r.last_stats)
            peer.done()
        else:
            r.render_pixels(cam, 1, 0, pixels=pix, out=out[:n_local])
            st = dict(r.last_stats)
            gather.gather()                # frame assembled on rank 0 (NCCL all-gather)
        if timed:
            e1.record(stream)
            e1.synchronize()
            st["step_ms"] = e0.elapsed_time(e1)
        return st

    for k in range(args.warmup):
        step(k, False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
    clocks.start()
    t_wall = time.perf_counter()
    steps = [step(args.warmup + k, True) for k in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall
    clk = clocks.stop()

    dev_ms = sum(s["step_ms"] for s in steps)
    samples = sum(s["nerf_samples"] for s in steps)
    paths = sum(s["paths"] for s in steps)
    march_ms = sum(s["field_ms"] for s in steps)
    march_n = sum(s["field_launches"] for s in steps)
    evaluated = sum(s["evaluated"] for s in steps)
    launches = sum(s["launches"] for s in steps)
    t = torch.tensor([dev_ms, samples, paths, march_ms, march_n, launches], dtype=torch.float64,
                     device=dev)
    tmax = t.clone()
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    max_ms = float(tmax[0])
    tot_samples, tot_paths = float(t[1]), float(t[2])
    value = tot_samples / (max_ms * 1e-3)

    # ---- e2e: the public host-buffer C-ABI call, H2D + D2H inside --------
    host_pix = Renderer.pinned((n_local,), np.int32)             # pinned host buffers (contract)
    host_pix[:] = pix_host
    host_out = Renderer.pinned((n_local, 3), np.float64)
    r.render_host(cams[0], 1, 0, pixels=host_pix, out=host_out)          # warm
    e2e_ms = []
    e2e_samples = 0
    for k in range(args.steps):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r.render_host(cams[(args.warmup + k) % len(cams)], 1, 0, pixels=host_pix, out=host_out)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_samples += r.last_stats["nerf_samples"]
    e2 = torch.tensor([sum(e2e_ms), e2e_samples], dtype=torch.float64, device=dev)
    e2max = e2.clone()
    if world > 1:
        dist.all_reduce(e2, op=dist.ReduceOp.SUM)
        dist.all_reduce(e2max, op=dist.ReduceOp.MAX)
    e2e_value = float(e2[1]) / (float(e2max[0]) * 1e-3)

    # ---- untimed extras: per-stage breakdown of one frame, gather roofline probe
    r.set_profile(True)
    r.render_pixels(cams[0], 1, 0, pixels=pix, out=out[:n_local])
    stages = {k: round(v, 3) for k, v in r.last_stats["stage_ms"].items()}
    stage_frame_ms = r.last_stats["ms"]
    r.set_profile(False)
    gather_gbs = r.gather_peak(2)

    if rank == 0:
        hbm, tflops, peak_src = peaks()
        enc_bytes = 8 * field.n_levels * field.n_features * 4            # 1024 B / sample
        mlp_flop = 2 * (field.enc_dim * 64 + 64 * 16 + 31 * 64 + 64 * 64 + 64 * 3)
        march_samples = evaluated                                          # rank-0 field-engine evaluations
        achieved = march_samples * enc_bytes / (march_ms * 1e-3) / 1e9
        traffic = ncu_traffic() or {}
        field_sps = march_samples / (march_ms * 1e-3)                      # samples/s inside the engine
        sec_per_sample = traffic.get("l2_sectors_per_sample")
        req_per_sample = traffic.get("l2_requests_per_sample")
        peak_requests = gather_gbs * 1e9 / 8.0                             # one request per random 8-B gather
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 rays/compositing, f32 hash encode, f16 tcgen05 MMA (f32 accum)",
            "data": "synthetic (seeded random-init NeRF + procedural meshes, SURVEY Appendix B)",
            "mrays_per_s": tot_paths / (max_ms * 1e-3) / 1e6,
            "nerf_samples_per_frame": tot_samples / args.steps,
            "config": {"workload": WORKLOAD, "frame": [w, h], "tile": TILE,
                       "parallelism": f"16x16 pixel tiles round-robin over {world} GPU(s); " + (
                           "each rank's k_accumulate stores its pixels into rank 0's frame over peer memory "
                           "(CUDA IPC / NVLink), then a barrier" if peer is not None
                           else "NCCL all-gather to rank 0"),
                       "l2": "256 MB buffer written before every timed step, outside the CUDA-event window",
                       "wall_s_timed_region": t_wall},
            "gpu_launches": int(launches),
            "roofline": {
                "bound": "hbm", "kernel": "fws::k_field_ws<32,2> (warp-specialized hash encode + 5-layer tcgen05 MLP, TMEM operands)",
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic.get("dram_bytes_per_launch"),
                "bytes_per_sample": enc_bytes, "launches": int(march_n),
                "avg_launch_ms": march_ms / max(1, march_n),
                "peak_source": peak_src + " hbm_gbs (burst copy); the 46.5 MiB table is L2-resident, "
                               "so frac > 1 vs HBM: the real limiter is roofline_gather",
            },
            "roofline_gather": {
                "bound": "L1 miss requests to L2 (random gathers, ~1 request/clk/SM)",
                "achieved": field_sps * req_per_sample if req_per_sample else None,
                "peak": peak_requests, "unit": "requests/s",
                "frac": field_sps * req_per_sample / peak_requests if req_per_sample else None,
                "requests_per_sample": req_per_sample, "sectors_per_sample": sec_per_sample,
                "peak_source": "hrt_gather_peak (live, this run): independent random 8-B gathers over the "
                               f"same table, {gather_gbs:.0f} GB/s useful = 1 request each; requests/sample from "
                               "profiles/r01e_field_traffic.json (ncu lts__t_requests_srcunit_tex_op_read over a "
                               "frame's field-engine launches)",
            },
            "roofline_mlp": {"bound": "tensor", "achieved": march_samples * mlp_flop / (march_ms * 1e-3) / 1e12,
                             "peak": tflops, "unit": "TFLOP/s",
                             "frac": march_samples * mlp_flop / (march_ms * 1e-3) / 1e12 / tflops,
                             "flop_per_sample": mlp_flop, "peak_source": peak_src + " bf16_tflops_sustained"},
            "e2e": {"value": e2e_value, "unit": "samples/s",
                    "h2d_bytes_per_step": int(4 * n_local), "d2h_bytes_per_step": int(24 * n_local),
                    "path": "hrt_render_host (pinned host pixel list in, pinned host float64 frame out, direct DMA both ways), wall clock"},
            "clocks": clk,
            "stages_ms": {"frame_ms": stage_frame_ms, **stages,
                          "note": "one untimed camera-0 frame with hrt_set_profile (event pair per launch)"},
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_block(args.cpu_tiles)
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    r.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
