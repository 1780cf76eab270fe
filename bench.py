#!/usr/bin/env python
"""Benchmark: NeRF samples/s and Mrays/s per frame for the hybrid NeRF/mesh
render path (BASELINE.json metric) on BASELINE config 3 - the config the
metric's "per frame at 1/2/4/8 B200" and the north star's "1->8-GPU Mrays/s
scaling at 1080p" are quoted on:

  200 icospheres s4 (1,024,000 triangles; mirror / glass / diffuse) moving
  rigidly inside the L16 F2 T2^19 hash-grid NeRF, 1920x1080, 8 spp, 4 bounces.

One step = one frame of the 30-frame seeded motion (frame = step mod 30):
`hrt_refit_rigid` (per-mesh transforms -> world faces -> BVH refit on the GPU,
the reference's per-frame `sim.sync_to_renderer -> Scene.rebuild_bvh`,
`sim.py:673-698`, `scene.py:475-479`), then the full frame
(`render.py:372-380`), with scene and network resident in HBM. With N GPUs
(one process per GPU) the frame is split into 16x16 pixel tiles dealt
round-robin to ranks (`render.py:353-369`'s tile split); every
rank's accumulate kernel stores its pixels straight into rank 0's frame over
peer memory (CUDA IPC over NVLink) - `--gather nccl` uses an NCCL all-gather
instead (strong scaling: the frame is fixed).

`python bench.py --gpus N` without torchrun re-launches itself under
`torch.distributed.run` with N ranks. `--config cfg1` times BASELINE config 1
instead (cfg1 is also reported as an extra key of the default run).
`--impl reference` times the CPU oracle port of the reference path (oracle/,
numpy) on the host cores, on seeded crops of the same config.

Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NeRF samples/sec and Mrays/sec per frame at 1/2/4/8 B200 vs CPU ref"
TILE = 16
WORKLOADS = {
    "cfg3": "cfg3: 200 moving icospheres s4 (1,024,000 tris; mirror/glass/diffuse, seed 3) in the "
            "L16 F2 T2^19 16->2048 hash-grid NeRF (seed 1), 1920x1080, 8 spp, 4 bounces, 128^3 "
            "occupancy, 1024-sample cap, early-out 1e-4; each step = GPU rigid refit of the next of "
            "30 seeded motion frames + the full frame",
    "cfg4": "cfg4: emissive quad (radiance 10, r_src 1) + shadow rays occluded by a 300k-triangle displaced "
            "torus in the L16 F4 T2^21 16->4096 softplus HDR NeRF (seed 4), 3840x2160, 64 spp (8x8 stratified), "
            "6 bounces; each step = one full 4K frame",
    "cfg1": "cfg1: glass icosphere s5 (20480 tris, IOR 1.5) in L16 F2 T2^19 16->2048 hash-grid NeRF, "
            "800x800, 1 spp, 4 bounces, 128^3 occupancy, 1024-sample cap, early-out 1e-4, 100 seeded "
            "cameras (step k = camera k mod 100)",
}
CFG3_FRAMES = 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["cfg3", "cfg1", "cfg4"], default="cfg3")
    ap.add_argument("--cpu-tiles", type=int, default=0,
                    help="16x16 tiles per CPU sample (0 = scaled to the worker count)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg1 extra key")
    ap.add_argument("--gather", choices=["peer", "nccl"], default="peer",
                    help="frame assembly: peer-memory stores from the render (default) or NCCL all-gather")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args):
    """`bench.py --gpus N` outside torchrun: re-launch under
    torch.distributed.run with N ranks (one per GPU) and exit with its code.
    Fails loudly when fewer than N GPUs are visible (HRT_DIST_BACKEND=gloo
    lets N ranks share fewer GPUs to exercise the multi-rank flow)."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1 or args.impl == "reference":
        return
    backend = os.environ.get("HRT_DIST_BACKEND", "nccl")
    if backend == "nccl":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n} "
                  "(HRT_DIST_BACKEND=gloo shares GPUs for a functional multi-rank run)",
                  file=sys.stderr, flush=True)
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=dict(os.environ)))


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


# Tables above this size cannot stay L2-resident next to the streaming batch rows
# (126 MB L2 per B200, two 63 MB halves): their roofline is HBM, not the L2 peak.
L2_RESIDENT_BYTES = 96 << 20


def ncu_traffic(config):
    """Field-engine L2 traffic per sample from the newest committed ncu
    capture of this config (profiles/*_field_traffic_<config>.json, made by
    tools/field_traffic.py from an ncu run over every k_field_ws launch of
    one frame; the file names the commit it was captured at)."""
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*field_traffic_{config}.json")))
    if not paths:
        return None, None
    try:
        with open(paths[-1]) as f:
            return json.load(f), os.path.relpath(paths[-1], ROOT)
    except (OSError, ValueError):
        return None, None


# --------------------------------------------------- CPU baseline (oracle) -

_CPU = {}


def _cpu_scene(config):
    """Oracle scene of the config, built once in the parent (scene build,
    BVH and occupancy are outside the timed sample, as for the GPU arm) and
    inherited by the forked workers."""
    if config not in _CPU:
        from oracle import tracer
        from paper_2309_04581_b200 import configs
        from paper_2309_04581_b200.pack import pack_camera, pack_scene
        scene = {"cfg3": configs.cfg3, "cfg1": configs.cfg1, "cfg4": configs.cfg4}[config]()
        _CPU[config] = (tracer.OracleScene(pack_scene(scene)), pack_camera(scene.camera))
    return _CPU[config]


def _occ_rows(args):
    config, lo, hi = args
    import numpy as np
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle.field import neural_encode, neural_mlp
    fp = _cpu_scene(config)[0].field
    g = int(fp["occ_res"])
    c = np.arange(lo, hi)
    ijk = np.stack([c % g, (c // g) % g, c // (g * g)], axis=1).astype(np.float64)
    pf = fp["bbox_lo"] + (ijk + 0.5) * ((fp["bbox_hi"] - fp["bbox_lo"]) / g)
    sigma, _ = neural_mlp(fp, neural_encode(fp, pf), None, density_only=True)
    return lo, sigma > fp["occ_threshold"]


def _cpu_occupancy(config, pool):
    """The oracle's occupancy bitfield (oracle.field.build_occupancy, cell i =
    x + G*(y + G*z)), computed in slices over the worker pool."""
    import numpy as np
    fp = _cpu_scene(config)[0].field
    if "_occ_cache" in fp or fp.get("occ_bits") is not None:
        return
    g = int(fp["occ_res"])
    n = g ** 3
    step = 1 << 14
    occ = np.zeros(n, bool)
    for lo, m in pool.map(_occ_rows, [(config, a, min(n, a + step)) for a in range(0, n, step)]):
        occ[lo:lo + len(m)] = m
    words = np.zeros((n + 31) // 32, np.uint32)
    idx = np.nonzero(occ)[0]
    np.bitwise_or.at(words, idx >> 5, (np.uint32(1) << (idx & 31).astype(np.uint32)))
    fp["_occ_cache"] = words


def _cpu_tile(args):
    config, frame_cam, pixels, spp = args
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)                 # one BLAS thread per worker process
    from oracle import tracer
    sc, cam = _cpu_scene(config)
    if config == "cfg1":
        from paper_2309_04581_b200 import configs
        from paper_2309_04581_b200.pack import pack_camera
        cam = pack_camera(configs.cfg1_cameras()[frame_cam])
    st = {}
    tracer.render(sc, cam, spp, 0, pixels=pixels, stats=st)
    return st["nerf_samples"], st["paths"]


def _warm(_):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    from oracle import tracer  # noqa: F401
    return 0


def cpu_pool(config, workers):
    """One forked worker per core, created once (scene inherited, imports
    warmed by a tiny job) so timed samples measure tracing, not start-up;
    the oracle occupancy grid is built on the pool before it is forked
    again for the tiles."""
    import multiprocessing as mp
    _cpu_scene(config)
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as p:
        _cpu_occupancy(config, p)
    pool = ctx.Pool(workers)              # forked after the occupancy cache exists
    pool.map(_warm, range(workers))
    return pool


def _frame_shape(config):
    return {"cfg3": ((1920, 1080), 8), "cfg1": ((800, 800), 1), "cfg4": ((3840, 2160), 64)}[config]


def _cpu_tile_size(config):
    return 8 if config == "cfg4" else TILE          # (a 16x16 x 64 spp cfg4 tile is minutes of CPU)


def cpu_sample(config, n_tiles, pool, cam_index=0, seed=0):
    """Oracle (numpy port of the reference path) on `n_tiles` seeded 16x16
    tiles of the config's frame, one process per core."""
    import numpy as np
    (w, h), spp = _frame_shape(config)
    rng = np.random.default_rng(seed)
    ts = _cpu_tile_size(config)
    tx = w // ts
    chosen = rng.choice(tx * (h // ts), n_tiles, replace=False)
    jobs = []
    for t in chosen:
        x0, y0 = (t % tx) * ts, (t // tx) * ts
        ys, xs = np.meshgrid(np.arange(y0, y0 + ts), np.arange(x0, x0 + ts), indexing="ij")
        jobs.append((config, cam_index, (ys * w + xs).reshape(-1), spp))
    t0 = time.perf_counter()
    res = pool.map(_cpu_tile, jobs, chunksize=1)
    dt = time.perf_counter() - t0
    return sum(r[0] for r in res), sum(r[1] for r in res), dt


def cpu_workers():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def shipped_block(workers):
    """The unmodified reference (baseline/_ref) with a dense-grid stand-in on
    seeded cfg3 tiles, one process per core (oracle/shipped.py)."""
    import multiprocessing as mp

    import numpy as np

    from oracle import shipped
    try:
        where = shipped.import_reference()
    except Exception as e:          # noqa: BLE001 - context only
        return {"unavailable": f"reference import failed: {e}"}
    if where is None:
        return {"unavailable": "hybridrt not installed in baseline/_ref"}
    t0 = time.perf_counter()
    shipped.scene()                  # reference Bvh build over 1.02 M triangles (outside the timing)
    build_s = time.perf_counter() - t0
    tiles = list(np.random.default_rng(7).choice((1920 // TILE) * (1080 // TILE), 2 * workers,
                                                  replace=False))
    with mp.get_context("fork").Pool(workers) as pool:
        pool.map(shipped.tile_job, tiles[:workers])          # warm
        t0 = time.perf_counter()
        res = pool.map(shipped.tile_job, tiles, chunksize=1)
        dt = time.perf_counter() - t0
    samples = sum(r[0] for r in res)
    paths = sum(r[1] for r in res)
    return {"value": samples / dt, "unit": "field samples/s", "mrays_per_s": paths / dt / 1e6,
            "cores": workers, "kind": "reference",
            "sample": f"{len(tiles)} seeded 16x16 x 8 spp tiles of the cfg3 frame-0 geometry through the "
                      f"UNMODIFIED reference tracer (hybridrt from {os.path.relpath(where, ROOT) if where.startswith(ROOT) else where}: "
                      "_sample_jitter -> Camera.primary_rays -> _trace_batch_hybrid) with a dense 64^3 "
                      f"RadianceGrid fog in place of the NeRF it does not implement; one process per core, "
                      f"{dt:.1f} s wall ({paths} paths, {samples} field samples; reference Bvh build "
                      f"{build_s:.1f} s not timed)"}


def cpu_baseline_block(config, n_tiles=0):
    workers = cpu_workers()
    (w, h), spp = _frame_shape(config)
    n_tiles = n_tiles or {"cfg3": 4 * workers, "cfg4": workers}.get(config, max(16, 8 * workers))  # ~10-30 s
    pool = cpu_pool(config, workers)
    samples, paths, dt = cpu_sample(config, n_tiles, pool)
    pool.close()
    pool.join()
    return {"value": samples / dt, "unit": "samples/s", "cores": workers, "kind": "port",
            "cpu": cpu_model(), "mrays_per_s": paths / dt / 1e6,
            "sample": f"{n_tiles} seeded {_cpu_tile_size(config)}x{_cpu_tile_size(config)} x {spp} spp tiles ({paths} paths, {samples} NeRF samples) "
                      f"of the {config} frame-0 {w}x{h} frame, oracle/ numpy port of the reference "
                      f"render loop + neural field, one process per core, {dt:.1f} s wall",
            "reference_as_shipped": shipped_block(workers) if config == "cfg3" else None}


# ------------------------------------------------------------ arms ------

def run_reference(args, rank, world):
    if rank != 0:
        return
    workers = cpu_workers()
    (w, h), spp = _frame_shape(args.config)
    n_tiles = args.cpu_tiles or {"cfg3": workers, "cfg4": workers // 2 or 1}.get(args.config, max(8, 4 * workers))
    pool = cpu_pool(args.config, workers)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(args.config, max(1, workers), pool)
    tot_s = tot_p = tot_t = 0.0
    for k in range(args.steps):
        s, p, dt = cpu_sample(args.config, n_tiles, pool, cam_index=k % 100, seed=k)
        tot_s, tot_p, tot_t = tot_s + s, tot_p + p, tot_t + dt
    pool.close()
    pool.join()
    value = tot_s / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "mrays_per_s": tot_p / tot_t / 1e6,
        "config": {"workload": WORKLOADS[args.config] + f"; CPU sample per step = {n_tiles} seeded "
                                                        f"16x16 x {spp} spp tiles of frame 0",
                   "frame": [w, h]},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": workers, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"{n_tiles} seeded 16x16 x {spp} spp tiles per step x {args.steps} "
                                   f"steps, oracle/ numpy port of the reference render loop + neural "
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


class Workload:
    """The timed scene: renderer + per-step inputs (camera, spp, motion)."""

    def __init__(self, config, dev):
        import numpy as np

        from paper_2309_04581_b200 import assets, configs
        from paper_2309_04581_b200.renderer import Renderer
        self.config = config
        if config == "cfg3":
            self.scene = configs.cfg3()
            self.r = Renderer(self.scene)
            base_v, base_f = assets.icosphere(1.0, 4)
            n = len(self.scene.meshes)
            self.r.set_rigid_base([base_v] * n, [base_f] * n)
            # the 30 frames' transforms in page-locked host memory (e2e H2D source)
            self.xf = [Renderer.pinned((n, 3, 4), np.float64) for _ in range(CFG3_FRAMES)]
            for f in range(CFG3_FRAMES):
                self.xf[f][:] = configs.cfg3_transforms(f)
            self.cams = [self.scene.camera]
            self.spp = self.scene.render.spp
        elif config == "cfg4":
            self.scene = configs.cfg4()
            self.r = Renderer(self.scene)
            self.xf = None
            self.cams = [self.scene.camera]
            self.spp = self.scene.render.spp
        else:
            self.scene = configs.cfg1()
            self.r = Renderer(self.scene)
            self.xf = None
            self.cams = configs.cfg1_cameras()
            self.spp = 1
        self.field = self.scene.field
        self.w, self.h = self.cams[0].resolution

    def prepare(self, k):
        """Per-frame scene update (cfg3: refit to motion frame k mod 30)."""
        if self.xf is not None:
            self.r.refit_rigid(self.xf[k % CFG3_FRAMES])

    def camera(self, k):
        return self.cams[k % len(self.cams)]

    def h2d_update_bytes(self):
        return 0 if self.xf is None else int(self.xf[0].nbytes)


def time_frames(wl, steps, warmup, pix, peer, out, gather, flush, stream, k0=0):
    """Device time of `steps` frames (after `warmup`): per step the scene
    update + the render of this rank's tiles (+ the NCCL gather when there is
    no peer frame), CUDA events on the launching stream."""
    import torch
    n_local = int(pix.numel())
    res = []

    def step(k, timed):
        if timed:
            flush.fill_(float(k))          # evict L2 between timed steps (outside the events)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
        wl.prepare(k)
        if timed:
            e1.record(stream)
        if peer is not None:               # pixels stored into rank 0's frame (peer memory)
            wl.r.render_pixels(wl.camera(k), wl.spp, 0, pixels=pix, frame_ptr=peer.ptr)
            st = dict(wl.r.last_stats)
            if timed:
                e2.record(stream)
            peer.done()                    # stream sync + barrier: rank 0's frame complete
        else:
            wl.r.render_pixels(wl.camera(k), wl.spp, 0, pixels=pix, out=out[:n_local])
            st = dict(wl.r.last_stats)
            gather.gather()                # frame assembled on rank 0 (NCCL all-gather)
            if timed:
                e2.record(stream)
        if timed:
            e2.synchronize()
            st["step_ms"] = e0.elapsed_time(e2)
            st["refit_ms"] = e0.elapsed_time(e1)
        return st

    for k in range(warmup):
        step(k0 + k, False)
    return [step(k0 + warmup + k, True) for k in range(steps)]


def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2309_04581_b200.renderer import Renderer, finalize_device
    from paper_2309_04581_b200.tiles import FrameGather, tile_pixels

    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    # one process per GPU; HRT_DIST_BACKEND=gloo lets several ranks share one GPU to test the
    # multi-rank flow where only one device exists (timings then mean nothing)
    dev_index = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    backend = os.environ.get("HRT_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")          # NVLink / NVLS transport choice in the log
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    wl = Workload(args.config, dev)
    w, h = wl.w, wl.h
    pix_host = tile_pixels(w, h, rank, world)
    pix = torch.as_tensor(pix_host, device=dev)
    n_local = len(pix_host)
    gather = FrameGather(w, h, rank, world, dev)
    out = gather.local
    peer = open_peer_frame(w, h, rank, world) if args.gather == "peer" else None
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev_index)
    clocks.start()
    t_wall = time.perf_counter()
    steps = time_frames(wl, args.steps, args.warmup, pix, peer, out, gather, flush, stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall
    clk = clocks.stop()

    # frame time = the slowest rank's step time, per step (max over ranks)
    per_step = torch.tensor([s["step_ms"] for s in steps], dtype=torch.float64, device=dev)
    sums = torch.tensor([sum(s[k] for s in steps) for k in
                         ("nerf_samples", "paths", "field_ms", "field_launches", "launches", "evaluated",
                          "refit_ms")], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(per_step, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    max_ms = float(per_step.sum())
    tot_samples, tot_paths = float(sums[0]), float(sums[1])
    value = tot_samples / (max_ms * 1e-3)
    rank0 = {k: sum(s[k] for s in steps) for k in ("field_ms", "field_launches", "evaluated", "launches",
                                                   "refit_ms")}

    # ---- e2e: the public API from host inputs to the host result --------
    # per step: H2D of the frame's transforms (pinned) -> hrt_refit_rigid, H2D of the rank's
    # pixel ids (pinned), render into rank 0's frame (peer stores or NCCL gather), then rank 0
    # encodes the frame (hrt_finalize, PFM = the CLI's output) and reads it back to host.
    pix_pinned = torch.from_numpy(Renderer.pinned((n_local,), np.int32))
    pix_pinned.numpy()[:] = pix_host
    pix_e2e = torch.empty_like(pix)
    pfm_host = None
    e2e_ms, e2e_samples, d2h = [], 0, 0

    def e2e_step(k):
        nonlocal pfm_host, d2h
        wl.prepare(k)                                    # H2D transforms inside (cfg3)
        pix_e2e.copy_(pix_pinned, non_blocking=True)
        if peer is not None:
            wl.r.render_pixels(wl.camera(k), wl.spp, 0, pixels=pix_e2e, frame_ptr=peer.ptr)
            st = dict(wl.r.last_stats)
            peer.done()
            frame = peer.frame() if rank == 0 else None
        else:
            wl.r.render_pixels(wl.camera(k), wl.spp, 0, pixels=pix_e2e, out=out[:n_local])
            st = dict(wl.r.last_stats)
            frame = gather.gather()
        if rank == 0:
            pfm = finalize_device(frame, w, h, hdr_output=True)
            if pfm_host is None:
                pfm_host = torch.empty(pfm.shape, dtype=torch.uint8, pin_memory=True)
            pfm_host.copy_(pfm)                          # D2H of the encoded frame
            d2h = int(pfm.numel())
        return st

    e2e_step(0)                                          # warm (finalize buffers)
    for k in range(args.steps):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        st = e2e_step(args.warmup + k)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_samples += st["nerf_samples"]
    e2 = torch.tensor(e2e_ms + [e2e_samples], dtype=torch.float64, device=dev)
    if world > 1:
        mx = e2.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(e2, op=dist.ReduceOp.SUM)
        e2[:-1] = mx[:-1]
    e2e_value = float(e2[-1]) / (float(e2[:-1].sum()) * 1e-3)

    # ---- untimed extras: per-stage breakdown of one frame, L2 / gather peaks, cfg1
    wl.r.set_profile(True)
    wl.prepare(args.warmup)
    wl.r.render_pixels(wl.camera(args.warmup), wl.spp, 0, pixels=pix, out=out[:n_local])
    stages = {k: round(v, 3) for k, v in wl.r.last_stats["stage_ms"].items()}
    stage_frame_ms = wl.r.last_stats["ms"]
    rrows, rsmp, rms = wl.r.round_rows()               # per march round: batch rows, samples, engine ms
    wl.r.set_profile(False)
    live = rrows > 0
    rounds_block = {
        "rounds": int(live.sum()), "batch_rows": int(rrows.sum()), "samples": int(rsmp.sum()),
        "hole_fraction": float(1.0 - rsmp.sum() / max(1, rrows.sum())),
        "first_rounds_G_samples_per_s": [round(float(rsmp[i] / (rms[i] * 1e-3) / 1e9), 2)
                                         for i in np.nonzero(live)[0][:8]],
        "note": "hrt_round_rows of the profiled frame (first chunk's rounds): the first rounds carry the "
                "coherent primary rays, the later ones the incoherent bounces (DESIGN 4.1)"}
    gather_gbs = wl.r.gather_peak(2)          # random one-entry gathers (8 B F = 2, 16 B F = 4), LSU + TEX
    l2 = wl.r.l2_peak()

    extra = None
    if rank == 0 and world == 1 and args.config == "cfg3" and not args.no_extra:
        wl.r.close()
        w1 = Workload("cfg1", dev)
        p1 = torch.as_tensor(tile_pixels(w1.w, w1.h, 0, 1), device=dev)
        o1 = torch.empty((p1.numel(), 3), dtype=torch.float64, device=dev)
        s1 = time_frames(w1, 10, 3, p1, None, o1, _NoGather(), flush, stream)
        ms1 = sum(s["step_ms"] for s in s1)
        extra = {"workload": WORKLOADS["cfg1"], "steps": 10, "ms_per_step": ms1 / 10,
                 "value": sum(s["nerf_samples"] for s in s1) / (ms1 * 1e-3), "unit": "samples/s",
                 "mrays_per_s": sum(s["paths"] for s in s1) / (ms1 * 1e-3) / 1e6}
        w1.r.close()

    if rank == 0:
        hbm, tflops, peak_src = peaks()
        field = wl.field
        enc_bytes = 8 * field.n_levels * field.n_features * 4            # 1024 B / sample
        mlp_flop = 2 * (field.enc_dim * 64 + 64 * 16 + 31 * 64 + 64 * 64 + 64 * 3)
        march_ms, march_samples = rank0["field_ms"], rank0["evaluated"]   # rank-0 field engine
        field_sps = march_samples / (march_ms * 1e-3)                      # samples/s inside the engine
        achieved = field_sps * enc_bytes / 1e9
        traffic, traffic_src = ncu_traffic(args.config)
        traffic = traffic or {}
        req_per_sample = traffic.get("l2_requests_per_sample")
        entry_bytes = 4 * field.n_features
        peak_requests = gather_gbs * 1e9 / entry_bytes if gather_gbs else None   # one request per random gather
        table_bytes = int(field.table.nbytes)
        roof_peak = l2["read_gbs"]
        gather_frac = field_sps * req_per_sample / peak_requests if req_per_sample and peak_requests else None
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 rays/compositing, f32 hash encode, f16 tcgen05 MMA (f32 accum)",
            "data": "synthetic (seeded random-init NeRF + procedural meshes, SURVEY Appendix B)",
            "mrays_per_s": tot_paths / (max_ms * 1e-3) / 1e6,
            "nerf_samples_per_frame": tot_samples / args.steps,
            "config": {"workload": WORKLOADS[args.config], "frame": [w, h], "spp": wl.spp, "tile": TILE,
                       "parallelism": f"16x16 pixel tiles round-robin over {world} GPU(s); " + (
                           "each rank's k_accumulate stores its pixels into rank 0's frame over peer memory "
                           "(CUDA IPC / NVLink), then a barrier" if peer is not None
                           else "NCCL all-gather to rank 0"),
                       "step": "refit (hrt_refit_rigid) + frame; frame time = max over ranks per step"
                               if args.config == "cfg3" else "frame; max over ranks per step",
                       "l2": "256 MB buffer written before every timed step, outside the CUDA-event window",
                       "wall_s_timed_region": t_wall,
                       "refit_ms_per_step": rank0["refit_ms"] / args.steps},
            "gpu_launches": int(rank0["launches"]),
            "roofline": {
                "bound": "l2",
                "kernel": f"fws::k_field_ws<{field.enc_dim},{field.n_features},T> (warp-specialized hash encode + "
                          "5-layer tcgen05 MLP, TMEM operands; T = 2 encode teams in the first march rounds)",
                "achieved": achieved, "peak": roof_peak, "unit": "GB/s",
                "frac": achieved / roof_peak,
                "traffic": traffic.get("dram_bytes_per_launch"),
                "l2_bytes_per_launch": traffic.get("l2_bytes_per_launch"),
                "bytes_per_sample": enc_bytes, "launches": int(rank0["field_launches"]),
                "avg_launch_ms": march_ms / max(1, rank0["field_launches"]),
                "peak_source": f"hrt_l2_peak (live, this run): coalesced 16-B reads of {l2['bytes'] / 2**20:.0f} MiB "
                               f"of the {table_bytes / 2**20:.1f} MiB hash table, L2-resident, by every SM; "
                               "achieved = algorithmic encode bytes (8 corners x L x F x 4 B) x field-engine "
                               "samples/s (L1 hits included, so this is an upper view of the L2 load); "
                               "traffic = ncu dram bytes per field-engine launch (" +
                               (traffic_src or "no capture") + ")",
                "hbm": {"peak": hbm, "frac": achieved / hbm, "source": peak_src + " hbm_gbs (burst copy)"},
                "l2_read_gbs": l2["read_gbs"],
            },
            "roofline_gather": {
                "bound": "L1 miss requests to L2 (random gathers, ~1 request/clk/SM)",
                "achieved": field_sps * req_per_sample if req_per_sample else None,
                "peak": peak_requests, "unit": "requests/s",
                "frac": gather_frac,
                "requests_per_sample": req_per_sample,
                "sectors_per_sample": traffic.get("l2_sectors_per_sample"),
                "random_sector_gbs": l2["gather_sector_gbs"],
                "peak_source": f"hrt_gather_peak (live, this run): independent random {entry_bytes}-B gathers over an "
                               f"L2-resident window (<= 64 MiB) of the same table, {gather_gbs or 0:.0f} GB/s useful = "
                               "1 request each; requests/sample from "
                               f"{traffic_src} (ncu lts__t_requests_srcunit_tex_op_read over every field-engine "
                               f"launch of one frame, commit {traffic.get('commit')})",
            },
            "roofline_mlp": {"bound": "tensor", "achieved": field_sps * mlp_flop / 1e12,
                             "peak": tflops, "unit": "TFLOP/s",
                             "frac": field_sps * mlp_flop / 1e12 / tflops,
                             "flop_per_sample": mlp_flop, "peak_source": peak_src + " bf16_tflops_sustained"},
            "e2e": {"value": e2e_value, "unit": "samples/s",
                    "h2d_bytes_per_step": int(wl.h2d_update_bytes() + 4 * n_local),
                    "d2h_bytes_per_step": d2h,
                    "path": "per step: transforms (pinned) -> hrt_refit_rigid, pixel ids (pinned) H2D, "
                            "hrt_render of the rank's tiles into rank 0's frame, barrier, rank 0 "
                            "hrt_finalize (PFM) + D2H to pinned host; wall clock, max over ranks"},
            "clocks": clk,
            "stages_ms": {"frame_ms": stage_frame_ms, **stages,
                          "note": "one untimed frame with hrt_set_profile (event pair per launch)"},
            "field_rounds": rounds_block,
        }
        if table_bytes > L2_RESIDENT_BYTES and traffic.get("samples"):
            # The 344 MiB cfg4 table does not fit L2 (the encode streams its fine levels from
            # HBM) and L1 / L2 serve most of the algorithmic gather bytes, so bytes / L2 peak
            # (a 64 MiB L2-resident window) is no efficiency - the same frame measured 0.85
            # and 1.1 of it on two boxes. The bound resource is then HBM: achieved = the DRAM bytes
            # per sample ncu measured over every field-engine launch of one frame (same
            # commit) x this run's field-engine samples/s, against the measured HBM peak.
            alg = line["roofline"]
            dram_ps = (traffic["dram_read_bytes"] + traffic["dram_write_bytes"]) / traffic["samples"]
            hbm_ach = field_sps * dram_ps / 1e9
            line["roofline"] = {
                "bound": "hbm", "kernel": alg["kernel"],
                "achieved": hbm_ach, "peak": hbm, "unit": "GB/s", "frac": hbm_ach / hbm,
                "traffic": alg["traffic"], "dram_bytes_per_sample": dram_ps,
                "launches": alg["launches"], "avg_launch_ms": alg["avg_launch_ms"],
                "peak_source": peak_src + " hbm_gbs (burst copy); achieved = ncu DRAM bytes per sample "
                               f"({dram_ps:.0f} B, {traffic_src}, commit {traffic.get('commit')}) x field-engine "
                               "samples/s of this run. The algorithmic-bytes view exceeds the L2 peak (cache hits) "
                               "and is kept under 'algorithmic'; the random-gather probe over this table is in "
                               "roofline_gather (the encode beats random gathers through L1 / L2 locality)",
                "algorithmic": {"achieved": achieved, "peak": roof_peak, "frac": achieved / roof_peak,
                                "bytes_per_sample": enc_bytes, "bound": "l2 (live hrt_l2_peak)"}}
        if extra:
            line["cfg1"] = extra
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_block(args.config, args.cpu_tiles)
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    wl.r.close()
    if world > 1:
        dist.destroy_process_group()


class _NoGather:
    def gather(self):
        return None


def main():
    args = parse()
    maybe_spawn(args)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
