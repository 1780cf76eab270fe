"""Dev aid: predict strong scaling of the bench workload (cfg1 800x800 frame)
on one GPU by rendering the pixel tiles ONE rank of an N-GPU job would
own (tiles.tile_pixels) and timing it with CUDA events, cameras cycling as in
bench.py. Every rank of an N-GPU run has this much work, so N * t(1) / t(N)
estimates the efficiency the multi-GPU bench can reach (minus the frame
barrier). Usage: python tools/scale_probe.py [frames] [worlds] [cfg]
(cfg 1: the bench workload, cameras cycling; cfg 3: the 1080p 8-spp frame of
the dynamic scene, its own camera)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.renderer import Renderer  # noqa: E402
from paper_2309_04581_b200.tiles import tile_pixels  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 10
worlds = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 1
scene = configs.BUILDERS[cfg]()
cams = configs.cfg1_cameras() if cfg == 1 else [scene.camera]
spp = 1 if cfg == 1 else scene.render.spp
r = Renderer(scene)
w, h = cams[0].resolution
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
base = None
for world in worlds:
    pix = torch.as_tensor(tile_pixels(w, h, 0, world), device="cuda")
    out = torch.empty((pix.numel(), 3), dtype=torch.float64, device="cuda")
    for k in range(3):
        r.render_pixels(cams[k % len(cams)], spp, 0, pixels=pix, out=out)
    ms = []
    syncs = []
    for k in range(frames):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r.render_pixels(cams[(3 + k) % len(cams)], spp, 0, pixels=pix, out=out)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        syncs.append(r.last_stats.get("rounds", 0))
    t = sum(ms) / len(ms)
    r.set_profile(True)
    r.render_pixels(cams[3 % len(cams)], spp, 0, pixels=pix, out=out)
    stages = " ".join(f"{k}={v:.2f}" for k, v in r.last_stats["stage_ms"].items())
    r.set_profile(False)
    if base is None:
        base = t * world
    print(f"world {world}: rank-0 share {pix.numel():7d} px  {t:7.3f} ms/frame  "
          f"rounds {sum(syncs) / len(syncs):.0f}  launches {r.last_stats['launches']}  "
          f"predicted efficiency {base / (world * t):.3f} (vs the first world listed)\n    stages ms: {stages}", flush=True)
