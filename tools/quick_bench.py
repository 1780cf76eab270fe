"""Quick device timing of one config's frames (development aid; bench.py is
the contract)."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.renderer import Renderer  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
res = tuple(int(v) for v in sys.argv[2].split("x")) if len(sys.argv) > 2 else None
spp = int(sys.argv[3]) if len(sys.argv) > 3 else None
t0 = time.time()
scene = configs.BUILDERS[cfg](res=res) if res and cfg in (3, 4) else configs.BUILDERS[cfg]()
if spp:
    scene.render.spp = spp
r = Renderer(scene)
r.set_profile(True)
if os.environ.get("HRT_MARCH") == "bounce":      # the reference's bounce-by-bounce loop
    r.set_march(False)
print(f"cfg{cfg} setup {time.time() - t0:.2f}s", flush=True)
for it in range(int(sys.argv[4]) if len(sys.argv) > 4 else 4):
    torch.cuda.synchronize()
    t = time.time()
    out = r.render_pixels(scene.camera, scene.render.spp, 0)
    torch.cuda.synchronize()
    dt = time.time() - t
    s = r.last_stats
    print(f"iter {it}: wall {dt*1e3:.1f} ms dev {s['ms']:.1f} ms samples {s['nerf_samples']:,} "
          f"({s['nerf_samples']/s['ms']*1e3/1e9:.3f} G/s) paths {s['paths']:,} "
          f"Mrays/s {s['paths']/s['ms']*1e3/1e6:.2f} mean {out.mean().item():.4f} | field {s['field_ms']:.1f} ms "
          f"x{s['field_launches']} evaluated {s['evaluated']:,} rounds {s['rounds']} launches {s['launches']} rows {s['batch_rows']:,}",
          flush=True)
    print("   stages ms: " + " ".join(f"{k}={v:.1f}" for k, v in s["stage_ms"].items()), flush=True)
