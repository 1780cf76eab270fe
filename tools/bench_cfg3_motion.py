"""cfg3 dynamic scene (BASELINE config 3): 30 frames of seeded rigid motion
with a GPU BVH refit per frame; prints per-frame update, refit and render
device time. Default: transforms only (hrt_refit_rigid); --host: move the
meshes on the host and refit from the uploaded world faces."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.renderer import renderer_for  # noqa: E402

res = tuple(int(v) for v in sys.argv[1].split("x")) if len(sys.argv) > 1 else (1920, 1080)
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 30
host = "--host" in sys.argv
scene = configs.cfg3(res=res)
r = renderer_for(scene)
if not host:
    from paper_2309_04581_b200 import assets  # noqa: E402
    base_v, base_f = assets.icosphere(1.0, 4)
    r.set_rigid_base([base_v] * len(scene.meshes), [base_f] * len(scene.meshes))
r.render_pixels(scene.camera, scene.render.spp, 0)            # warm
tot = {"move": 0.0, "refit": 0.0, "render": 0.0}
for f in range(frames):
    t0 = time.perf_counter()
    if host:
        configs.cfg3_move(scene, f)
        t1 = time.perf_counter()
        r = renderer_for(scene)                              # geometry changed -> hrt_refit
    else:
        xf = configs.cfg3_transforms(f)
        t1 = time.perf_counter()
        r.refit_rigid(xf)                                    # hrt_refit_rigid
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    r.render_pixels(scene.camera, scene.render.spp, 0)
    s = r.last_stats
    tot["move"] += t1 - t0
    tot["refit"] += t2 - t1
    tot["render"] += s["ms"] * 1e-3
    print(f"frame {f:2d}: move {1e3*(t1-t0):7.1f} ms  refit {1e3*(t2-t1):7.1f} ms  "
          f"render {s['ms']:7.1f} ms  {s['paths']/s['ms']/1e3:6.1f} Mrays/s", flush=True)
print({k: round(v / frames * 1e3, 2) for k, v in tot.items()}, "ms per frame (mean)")
