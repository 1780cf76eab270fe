"""Dev aid: wall time of one cfg1 frame through the device API vs the host
API (hrt_render_host) with pageable and with page-locked caller buffers."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.renderer import Renderer  # noqa: E402
from paper_2309_04581_b200.tiles import tile_pixels  # noqa: E402

scene = configs.cfg1()
r = Renderer(scene)
cam = scene.camera
pix = tile_pixels(800, 800, 0, 1)
P = torch.as_tensor(pix, device="cuda")
out = np.empty((len(pix), 3))
pin_pix = Renderer.pinned((len(pix),), np.int32)
pin_pix[:] = pix
pin_out = Renderer.pinned((len(pix), 3), np.float64)
for name, fn in (("device", lambda: r.render_pixels(cam, 1, 0, pixels=P)),
                 ("host pageable", lambda: r.render_host(cam, 1, 0, pixels=pix, out=out)),
                 ("host pinned", lambda: r.render_host(cam, 1, 0, pixels=pin_pix, out=pin_out))):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"{name:14s}", [f"{x:.2f}" for x in ts], "dev ms", f"{r.last_stats['ms']:.2f}")
