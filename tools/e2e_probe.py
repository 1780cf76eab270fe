import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs
from paper_2309_04581_b200.renderer import Renderer
from paper_2309_04581_b200.tiles import tile_pixels
scene = configs.cfg1(); r = Renderer(scene); cam = scene.camera
pix = tile_pixels(800, 800, 0, 1); P = torch.as_tensor(pix, device="cuda")
out = np.empty((len(pix), 3))
for name, fn in (("device", lambda: r.render_pixels(cam, 1, 0, pixels=P)), ("host", lambda: r.render_host(cam, 1, 0, pixels=pix, out=out))):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    print(name, [f"{x:.1f}" for x in ts], "dev ms", f"{r.last_stats['ms']:.1f}")
