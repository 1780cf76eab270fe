"""Per-round field-engine throughput of one frame (hrt_round_rows): batch
rows (holes included), engine time, rows/s. With a HRT_SYNTH_ENCODE=1 build
(features from the position, no table gathers) the same table gives the MLP
pipeline's own ceiling. Usage: python tools/round_profile.py [cfg] [WxH] [spp]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.renderer import Renderer  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
res = tuple(int(v) for v in sys.argv[2].split("x")) if len(sys.argv) > 2 else None
scene = configs.BUILDERS[cfg](res=res) if res and cfg in (3, 4) else configs.BUILDERS[cfg]()
spp = int(sys.argv[3]) if len(sys.argv) > 3 else scene.render.spp
r = Renderer(scene)
r.render_pixels(scene.camera, spp, 0)
torch.cuda.synchronize()
r.render_pixels(scene.camera, spp, 0)
st = r.last_stats
rows, smp, ms = r.round_rows()
live = rows > 0
out = {"cfg": cfg, "frame_ms": st["ms"], "field_ms": st["field_ms"], "samples": st["nerf_samples"],
       "batch_rows": int(rows.sum()), "rounds": int(live.sum()),
       "rows_per_s_frame": float(rows.sum() / (ms.sum() * 1e-3)),
       "per_round": [{"i": i, "rows": int(rows[i]), "samples": int(smp[i]), "ms": round(float(ms[i]), 4),
                      "G_rows_per_s": round(float(rows[i] / (ms[i] * 1e-3) / 1e9), 3) if ms[i] > 0 else None}
                     for i in range(len(rows)) if rows[i] > 0]}
print(json.dumps(out))
