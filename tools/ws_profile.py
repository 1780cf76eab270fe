"""Per-role cycle accounting of the field engine (HRT_WS_PROFILE build)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from paper_2309_04581_b200 import _lib, configs
from paper_2309_04581_b200.renderer import Renderer
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
scene = configs.BUILDERS[cfg]()
r = Renderer(scene)
r.render_pixels(scene.camera, scene.render.spp, 0); lib.hrt_ws_profile(buf)
r.render_pixels(scene.camera, scene.render.spp, 0); torch.cuda.synchronize()
lib.hrt_ws_profile(buf)
v = [buf[i] for i in range(8)]
enc_warps, epi_warps, mma = 16 * 148, 8 * 148, 148
print(f"cfg{cfg} frame {r.last_stats['ms']:.2f} ms field {r.last_stats['field_ms']:.2f} ms")
print(f" encode warps: total {v[0]/enc_warps/1e6:.2f} Mcyc/warp, waiting empty {100*v[1]/max(v[0],1):.1f}%")
print(f" epilogue warps: total {v[2]/epi_warps/1e6:.2f} Mcyc/warp, waiting accf {100*v[3]/max(v[2],1):.1f}%")
print(f" mma thread: total {v[4]/mma/1e6:.2f} Mcyc, waiting full {100*v[5]/max(v[4],1):.1f}%, waiting actr {100*v[6]/max(v[4],1):.1f}%")
