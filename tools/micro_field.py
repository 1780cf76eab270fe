"""Microbenchmark of the field kernels on ray-coherent sample streams:
hash encode alone (hrt_field_encode) vs encode + tcgen05 MLP (hrt_field_sample, the field engine)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.pack import pack_camera  # noqa: E402
from paper_2309_04581_b200.renderer import Renderer  # noqa: E402

from oracle import tracer  # noqa: E402


def coherent_points(cam, n_rays, per_ray, step):
    w, h = cam.resolution
    pix = np.linspace(0, w * h - 1, n_rays).astype(np.int64)
    o, d = tracer.primary_rays(pack_camera(cam), pix, np.full(n_rays, 0.5), np.full(n_rays, 0.5))
    t0, _ = tracer.ray_slab(np.full(3, -1.5), np.full(3, 1.5), o, d)
    t = np.maximum(t0, 0)[:, None] + (np.arange(per_ray)[None, :] + 0.5) * step
    p = o[:, None, :] + t[..., None] * d[:, None, :]
    dd = np.repeat(d[:, None, :], per_ray, 1)
    return p.reshape(-1, 3), dd.reshape(-1, 3)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
  for cfg in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "10")]:
      scene = configs.BUILDERS[cfg]()
      r = Renderer(scene)
      cam = scene.camera
      for layout in ("ray-major", "sample-major", "random"):
          p, d = coherent_points(cam, 65536, 128, configs.MARCH_STEP)
          if layout == "sample-major":       # 128 consecutive threads = 128 rays at one step
              p = p.reshape(65536, 128, 3).transpose(1, 0, 2).reshape(-1, 3)
              d = d.reshape(65536, 128, 3).transpose(1, 0, 2).reshape(-1, 3)
          elif layout == "random":
              perm = np.random.default_rng(0).permutation(len(p))
              p, d = p[perm], d[perm]
          P = torch.as_tensor(np.ascontiguousarray(p), device="cuda")
          D = torch.as_tensor(np.ascontiguousarray(d), device="cuda")
          n = len(p)
          t_enc = timeit(lambda: r.field_encode(P, with_index=False))
          t_full = timeit(lambda: r.field_sample(P, D))
          t_den = timeit(lambda: r.field_sample(P, None))
          print(f"cfg{cfg} {layout:12s} n={n/1e6:.1f}M  encode-only {n/t_enc/1e6:.2f} G/s  "
                f"encode+density {n/t_den/1e6:.2f} G/s  encode+full MLP {n/t_full/1e6:.2f} G/s",
                flush=True)
      r.close()


if __name__ == '__main__':
    main()
