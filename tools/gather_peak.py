"""Dev aid: hrt_gather_peak on the cfg1 table (LSU, TEX, both)."""
import sys

sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs  # noqa: E402
from paper_2309_04581_b200.renderer import Renderer  # noqa: E402

r = Renderer(configs.cfg1())
for mode, name in ((0, "LSU"), (1, "TEX"), (2, "LSU+TEX")):
    print(f"{name:8s} {r.gather_peak(mode):8.1f} GB/s useful (8 B per random gather)", flush=True)
