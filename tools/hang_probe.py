import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2309_04581_b200 import configs
from paper_2309_04581_b200.renderer import Renderer
cfg = int(sys.argv[1]); n = int(float(sys.argv[2])); dens = sys.argv[3] == "1"
scene = configs.BUILDERS[cfg]()
r = Renderer(scene)
g = np.random.default_rng(0)
P = torch.as_tensor(g.uniform(-1.5, 1.5, (n, 3)), device="cuda")
D = torch.as_tensor(g.normal(size=(n, 3)), device="cuda")
D = D / D.norm(dim=1, keepdim=True)
torch.cuda.synchronize(); t = time.time()
s, c, e = r.field_sample(P, None if dens else D)
torch.cuda.synchronize()
print(f"cfg{cfg} n={n} density_only={dens} {time.time()-t:.3f}s sigma_mean={s.mean().item():.4f}", flush=True)
