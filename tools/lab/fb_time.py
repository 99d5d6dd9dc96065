import math, os, sys
sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1405_2270_b200 as L
dev = torch.device("cuda", 0)
spec4 = L.LatticeSpec((256, 256, 256), L.GridSpec(10.0, 256), [L.Charge((0.0, 0.0, 0.0), 1.0)])
rule4 = L.sinc_quadrature(1e-6, spec4.unit.h, math.sqrt(3.0) * 256 * 10.0, 20, 1.0)
p4 = L.DevicePipeline(spec4, rule4, mode="erf", periodic=True, device=dev)
p4.generate(); p4.assemble()
rng = np.random.default_rng(4)
G = [torch.as_tensor(rng.uniform(size=(256, 1024)), device=dev) for _ in range(3)]
for _ in range(5):
    L.DevicePipeline.functional_batch_device([p4.factor(l).T for l in range(3)], p4.w, G)
torch.cuda.synchronize()
