import math, os, sys
sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np, torch
import bench
import paper_1405_2270_b200 as L
dev = torch.device("cuda", 0)
B = 10.0
spec4 = L.LatticeSpec((256, 256, 256), L.GridSpec(B, 256), [L.Charge((0.0, 0.0, 0.0), 1.0)])
rule4 = L.sinc_quadrature(1e-6, spec4.unit.h, math.sqrt(3.0) * 256 * B, 20, 1.0)
p4 = L.DevicePipeline(spec4, rule4, mode="erf", periodic=True, device=dev)
rng = np.random.default_rng(4)
G = [torch.as_tensor(rng.uniform(size=(256, 1024)), device=dev) for _ in range(3)]
fb = lambda: L.DevicePipeline.functional_batch_device([p4.factor(l) for l in range(3)], p4.w, G)
p4.generate(); p4.assemble()
a = fb().clone(); b = fb().clone()
print("eager repeat equal:", torch.equal(a, b))
f0 = [p4.factor(l).clone() for l in range(3)]
bench._ev_ms(lambda: (p4.generate(), p4.assemble()))
print("factors after eager gen+asm equal:", all(torch.equal(f0[l], p4.factor(l)) for l in range(3)), "fb equal:", torch.equal(fb(), a))
ms, how = bench._graph_ms(lambda: (p4.generate(), p4.assemble()))
print(how, "factors after graph gen+asm equal:", all(torch.equal(f0[l], p4.factor(l)) for l in range(3)), "fb equal:", torch.equal(fb(), a))
ms, how = bench._graph_ms(fb)
c = fb()
print(how, "fb after graph fb equal:", torch.equal(c, a), float((c - a).abs().max()), float(a.abs().max()))
ms, how = bench._graph_ms(lambda: p4.grid_functional_batch(G))
print(how, "after graph gfb:", torch.equal(fb(), a), all(torch.equal(f0[l], p4.factor(l)) for l in range(3)))
