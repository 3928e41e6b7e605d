import sys, os, time, hashlib
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1909_12234_b200 as M
from paper_1909_12234_b200 import multigrid as MG
geo = M.LatticeGeometry((16, 16, 16, 16), "antiperiodic")
op = M.build_wilson(M.generate_gauge(geo, "su3", eps=0.2, seed=0), 0.1)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    nv = MG.generate_null_vectors(op, 24, tol=1e-12, max_iter=8, seed=7)
    torch.cuda.synchronize(); el = time.perf_counter() - t0
print("null vectors 16^4 x24:", round(el, 4), "s  sha", hashlib.sha1(nv.vectors.cpu().numpy().tobytes()).hexdigest()[:16],
      "ratios", nv.residual_ratios[:3])
