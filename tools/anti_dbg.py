import sys, os, numpy as np, torch
sys.path[:0]=['/root/repo','/root/repo/tests']
import oracle as O, paper_0901_0638_b200 as Q
from synth import inputs as I
from _parity import ulp_errors
dtype=np.float32
n=(1<<23)+37
u = np.concatenate([I.edge_values(dtype), I.uniform_grid(n, dtype=dtype), I.edge_values(dtype)])
for alg, f in [(Q.BREAKLESS77, O.A77), (Q.BREAKLESS, O.C55)]:
    ref = O.normal_antithetic(u.astype(np.float64), f, 32)
    for rep in range(int(os.environ.get("REPS", "5"))):
        g = Q.qm_normal_antithetic(torch.from_numpy(u).cuda(), alg=alg).cpu().numpy()
        err = ulp_errors(g, ref, dtype)
        bad = np.nonzero(err > 4)[0]
        print(alg, rep, err.max(), len(bad), bad[:10], g[bad[:4]] if len(bad) else '', ref[bad[:4]].astype(np.float64) if len(bad) else '')
