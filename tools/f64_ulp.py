"""Max and tail-quantile ulp error of the fp64 breakless maps against the oracle
(measurement helper, not a test): python tools/f64_ulp.py [log2 n]
Inputs: half odd-grid uniforms, half tail-stratified (min(u, 1-u) log-uniform
down to 2^-53), the parity tests' recipe at a larger size.  One JSON line per formula."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as O  # noqa: E402
import paper_0901_0638_b200 as Q  # noqa: E402
from _parity import ulp_errors  # noqa: E402
from synth import inputs as I  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
deep = len(sys.argv) > 2 and sys.argv[2] == "deep"    # off the 2^-53 grid: u = 10^U(-320, -16), z = 36 .. 736
if deep:
    u = 10.0 ** np.random.default_rng(5).uniform(-320, -16, n)
else:
    u = np.concatenate([I.uniform_grid(n // 2, dtype=np.float64), I.tail_stratified(n - n // 2, dtype=np.float64)])
ud = torch.from_numpy(u).cuda()
cases = (("D13", Q.BREAKLESS, O.D13), ("F1212", Q.BREAKLESS1212, O.F1212), ("A77", Q.BREAKLESS77, O.A77))
if deep:
    cases = (("D13", Q.BREAKLESS, O.D13), ("D13_tail_composite", Q.BREAKLESS_TAIL, O.D13))
for name, alg, form in cases:
    z = Q.qm_normal_quantile(ud, alg=alg).cpu().numpy()
    ref = (O.normal_breakless_tail(u, form, 64, 86.75) if alg == Q.BREAKLESS_TAIL else O.normal_breakless(u, form, 64))
    e = ulp_errors(z, ref, np.float64)
    zz = -np.log(2 * np.minimum(u, 1 - u))
    worst = float(zz[np.argmax(e)])
    print(json.dumps({"formula": name, "inputs": "deep" if deep else "grid+tail", "n": int(n), "max_ulp": float(e.max()),
                      "z_at_max": worst,
                      "p99999_ulp": float(np.quantile(e, 0.99999)), "mean_ulp": float(e.mean()),
                      "lib": os.environ.get("QM_LIB_PATH", "libqm.so")}), flush=True)
