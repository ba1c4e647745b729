"""Config-2 parity report vs the reference fixture (tests/golden/config2_parity.npz):
device iterations at RMS 1e-6 per seed next to the reference's and its
split-summation floor, and the relative L2 at RMS 1e-10 (seed 0)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth  # noqa: E402
from oracle import port  # noqa: E402
from test_gpu_parity_config2 import inputs, FIX  # noqa: E402

d = synth.config_design(2, seed=0)
X, Xo = d.matrix(), port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
fx = np.load(FIX)
for k, seed in enumerate(fx["seeds"]):
    cond, b = inputs(d, Xo, int(seed))
    phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
    rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-6), residual_scale=cond["scale"])
    tr = rep.rms_precond_residual_trace
    print(f"seed {seed}: device {rep.iterations} reference {int(fx['iters_ref'][k])} split {int(fx['iters_split'][k])}"
          f" extended precision {int(fx['iters_accurate'][k])}"
          f" | device RMS trace last 4: {np.array2string(tr[-4:], precision=2)}", flush=True)
    if k == 0:
        tight = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=cond["scale"])
        x = fx["x_1e10"]
        print(f"seed 0 RMS 1e-10: relative L2 {np.linalg.norm(tight.solution - x) / np.linalg.norm(x):.2e}, "
              f"iterations {tight.iterations} vs {int(fx['iters_1e10'])}", flush=True)
