"""Device vs CPU-oracle PCG sequences (alpha, beta, RMS trace) at config 2,
seed 0 of the parity recipe: where do they part?"""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth  # noqa: E402
from oracle import port  # noqa: E402
from test_gpu_parity_config2 import inputs  # noqa: E402

ref = np.load(ROOT / "tools" / "data" / "seq_seed0.npz")
d = synth.config_design(2, seed=0)
X, Xo = d.matrix(), port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
cond, b = inputs(d, Xo, 0)
phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-6), residual_scale=cond["scale"])
ra, rb, rt = ref["alphas"], ref["betas"], ref["trace"]
n = min(len(ra), len(rep.alphas))
da = np.abs(rep.alphas[:n] / ra[:n] - 1)
db = np.abs(rep.betas[:min(len(rb), len(rep.betas))] / rb[:min(len(rb), len(rep.betas))] - 1)
dt = np.abs(rep.rms_precond_residual_trace[:n + 1] / rt[:n + 1] - 1)
for k in [0, 1, 2, 3, 5, 10, 20, 40, 60, 80, 100, 120, 150, 180]:
    if k < n:
        print(f"k={k:3d} rel alpha {da[k]:.2e} beta {db[k] if k < len(db) else float('nan'):.2e} "
              f"trace {dt[k]:.2e}  dev trace {rep.rms_precond_residual_trace[k]:.3e} ref {rt[k]:.3e}")
print("iterations device", rep.iterations, "cpu", int(ref["iters"]))
# one Phi-apply of the same vector on both sides
v = np.random.default_rng(3).standard_normal(d.p + 1)
a1 = phi.apply(v); a2 = port.phi_apply(Xo, cond["omega"], cond["prior_diag"], v)
print("Phi v rel diff", np.linalg.norm(a1 - a2) / np.linalg.norm(a2))
