"""Config-2 parity probe: for every fixture
seed, the device's iterations to RMS 1e-6, its recursive RMS at the stop, the
TRUE scaled residual of its solution (oracle.port.true_rms: Phi x in long
double) and its relative error vs the reference's RMS-1e-10 solution, next to
the reference's own numbers from tests/golden/config2_parity.npz.
Prints one JSON line per seed (tools/ only; the gate is
tests/test_gpu_parity_config2.py)."""
import json
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
multi = fx["x_1e10"].ndim == 2
for k, seed in enumerate(fx["seeds"]):
    cond, b = inputs(d, Xo, int(seed))
    phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
    row = {"seed": int(seed)}
    for rtol in (1e-6, 1e-8):
        rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=rtol), residual_scale=cond["scale"])
        x = rep.solution
        tr = port.true_rms(Xo, cond["omega"], cond["prior_diag"], b, x, cond["scale"])
        row[f"dev_{rtol:g}"] = {"iters": rep.iterations, "rec_rms": float(rep.rms_precond_residual_trace[-1]),
                                "true_rms": tr}
        if multi or k == 0:
            xs = fx["x_1e10"][k] if multi else fx["x_1e10"]
            row[f"dev_{rtol:g}"]["err"] = float(np.linalg.norm(x - xs) / np.linalg.norm(xs))
    ref_keys = [key for key in fx.files if key.startswith("iters_") and fx[key].ndim == 1]
    row["cpu"] = {key[6:]: int(fx[key][k]) for key in ref_keys}
    for key in ("ref_true_rms", "ref_err"):
        if key in fx.files:
            row[key] = float(fx[key][k])
    print(json.dumps(row), flush=True)
