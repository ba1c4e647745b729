"""Per chain-iteration time of the batched PCG (csrc/sliced.cu, R chains in one
persistent kernel) against the single-chain k_pcg, config-2 design, every
solve pinned to `--iters` iterations (rtol 0) so the counts are equal.
Prints one JSON line per configuration (tools/ only)."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import batched, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--R", default="1,2,4,8")
ap.add_argument("--profile", action="store_true", help="phase stamps of the batched kernel")
ap.add_argument("--sliced1", action="store_true", help="R = 1 through the sliced batched kernel")
a = ap.parse_args()

d = synth.config_design(2, seed=0)
X = d.matrix()
rng = np.random.default_rng(0)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for R in (int(v) for v in a.R.split(",")):
    om = rng.uniform(0.05, 0.3, (max(R, 1), d.n))
    lam = np.abs(rng.standard_cauchy((max(R, 1), d.p))) + 0.05
    diag = np.concatenate([np.zeros((max(R, 1), 1)), (0.01 * lam) ** -2.0], axis=1)
    minv = 1.0 / np.maximum(diag, 1e-2)
    B = rng.standard_normal((max(R, 1), d.p + 1))
    cfg = pk.CGConfig(rtol=1e-300, max_iter=a.iters)
    if R == 1 and not a.sliced1:
        phi = pk.PrecisionOperator(X, om[0], diag[0])
        M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv[0])
        bt = torch.from_numpy(B[0]).cuda()
        ms = timed(lambda: pk.pcg_solve(phi, bt, M, config=cfg, residual_scale=np.sqrt(minv[0])))
        info = X.device_store().describe()
    else:
        op = batched.BatchedPrecisionOperator(X, om, diag)
        dev = op.dev
        Bc = batched._to_dev_cm(B, dev)
        Mc = batched._to_dev_cm(minv, dev)
        Sc = batched._to_dev_cm(np.sqrt(minv), dev)
        ms = timed(lambda: batched.batched_pcg_device(op, Bc, Mc, Sc, max_iter=a.iters, rtol=1e-300))
        info = op.store.describe()
        if a.profile:
            from paper_1810_12437_b200 import _lib
            buf = torch.zeros(8 * 64, dtype=torch.int64, device=dev)
            _lib.lib().pcgs_batch_debug_profile(buf.data_ptr())
            batched.batched_pcg_device(op, Bc, Mc, Sc, max_iter=a.iters, rtol=1e-300)
            torch.cuda.synchronize()
            _lib.lib().pcgs_batch_debug_profile(None)
            st = buf.cpu().numpy().reshape(64, 8).astype(np.float64)
            rows = st[2:min(a.iters, 60)]
            ph = {name: float(np.mean(rows[:, k + 1] - rows[:, k])) / 1e3
                  for k, name in enumerate(["csr", "combine", "csc", "step", "direction"])}
            ph["iteration"] = float(np.mean(rows[1:, 0] - rows[:-1, 0])) / 1e3
            info["phases_us"] = ph
    per_apply = ms * 1e3 / (a.iters + 1)
    print(json.dumps({"R": R, "iters": a.iters, "ms_per_solve": ms, "us_per_apply": per_apply,
                      "us_per_chain_iteration": per_apply / R, "store": info}), flush=True)
