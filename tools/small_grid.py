"""Config 1 (n=2,000, p=500): Gibbs scans/s and PCG us/iteration vs the CTA
count the store is planned for (small designs are latency-bound; tools/ only)."""
import json
import math
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1810_12437_b200 import gibbs, synth  # noqa: E402

d = synth.config_design(int(sys.argv[1]) if len(sys.argv) > 1 else 1, seed=0)
y, _ = synth.simulate_outcomes(d, seed=0, n_signal=10)
X = d.matrix()
cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(math.inf,))
for G in (4, 8, 16, 32, 74, 148):
    ch = gibbs.DeviceChain(X, y, cfg, 205, burn_in=5, seed=0, cg_config=gibbs.CGConfig(rtol=1e-6), grid=G)
    for t in range(1, 6):
        ch.scan(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(6, 206):
        ch.scan(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    cg = ch.results.view(-1, 8).cpu().numpy()[5:205, 0]
    print(json.dumps({"grid": G, "scans_per_s": 200 / (ms * 1e-3), "ms_per_scan": ms / 200,
                      "cg_mean": float(cg.mean()), "us_per_cg_iter_incl_scan": ms * 1e3 / 200 / (cg.mean() + 1)}))
