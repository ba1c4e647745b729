import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import gibbs, synth  # noqa: E402
d = synth.config_design(3, seed=0)
y, _ = synth.simulate_outcomes(d, seed=0, rate=0.02)
X = d.matrix()
X.device_store()
for name, cfg in (("bridge", gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,))),
                  ("horseshoe", gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,)))):
    ch = gibbs.DeviceChain(X, y, cfg, 60, seed=1)
    for t in range(1, 11):
        ch.scan(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(11, 61):
        ch.scan(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res = ch.results.view(-1, 8).cpu().numpy()[10:60]
    print(f"{name}: {50 / (ms * 1e-3):.1f} scans/s, mean CG {res[:, 0].mean():.1f}, "
          f"{ms / 50 * 1e3:.0f} us/scan, applies {res[:, 3].sum()}")
