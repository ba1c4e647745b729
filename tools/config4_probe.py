"""Chains side by side vs one after another, full horseshoe scans at config 3:
(a) the normal stopping rule, (b) every solve pinned to 100 iterations (the
chains' solves then have equal lengths, as in tools/concurrent_chains.py)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import gibbs, parallel, synth  # noqa: E402

d = synth.config_design(3, seed=0)
y, _ = synth.simulate_outcomes(d, seed=0, n_signal=10, rate=0.02)
X = d.matrix()
cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))
dev = torch.device("cuda", 0)
W, K = 3, 8


def run(R, cgc):
    grid = 0 if R == 1 else 148 // R
    total, its = 0.0, 0
    for w0 in range(0, 8, R):
        streams = [torch.cuda.Stream(dev) for _ in range(R)]
        chains = []
        for c, s in zip(range(w0, w0 + R), streams):
            with torch.cuda.stream(s):
                chains.append(gibbs.DeviceChain(X, y, cfg, W + K, burn_in=W, seed=parallel.chain_seed(0, c),
                                                cg_config=cgc, device=dev, grid=grid))
        for t in range(1, W + 1):
            for ch, s in zip(chains, streams):
                with torch.cuda.stream(s):
                    ch.scan(t)
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for s in streams:
            s.wait_stream(cur)
        import time
        h0 = time.perf_counter()
        for t in range(W + 1, W + K + 1):
            for ch, s in zip(chains, streams):
                with torch.cuda.stream(s):
                    ch.scan(t)
        for s in streams:
            cur.wait_stream(s)
        e1.record(cur)
        host = time.perf_counter() - h0
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
        print(f"   R={R} wave {w0}: host issue {host * 1e3:.1f} ms, GPU {e0.elapsed_time(e1):.1f} ms", flush=True)
        for ch in chains:
            its += int(ch.results.view(-1, 8).cpu().numpy()[W:W + K, 3].sum())
    return 8 * K / (total * 1e-3), total * 1e3 / its


for name, cgc in (("rtol 1e-6", gibbs.CGConfig(rtol=1e-6)), ("100 iterations", gibbs.CGConfig(rtol=1e-30, max_iter=100))):
    for R in (1, 4):
        rate, us = run(R, cgc)
        print(f"{name}, R={R}: {rate:.1f} chain-scans/s, {us:.1f} us per Phi-apply (all kernels of the scan)", flush=True)
