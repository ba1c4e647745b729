"""Phase profile of the fused batched Gibbs kernel (pcgs_batch_gibbs_run,
csrc/sgibbs.cu) on the bench's config-3 workload, 8 chains: %globaltimer
stamps of CTA 0 after each grid barrier for the first 64 iterations of a
launch, plus the launch's wall time per scan (tools/ only)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1810_12437_b200 import _lib, gibbs, parallel  # noqa: E402
import bench  # noqa: E402

d, y, cfg = bench.workload("horseshoe")
X = d.matrix()
dev = torch.device("cuda", 0)
W, K = 3, int(sys.argv[1]) if len(sys.argv) > 1 else 4
seeds = [parallel.chain_seed(0, c) for c in range(8)]
B = gibbs.BatchedChains(X, y, cfg, W + K + 1, seeds, device=dev, burn_in=W, cg_config=gibbs.CGConfig(rtol=1e-6))
B.run(1, W)
torch.cuda.synchronize()
buf = torch.zeros(8 * 64, dtype=torch.int64, device=dev)
_lib.lib().pcgs_batch_debug_profile(buf.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
B.run(W + 1, W + K)
e1.record()
torch.cuda.synchronize()
_lib.lib().pcgs_batch_debug_profile(None)
ms = e0.elapsed_time(e1)
st = buf.cpu().numpy().reshape(64, 8).astype(np.float64)
rows = st[1:63]
names = ["csr", "combine", "csc", "step", "direction"]
ph = {nm: float(np.mean(rows[:, k + 1] - rows[:, k])) / 1e3 for k, nm in enumerate(names)}
ph["iteration"] = float(np.mean(rows[1:, 0] - rows[:-1, 0])) / 1e3
cg = [int(v) for ch in B.chains for v in ch.results.view(-1, 8).cpu().numpy()[W:W + K, 0]]
iters_est = max(sum(ch.results.view(-1, 8).cpu().numpy()[W:W + K, 0] + 2) for ch in B.chains)
print(json.dumps({"scans": K, "ms": ms, "chain_iter_per_s": 8 * K / (ms * 1e-3), "cg_mean": float(np.mean(cg)),
                  "slowest_chain_iterations": int(iters_est), "us_per_batched_iteration": ms * 1e3 / iters_est,
                  "phases_us_first_64": ph}))
