"""Per-CTA pass work (barrier trace, iteration 10, config 2) grouped by CSC
slab group: is the CSC spread between slab groups or inside them?"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth, _lib  # noqa: E402

des = synth.config_design(2, seed=0)
X = des.matrix()
cond = synth.config2_conditioning(des, seed=0)
phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
dev = phi.store.device
G = phi.store.describe()["grid"]
b = torch.tensor(np.random.default_rng(7).standard_normal(des.p + 1) * 10, device=dev)
mt, st = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)
buf = torch.zeros(16 * G, dtype=torch.int64, device=dev)
L = _lib.lib()
L.pcgs_debug_sync_times(buf.data_ptr())
L.pcgs_debug_option(1, 128)
W = []
for _ in range(6):
    pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=20)
    torch.cuda.synchronize()
    r = buf.cpu().numpy().reshape(G, 16).astype(np.float64)[:, :8].reshape(G, 4, 2)
    W.append(np.stack([r[:, 1, 0] - r[:, 0, 1], r[:, 2, 0] - r[:, 1, 1]]) / 1e3)
L.pcgs_debug_option(1, 0)
W = np.mean(W[1:], axis=0)
# slab of each CTA in the CSC plan: cta_task_ptr -> task slab (read back through the selftest-free path:
# recompute the proportional allocation from the reported slab count is not exposed, so infer from the
# per-CTA work jumps); print the CSC work in CTA order
print("csr:", " ".join(f"{x:.1f}" for x in W[0]))
print("csc:", " ".join(f"{x:.1f}" for x in W[1]))
