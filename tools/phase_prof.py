"""Per-phase timeline of the persistent PCG kernel at config 2 (globaltimer
stamps of CTA 0, pcgs_debug_profile): A = CSR pass, B = CSC pass (+ the grid
sync after A), syncB, C = assembly/step/convergence + direction update."""
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
b = torch.tensor(np.random.default_rng(7).standard_normal(des.p + 1) * 10, device=dev)
mt, st = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)
pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=70)
prof = torch.zeros(4 * 64, dtype=torch.int64, device=dev)
_lib.lib().pcgs_debug_profile(prof.data_ptr())
pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=70)
torch.cuda.synchronize()
_lib.lib().pcgs_debug_profile(None)
pr = prof.cpu().numpy().reshape(-1, 4).astype(np.float64) / 1e3
sel = range(5, 60)
A = np.mean([pr[a, 1] - pr[a, 0] for a in sel])
B = np.mean([pr[a, 2] - pr[a, 1] for a in sel])
S = np.mean([pr[a, 3] - pr[a, 2] for a in sel])
C = np.mean([pr[a + 1, 0] - pr[a, 3] for a in sel])
print(f"A(csr) {A:.1f}  syncA+B(csc) {B:.1f}  syncB {S:.1f}  C+sync+dir {C:.1f}  total {A+B+S+C:.1f} us")
