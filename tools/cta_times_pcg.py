"""Per-CTA [start, filled, end] of the last CSC pass inside the persistent
PCG kernel at config 2 (debug option bit 64)."""
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
buf = torch.zeros(3 * 148, dtype=torch.int64, device=dev)
_lib.lib().pcgs_debug_cta_times(buf.data_ptr())
_lib.lib().pcgs_debug_option(1, 64)
ends, fills, starts = [], [], []
for it in (20, 21, 22, 23, 24):
    pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=it)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(-1, 3).astype(np.float64)
    t0 = t[:, 0].min()
    starts.append((t[:, 0] - t0) / 1e3)
    fills.append((t[:, 1] - t[:, 0]) / 1e3)
    ends.append((t[:, 2] - t0) / 1e3)
_lib.lib().pcgs_debug_option(1, 0)
s, f, e = (np.median(np.array(x), axis=0) for x in (starts, fills, ends))
print(f"start spread {s.max():.1f} us, fill median {np.median(f):.1f} max {f.max():.1f}, "
      f"end min {e.min():.1f} med {np.median(e):.1f} max {e.max():.1f}")
print("end by CTA group of 4:", " ".join(f"{x:.0f}" for x in e.reshape(-1, 4).mean(1)))
print("fill by CTA group of 4:", " ".join(f"{x:.1f}" for x in f.reshape(-1, 4).mean(1)))
info = phi.store.describe()
print(info)
