"""Arrival / departure of every CTA at the four grid barriers of PCG
iteration 10 (config 2, or `python tools/sync_times_pcg.py 1` for config 1):
how much of each phase is load imbalance vs barrier."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth, _lib  # noqa: E402

des = synth.config_design(int(sys.argv[1]) if len(sys.argv) > 1 else 2, seed=0)
X = des.matrix()
cond = synth.config2_conditioning(des, seed=0)
phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
dev = phi.store.device
b = torch.tensor(np.random.default_rng(7).standard_normal(des.p + 1) * 10, device=dev)
mt, st = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)
buf = torch.zeros(16 * 148, dtype=torch.int64, device=dev)
_lib.lib().pcgs_debug_sync_times(buf.data_ptr())
_lib.lib().pcgs_debug_option(1, 128)
runs = []
for _ in range(5):
    pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=20)
    torch.cuda.synchronize()
    runs.append(buf.cpu().numpy().reshape(148, 16).astype(np.float64))
_lib.lib().pcgs_debug_option(1, 0)
names = ["dir", "csr", "csc", "stepC"]
for rr in runs[2:]:
    r = rr[:, :8].reshape(148, 4, 2)
    c = rr[:, 8:13]
    dep2 = r[:, 2, 1]
    print("phase C stamps after sync2 (median us): stage-start %.2f staged %.2f dAd %.2f loop %.2f sum %.2f" %
          tuple(np.median(c[:, k] - dep2) / 1e3 for k in range(5)))
    t0 = r[:, 0, 1].max()   # everyone left barrier 0 (start of the CSR pass)
    line = []
    prev_dep = r[:, 0, 1]
    for k in (1, 2, 3):
        arr, dep = r[:, k, 0], r[:, k, 1]
        work = arr - prev_dep
        line.append(f"{names[k]}: work min {work.min()/1e3:.1f} med {np.median(work)/1e3:.1f} max {work.max()/1e3:.1f}"
                    f" | last arrival->first departure {(dep.min() - arr.max())/1e3:.2f} | departure spread {(dep.max()-dep.min())/1e3:.2f}")
        prev_dep = dep
    print("\n".join(line))
    print("---")
