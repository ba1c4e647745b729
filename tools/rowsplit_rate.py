"""us per PCG iteration of the fused row-split kernel with G shards hosted by
one grid (config 2), next to the single-design k_pcg."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import parallel, synth  # noqa: E402

d = synth.config_design(2, seed=0)
X = d.matrix()
cond = synth.config2_conditioning(d, seed=0)
phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
dev = phi.store.device
b = torch.tensor(np.random.default_rng(7).standard_normal(d.p + 1) * 10, device=dev)
mt, st = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / int(out[4][3])


print(f"k_pcg: {timed(lambda: pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=100)):.1f} us/iter")
for G in [int(g) for g in sys.argv[1:]] or [1, 2, 4, 8]:
    parts = parallel.row_partition(d.row_ptr, G)
    shards = [parallel.local_rows(X, lo, hi) for lo, hi in parts]
    rs = parallel.RowSplitPCG(shards, device=dev)
    oms = [torch.tensor(cond["omega"][lo:hi], device=dev) for lo, hi in parts]
    us = timed(lambda: rs.solve(oms, phi.device_diag(), mt, st, b, rtol=1e-30, max_iter=100))
    print(f"row split G={G} (one grid): {us:.1f} us/iter")
