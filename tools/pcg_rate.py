import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth, _lib  # noqa: E402
d = synth.config_design(2, seed=0)
X = d.matrix()
cond = synth.config2_conditioning(d, seed=0)
phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
dev = phi.store.device
b = torch.tensor(np.random.default_rng(7).standard_normal(d.p + 1) * 10, device=dev)
mt, st = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)
for mode in [int(x) for x in sys.argv[1:]] or [0]:
    _lib.lib().pcgs_debug_option(1, mode)
    phi.store.matvec(torch.zeros(d.p + 1, dtype=torch.float64, device=dev))
    for _ in range(2):
        out = pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=100)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = pk.cg.pcg_solve_device(phi, b, mt, st, rtol=1e-30, max_iter=100)
    e1.record()
    torch.cuda.synchronize()
    print(f"mode {mode}: {e0.elapsed_time(e1) / int(out[4][3]) * 1e3:.1f} us/iter")
_lib.lib().pcgs_debug_option(1, 0)
