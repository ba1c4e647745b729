import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import batched, synth  # noqa: E402
d = synth.config_design(2, seed=0)
X = d.matrix()
cond = synth.config2_conditioning(d, seed=0)
for R in [int(x) for x in sys.argv[1:]] or (2, 4, 8):
    om = np.tile(cond["omega"], (R, 1))
    diag = np.tile(cond["prior_diag"], (R, 1))
    minv = np.tile(cond["minv"], (R, 1))
    rng = np.random.default_rng(7)
    B = rng.standard_normal((R, d.p + 1)) * 10
    op = batched.BatchedPrecisionOperator(X, om, diag)
    dev = op.dev
    Bc, Mc, Sc = (batched._to_dev_cm(a, dev) for a in (B, minv, np.sqrt(minv)))
    for _ in range(2):
        out = batched.batched_pcg_device(op, Bc, Mc, Sc, max_iter=60, rtol=1e-30)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = batched.batched_pcg_device(op, Bc, Mc, Sc, max_iter=60, rtol=1e-30)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    applies = int(out[4][0, 3])
    print(f"R={R}: {ms/applies*1e3:.1f} us per batched iteration, {ms/applies/R*1e3:.1f} us per chain-iteration "
          f"(applies {applies}); store {op.store.describe()['csr_slabs']}x{op.store.describe()['csc_slabs']} slabs")
