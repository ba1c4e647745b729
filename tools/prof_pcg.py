"""Runs the config-2 PCG solve (ncu target)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth  # noqa: E402

des = synth.config_design(2, seed=0)
X = des.matrix()
st = X.device_store()
dev = st.device
cond = synth.config2_conditioning(des, seed=0)
phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
rng = np.random.default_rng(7)
b = torch.tensor(rng.standard_normal(st.p_total) * 10, device=dev)
mt, stt = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)
for _ in range(2):
    out = pk.cg.pcg_solve_device(phi, b, mt, stt, rtol=1e-6, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else None)
torch.cuda.synchronize()
print("ok", out[4].cpu().numpy())
