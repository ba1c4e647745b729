"""Runs the config-2 standalone passes a few times (ncu target)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import synth  # noqa: E402

des = synth.config_design(2, seed=0)
X = des.matrix()
st = X.device_store()
dev = st.device
v = torch.randn(st.p_total, dtype=torch.float64, device=dev)
w = torch.randn(des.n, dtype=torch.float64, device=dev)
om = torch.rand(des.n, dtype=torch.float64, device=dev)
d = torch.rand(st.p_total, dtype=torch.float64, device=dev)
for _ in range(3):
    st.matvec(v)
    st.matvec_t(w)
    st.phi_apply(om, d, v)
torch.cuda.synchronize()
print("ok")
