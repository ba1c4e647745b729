import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import synth, _lib  # noqa: E402
des = synth.config_design(2, seed=0)
st = des.matrix().device_store()
v = torch.randn(st.p_total, dtype=torch.float64, device=st.device)
for mode in [int(x) for x in sys.argv[1:]]:
    _lib.lib().pcgs_debug_option(1, mode)
    for _ in range(2):
        st.matvec(v)
torch.cuda.synchronize()
print("ok")
