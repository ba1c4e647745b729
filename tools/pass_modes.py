"""Time the standalone passes under debug modes (skip gathers / skip reduce)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import synth, _lib  # noqa: E402

des = synth.config_design(2, seed=0)
X = des.matrix()
st = X.device_store()
dev = st.device
v = torch.randn(st.p_total, dtype=torch.float64, device=dev)
w = torch.randn(des.n, dtype=torch.float64, device=dev)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts), np.min(ts)


for mode in [int(x) for x in sys.argv[1:]] or (0, 1, 2, 3):
    _lib.lib().pcgs_debug_option(1, mode)
    a = timed(lambda: st.matvec(v))
    b = timed(lambda: st.matvec_t(w))
    print(f"mode {mode}: csr {a[0]:.1f}/{a[1]:.1f} us  csc {b[0]:.1f}/{b[1]:.1f} us")
_lib.lib().pcgs_debug_option(1, 0)
