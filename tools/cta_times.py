import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import synth, _lib  # noqa: E402
des = synth.config_design(2, seed=0)
st = des.matrix().device_store()
v = torch.randn(st.p_total, dtype=torch.float64, device=st.device)
w = torch.randn(des.n, dtype=torch.float64, device=st.device)
buf = torch.zeros(3 * 148, dtype=torch.int64, device=st.device)
_lib.lib().pcgs_debug_cta_times(buf.data_ptr())
for mode in [int(x) for x in sys.argv[1:]]:
    _lib.lib().pcgs_debug_option(1, mode | 64)
    for name, fn in (("csr", lambda: st.matvec(v)), ("csc", lambda: st.matvec_t(w))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t = buf.cpu().numpy().reshape(-1, 3).astype(np.float64)
        t0 = t[:, 0].min()
        start, filled, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
        print(f"mode {mode} {name}: start max {start.max():.1f}us fill {np.median(filled-start):.1f}us "
              f"end min {end.min():.1f} med {np.median(end):.1f} p90 {np.percentile(end,90):.1f} max {end.max():.1f}")
        print("   slowest CTAs", np.argsort(-end)[:8], "fastest", np.argsort(end)[:8])
_lib.lib().pcgs_debug_option(1, 0)
if len(sys.argv) > 1 and sys.argv[1] == "0":
    # end-time profile along the CTA index (CTAs are assigned to slabs in order)
    _lib.lib().pcgs_debug_option(1, 64)
    for name, fn in (("csr", lambda: st.matvec(v)), ("csc", lambda: st.matvec_t(w))):
        ends = []
        for _ in range(5):
            fn()
            torch.cuda.synchronize()
            t = buf.cpu().numpy().reshape(-1, 3).astype(np.float64)
            ends.append((t[:, 2] - t[:, 0].min()) / 1e3)
        e = np.median(np.array(ends), axis=0)
        print(name, "end by CTA group of 8:", " ".join(f"{x:.0f}" for x in e.reshape(-1, 4).mean(1)[:37]))
    _lib.lib().pcgs_debug_option(1, 0)
