"""Per-CTA phases of the standalone CSR / CSC passes at config 2 (debug option
key 1 bit 64: globaltimer stamps at pass start, after the slab fill and at the
end): median fill and streaming times over the CTAs, and the event-timed
kernel (tools/ only)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import synth, _lib  # noqa: E402

des = synth.config_design(int(sys.argv[1]) if len(sys.argv) > 1 else 2, seed=0)
X = des.matrix()
st = X.device_store()
dev = st.device
v = torch.randn(st.p_total, dtype=torch.float64, device=dev)
w = torch.randn(des.n, dtype=torch.float64, device=dev)
buf = torch.zeros(3 * 148, dtype=torch.int64, device=dev)
L = _lib.lib()
L.pcgs_debug_cta_times(buf.data_ptr())
for name, fn in (("csr", lambda: st.matvec(v)), ("csc", lambda: st.matvec_t(w))):
    L.pcgs_debug_option(1, 0)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    L.pcgs_debug_option(1, 64)
    rows = []
    for _ in range(5):
        fn()
        torch.cuda.synchronize()
        t = buf.cpu().numpy().reshape(148, 3).astype(np.float64) / 1e3
        rows.append((np.median(t[:, 1] - t[:, 0]), np.median(t[:, 2] - t[:, 1]), (t[:, 2] - t[:, 1]).min(),
                     (t[:, 2] - t[:, 1]).max(), t[:, 2].max() - t[:, 0].min()))
    r = np.median(np.array(rows), axis=0)
    print(f"{name}: call {np.median(ts):.1f} us (min {np.min(ts):.1f}) | fill {r[0]:.2f} | stream med {r[1]:.2f} "
          f"min {r[2]:.2f} max {r[3]:.2f} | first start -> last end {r[4]:.2f}")
L.pcgs_debug_option(1, 0)
