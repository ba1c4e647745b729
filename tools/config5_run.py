"""BASELINE config 5 at full scale on one GPU: n=1,000,000, p=100,000,
log-uniform rates [1e-5, 0.1] (~1.09e9 nonzeros), 1 % positives, horseshoe.
Prints generation/build time, Phi-apply and PCG timing and Gibbs scans/s."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import gibbs, synth  # noqa: E402

t0 = time.time()
d = synth.config_design(5, seed=0)
print(f"design nnz {d.nnz:,} generated in {time.time() - t0:.0f}s", flush=True)
t0 = time.time()
X = d.matrix()
st = X.device_store()
print(f"store built in {time.time() - t0:.0f}s: {st.describe()}", flush=True)
dev = st.device
rng = np.random.default_rng(0)
om = torch.rand(d.n, dtype=torch.float64, device=dev) * 0.2 + 0.05
diag = torch.rand(d.p + 1, dtype=torch.float64, device=dev) * 1e4 + 1.0
v = torch.randn(d.p + 1, dtype=torch.float64, device=dev)
out = torch.empty_like(v)
for _ in range(3):
    st.phi_apply(om, diag, v, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    st.phi_apply(om, diag, v, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
canon = 8 * d.nnz + 8 * (d.n + 1) + 8 * (d.p + 1) + 8 * (3 * d.n + 4 * d.p)
print(f"phi_apply {ms:.2f} ms; canonical {canon / 1e9:.2f} GB -> {canon / ms / 1e6:.0f} GB/s", flush=True)
# a check of Phi v through the transposed identity <X v, w> = <v, X' w>
w = torch.randn(d.n, dtype=torch.float64, device=dev)
a = float(torch.dot(st.matvec(v), w))
b = float(torch.dot(v, st.matvec_t(w)))
print(f"adjoint check rel {abs(a - b) / abs(a):.2e}", flush=True)
y, _ = synth.simulate_outcomes(d, seed=0, rate=0.01)
print(f"positives {y.mean():.4f}", flush=True)
for name, cfg, n_scans in (("bridge", gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,)), 12),
                           ("horseshoe", gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,)), 6)):
    ch = gibbs.DeviceChain(X, y, cfg, n_scans + 2, seed=1, device=dev)
    for t in (1, 2):
        ch.scan(t)
    torch.cuda.synchronize()
    e0.record()
    for t in range(3, n_scans + 3):
        ch.scan(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ch.check(1, n_scans + 2, allow_max_iter=True)
    res = ch.results.view(-1, 8).cpu().numpy()[2:n_scans + 2]
    print(f"config5 {name}: {n_scans / (ms * 1e-3):.2f} scans/s, CG iters {res[:, 0].tolist()}, "
          f"{ms / res[:, 3].sum() * 1e3:.0f} us per PCG iteration (incl. scan overhead)", flush=True)
