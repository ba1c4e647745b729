import sys
sys.path.insert(0, '/root/repo')
exec(open('/root/repo/tools/sync_times_pcg.py').read().split("names = ")[0])
import numpy as np
W = []
for rr in runs:
    r = rr[:, :8].reshape(148, 4, 2)
    W.append(np.stack([r[:, 1, 0] - r[:, 0, 1], r[:, 2, 0] - r[:, 1, 1]]) / 1e3)
W = np.array(W)  # runs x 2 x 148
for k, nm in enumerate(["csr", "csc"]):
    a = W[:, k, :]
    c = np.corrcoef(a)
    print(nm, "work per CTA, run-to-run correlation:", np.round(c[0, 1:], 2), "spread", np.round(a.max(1) - a.min(1), 1))
    print(nm, "slowest CTAs per run:", [list(np.argsort(-x)[:6]) for x in a[:3]])
a = W[:, 1, :].mean(0)
b = W[:, 0, :].mean(0)
print("csc mean work by CTA quarter:", [round(float(a[i*37:(i+1)*37].mean()), 2) for i in range(4)])
print("csc work by CTA (avg over runs):", " ".join(f"{x:.1f}" for x in a))
print("csr mean work by CTA quarter:", [round(float(b[i*37:(i+1)*37].mean()), 2) for i in range(4)])
