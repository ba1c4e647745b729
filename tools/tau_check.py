import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1810_12437_b200 import gibbs, synth  # noqa: E402
from oracle import port  # noqa: E402
des = synth.config_design(1, seed=0)
y, truth = synth.simulate_outcomes(des, seed=0, n_signal=10, rate=None)
X = des.matrix()
Xo = port.design_from_pattern(des.n, des.p, des.row_ptr, des.col_idx)
cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))
n, burn = 4000, 1000
g = [gibbs.gibbs_run(X, y, cfg, n, burn_in=burn, seed=100 + k) for k in range(8)]
gt = np.array([o.tau_draws.mean() for o in g])
print("gpu tau chain means", np.round(gt, 5), "mean", gt.mean(), "se", gt.std(ddof=1) / np.sqrt(len(gt)))
t0 = time.time()
c = [port.gibbs_horseshoe(Xo, y, n, seed=200 + k, burn_in=burn, unshrunk_sd=(np.inf,)) for k in range(4)]
ct = np.array([o.tau_draws.mean() for o in c])
print("cpu tau chain means", np.round(ct, 5), "mean", ct.mean(), "se", ct.std(ddof=1) / np.sqrt(len(ct)), time.time() - t0)
gl = np.array([o.logdensity_trace[burn:].mean() for o in g]); cl = np.array([o.logdens[burn:].mean() for o in c])
print("logdens gpu", gl.mean(), gl.std(ddof=1)/np.sqrt(8), "cpu", cl.mean(), cl.std(ddof=1)/2)
