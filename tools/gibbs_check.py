"""Quick GPU Gibbs check: device chains vs the CPU oracle (development tool)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import gibbs, synth  # noqa: E402
from oracle import port  # noqa: E402


def batch_se(x, nb=20):
    n = (len(x) // nb) * nb
    m = x[:n].reshape(nb, -1).mean(1)
    return m.std(ddof=1) / np.sqrt(nb)


def compare(name, a, b):
    ma, mb = a.mean(0), b.mean(0)
    se = np.sqrt(np.array([batch_se(a[:, j]) ** 2 + batch_se(b[:, j]) ** 2 for j in range(a.shape[1])]))
    z = (ma - mb) / np.maximum(se, 1e-12)
    big = np.argsort(-np.abs(ma))[:8]
    print(f"{name}: |z| mean {np.mean(np.abs(z)):.2f} max {np.max(np.abs(z)):.2f} "
          f"frac|z|>3 {np.mean(np.abs(z) > 3):.3f}")
    for j in big:
        print(f"   j={j:4d} gpu {ma[j]: .4f} cpu {mb[j]: .4f} z {z[j]: .2f}")


def main():
    des = synth.config_design(1, seed=0)
    y, truth = synth.simulate_outcomes(des, seed=0, n_signal=10, rate=None)
    X = des.matrix()
    Xo = port.design_from_pattern(des.n, des.p, des.row_ptr, des.col_idx)
    n_iter, burn = 3000, 500
    for prior in ("bridge", "horseshoe"):
        t0 = time.time()
        if prior == "bridge":
            cfg = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,))
            out = gibbs.gibbs_run(X, y, cfg, n_iter, burn_in=burn, seed=1)
        else:
            cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))
            out = gibbs.gibbs_run(X, y, cfg, n_iter, burn_in=burn, seed=1)
        torch.cuda.synchronize()
        tg = time.time() - t0
        t0 = time.time()
        if prior == "bridge":
            ref = port.gibbs_bridge(Xo, y, n_iter, seed=2, burn_in=burn, unshrunk_sd=(np.inf,))
        else:
            ref = port.gibbs_horseshoe(Xo, y, n_iter, seed=2, burn_in=burn, unshrunk_sd=(np.inf,))
        tc = time.time() - t0
        print(f"[{prior}] gpu {n_iter/tg:.0f} iter/s, cpu {n_iter/tc:.0f} iter/s; "
              f"cg iters gpu mean {out.cg_iteration_counts.mean():.1f} cpu {ref.cg_iters.mean():.1f}; "
              f"logdens gpu {out.logdensity_trace[burn:].mean():.2f} cpu {ref.logdens[burn:].mean():.2f}; "
              f"tau gpu {out.tau_draws.mean():.4g} cpu {ref.tau_draws.mean():.4g}")
        compare(f"[{prior}] beta mean", out.draws, ref.draws)
        compare(f"[{prior}] beta^2 mean", out.draws ** 2, ref.draws ** 2)
        print("   truth nonzeros:", np.flatnonzero(truth)[:12])

    # paper scale timing (config 3 design, horseshoe, rare outcome)
    t0 = time.time()
    des3 = synth.config_design(3, seed=0)
    y3, _ = synth.simulate_outcomes(des3, seed=0, n_signal=10, rate=0.02)
    X3 = des3.matrix()
    X3.device_store()
    print(f"config3 setup {time.time()-t0:.1f}s, positives {y3.mean():.4f}")
    for prior, cfg in (("horseshoe", gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))),
                       ("bridge", gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,)))):
        n3 = 60
        gibbs.gibbs_run(X3, y3, cfg, 3, seed=3)
        torch.cuda.synchronize()
        t0 = time.time()
        out3 = gibbs.gibbs_run(X3, y3, cfg, n3, seed=3)
        torch.cuda.synchronize()
        dt = time.time() - t0
        print(f"config3 {prior}: {n3/dt:.1f} iter/s; cg iters {out3.cg_iteration_counts.tolist()[:12]} ... "
              f"{out3.cg_iteration_counts[-10:].tolist()}; mean {out3.cg_iteration_counts.mean():.1f}")


if __name__ == "__main__":
    main()
