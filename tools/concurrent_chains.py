"""Config 2 PCG: R independent solves run concurrently on R streams, each on a
store planned for 148/R CTAs, vs the same R solves one after another on the
full-grid store (aggregate chain-iterations per second)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth  # noqa: E402

d = synth.config_design(2, seed=0)
cond = synth.config2_conditioning(d, seed=0)
dev = torch.device("cuda", 0)
mt, st = torch.tensor(cond["minv"], device=dev), torch.tensor(cond["scale"], device=dev)
ITER = 100


class Op:  # the operator view pcg_solve_device needs, on a store of a chosen grid
    def __init__(self, store, omega, diag):
        self.store, self._om, self._dg = store, omega, diag

    def device_omega(self):
        return self._om

    def device_diag(self):
        return self._dg


def run(R, grid, stagger_us=0.0):
    X = d.matrix()
    store = X.device_store(dev, grid=grid)
    om = torch.tensor(cond["omega"], device=dev)
    dg = torch.tensor(cond["prior_diag"], device=dev)
    phis = [Op(store, om.clone(), dg.clone()) for _ in range(R)]
    bs = [torch.tensor(np.random.default_rng(7 + c).standard_normal(d.p + 1) * 10, device=dev) for c in range(R)]
    streams = [torch.cuda.Stream(dev) for _ in range(R)]

    def once():
        outs = []
        for c in range(R):
            with torch.cuda.stream(streams[c] if grid else torch.cuda.current_stream(dev)):
                if stagger_us and grid:
                    torch.cuda._sleep(int(c * stagger_us * 1965))   # ~cycles at 1.965 GHz
                outs.append(pk.cg.pcg_solve_device(phis[c], bs[c], mt, st, rtol=1e-30, max_iter=ITER))
        return outs
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_stream(torch.cuda.current_stream(dev))
    outs = once()
    for s in streams:
        torch.cuda.current_stream(dev).wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    its = sum(int(o[4][3]) for o in outs)
    return e0.elapsed_time(e1) * 1e3 / its


print(f"sequential, full grid: {run(2, 0):.1f} us per chain-iteration")
for R in (2, 3, 4, 6, 8):
    print(f"{R} concurrent chains on {148 // R}-CTA stores: {run(R, 148 // R):.1f} us per chain-iteration")
# the same 4 solves with chain c started c x 45 us (about one pass of L2 residency) later
print(f"4 chains, staggered starts: {run(4, 37, 45.0):.1f} us per chain-iteration (incl. the stagger)")
