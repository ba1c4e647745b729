"""Quick GPU parity + timing probe (development tool; not the test suite)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import synth  # noqa: E402
from oracle import port  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def random_pattern(rng, n, p, density):
    mask = rng.random((n, p)) < density
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    ci = np.nonzero(mask)[1].astype(np.int32)
    return rp, ci


def check_small():
    rng = np.random.default_rng(0)
    worst = 0.0
    for trial in range(40):
        n, p = (int(x) for x in rng.integers(1, 300, size=2))
        dens = float(rng.uniform(0.0, 0.9))
        rp, ci = random_pattern(rng, n, p, dens)
        for icpt in (True, False):
            for slab_max in (0, 16, 48):
                X = pk.SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=icpt)
                X.slab_max = slab_max
                Xo = port.design_from_pattern(n, p, rp, ci, intercept=icpt)
                v = rng.standard_normal(X.n_cols)
                w = rng.standard_normal(n)
                om = rng.uniform(0.05, 2.0, size=n)
                d = rng.uniform(0.0, 3.0, size=X.n_cols)
                e1 = rel(X.matvec(v), port.matvec(Xo, v))
                e2 = rel(X.matvec_t(w), port.matvec_t(Xo, w))
                phi = pk.PrecisionOperator(X, om, d)
                e3 = rel(phi.apply(v), port.phi_apply(Xo, om, d, v))
                e4 = rel(X.gram_diagonal(om), port.gram_diagonal(Xo, om))
                worst = max(worst, e1, e2, e3, e4)
                if max(e1, e2, e3, e4) > 1e-12:
                    print("MISMATCH", n, p, dens, icpt, slab_max, e1, e2, e3, e4)
    print(f"small designs: worst rel err {worst:.2e}")


def check_pcg_config1():
    des = synth.config_design(1, seed=0)
    X = des.matrix()
    Xo = port.design_from_pattern(des.n, des.p, des.row_ptr, des.col_idx)
    cond = synth.config2_conditioning(des, seed=0, pg_sampler=port.pg_batch)
    om, d, minv, scale = cond["omega"], cond["prior_diag"], cond["minv"], cond["scale"]
    rng = np.random.default_rng(5)
    lin = port.matvec_t(Xo, cond["kappa"])
    b = port.rhs(Xo, lin, om, d, rng)
    phi = pk.PrecisionOperator(X, om, d)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    for rtol in (1e-6, 1e-10):
        ref = port.pcg(lambda v: port.phi_apply(Xo, om, d, v), b, minv, scale, rtol=rtol)
        rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=rtol), residual_scale=scale)
        print(f"config1 rtol={rtol}: iters gpu {rep.iterations} ref {ref.iterations}; "
              f"relL2 {rel(rep.solution, ref.x):.2e}; matvecs {rep.matvec_count}; "
              f"trace0 {rep.rms_precond_residual_trace[0]:.6e} vs {ref.trace[0]:.6e}")


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(np.min(ts))


def check_config2(run_oracle=False):
    t0 = time.time()
    des = synth.config_design(2, seed=0)
    print(f"config2 design nnz {des.nnz} in {time.time() - t0:.1f}s")
    X = des.matrix()
    t0 = time.time()
    st = X.device_store()
    print(f"store build {time.time() - t0:.1f}s", st.describe())
    cond = synth.config2_conditioning(des, seed=0)
    om, d, minv, scale = cond["omega"], cond["prior_diag"], cond["minv"], cond["scale"]
    dev = st.device
    omt, dt = torch.tensor(om, device=dev), torch.tensor(d, device=dev)
    v = torch.randn(st.p_total, dtype=torch.float64, device=dev)
    out = torch.empty_like(v)
    med, mn = timed(lambda: st.phi_apply(omt, dt, v, out))
    nnz = des.nnz
    canon = 8 * nnz + 8 * (des.n + 1) + 8 * (des.p + 1) + 8 * (3 * des.n + 4 * des.p)
    print(f"phi_apply median {med*1e3:.1f} us min {mn*1e3:.1f} us; canonical {canon/1e6:.1f} MB -> "
          f"{canon / (mn * 1e-3) / 1e9:.0f} GB/s; store idx bytes {st.info[13]/1e6:.1f} MB -> "
          f"{st.info[13] / (mn * 1e-3) / 1e9:.0f} GB/s")
    w = torch.randn(des.n, dtype=torch.float64, device=dev)
    med, mn = timed(lambda: st.matvec(v))
    print(f"matvec median {med*1e3:.1f} us min {mn*1e3:.1f}")
    med, mn = timed(lambda: st.matvec_t(w))
    print(f"matvec_t median {med*1e3:.1f} us min {mn*1e3:.1f}")
    # parity of Phi v against the oracle
    Xo = port.design_from_pattern(des.n, des.p, des.row_ptr, des.col_idx)
    vh = v.cpu().numpy()
    t0 = time.time()
    ref = port.phi_apply(Xo, om, d, vh)
    print(f"phi parity rel {rel(out.cpu().numpy(), ref):.2e} (oracle {time.time()-t0:.2f}s)")
    # PCG
    rng = np.random.default_rng(7)
    lin = port.matvec_t(Xo, cond["kappa"])
    b = port.rhs(Xo, lin, om, d, rng)
    phi = pk.PrecisionOperator(X, om, d)
    bt = torch.tensor(b, device=dev)
    mt, stt = torch.tensor(minv, device=dev), torch.tensor(scale, device=dev)
    from paper_1810_12437_b200 import _lib
    for mode in (0, 1):
        _lib.lib().pcgs_debug_option(0, mode)
        prof = torch.zeros(256, dtype=torch.int64, device=dev)
        _lib.lib().pcgs_debug_profile(prof.data_ptr())
        pk.cg.pcg_solve_device(phi, bt, mt, stt, rtol=1e-6)
        torch.cuda.synchronize()
        _lib.lib().pcgs_debug_profile(None)
        pr = prof.cpu().numpy().reshape(-1, 4).astype(np.float64)
        print(f"  tma_dir={mode}")
        for a in (0, 1, 2, 10, 20):
            t0 = pr[a, 0]
            nxt = pr[a + 1, 0]
            print(f"  apply {a}: A {(pr[a,1]-t0)/1e3:.1f}  syncA+B {(pr[a,2]-pr[a,1])/1e3:.1f}"
                  f"  syncB {(pr[a,3]-pr[a,2])/1e3:.1f}  C+syncC+dir {(nxt-pr[a,3])/1e3:.1f}  total {(nxt-t0)/1e3:.1f} us")
        res = {}

        def solve():
            res["o"] = pk.cg.pcg_solve_device(phi, bt, mt, stt, rtol=1e-6)
        med, mn = timed(solve, reps=5, warm=1)
        r = res["o"][4].cpu().numpy()
        print(f"  tma_dir={mode} PCG iters {r[0]} time {med:.2f} ms ({med / max(r[3],1) * 1e3:.1f} us/iter)")
    for rtol in (1e-6, 1e-10):
        res = {}

        def solve():
            res["o"] = pk.cg.pcg_solve_device(phi, bt, mt, stt, rtol=rtol)
        med, mn = timed(solve, reps=5, warm=1)
        r = res["o"][4].cpu().numpy()
        iters = int(r[0])
        print(f"config2 PCG rtol={rtol}: iters {iters} status {r[1]} applies {r[3]} "
              f"time {med:.2f} ms ({med / max(r[3],1) * 1e3:.1f} us/iter)")
        x = res["o"][0].cpu().numpy()
        resid = b - port.phi_apply(Xo, om, d, x)
        print(f"   true rms scaled residual {np.sqrt(np.mean((scale*resid)**2)):.3e}; "
              f"trace end {res['o'][1][iters].item():.3e}")
        if run_oracle:
            t0 = time.time()
            ref = port.pcg(lambda vv: port.phi_apply(Xo, om, d, vv), b, minv, scale, rtol=rtol)
            print(f"   oracle iters {ref.iterations} ({time.time()-t0:.1f}s) relL2 {rel(x, ref.x):.2e}")


if __name__ == "__main__":
    check_small()
    check_pcg_config1()
    check_config2(run_oracle="--oracle" in sys.argv)
