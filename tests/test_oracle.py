"""The CPU oracle (oracle/port.py) against golden vectors written by the
reference itself (tests/golden/make_golden.py).  Where the reference is
deterministic the port must reproduce it bit for bit."""
import numpy as np
import pytest

from oracle import port


def design(g, k):
    return port.design_from_pattern(int(g[f"c{k}_n"]), int(g[f"c{k}_p"]), g[f"c{k}_rp"], g[f"c{k}_ci"],
                                    intercept=bool(g[f"c{k}_icpt"]))


class TestSparseOracle:
    def test_matvec_bitwise(self, golden):
        g = golden("sparse")
        for k in range(int(g["ncases"])):
            X = design(g, k)
            np.testing.assert_array_equal(port.matvec(X, g[f"c{k}_v"]), g[f"c{k}_Xv"])

    def test_matvec_t_bitwise(self, golden):
        g = golden("sparse")
        for k in range(int(g["ncases"])):
            np.testing.assert_array_equal(port.matvec_t(design(g, k), g[f"c{k}_w"]), g[f"c{k}_Xtw"])

    def test_phi_apply_bitwise(self, golden):
        g = golden("sparse")
        for k in range(int(g["ncases"])):
            got = port.phi_apply(design(g, k), g[f"c{k}_om"], g[f"c{k}_d"], g[f"c{k}_v"])
            np.testing.assert_array_equal(got, g[f"c{k}_phiv"])

    def test_gram_diagonal(self, golden):
        g = golden("sparse")
        for k in range(int(g["ncases"])):
            np.testing.assert_allclose(port.gram_diagonal(design(g, k), g[f"c{k}_om"]), g[f"c{k}_gdiag"],
                                       rtol=1e-14, atol=0)


class TestPcgOracle:
    def setup_method(self):
        pass

    def _problem(self, g):
        X = port.design_from_pattern(int(g["n"]), int(g["p"]), g["rp"], g["ci"])
        apply = lambda v: port.phi_apply(X, g["om"], g["prior"], v)  # noqa: E731
        return X, apply

    @pytest.mark.parametrize("tag,rtol", [("r6", 1e-6), ("r10", 1e-10)])
    def test_solution_trace_coefficients_bitwise(self, golden, tag, rtol):
        g = golden("pcg")
        _, apply = self._problem(g)
        res = port.pcg(apply, g["b"], g["minv"], g["scale"], rtol=rtol)
        assert res.iterations == int(g[f"{tag}_iters"])
        assert res.applies == int(g[f"{tag}_mv"]) == res.iterations + 1
        np.testing.assert_array_equal(res.x, g[f"{tag}_x"])
        np.testing.assert_array_equal(res.trace, g[f"{tag}_trace"])
        np.testing.assert_array_equal(res.alphas, g[f"{tag}_alphas"])
        np.testing.assert_array_equal(res.betas, g[f"{tag}_betas"])

    def test_max_iter_and_warm_start(self, golden):
        g = golden("pcg")
        _, apply = self._problem(g)
        res = port.pcg(apply, g["b"], g["minv"], g["scale"], x0=g["mi_x0"], max_iter=7, rtol=1e-8)
        assert res.termination == str(g["mi_term"]) == "max_iter"
        assert res.iterations == int(g["mi_iters"]) == 7
        np.testing.assert_array_equal(res.x, g["mi_x"])
        np.testing.assert_array_equal(res.betas, g["mi_betas"])

    def test_linear_term_and_rhs_stream_order(self, golden):
        g = golden("pcg")
        X, _ = self._problem(g)
        lin = port.matvec_t(X, g["om"] * ((g["y"] - 0.5) / g["om"]))
        np.testing.assert_array_equal(lin, g["lin"])
        b = port.rhs(X, lin, g["om"], g["prior"], np.random.default_rng(99))
        np.testing.assert_array_equal(b, g["rhs_b"])
        b2 = port.rhs_given_noise(X, lin, g["om"], g["prior"], g["rhs_eta"], g["rhs_delta"])
        np.testing.assert_array_equal(b2, g["rhs_b"])


class TestPolyaGammaOracle:
    def test_draws_bitwise(self, golden):
        g = golden("pg")
        for s in (0, 1, 2):
            np.testing.assert_array_equal(port.pg_batch(g["z"], np.random.default_rng(s)), g[f"draw_{s}"])

    def test_mean(self, golden):
        g = golden("pg")
        np.testing.assert_allclose(port.pg_mean(g["zz"]), g["mean_zz"], rtol=1e-15, atol=0)


class TestGibbsOracle:
    def test_bridge_chain_bitwise(self, golden):
        g = golden("gibbs")
        X = port.design_from_pattern(int(g["n"]), int(g["p"]), g["rp"], g["ci"])
        ch = port.gibbs_bridge(X, g["y"], 30, seed=3, burn_in=10, thin=2, unshrunk_sd=(np.inf,))
        np.testing.assert_array_equal(ch.cg_iters, g["iters"])
        np.testing.assert_array_equal(ch.draws, g["draws"])
        np.testing.assert_array_equal(ch.tau_draws, g["tau_draws"])
        np.testing.assert_array_equal(ch.logdens, g["logdens"])
        np.testing.assert_array_equal(ch.extra["stats_mean"], g["mean"])

    def test_scale_conditionals_bitwise(self, golden):
        g = golden("gibbs")
        bs = g["bs"]
        taus = [port.bridge_tau(bs, 1.0, 1.0, 1.0, np.random.default_rng(s)) for s in range(20)]
        np.testing.assert_array_equal(taus, g["tau_draws_cond"])
        lams = np.stack([port.bridge_lambda(bs, 0.7, np.random.default_rng(s)) for s in range(5)])
        np.testing.assert_array_equal(lams, g["lam_draws_cond"])
