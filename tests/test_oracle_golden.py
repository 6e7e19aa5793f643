"""The CPU oracle reproduces the reference's own outputs (golden fixtures from tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import blockstat_oracle as orc


def _names(golden, prefix):
    return sorted({k[len(prefix):].rsplit("_", 1)[0] for k in golden if k.startswith(prefix) and k.endswith("_meta")})


@pytest.mark.parametrize("seed", [1, 7, 4242])
def test_philox_raw_words(golden, seed):
    np.testing.assert_array_equal(orc.philox_raw(seed, 16), golden[f"philox_raw_{seed}"])


@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
@pytest.mark.parametrize("p", [1, 3])
def test_rand_fill_common_init(golden, tag, dt, p):
    want = golden[f"rand_fill_{tag}_p{p}"]
    np.testing.assert_array_equal(orc.rand_fill_common((5, 7), 3, dt), want)
    flat = orc.philox_uniform(3, 35, dt)
    np.testing.assert_array_equal(flat.reshape((5, 7), order="F"), want)


def test_nmf_matches_reference(golden):
    names = _names(golden, "nmf_")
    assert len(names) == 6
    for name in names:
        m, n, r, seed, iters, algo, p = golden[f"nmf_{name}_meta"]
        x = golden[f"nmf_{name}_x"]
        np.testing.assert_array_equal(x, orc.rand_fill_common((m, n), seed, x.dtype))
        vt0, w0 = orc.nmf_init(x, r, seed + 1)
        np.testing.assert_array_equal(vt0, golden[f"nmf_{name}_vt0"])
        np.testing.assert_array_equal(w0, golden[f"nmf_{name}_w0"])
        fn = orc.nmf_multiplicative if algo == 0 else orc.nmf_apg
        vt, w, tr = fn(x, vt0, w0, iters)
        tol = 1e-9 if x.dtype == np.float64 else 2e-5
        np.testing.assert_allclose(tr, golden[f"nmf_{name}_trace"], rtol=tol, err_msg=name)
        np.testing.assert_allclose(vt, golden[f"nmf_{name}_vt"], rtol=tol * 10, atol=tol, err_msg=name)
        np.testing.assert_allclose(w, golden[f"nmf_{name}_w"], rtol=tol * 10, atol=tol, err_msg=name)


def test_mds_matches_reference(golden):
    names = _names(golden, "mds_")
    assert len(names) == 3
    for name in names:
        d, n, q, seed, iters, p = golden[f"mds_{name}_meta"]
        x = golden[f"mds_{name}_x"]
        np.testing.assert_array_equal(x, orc.rand_fill_common((d, n), seed, x.dtype))
        y = orc.pairwise_euclidean(x)
        tol = 1e-12 if x.dtype == np.float64 else 1e-6
        np.testing.assert_allclose(y, golden[f"mds_{name}_y"], rtol=tol, atol=tol)
        th0 = orc.mds_init(golden[f"mds_{name}_y"], q, seed + 1)
        np.testing.assert_array_equal(th0, golden[f"mds_{name}_theta0"])
        th, tr = orc.mds_fit(golden[f"mds_{name}_y"], th0, iters)
        tol = 1e-9 if x.dtype == np.float64 else 1e-4
        np.testing.assert_allclose(tr, golden[f"mds_{name}_trace"], rtol=tol, err_msg=name)
        np.testing.assert_allclose(th, golden[f"mds_{name}_theta"], rtol=tol, atol=tol, err_msg=name)


@pytest.mark.parametrize("name", ["m40_n12_lam01", "m40_n12_powersigma", "m40_n12_f32", "m40_n12_breslow"])
def test_cox_matches_reference(golden, name):
    x = golden[f"cox_{name}_x"]
    y = golden[f"cox_{name}_y"]
    delta = golden[f"cox_{name}_delta"].astype(x.dtype)
    lam, sigma, iters, breslow, p = golden[f"cox_{name}_meta"]
    cuts = orc.tie_cuts(y) if breslow else np.arange(len(y))
    if sigma < 0:
        norm = orc.opnorm_l2_power(x)
        sigma = 1.0 / (2.0 * norm * norm)
    np.testing.assert_allclose(sigma, golden[f"cox_{name}_sigma"][0], rtol=1e-12)
    clamp = 700.0 if x.dtype == np.float64 else 85.0
    beta, grad, tr = orc.cox_fit(x, delta, cuts, lam, sigma, int(iters), clamp=clamp)
    tol = 1e-10 if x.dtype == np.float64 else 1e-4
    np.testing.assert_allclose(tr, golden[f"cox_{name}_trace"], rtol=tol)
    np.testing.assert_allclose(beta, golden[f"cox_{name}_beta"], rtol=tol * 10, atol=tol)
    np.testing.assert_allclose(grad, golden[f"cox_{name}_grad"], rtol=tol * 10, atol=tol)


@pytest.mark.parametrize("p", [1, 3])
def test_pi_delta_partials_sum_to_reference(golden, p):
    w, W, d, cuts = golden["pid_w"], golden["pid_W"], golden["pid_delta"], golden["pid_cuts"]
    b = orc.partition_of(23, p)
    total = sum(orc.pi_delta(w, W, d, b[r], b[r + 1], cuts) for r in range(p))
    np.testing.assert_allclose(total, golden[f"pid_out_p{p}"], rtol=1e-13, atol=1e-15)


def test_opnorm_power_iteration(golden):
    np.testing.assert_allclose(orc.opnorm_l2_power(golden["opnorm_a"]), golden["opnorm_l2"][0], rtol=1e-13)


def test_partition_of():
    assert orc.partition_of(7, 4) == (0, 2, 4, 6, 7)
    assert orc.partition_of(2, 4) == (0, 1, 2, 2, 2)
