"""Generates the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is importable from
/root/reference/pkg/src; it does not exist on the GPU box):

    python tests/golden/make_golden.py

Each case runs blockstat's own public API (inproc backend, several rank
counts) on seeded inputs and stores inputs + outputs in ``golden.npz``.  The
fixtures pin the oracle (tests/test_oracle_golden.py) and the CUDA path
(tests/test_*_gpu.py).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"


def main():
    sys.path.insert(0, str(REF))
    import blockstat as bs  # the reference implementation

    g = {}

    # -- Philox / rand_fill (distarray.py:170-208) ---------------------------------
    for seed in (1, 7, 4242):
        g[f"philox_raw_{seed}"] = np.random.Philox(seed).random_raw(16)
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        for p in (1, 3):
            def fill(comm, dt=dt):
                a = bs.empty((5, 7), comm, dt)
                bs.rand_fill(a, seed=3, common_init=True)
                return bs.gather_full(a)
            g[f"rand_fill_{tag}_p{p}"] = bs.run_inproc(p, fill)[0]

    # -- NMF (solvers.py:97-185) ---------------------------------------------------
    def nmf_case(comm, m, n, r, seed, iters, algo, dt):
        x = bs.empty((m, n), comm, dt)
        bs.rand_fill(x, seed=seed, common_init=True)
        st = bs.nmf_init(x, r, seed=seed + 1)
        vt0, w0 = bs.gather_full(st.Vt), bs.gather_full(st.W)
        (bs.nmf_multiplicative if algo == "mu" else bs.nmf_apg)(st, iters)
        return bs.gather_full(x), vt0, w0, np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)

    nmf_cases = [
        ("mu_16x16_r2", 16, 16, 2, 5000, 60, "mu", np.float64, 2),
        ("apg_16x16_r4", 16, 16, 4, 5017, 60, "apg", np.float64, 1),
        ("mu_60x44_r6", 60, 44, 6, 77, 40, "mu", np.float64, 3),
        ("apg_60x44_r6", 60, 44, 6, 78, 40, "apg", np.float64, 3),
        ("mu_50x30_r5_f32", 50, 30, 5, 91, 30, "mu", np.float32, 1),
        ("apg_50x30_r5_f32", 50, 30, 5, 92, 30, "apg", np.float32, 2),
    ]
    for name, m, n, r, seed, iters, algo, dt, p in nmf_cases:
        x, vt0, w0, tr, vt, w = bs.run_inproc(p, nmf_case, m, n, r, seed, iters, algo, dt)[0]
        g[f"nmf_{name}_meta"] = np.array([m, n, r, seed, iters, 0 if algo == "mu" else 1, p], dtype=np.int64)
        g[f"nmf_{name}_x"] = x
        g[f"nmf_{name}_vt0"] = vt0
        g[f"nmf_{name}_w0"] = w0
        g[f"nmf_{name}_trace"] = tr
        g[f"nmf_{name}_vt"] = vt
        g[f"nmf_{name}_w"] = w

    # -- MDS (solvers.py:209-305) + pairwise_euclidean (distlinalg.py:442-468) -----
    def mds_case(comm, d, n, q, seed, iters, dt):
        x = bs.empty((d, n), comm, dt)
        bs.rand_fill(x, seed=seed, common_init=True)
        y = bs.empty((n, n), comm, dt)
        bs.pairwise_euclidean(y, x)
        st = bs.mds_init(y, q, seed=seed + 1)
        th0 = bs.gather_full(st.theta)
        bs.mds_fit(st, iters)
        return bs.gather_full(x), bs.gather_full(y), th0, np.asarray(st.trace), bs.gather_full(st.theta)

    mds_cases = [
        ("d5_n12_q2", 5, 12, 2, 6000, 60, np.float64, 2),
        ("d8_n40_q3", 8, 40, 3, 6100, 40, np.float64, 3),
        ("d6_n30_q2_f32", 6, 30, 2, 6200, 30, np.float32, 1),
    ]
    for name, d, n, q, seed, iters, dt, p in mds_cases:
        x, y, th0, tr, th = bs.run_inproc(p, mds_case, d, n, q, seed, iters, dt)[0]
        g[f"mds_{name}_meta"] = np.array([d, n, q, seed, iters, p], dtype=np.int64)
        g[f"mds_{name}_x"] = x
        g[f"mds_{name}_y"] = y
        g[f"mds_{name}_theta0"] = th0
        g[f"mds_{name}_trace"] = tr
        g[f"mds_{name}_theta"] = th

    # -- Cox (solvers.py:337-450), opnorm (distlinalg.py:375-423) --------------------
    def survival(seed, m, n, beta_true=None):
        gen = np.random.Generator(np.random.Philox(seed))
        x = gen.standard_normal((m, n))
        eta = x @ beta_true if beta_true is not None else np.zeros(m)
        times = gen.exponential(1.0 / np.exp(eta))
        delta = (gen.random(m) > 0.3).astype(np.float64)
        order = np.argsort(-times)
        return x[order], times[order], delta[order]

    def cox_case(comm, x, y, delta, lam, sigma, iters, ties, dt):
        xd = bs.distribute(x.astype(dt) if comm.rank == 0 else None, comm)
        st = bs.cox_init(xd, y, delta, lam=lam, sigma=sigma, ties=ties)
        sig = st.sigma
        bs.cox_fit(st, iters)
        return (np.asarray(st.trace), bs.gather_full(st.beta), bs.gather_full(st.grad), sig,
                np.asarray(st.w), np.asarray(st.W), np.asarray(st.pd))

    bt = np.zeros(12)
    bt[[1, 4, 7]] = [0.8, -0.6, 0.5]
    x, y, delta = survival(7001, 40, 12, bt)
    cox_cases = [
        ("m40_n12_lam01", x, y, delta, 0.1, 0.01, 60, "none", np.float64, 2),
        ("m40_n12_powersigma", x, y, delta, 0.05, None, 40, "none", np.float64, 3),
        ("m40_n12_f32", x, y, delta, 0.1, 0.01, 40, "none", np.float32, 1),
    ]
    yt = np.round(y * 2) / 2  # heavy ties
    yt = -np.sort(-yt)
    cox_cases.append(("m40_n12_breslow", x, yt, delta, 0.02, 0.01, 50, "breslow", np.float64, 2))
    for name, xx, yy, dd, lam, sigma, iters, ties, dt, p in cox_cases:
        tr, beta, grad, sig, w, W, pd = bs.run_inproc(p, cox_case, xx, yy, dd, lam, sigma, iters, ties, dt)[0]
        g[f"cox_{name}_x"] = xx.astype(dt)
        g[f"cox_{name}_y"] = yy
        g[f"cox_{name}_delta"] = dd
        g[f"cox_{name}_meta"] = np.array([lam, -1.0 if sigma is None else sigma, iters,
                                          1.0 if ties == "breslow" else 0.0, p], dtype=np.float64)
        g[f"cox_{name}_trace"] = tr
        g[f"cox_{name}_beta"] = beta
        g[f"cox_{name}_grad"] = grad
        g[f"cox_{name}_sigma"] = np.array([sig])
        g[f"cox_{name}_w"] = w
        g[f"cox_{name}_W"] = W
        g[f"cox_{name}_pd"] = pd

    # pi_delta partials over rank ranges (solvers.py:401-419)
    gen = np.random.Generator(np.random.Philox(7300))
    w = np.exp(gen.standard_normal(23) * 0.3)
    W = np.cumsum(w)
    dl = (gen.random(23) > 0.4).astype(np.float64)
    yy = -np.sort(-np.round(gen.random(23) * 6))
    cuts = np.searchsorted(-yy, -yy, side="right").astype(np.int64) - 1
    g["pid_w"], g["pid_W"], g["pid_delta"], g["pid_cuts"] = w, W, dl, cuts
    for p in (1, 3):
        def pid(comm):
            part = bs.partition_of(23, comm.size)
            out = np.empty(23)
            bs.pi_delta(out, w, W, dl, part.lo(comm.rank), part.hi(comm.rank), comm, cuts=cuts)
            return out
        g[f"pid_out_p{p}"] = bs.run_inproc(p, pid)[0]

    # operator norm by power iteration
    a = np.random.Generator(np.random.Philox(4001)).standard_normal((30, 17))
    g["opnorm_a"] = a
    g["opnorm_l2"] = np.array([bs.run_inproc(2, lambda c: bs.opnorm(bs.distribute(a if c.rank == 0 else None, c)))[0]])

    # .dsta matrix files written by the reference's own writer (cli.py:63-78)
    import tempfile

    from blockstat.cli import write_matrix

    for dt, tag in ((np.float32, "f32"), (np.float64, "f64"), (np.int64, "i64")):
        data = (np.random.Generator(np.random.Philox(4100)).random((3, 7)) * 10).astype(dt)
        with tempfile.TemporaryDirectory() as d:
            path = Path(d) / "m.dsta"
            write_matrix(path, data)
            g[f"dsta_{tag}_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()
        g[f"dsta_{tag}_data"] = data

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({len(g)} arrays)")


if __name__ == "__main__":
    main()
