"""Golden fixtures at BASELINE scale, produced by running the REFERENCE package itself.

Run in the build container (the reference lives at /root/reference/pkg/src and
does not exist on the GPU box):

    python tests/golden/make_golden_scale.py            # all cases
    python tests/golden/make_golden_scale.py c1_full    # one case

Inputs are never stored: every case draws its data from seeds, and the GPU tests
(tests/test_scale_gpu.py) regenerate the same bytes on the device with the
bit-exact Philox ``rand_fill`` (or with numpy for the planted case).  Only traces,
final iterates (or, for the 200,000-row factor, a strided sample plus row sums)
and a float64 re-evaluation of the reference's final objective are stored.

Cases (SURVEY.md §8(c) parity protocol; VERDICT r01 "Next round" item 1):
  c1_full            NMF-MU float64, X 10,000 x 10,000, r = 20, 1,000 iterations,
                     trace every 50 — BASELINE configs[0] exactly (solvers.py:144-162)
  c2k_slice          NMF-APG float32, X 200,000 x 1,024, r = 60, 20 iterations: scn a
                     reduces over K = m = 200,000 as in C2 (solvers.py:165-185,
                     distlinalg.py:239-243)
  nmf_apg_f64_r60    NMF-APG float64, 20,000 x 2,000, r = 60 (C2's rank), 20 iterations
  nmf_mu_f32         NMF-MU float32, 2,000 x 1,500, r = 20, 100 iterations
  nmf_planted_*      float32 X = V*^T W* + 1e-3 noise started next to (V*, W*): the
                     objective is ~1e-6 of ||X||^2, where a Gram-identity objective
                     cancels catastrophically
  mds_n2000_{f32,f64} MDS, 2,000 points from 100-dim data, q = 20, 100 iterations
                     (solvers.py:269-305)
  mds_n8000_f32      MDS, 8,000 points, q = 20, 20 iterations, float32 (several row
                     segments and column blocks per rank in the tensor-core pass)
  cox_breslow_f64    Cox, X 4,000 x 3,000 (uniform - 0.5), Breslow ties, default
                     power-iteration sigma, 100 iterations (solvers.py:337-450)
  cox_f32            same X in float32, explicit sigma, 100 iterations
  cox_f32_fused      Cox float32, X 20,000 x 2,000 (uniform - 0.5), Breslow, explicit sigma,
                     50 iterations: large enough for the one-stream fused pass (C4's kernel)
  cox_geno_long_f64  Cox on genotypes, 200,000 x 1,024, float64, 10 iterations (long K for
                     the packed tensor-core passes)
  cox_geno_f64       Cox on genotypes (the counter-based generator of this build, values
                     0/1/2 handed to the reference as float64 — it has no int8 arithmetic),
                     4,000 x 3,000, Breslow ties, default sigma, 100 iterations: pins the
                     packed-genotype tensor-core passes in float64 against the reference
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden_scale.npz"


def planted(m, n, r, seed, noise):
    """Planted nonnegative low-rank data (shared with tests/test_scale_gpu.py)."""
    g = np.random.Generator(np.random.Philox(seed))
    vt = g.random((r, m))
    w = g.random((r, n))
    x = (vt.T @ w + noise * g.random((m, n))).astype(np.float32)
    vt0 = (vt * (1.0 + 0.01 * g.random((r, m)))).astype(np.float32)
    w0 = (w * (1.0 + 0.01 * g.random((r, n)))).astype(np.float32)
    return np.asfortranarray(x), vt0, w0


def cox_inputs(m, n, seed):
    """Cox data: X = U(0,1) - 0.5 (rand_fill stream, column-major), tied y, delta = U > 0.3."""
    x = np.random.Generator(np.random.Philox(seed)).random(m * n).reshape((m, n), order="F") - 0.5
    y = np.floor(np.arange(m, 0, -1) / 3.0)
    delta = (np.random.Generator(np.random.Philox(seed + 1)).random(m) > 0.3).astype(np.float64)
    return x, y, delta


def main(only=None):
    sys.path.insert(0, str(REF))
    import blockstat as bs  # the reference implementation

    out = {}
    if OUT.exists():
        with np.load(OUT) as old:
            out.update({k: old[k] for k in old.files})

    def want(name):
        return only is None or name in only

    def obj64(x, vt, w):
        d = np.asarray(x, dtype=np.float64) - np.asarray(vt, dtype=np.float64).T @ np.asarray(w, dtype=np.float64)
        return float(np.einsum("ij,ij->", d, d))

    def nmf_run(comm, m, n, r, xseed, fseed, dt, algo, iters, every, start=None, xdata=None):
        if xdata is None:
            x = bs.empty((m, n), comm, dt)
            bs.rand_fill(x, seed=xseed, common_init=True)
        else:
            x = bs.distribute(xdata if comm.rank == 0 else None, comm)
        st = bs.nmf_init(x, r, seed=fseed)
        if start is not None:
            vt0, w0 = start
            st.Vt.local[...] = vt0[:, st.Vt.lo:st.Vt.hi]
            st.W.local[...] = w0[:, st.W.lo:st.W.hi]
        (bs.nmf_multiplicative if algo == "mu" else bs.nmf_apg)(st, iters, trace_every=every)
        return np.asarray(st.trace), bs.gather_full(st.Vt), bs.gather_full(st.W)

    t0 = time.time()
    if want("c1_full"):
        tr, vt, w = bs.run_inproc(1, nmf_run, 10000, 10000, 20, 2010, 2011, np.float64, "mu", 1000, 50)[0]
        out["c1_full_meta"] = np.array([10000, 10000, 20, 2010, 2011, 1000, 50, 0], dtype=np.int64)
        out["c1_full_trace"], out["c1_full_vt"], out["c1_full_w"] = tr, vt, w
        print(f"c1_full {time.time() - t0:.0f}s trace[-1]={tr[-1]:.12e}", flush=True)

    if want("c2k_slice"):
        m, n, r = 200000, 1024, 60
        tr, vt, w = bs.run_inproc(1, nmf_run, m, n, r, 2020, 2021, np.float32, "apg", 20, 1)[0]
        x = np.random.Generator(np.random.Philox(2020)).random(m * n, dtype=np.float32).reshape((m, n), order="F")
        out["c2k_slice_meta"] = np.array([m, n, r, 2020, 2021, 20, 1, 1], dtype=np.int64)
        out["c2k_slice_trace"] = tr
        out["c2k_slice_w"] = w
        out["c2k_slice_vt_sample"] = np.ascontiguousarray(vt[:, ::50])
        out["c2k_slice_vt_rowsum"] = vt.astype(np.float64).sum(axis=1)
        out["c2k_slice_obj64"] = np.array([obj64(x, vt, w)])
        print(f"c2k_slice {time.time() - t0:.0f}s trace[-1]={tr[-1]:.9e} obj64={out['c2k_slice_obj64'][0]:.9e}",
              flush=True)
        del x

    if want("nmf_apg_f64_r60"):
        # C2's rank in float64: the cp.async m16n8k16 DMMA kernel at RP = 64
        tr, vt, w = bs.run_inproc(2, nmf_run, 20000, 2000, 60, 2035, 2036, np.float64, "apg", 20, 1)[0]
        out["nmf_apg_f64_r60_meta"] = np.array([20000, 2000, 60, 2035, 2036, 20, 1, 1], dtype=np.int64)
        out["nmf_apg_f64_r60_trace"], out["nmf_apg_f64_r60_w"] = tr, w
        out["nmf_apg_f64_r60_vt_sample"] = np.ascontiguousarray(vt[:, ::20])  # keeps the fixture small
        out["nmf_apg_f64_r60_vt_rowsum"] = vt.sum(axis=1)
        print(f"nmf_apg_f64_r60 {time.time() - t0:.0f}s", flush=True)

    if want("nmf_mu_f32"):
        tr, vt, w = bs.run_inproc(2, nmf_run, 2000, 1500, 20, 2030, 2031, np.float32, "mu", 100, 10)[0]
        out["nmf_mu_f32_meta"] = np.array([2000, 1500, 20, 2030, 2031, 100, 10, 0], dtype=np.int64)
        out["nmf_mu_f32_trace"], out["nmf_mu_f32_vt"], out["nmf_mu_f32_w"] = tr, vt, w
        print(f"nmf_mu_f32 {time.time() - t0:.0f}s", flush=True)

    for algo in ("mu", "apg"):
        name = f"nmf_planted_{algo}"
        if not want(name):
            continue
        m, n, r = 4096, 1024, 20
        x, vt0, w0 = planted(m, n, r, 2040, 1e-3)
        tr, vt, w = bs.run_inproc(1, nmf_run, m, n, r, 0, 2041, np.float32, algo, 10, 1, (vt0, w0), x)[0]
        out[f"{name}_meta"] = np.array([m, n, r, 2040, 2041, 10, 1, 0 if algo == "mu" else 1], dtype=np.int64)
        out[f"{name}_trace"], out[f"{name}_vt"], out[f"{name}_w"] = tr, vt, w
        out[f"{name}_obj64"] = np.array([obj64(x, vt, w)])
        out[f"{name}_xsq"] = np.array([float(np.sum(x.astype(np.float64) ** 2))])
        print(f"{name} {time.time() - t0:.0f}s obj/|X|^2={tr[-1] / out[f'{name}_xsq'][0]:.3e}", flush=True)

    def mds_run(comm, d, n, q, xseed, tseed, dt, iters):
        x = bs.empty((d, n), comm, dt)
        bs.rand_fill(x, seed=xseed, common_init=True)
        y = bs.empty((n, n), comm, dt)
        bs.pairwise_euclidean(y, x)
        st = bs.mds_init(y, q, seed=tseed)
        bs.mds_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.theta)

    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        name = f"mds_n2000_{tag}"
        if not want(name):
            continue
        tr, th = bs.run_inproc(2, mds_run, 100, 2000, 20, 2050, 2051, dt, 100)[0]
        out[f"{name}_meta"] = np.array([100, 2000, 20, 2050, 2051, 100], dtype=np.int64)
        out[f"{name}_trace"], out[f"{name}_theta"] = tr, th
        print(f"{name} {time.time() - t0:.0f}s", flush=True)

    if want("mds_n8000_f32"):
        # more points than one segment of the tensor-core pass holds: several row segments
        # and column blocks per rank, 20 iterations, float32
        tr, th = bs.run_inproc(2, mds_run, 100, 8000, 20, 2080, 2081, np.float32, 20)[0]
        out["mds_n8000_f32_meta"] = np.array([100, 8000, 20, 2080, 2081, 20], dtype=np.int64)
        out["mds_n8000_f32_trace"], out["mds_n8000_f32_theta"] = tr, th
        # The reference's float32 stress is a float32 dot over n^2 = 64M terms: 1.5e-4 low at
        # theta0 against the same float32 terms summed in float64.  Store that float64 sum for
        # the first trace entry (the same float32 Y, theta0 and Gram-identity distances).
        sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
        from oracle import blockstat_oracle as orc

        xf = orc.rand_fill_common((100, 8000), 2080, np.float32)
        yf = orc.pairwise_euclidean(xf)
        th0 = orc.mds_init(yf, 20, 2081)
        g0 = th0.T @ th0
        nr = np.diag(g0)
        d0 = np.sqrt(np.maximum(nr[:, None] + nr[None, :] - 2 * g0, 0)).astype(np.float32)
        np.fill_diagonal(d0, 0)
        out["mds_n8000_f32_stress0_f64"] = np.array([float(np.sum((yf.astype(np.float64) - d0) ** 2))])
        print(f"mds_n8000_f32 {time.time() - t0:.0f}s  reference trace[0] / float64 sum - 1 = "
              f"{tr[0] / out['mds_n8000_f32_stress0_f64'][0] - 1:.2e}", flush=True)

    def cox_run(comm, x, y, delta, lam, sigma, iters, dt):
        xd = bs.distribute(x.astype(dt) if comm.rank == 0 else None, comm)
        st = bs.cox_init(xd, y, delta, lam=lam, sigma=sigma, ties="breslow")
        bs.cox_fit(st, iters)
        return np.asarray(st.trace), bs.gather_full(st.beta), st.sigma

    m, n = 4000, 3000
    x, y, delta = cox_inputs(m, n, 2060)
    for name, dt, sigma, lam in (("cox_breslow_f64", np.float64, None, 0.008), ("cox_f32", np.float32, 2e-4, 0.004)):
        if not want(name):
            continue
        tr, beta, sig = bs.run_inproc(2, cox_run, x, y, delta, lam, sigma, 100, dt)[0]
        out[f"{name}_meta"] = np.array([m, n, 2060, lam, -1.0 if sigma is None else sigma, 100], dtype=np.float64)
        out[f"{name}_trace"], out[f"{name}_beta"], out[f"{name}_sigma"] = tr, beta, np.array([sig])
        print(f"{name} {time.time() - t0:.0f}s nnz={np.count_nonzero(beta)} sigma={sig:.6e}", flush=True)

    if want("cox_geno_long_f64"):
        # long K for the packed tensor-core passes: 200,000 samples (98 groups of 2,048 rows in
        # the gradient), 1,024 variants, float64, default sigma, 10 iterations
        sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
        from oracle import blockstat_oracle as orc

        m3, n3, seed3 = 200000, 1024, 2095
        xg3 = orc.genotype_fill(m3, n3, seed3).astype(np.float64)
        y3 = np.floor(np.arange(m3, 0, -1) / 4.0)
        delta3 = (np.random.Generator(np.random.Philox(seed3 + 7)).random(m3) < 0.3).astype(np.float64)
        tr, beta, sig = bs.run_inproc(2, cox_run, xg3, y3, delta3, 1e-7, None, 10, np.float64)[0]
        out["cox_geno_long_f64_meta"] = np.array([m3, n3, seed3, 1e-7, -1.0, 10], dtype=np.float64)
        out["cox_geno_long_f64_trace"], out["cox_geno_long_f64_beta"] = tr, beta
        out["cox_geno_long_f64_sigma"] = np.array([sig])
        print(f"cox_geno_long_f64 {time.time() - t0:.0f}s nnz={np.count_nonzero(beta)}", flush=True)
        del xg3

    if want("cox_f32_fused"):
        # float32 X large enough for the one-stream fused pass (m >= 4096, n >= 128): the C4
        # kernel (bs_cox_grad_xbeta) against the reference's float32 arithmetic
        m2, n2 = 20000, 2000
        x2, y2, delta2 = cox_inputs(m2, n2, 2090)
        tr, beta, sig = bs.run_inproc(2, cox_run, x2, y2, delta2, 2e-3, 1e-4, 50, np.float32)[0]
        out["cox_f32_fused_meta"] = np.array([m2, n2, 2090, 2e-3, 1e-4, 50], dtype=np.float64)
        out["cox_f32_fused_trace"], out["cox_f32_fused_beta"] = tr, beta
        print(f"cox_f32_fused {time.time() - t0:.0f}s nnz={np.count_nonzero(beta)}", flush=True)

    if want("cox_geno_f64"):
        sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
        from oracle import blockstat_oracle as orc

        m, n, seed = 4000, 3000, 2070
        xg = orc.genotype_fill(m, n, seed).astype(np.float64)
        y = np.floor(np.arange(m, 0, -1) / 4.0)
        delta = (np.random.Generator(np.random.Philox(seed + 7)).random(m) < 0.4).astype(np.float64)
        tr, beta, sig = bs.run_inproc(2, cox_run, xg, y, delta, 2e-6, None, 100, np.float64)[0]
        out["cox_geno_f64_meta"] = np.array([m, n, seed, 2e-6, -1.0, 100], dtype=np.float64)
        out["cox_geno_f64_trace"], out["cox_geno_f64_beta"], out["cox_geno_f64_sigma"] = tr, beta, np.array([sig])
        print(f"cox_geno_f64 {time.time() - t0:.0f}s nnz={np.count_nonzero(beta)} sigma={sig:.6e}", flush=True)
        # the same in float32 arithmetic (the C5 setting), with the float64 run's sigma
        tr, beta, sig = bs.run_inproc(2, cox_run, xg, y, delta, 2e-6, float(sig), 100, np.float32)[0]
        out["cox_geno_f32_trace"], out["cox_geno_f32_beta"], out["cox_geno_f32_sigma"] = tr, beta, np.array([sig])
        print(f"cox_geno_f32 {time.time() - t0:.0f}s nnz={np.count_nonzero(beta)}", flush=True)

    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({len(out)} arrays, {OUT.stat().st_size / 1e6:.1f} MB)")


if __name__ == "__main__":
    main(set(sys.argv[1:]) or None)
