"""Multi-process parity under torchrun (one process per rank).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/nccl_parity.py

BS_PARITY_BACKEND selects the communicator: ``nccl`` (default; one GPU per rank) or
``gloo+cuda`` (data on the GPU, collectives staged through the host, so several ranks
may share one GPU — tests/test_multiproc_gpu.py runs it with 2 ranks on a 1-GPU box).
The solver-level C ABI sections need NCCL and run only with ``nccl``.

Runs NMF (both algorithms, float32 tcgen05 path and float64), MDS and Cox through
the 'nccl' Communicator on column-sharded data and checks every rank's result
against the CPU oracle.  Exits non-zero on a mismatch.
"""

import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2010_16114_b200 as bs  # noqa: E402
from oracle import blockstat_oracle as orc  # noqa: E402


def check(name, got, want, tol):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-300)
    ok = err <= tol
    print(f"[rank {os.environ.get('RANK')}] {name}: rel err {err:.2e} (tol {tol:.0e}) {'OK' if ok else 'FAIL'}",
          flush=True)
    return ok


def main():
    backend = os.environ.get("BS_PARITY_BACKEND", "nccl")
    comm = bs.init(backend)
    ok = True
    for dt, tol, (m, n, r) in ((np.float64, 1e-9, (300, 257, 7)), (np.float32, 2e-5, (2048, 1501, 60))):
        x = orc.rand_fill_common((m, n), 5, dt)
        vt0, w0 = orc.nmf_init(x, r, 6)
        for algo, fn, ofn in ((0, bs.nmf_multiplicative, orc.nmf_multiplicative), (1, bs.nmf_apg, orc.nmf_apg)):
            xd = bs.empty((m, n), comm, dt)
            bs.rand_fill(xd, seed=5, common_init=True)
            st = bs.nmf_init(xd, r, seed=6)
            fn(st, 15)
            ovt, ow, otr = ofn(x.astype(np.float64), vt0.astype(np.float64), w0.astype(np.float64), 15)
            ok &= check(f"nmf algo={algo} {np.dtype(dt).name} trace", st.trace, otr, tol)
            ok &= check(f"nmf algo={algo} {np.dtype(dt).name} W", bs.gather_full(st.W), ow, tol * 10)
    # MDS
    pts = orc.rand_fill_common((6, 301), 7, np.float64)
    y = orc.pairwise_euclidean(pts)
    th0 = orc.mds_init(y, 3, 8)
    yd = bs.empty((301, 301), comm)
    pd = bs.empty((6, 301), comm)
    bs.rand_fill(pd, seed=7, common_init=True)
    bs.pairwise_euclidean(yd, pd)
    st = bs.mds_init(yd, 3, seed=8)
    bs.mds_fit(st, 12)
    oth, otr = orc.mds_fit(y, th0, 12)
    ok &= check("mds trace", st.trace, otr, 1e-9)
    ok &= check("mds theta", bs.gather_full(st.theta), oth, 1e-8)
    # Cox (float64 and int8 storage)
    xs, ys, ds = orc.survival_data(9, 500, 301, np.r_[0.4, -0.3, np.zeros(299)])
    sig = 0.5 / np.linalg.norm(xs, 2) ** 2
    xd = bs.distribute(xs if comm.rank == 0 else None, comm)
    st = bs.cox_init(xd, ys, ds, lam=0.01, sigma=sig)
    bs.cox_fit(st, 20)
    ob, og, otr = orc.cox_fit(xs, ds, np.arange(500), 0.01, sig, 20)
    ok &= check("cox trace", st.trace, otr, 1e-10)
    ok &= check("cox beta", bs.gather_full(st.beta), ob, 1e-8)
    ok &= check("cox sigma (power iteration)", bs.opnorm(xd), orc.opnorm_l2_power(xs), 1e-12)
    # Cox float32 (the fused one-stream pass, cox_fused2.cu), split over two calls so the
    # second reuses the last pass's X beta partial (allreduced at the start of the call)
    gen = np.random.Generator(np.random.Philox(12))
    xf = gen.standard_normal((8000, 1203)).astype(np.float32)
    df = (gen.random(8000) < 0.5).astype(np.float64)
    yf = np.arange(8000, 0, -1, dtype=np.float64)
    sgf = 2e-5
    xfd = bs.distribute(xf if comm.rank == 0 else None, comm)
    st = bs.cox_init(xfd, yf, df, lam=1e-4, sigma=sgf)
    bs.cox_fit(st, 6)
    bs.cox_fit(st, 6)
    ob, og, otr = orc.cox_fit(xf.astype(np.float64), df, np.arange(8000), 1e-4, sgf, 12)
    ok &= check("cox float32 fused: nonzero coefficients", [min(np.count_nonzero(ob), 1)], [1], 0)
    ok &= check("cox float32 fused trace", st.trace, otr, 2e-5)
    ok &= check("cox float32 fused beta", bs.gather_full(st.beta), ob, 2e-4)
    # packed genotypes (2-bit) against int8 storage of the same matrix
    gp = bs.genotype_fill(bs.PackedGenotypes(comm, (6000, 777)), 31)
    g8 = bs.genotype_fill(bs.empty((6000, 777), comm, np.int8), 31)
    yg = np.floor(np.arange(6000, 0, -1) / 4.0)
    dg = (np.random.Generator(np.random.Philox(3)).random(6000) < 0.3).astype(np.float64)
    tr = []
    for a in (gp, g8):
        st = bs.cox_init(a, yg, dg, lam=1e-6, sigma=2e-7, ties="breslow", dtype=np.float32)
        bs.cox_fit(st, 8)
        tr.append(np.asarray(st.trace))
        ok &= check("cox packed/int8: nonzero coefficients", [min(np.count_nonzero(bs.gather_full(st.beta)), 1)], [1], 0)
    ok &= check("cox packed genotypes vs int8 trace", tr[0], tr[1], 2e-5)
    if backend != "nccl":
        comm.barrier()
        import torch.distributed as dist

        dist.destroy_process_group()
        sys.exit(0 if ok else 1)
    # the solver-level C ABI (bs_ctx_create over NCCL + bs_cox_run) against cox_fit
    from paper_2010_16114_b200 import runtime

    for xs_, tol in ((xs, 1e-12), (xf, 1e-9)):
        res = []
        for native in (False, True):
            xd_ = bs.distribute(xs_ if comm.rank == 0 else None, comm)
            mm = xs_.shape[0]
            dd = ds if xs_ is xs else df
            yy = ys if xs_ is xs else yf
            st = bs.cox_init(xd_, yy, dd, lam=1e-4, sigma=sig if xs_ is xs else sgf)
            if native:
                with runtime.Context(comm) as ctx:
                    runtime.cox_run(ctx, st, 10)
            else:
                bs.cox_fit(st, 10)
            res.append((np.asarray(st.trace), bs.gather_full(st.beta)))
        name = np.dtype(xs_.dtype).name
        ok &= check(f"native bs_cox_run {name} trace (NCCL)", res[1][0], res[0][0], tol)
        ok &= check(f"native bs_cox_run {name} beta (NCCL)", res[1][1], res[0][1], tol * 1e3)
    # bs_nmf_run: grouped NCCL reduces / broadcasts for the uneven blocks (m = 301 over 2 ranks)
    for dt, tol in ((np.float64, 1e-12), (np.float32, 1e-5)):
        xn = orc.rand_fill_common((301, 200), 5, dt)
        res = []
        for native in (False, True):
            st = bs.nmf_init(bs.distribute(xn if comm.rank == 0 else None, comm), 6, seed=6)
            if native:
                with runtime.Context(comm) as ctx:
                    runtime.nmf_run(ctx, st, 8, algo="apg")
            else:
                bs.nmf_apg(st, 8)
            res.append((np.asarray(st.trace), bs.gather_full(st.W)))
        ok &= check(f"native bs_nmf_run {np.dtype(dt).name} trace (NCCL)", res[1][0], res[0][0], tol)
        ok &= check(f"native bs_nmf_run {np.dtype(dt).name} W (NCCL)", res[1][1], res[0][1], tol * 10)
    # bs_mds_run: theta all-gather by grouped broadcasts (n = 301 over 2 ranks)
    res = []
    for native in (False, True):
        st = bs.mds_init(yd, 3, seed=8)
        if native:
            with runtime.Context(comm) as ctx:
                runtime.mds_run(ctx, st, 12)
        else:
            bs.mds_fit(st, 12)
        res.append((np.asarray(st.trace), bs.gather_full(st.theta)))
    ok &= check("native bs_mds_run trace (NCCL)", res[1][0], res[0][0], 1e-12)
    ok &= check("native bs_mds_run theta (NCCL)", res[1][1], res[0][1], 1e-11)
    comm.barrier()
    import torch.distributed as dist

    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
