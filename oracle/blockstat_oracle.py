"""CPU oracle for the B200 hot path — TEST INFRASTRUCTURE ONLY.

A dense, single-process numpy restatement of the reference algorithm
(``/root/reference/pkg/src/blockstat``, "blockstat") for the three solvers and
the primitives they use.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg may import it, and only as the checker; the
product path (``paper_2010_16114_b200``) never imports it.

Parity pinning: every function here is checked against golden vectors produced
by running the reference package itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``, test
``tests/test_oracle_golden.py``).  The Philox restatement is additionally
checked bit-for-bit against numpy's generator.

Distributed semantics: the reference's results are independent of the rank
count up to floating-point reassociation; the oracle computes
the p = 1 arithmetic.  ``pi_delta`` keeps the [lo, hi) range semantics of the
reference because its contract is per-rank.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# partitions and random fill (distarray.py:55-65, 170-208)
# ---------------------------------------------------------------------------


def partition_of(extent, nranks):
    """Block boundaries: first extent % nranks ranks get one extra (distarray.py:55-65)."""
    base, rem = divmod(extent, nranks)
    b = [0]
    for r in range(nranks):
        b.append(b[-1] + base + (1 if r < rem else 0))
    return tuple(b)


def rand_fill_common(shape, seed, dtype=np.float64, dist="uniform01"):
    """rand_fill(common_init=True): whole array drawn in column-major order (distarray.py:195-204)."""
    n = int(np.prod(shape))
    gen = np.random.Generator(np.random.Philox(seed))
    if dist == "uniform01":
        vals = gen.random(n, dtype=dtype)
    else:
        vals = gen.standard_normal(n, dtype=dtype)
    return vals.reshape(shape, order="F")


# Philox4x64-10 restated in pure Python (numpy bit_generator/philox.h semantics):
# block b uses counter b+1 (the counter is incremented before each refill).
_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_MASK = (1 << 64) - 1


def philox_key(seed):
    st = np.random.Philox(seed).state["state"]["key"]
    return int(st[0]), int(st[1])


def philox_block(b, key, c1=0):
    c = [(b + 1) & _MASK, c1, 0, 0]
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> 64, p0 & _MASK
        hi1, lo1 = p1 >> 64, p1 & _MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


def philox_normal(seed, first, count):
    """Elements [first, first+count) of the counter-based normal stream of bs_philox_normal
    (no reference equivalent: numpy's ziggurat consumes a data-dependent number of words;
    SURVEY.md §8(f)1).  Element e: Box-Muller on Philox block (e // 2 + 1, 1, 0, 0)."""
    key = philox_key(seed)
    out = np.empty(count)
    for i, e in enumerate(range(first, first + count)):
        w = philox_block(e // 2, key, c1=1)
        u1 = ((w[0] >> 11) + 0.5) / 2.0 ** 53
        u2 = (w[1] >> 11) / 2.0 ** 53
        r = np.sqrt(-2.0 * np.log(u1))
        out[i] = r * (np.cos(2.0 * np.pi * u2) if e % 2 == 0 else np.sin(2.0 * np.pi * u2))
    return out


def philox_raw(seed, count):
    key = philox_key(seed)
    out = []
    b = 0
    while len(out) < count:
        out.extend(philox_block(b, key))
        b += 1
    return np.array(out[:count], dtype=np.uint64)


def philox_uniform(seed, count, dtype=np.float64, first=0):
    """Elements [first, first+count) of Generator(Philox(seed)).random(N, dtype)."""
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        words = philox_raw(seed, first + count)[first:]
        return (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    words = philox_raw(seed, (first + count + 1) // 2 + 1)
    halves = np.empty(2 * len(words), dtype=np.uint64)
    halves[0::2] = words & np.uint64(0xFFFFFFFF)
    halves[1::2] = words >> np.uint64(32)
    h = halves[first:first + count]
    return ((h >> np.uint64(8)).astype(np.float64) * (1.0 / 16777216.0)).astype(np.float32)


# ---------------------------------------------------------------------------
# NMF (solvers.py:97-185)
# ---------------------------------------------------------------------------


def nmf_init(x, rank, seed):
    """Factors drawn like nmf_init (solvers.py:97-121): Vt from seed, W from seed+1."""
    m, n = x.shape
    if np.min(x) < 0:
        raise ValueError("NMF requires nonnegative data")
    vt = rand_fill_common((rank, m), seed, x.dtype)
    w = rand_fill_common((rank, n), seed + 1, x.dtype)
    return vt, w


def nmf_objective(x, vt, w):
    """||X - Vt^T W||_F^2 (solvers.py:124-136)."""
    d = x - vt.T @ w
    return float(np.dot(np.ravel(d, order="F"), np.ravel(d, order="F")))


def nmf_multiplicative(x, vt, w, iters, eps=1e-10, trace_every=1):
    """Lee-Seung updates; objective traced after each update (solvers.py:144-162)."""
    vt, w = vt.copy(), w.copy()
    trace = []
    for it in range(iters):
        wxt = w @ x.T
        wwt = w @ w.T
        vt = vt * wxt / (wwt @ vt + eps)
        vtx = vt @ x
        vtv = vt @ vt.T
        w = w * vtx / (vtv @ w + eps)
        if trace_every and it % trace_every == 0:
            trace.append(nmf_objective(x, vt, w))
    return vt, w, trace


def nmf_apg(x, vt, w, iters, eps=1e-10, trace_every=1):
    """Alternating projected gradient (solvers.py:165-185): sigma from the old W, tau from the new Vt."""
    vt, w = vt.copy(), w.copy()
    trace = []
    for it in range(iters):
        wxt = w @ x.T
        wwt = w @ w.T
        sigma = 1.0 / (2.0 * float(np.sum(wwt ** 2)) + eps)
        vt = np.maximum(0.0, vt - sigma * (wwt @ vt - wxt))
        vtx = vt @ x
        vtv = vt @ vt.T
        tau = 1.0 / (2.0 * float(np.sum(vtv ** 2)) + eps)
        w = np.maximum(0.0, w - tau * (vtv @ w - vtx))
        if trace_every and it % trace_every == 0:
            trace.append(nmf_objective(x, vt, w))
    return vt, w, trace


# ---------------------------------------------------------------------------
# MDS (solvers.py:209-305) and its input (distlinalg.py:442-468)
# ---------------------------------------------------------------------------


def pairwise_euclidean(x):
    """Distances between the columns of x, direct differences, zero diagonal (distlinalg.py:442-468)."""
    n = x.shape[1]
    y = np.empty((n, n), dtype=x.dtype)
    for i in range(n):
        diff = x - x[:, i:i + 1]
        y[i, :] = np.sqrt((diff * diff).sum(axis=0))
    np.fill_diagonal(y, 0)
    return y


def mds_init(y, ndim, seed):
    """theta = 2 U(0,1) - 1 drawn with rand_fill (solvers.py:209-234)."""
    n = y.shape[0]
    if y.shape != (n, n) or n < 2:
        raise ValueError("MDS expects a square distance matrix of >= 2 points")
    if np.any(np.diag(y) != 0):
        raise ValueError("target distance matrix must have a zero diagonal")
    return 2.0 * rand_fill_common((ndim, n), seed, y.dtype) - 1.0


def embedding_distances(theta):
    """Gram-identity distances; the diagonal cancels to exactly 0 (solvers.py:237-247)."""
    g = theta.T @ theta
    dg = np.diag(g)
    return np.sqrt(np.maximum(dg[None, :] + dg[:, None] - 2.0 * g, 0.0))


def mds_stress(theta, y):
    """sum (Y - D)^2 (solvers.py:250-266)."""
    d = y - embedding_distances(theta)
    return float(np.dot(np.ravel(d, order="F"), np.ravel(d, order="F")))


class DegenerateConfigError(RuntimeError):
    pass


def mds_fit(y, theta, iters, perturb=False, trace_every=1):
    """MM updates; trace = stress of the iterate entering each update (solvers.py:269-305)."""
    theta = theta.copy()
    n = y.shape[0]
    wsum = float(n - 1)
    trace = []
    for it in range(iters):
        dist = embedding_distances(theta)
        d = y - dist
        stress = float(np.dot(np.ravel(d, order="F"), np.ravel(d, order="F")))
        zero_pairs = float((dist == 0.0).sum() - n)
        if trace_every and it % trace_every == 0:
            trace.append(stress)
        np.fill_diagonal(dist, np.inf)
        if zero_pairs > 0:
            if not perturb:
                raise DegenerateConfigError("coincident embedding points")
            dist = np.where(dist == 0.0, 1e-10, dist)
        z = y / dist
        zsum = z.sum(axis=0)
        wmz = 1.0 - z
        np.fill_diagonal(wmz, 0.0)
        t = theta @ wmz
        theta = (theta * (zsum[None, :] + wsum) + t) / (2.0 * wsum)
    return theta, trace


# ---------------------------------------------------------------------------
# l1-Cox (solvers.py:332-450) and the power-iteration step size (distlinalg.py:375-423)
# ---------------------------------------------------------------------------


def soft_threshold(x, lam):
    """sign(x) max(|x| - lam, 0) (solvers.py:48-51)."""
    x = np.asarray(x)
    return np.sign(x) * np.maximum(np.abs(x) - lam, 0)


def converged(history, f_new, window=10, rel_tol=1e-5):
    """Windowed relative-change rule (solvers.py:63-70)."""
    history.append(float(f_new))
    if len(history) <= window:
        return False
    return abs(history[-1] - history[-1 - window]) / (abs(history[-1]) + 1.0) < rel_tol


def tie_cuts(y):
    """Last index of each tied block (solvers.py:332-334)."""
    neg = -np.asarray(y, dtype=np.float64)
    return np.searchsorted(neg, neg, side="right").astype(np.int64) - 1


def risk_weights(xbeta, clamp):
    """w = exp(min(xbeta, clamp)), W = forward cumsum (solvers.py:379-390)."""
    clamped = bool(np.any(xbeta > clamp))
    w = np.exp(np.minimum(xbeta, clamp)) if clamped else np.exp(xbeta)
    if not np.all(np.isfinite(w)):
        raise FloatingPointError("nonfinite risk weights")
    return w, np.cumsum(w), clamped


def pi_delta(w, W, delta, lo, hi, cuts=None):
    """One rank's partial of P delta over [lo, hi) (solvers.py:401-419), before the allreduce."""
    m = len(delta)
    out = np.zeros(m, dtype=np.result_type(w, W, delta))
    if hi > lo:
        seg = np.arange(lo, hi) if cuts is None else cuts[lo:hi]
        contrib = delta[lo:hi] / W[seg]
        suffix = np.cumsum(contrib[::-1])[::-1]
        first = np.searchsorted(seg, np.arange(m), side="left")
        valid = first < (hi - lo)
        out[valid] = suffix[first[valid]]
        out *= w
    return out


def cox_loglik(x, beta, delta, cuts, clamp=700.0):
    """sum delta (X beta - log W[cuts]) (solvers.py:393-398)."""
    xb = x @ beta
    _, W, _ = risk_weights(xb, clamp)
    return float(np.sum(delta * (xb - np.log(W[cuts]))))


def cox_fit(x, delta, cuts, lam, sigma, iters, beta0=None, trace_every=1, window=None, clamp=700.0):
    """Proximal gradient (solvers.py:422-450); returns beta, grad, trace, iterations run."""
    m, n = x.shape
    beta = np.zeros(n, dtype=x.dtype) if beta0 is None else beta0.copy()
    grad = np.zeros(n, dtype=x.dtype)
    trace = []
    history = []
    for it in range(iters):
        xb = x @ beta
        w, W, _ = risk_weights(xb, clamp)
        if trace_every and it % trace_every == 0:
            loglik = float(np.sum(delta * (xb - np.log(W[cuts]))))
            obj = -loglik + lam * float(np.sum(np.abs(beta)))
            trace.append(obj)
            if window is not None and converged(history, obj, window=window):
                break
        pd = pi_delta(w, W, delta, 0, m, cuts)
        grad = x.T @ (delta - pd)
        beta = soft_threshold(beta + sigma * grad, lam)
    return beta, grad, trace


def opnorm_l2_power(a, tol=1e-6, maxiter=1000, seed=95376):
    """Power iteration on A^T A with the reference's start vector and stopping rule (distlinalg.py:403-423)."""
    m, n = a.shape
    gen = np.random.Generator(np.random.Philox(seed))
    v = gen.random(n)
    v /= np.linalg.norm(v)
    estimate, previous = 0.0, np.inf
    for _ in range(maxiter):
        u = (a @ v).astype(a.dtype)
        estimate = float(np.linalg.norm(u))
        if abs(estimate - previous) <= tol * max(estimate, np.finfo(float).tiny):
            break
        previous = estimate
        w = (a.T @ u).astype(a.dtype)
        nw = np.linalg.norm(w)
        if nw == 0:
            return 0.0
        v = w / nw
    return estimate


def survival_data(seed, m, n, beta_true=None):
    """Synthetic sorted survival data in the style of the reference tests (test_solvers.py:311-317)."""
    gen = np.random.Generator(np.random.Philox(seed))
    x = gen.standard_normal((m, n))
    eta = x @ beta_true if beta_true is not None else np.zeros(m)
    times = gen.exponential(1.0 / np.exp(eta))
    delta = (gen.random(m) > 0.3).astype(np.float64)
    order = np.argsort(-times)
    return x[order], times[order], delta[order]


def genotype_fill(m, n, seed, maf_range=(0.05, 0.5)):
    """Counter-based genotypes (this build's C5 input; the reference has no int8 fill):
    p_j = lo + (hi - lo) * Generator(Philox(seed + 1)).random(n)[j];
    X[i, j] = [u[2e] < p_j] + [u[2e + 1] < p_j], e = j*m + i, u = Generator(Philox(seed)).random(2mn).
    Small sizes only (test infrastructure)."""
    lo, hi = maf_range
    p = lo + (hi - lo) * np.random.Generator(np.random.Philox(seed + 1)).random(n)
    u = np.random.Generator(np.random.Philox(seed)).random(2 * m * n).reshape(m * n, 2)
    pe = np.repeat(p, m)
    x = (u[:, 0] < pe).astype(np.int8) + (u[:, 1] < pe).astype(np.int8)
    return x.reshape((m, n), order="F")


def pack_genotypes_u2(x):
    """2-bit packing of an (m, n) genotype matrix (this build's BS_U2 layout, include/bsb200.h):
    column j is ceil(m/64)*16 bytes, genotype i in bits 2(i%4)..+1 of byte i//4, zero pad.
    Returns the (ld, n) uint8 block, column-major like the device block."""
    x = np.asarray(x)
    m, n = x.shape
    ld = ((m + 63) // 64) * 16
    g = np.zeros((ld * 4, n), dtype=np.uint8)
    g[:m] = x.astype(np.uint8) & 3
    q = g.reshape(ld, 4, n)
    return (q[:, 0] | (q[:, 1] << 2) | (q[:, 2] << 4) | (q[:, 3] << 6)).astype(np.uint8)
