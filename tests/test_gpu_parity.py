"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

All inputs are seeded.  Sizes span several tiles and ragged batches; the
config-sized cases run at BASELINE.json's full sizes and compare sampled
transforms / positions with the oracle (whole transforms where the oracle is
fast enough) plus size-independent properties.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_util import P30, P62, P62G, RNS, bitrev, rand_residues, root, to_dev, to_host  # noqa: E402


@pytest.fixture(scope="module")
def ntt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1205_2926_b200 as P
    return P


NTHREADS = oracle.default_threads()


def _roundtrip_case(ntt, p, bits, ell, batch, seed, top=False):
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits)
    rng = np.random.default_rng(seed)
    x = rand_residues(rng, p, (batch, L))
    if top:  # Alg. 3 accepts [0,2p): exercise the top of the range
        x = np.where(rng.random((batch, L)) < 0.5, x + np.uint64(p), x)
        x[:, 0] = 2 * p - 1
    d = to_dev(x, bits)
    plan.forward(d)
    got = to_host(d)
    ref = oracle.ntt_forward(p, w, x, nthreads=NTHREADS)
    assert np.array_equal(got, ref), f"forward mismatch p={p} ell={ell} batch={batch}"
    # inverse accepts [0,4p): feed redundant representatives of the forward output
    y = got.copy()
    if top:
        y = y + np.uint64(p) * rng.integers(0, 4, size=y.shape, dtype=np.uint64)
    d2 = to_dev(y, bits)
    plan.inverse(d2)
    got_inv = to_host(d2)
    ref_inv = oracle.ntt_inverse(p, w, got, nthreads=NTHREADS)
    assert np.array_equal(got_inv, ref_inv), f"inverse mismatch p={p} ell={ell}"
    xr = x.astype(object) % p
    assert np.array_equal(got_inv.astype(object), (xr * L) % p)  # inverse o forward = L x


@pytest.mark.parametrize("ell", list(range(0, 16)))
def test_single_pass_u32(ntt, ell):
    _roundtrip_case(ntt, P30, 32, ell, batch=3 if ell > 10 else 37, seed=ell, top=True)


@pytest.mark.parametrize("ell", list(range(0, 15)))
def test_single_pass_u64(ntt, ell):
    _roundtrip_case(ntt, P62, 64, ell, batch=3 if ell > 10 else 37, seed=100 + ell, top=True)


@pytest.mark.parametrize("p,bits,ell,batch", [
    (P30, 32, 16, 2), (RNS[0], 32, 17, 1), (RNS[1], 32, 20, 1),
    (P62, 64, 15, 3), (P62, 64, 16, 1), (P62, 64, 18, 1), (P62, 64, 21, 1),
])
def test_multi_pass(ntt, p, bits, ell, batch):
    _roundtrip_case(ntt, p, bits, ell, batch, seed=ell * 7 + bits, top=True)


@pytest.mark.parametrize("ell,batch", [(4, 9), (9, 7), (12, 5), (13, 3), (14, 2), (15, 2), (16, 1), (20, 1), (24, 1)])
def test_generic_u64_prime(ntt, ell, batch):
    """p = 2305843009146585089 (not 1 mod 2^32): the generic lo64(Qp) path of every kernel."""
    _roundtrip_case(ntt, P62G, 64, ell, batch, seed=500 + ell, top=True)


def test_cross_width_identity(ntt):
    """The same p = 998244353 at beta = 2^32 and 2^64 gives identical outputs."""
    p, ell = P30, 12
    w = root(p, 1 << ell)
    x = rand_residues(np.random.default_rng(9), p, (5, 1 << ell))
    outs = []
    for bits in (32, 64):
        d = to_dev(x, bits)
        ntt.Plan(p, w, ell, bits).forward(d)
        outs.append(to_host(d))
    assert np.array_equal(outs[0], outs[1])


def test_closed_form_delta_and_constant(ntt):
    """Delta -> all ones; constant c -> (Lc, 0, ...) at a multi-pass length."""
    for p, bits, ell in ((P62, 64, 20), (P30, 32, 18)):
        L = 1 << ell
        plan = ntt.Plan(p, root(p, L), ell, bits)
        x = np.zeros((2, L), dtype=np.uint64)
        x[0, 0] = 1
        x[1, :] = 5
        d = to_dev(x, bits)
        plan.forward(d)
        got = to_host(d)
        assert (got[0] == 1).all()
        assert int(got[1, 0]) == 5 * L % p and not got[1, 1:].any()


# ------------------------------------------------------------------ BASELINE configs
def test_config1_single_2p10_u32(ntt):
    """C1: one forward NTT, L = 2^10, beta = 2^32, p = 998244353, seeded uniform input."""
    p, ell = P30, 10
    L = 1 << ell
    w = root(p, L)
    assert w == 258648936
    x = synth.uniform_mod(synth.config_seed(1), 0, 0, L, p)
    d = to_dev(x, 32)
    ntt.Plan(p, w, ell, 32).forward(d)
    got = to_host(d)
    assert np.array_equal(got, oracle.ntt_forward(p, w, x))
    b = oracle.dft_direct(p, w, x)  # the definition
    assert all(int(got[j]) == int(b[bitrev(j, ell)]) for j in range(L))


def test_config2_batched_2p12_u64_fwd_inv(ntt):
    """C2: 4096 transforms of L = 2^12, beta = 2^64; inverse o forward = L x (all 4096)."""
    p, ell, batch = P62, 12, 4096
    L = 1 << ell
    w = root(p, L)
    assert w == 3233568307201063014
    plan = ntt.Plan(p, w, ell, 64)
    d = torch.empty(batch * L, dtype=torch.uint64, device="cuda")
    ntt.synth_uniform(d, synth.config_seed(2), 0, bound=p)
    x = to_host(d).reshape(batch, L)
    plan.forward(d)
    fwd = to_host(d).reshape(batch, L)
    sample = np.r_[0:8, 2040:2048, batch - 8:batch]
    assert np.array_equal(fwd[sample], oracle.ntt_forward(p, w, x[sample], nthreads=NTHREADS))
    plan.inverse(d)
    inv = to_host(d).reshape(batch, L)
    assert np.array_equal(inv, ((x.astype(object) * L) % p).astype(np.uint64))


def test_config3_rns_convolution(ntt):
    """C3: 1024 pairs of 2^15-coefficient polynomials (coeffs < 2^20) zero-padded to 2^16,
    cyclic convolution mod each of the three primes; sampled pairs vs the oracle."""
    ell, npairs, half = 16, 1024, 1 << 15
    L = 1 << ell
    a = torch.zeros(npairs, L, dtype=torch.uint32, device="cuda")
    b = torch.zeros(npairs, L, dtype=torch.uint32, device="cuda")
    ah = synth.uniform_bits(synth.config_seed(3), 0, 0, npairs * half, 20).reshape(npairs, half)
    bh = synth.uniform_bits(synth.config_seed(3), 1, 0, npairs * half, 20).reshape(npairs, half)
    a[:, :half] = torch.from_numpy(ah.astype(np.uint32)).cuda()
    b[:, :half] = torch.from_numpy(bh.astype(np.uint32)).cuda()
    for p in RNS:
        plan = ntt.Plan(p, root(p, L), ell, 32)
        ca, cb = a.clone(), b.clone()
        plan.cyclic_convolve(ca, cb)
        got = to_host(ca)
        for i in (0, 511, npairs - 1):
            pa = np.zeros(L, dtype=np.uint64); pa[:half] = ah[i]
            pb = np.zeros(L, dtype=np.uint64); pb[:half] = bh[i]
            w = root(p, L)
            ref = oracle.ntt_inverse(p, w, oracle.pointwise(p, oracle.ntt_forward(p, w, pa), oracle.ntt_forward(p, w, pb),
                                                            scale_L=L))
            assert np.array_equal(got[i], ref)
            for k in (0, 1, half, L - 2, L - 1):  # the definition, coefficient by coefficient
                assert int(got[i, k]) == oracle.cyclic_conv_coeff(p, pa, pb, k)


def test_config4_batched_2p24_u64(ntt):
    """C4: 64 transforms of L = 2^24 (8 GiB); transforms 0 and 63 fully vs the oracle,
    sampled positions of others by Horner evaluation."""
    p, ell, batch = P62, 24, 64
    L = 1 << ell
    w = root(p, L)
    assert w == 3854271288527505563
    plan = ntt.Plan(p, w, ell, 64)
    d = torch.empty(batch * L, dtype=torch.uint64, device="cuda")
    ntt.synth_uniform(d, synth.config_seed(4), 0, bound=p)
    x0 = to_host(d[:L])
    x63 = to_host(d[63 * L:])
    x17 = to_host(d[17 * L:18 * L])
    plan.forward(d)
    assert np.array_equal(to_host(d[:L]), oracle.ntt_forward(p, w, x0, nthreads=NTHREADS))
    assert np.array_equal(to_host(d[63 * L:]), oracle.ntt_forward(p, w, x63, nthreads=NTHREADS))
    got17 = to_host(d[17 * L:18 * L])
    for j in (0, 1, 12345, L // 2 + 3, L - 1):
        assert int(got17[j]) == oracle.ntt_output_at(p, w, x17, j)


def test_config5_single_2p28_u64(ntt):
    """C5: one forward NTT of L = 2^28 (2 GiB) on one GPU; whole output vs the oracle."""
    p, ell = P62, 28
    L = 1 << ell
    w = root(p, L)
    assert w == 796245258878702573
    plan = ntt.Plan(p, w, ell, 64)
    d = torch.empty(L, dtype=torch.uint64, device="cuda")
    ntt.synth_uniform(d, synth.config_seed(5), 0, bound=p)
    x = to_host(d)
    plan.forward(d)
    got = to_host(d)
    del d
    torch.cuda.empty_cache()
    for j in (0, 1, 7, L // 3, L - 1):
        assert int(got[j]) == oracle.ntt_output_at(p, w, x, j)
    ref = oracle.ntt_forward(p, w, x, nthreads=NTHREADS)
    assert np.array_equal(got, ref)


# ------------------------------------------------------------------ pieces
def test_pointwise(ntt):
    for p, bits in ((P30, 32), (P62, 64)):
        ell = 8
        L = 1 << ell
        plan = ntt.Plan(p, root(p, L), ell, bits)
        rng = np.random.default_rng(3)
        a = rand_residues(rng, 2 * p, (4, L))  # [0,2p) accepted
        b = rand_residues(rng, 2 * p, (4, L))
        a[0, 0] = b[0, 0] = 2 * p - 1
        for scale in (False, True):
            da, db = to_dev(a, bits), to_dev(b, bits)
            dc = torch.empty_like(da)
            plan.pointwise_mul(dc, da, db, scale_inv_L=scale)
            ref = oracle.pointwise(p, a, b, scale_L=L if scale else 0)
            assert np.array_equal(to_host(dc), ref)
        # word-aligned but not 16-byte-aligned views (the scalar path of k_pointwise), and L = 2 with an
        # odd batch (the 16-byte path's tail)
        fa, fb = to_dev(a.reshape(-1), bits), to_dev(b.reshape(-1), bits)
        out = torch.zeros(4 * L + 1, dtype=fa.dtype, device="cuda")
        plan.pointwise_mul(out[1:L + 1], fa[1:L + 1], fb[1:L + 1], batch=1, scale_inv_L=True)
        assert np.array_equal(to_host(out[1:L + 1]),
                              oracle.pointwise(p, a.reshape(-1)[1:L + 1], b.reshape(-1)[1:L + 1], scale_L=L))
        rest = to_host(out)
        assert rest[0] == 0 and not rest[L + 1:].any(), "pointwise wrote outside its view"
        plan2 = ntt.Plan(p, root(p, 2), 1, bits)
        a2, b2 = rand_residues(rng, 2 * p, (7, 2)), rand_residues(rng, 2 * p, (7, 2))
        dc2 = torch.empty(14, dtype=fa.dtype, device="cuda")
        plan2.pointwise_mul(dc2, to_dev(a2, bits), to_dev(b2, bits))
        assert np.array_equal(to_host(dc2).reshape(7, 2), oracle.pointwise(p, a2, b2, scale_L=0))


def test_convolution_inverse_fused_variant(ntt, tmp_path):
    """The alternative cluster-size convolution (product fused into the inverse's load: NTT_CONV_INV_PW, read
    once per process, so run in a child process) equals the default path (product fused into b's forward)."""
    import os
    import subprocess
    import sys
    for bits, p, ell, batch in ((32, RNS[2], 16, 77), (64, P62, 15, 5)):
        L = 1 << ell
        rng = np.random.default_rng(bits + batch)
        a = rand_residues(rng, p, (batch, L))
        b = rand_residues(rng, p, (batch, L))
        np.save(tmp_path / "a.npy", a)
        np.save(tmp_path / "b.npy", b)
        child = (
            "import sys, numpy as np, torch; sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})\n"
            "import paper_1205_2926_b200 as ntt\nfrom gpu_util import root, to_dev, to_host\n"
            "a = np.load({pa!r}); b = np.load({pb!r})\n"
            "plan = ntt.Plan({p}, root({p}, {L}), {ell}, {bits})\n"
            "da, db = to_dev(a, {bits}), to_dev(b, {bits}); plan.cyclic_convolve(da, db)\n"
            "np.save({out!r}, to_host(da))\n"
        ).format(root=os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                 tests=os.path.dirname(os.path.abspath(__file__)), pa=str(tmp_path / "a.npy"),
                 pb=str(tmp_path / "b.npy"), p=p, L=L, ell=ell, bits=bits, out=str(tmp_path / "c.npy"))
        env = dict(os.environ, NTT_CONV_INV_PW="1")
        r = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        alt = np.load(tmp_path / "c.npy")
        plan = ntt.Plan(p, root(p, L), ell, bits)
        da, db = to_dev(a, bits), to_dev(b, bits)
        plan.cyclic_convolve(da, db)
        assert np.array_equal(to_host(da), alt)
        for i in (0, batch - 1):
            for k in (0, L - 1):
                assert int(alt[i, k]) == oracle.cyclic_conv_coeff(p, a[i], b[i], k)


def test_twiddle_table(ntt):
    """A1: W_e = omega^e and W'_e = floor(W_e beta/p), i.e. W' p <= W beta < (W'+1) p."""
    for p, bits, ell in ((P30, 32, 10), (P62, 64, 12), (P62, 64, 20)):
        L = 1 << ell
        w = root(p, L)
        W, Wp = ntt.Plan(p, w, ell, bits).twiddles()
        beta = 1 << bits
        for e in list(range(0, 64)) + list(range(L // 2 - 64, L // 2)):
            We, Wpe = int(W[e]), int(Wp[e])
            assert We == pow(w, e, p)
            assert Wpe * p <= We * beta < (Wpe + 1) * p


@pytest.mark.parametrize("bits,p", [(32, P30), (64, P62), (32, 167772161)])
def test_butterflies_bitexact_vs_paper_model(ntt, bits, p):
    """Each device butterfly reproduces the oracle's step-by-step model of Algorithms
    2-5 exactly (including the redundant representative)."""
    rng = np.random.default_rng(bits)
    n = 1 << 16
    plan = ntt.Plan(p, root(p, 4), 2, bits)
    beta = 1 << bits
    J = pow(p, -1, beta)
    W = rng.integers(1, p, size=n, dtype=np.uint64)
    for alg, in_b in ((2, 1), (3, 2), (4, 4), (5, 2), (31, 2), (41, 4)):
        X = rand_residues(rng, in_b * p, n)
        Y = rand_residues(rng, in_b * p, n)
        X[:4] = [0, in_b * p - 1, 0, in_b * p - 1]
        Y[:4] = [0, 0, in_b * p - 1, in_b * p - 1]
        Wa = np.ones(n, dtype=np.uint64) if alg in (31, 41) else W
        if alg == 5:
            Wp = np.array([(int(w_) * beta) % p for w_ in Wa], dtype=np.uint64)
        else:
            Wp = np.array([(int(w_) * beta) // p for w_ in Wa], dtype=np.uint64)
        dX, dY = to_dev(X, bits), to_dev(Y, bits)
        plan.debug_butterfly(alg, to_dev(Wa, bits), to_dev(Wp, bits), dX, dY)
        gx, gy = to_host(dX), to_host(dY)
        if alg in (31, 41):
            # W = 1 fast paths: congruence + range (their representative differs from Shoup's)
            if alg == 31:
                assert np.array_equal(gx.astype(object) % p, (X.astype(object) + Y) % p)
                assert np.array_equal(gy.astype(object) % p, (X.astype(object) - Y.astype(object)) % p)
                assert (gx < 2 * p).all() and (gy < 2 * p).all()
            else:
                assert np.array_equal(gx.astype(object) % p, (X.astype(object) + Y) % p)
                assert np.array_equal(gy.astype(object) % p, (X.astype(object) - Y.astype(object)) % p)
                assert (gx < 4 * p).all() and (gy < 4 * p).all()
            continue
        ox, oy = oracle.bfly(alg, bits, p, Wa, Wp, X, Y, J=J)
        assert np.array_equal(gx, ox) and np.array_equal(gy, oy), alg


def test_synth_matches_host_generator(ntt):
    for bits, bound, kbits in ((64, P62, 0), (32, P30, 0), (32, 0, 20), (64, 0, 61)):
        d = torch.empty(100_003, dtype=torch.uint64 if bits == 64 else torch.uint32, device="cuda")
        ntt.synth_uniform(d, 77, 5, start=1000, bound=bound, bits=kbits)
        host = (synth.uniform_mod(77, 5, 1000, d.numel(), bound) if bound
                else synth.uniform_bits(77, 5, 1000, d.numel(), kbits))
        assert np.array_equal(to_host(d), host)


def test_edge_cases(ntt):
    import ctypes
    p, ell = P62, 10
    plan = ntt.Plan(p, root(p, 1 << ell), ell, 64)
    d = torch.zeros(1 << ell, dtype=torch.uint64, device="cuda")
    plan.forward(d, batch=0)  # no-op
    lib = ntt.lib()
    # misaligned pointer -> NTT_ERR_ARG
    assert lib.ntt_forward(plan.handle, d.data_ptr() + 8, 1, 0) == -1
    assert lib.ntt_forward(plan.handle, None, 1, 0) == -1
    # ell = 0: identity (only normalisation)
    p0 = ntt.Plan(P30, 1, 0, 32)
    t = to_dev(np.array([5, P30 + 3, 2 * P30 - 1], dtype=np.uint64), 32)
    p0.forward(t)
    assert list(to_host(t)) == [5, 3, P30 - 1]
    # all-(2p-1) input at the edge of Alg. 3's range
    x = np.full((2, 1 << ell), 2 * p - 1, dtype=np.uint64)
    dx = to_dev(x, 64)
    plan.forward(dx)
    assert np.array_equal(to_host(dx), oracle.ntt_forward(p, root(p, 1 << ell), x))


# ---- F3: three-prime CRT
def test_crt3_parity(ntt):
    """ntt_crt3 vs the oracle's textbook CRT on random residues (incl. p-1 and 0), bit-exact, ragged n."""
    rng = np.random.default_rng(21)
    for n in (1, 1000, 100003):
        res = [rng.integers(0, q, n, dtype=np.uint64) for q in RNS]
        for r in res:
            r[0], r[-1] = 0, 0
        res[0][n // 2] = RNS[0] - 1
        res[2][n // 3] = RNS[2] - 1
        d = [torch.from_numpy(r.astype(np.uint32)).cuda() for r in res]
        out = torch.empty(2 * n, dtype=torch.uint64, device="cuda")
        ntt.crt3(out, *d, RNS)
        o = out.cpu().numpy().view(np.uint64).reshape(n, 2)
        got = [int(lo) + (int(hi) << 64) for lo, hi in o]
        idx = list(range(n)) if n <= 1000 else list(rng.integers(0, n, 2000)) + [0, n // 2, n // 3, n - 1]
        want = oracle.crt([r[idx] for r in res], RNS)
        assert [got[i] for i in idx] == want


def test_config3_exact_integer_product(ntt):
    """C3 + F3 end to end: three-prime cyclic convolutions of length 2^16 (2^15 coefficients < 2^20,
    zero-padded) lifted by ntt_crt3 equal numpy's exact integer convolution, on sampled pairs."""
    ell, npairs, half = 16, 16, 1 << 15
    L = 1 << ell
    ah = synth.uniform_bits(synth.config_seed(3), 0, 0, npairs * half, 20).reshape(npairs, half)
    bh = synth.uniform_bits(synth.config_seed(3), 1, 0, npairs * half, 20).reshape(npairs, half)
    a = torch.zeros(npairs, L, dtype=torch.uint32, device="cuda")
    b = torch.zeros(npairs, L, dtype=torch.uint32, device="cuda")
    a[:, :half] = torch.from_numpy(ah.astype(np.uint32)).cuda()
    b[:, :half] = torch.from_numpy(bh.astype(np.uint32)).cuda()
    res = []
    for p in RNS:
        plan = ntt.Plan(p, root(p, L), ell, 32)
        ca, cb = a.clone(), b.clone()
        plan.cyclic_convolve(ca, cb)
        res.append(ca.reshape(-1))
    out = torch.empty(2 * npairs * L, dtype=torch.uint64, device="cuda")
    ntt.crt3(out, *res, RNS)
    o = out.cpu().numpy().view(np.uint64).reshape(npairs, L, 2)
    assert (o[:, :, 1] == 0).all()  # every coefficient < 2^55 < 2^64
    for i in (0, npairs - 1):
        exact = np.convolve(ah[i].astype(np.int64), bh[i].astype(np.int64))
        assert np.array_equal(o[i, :2 * half - 1, 0].astype(np.int64), exact)
        assert (o[i, 2 * half - 1:, 0] == 0).all()


@pytest.mark.parametrize("p,bits,ell,batch", [(P62, 64, 15, 1), (P62, 64, 15, 149), (P62G, 64, 15, 75),
                                               (P30, 32, 16, 1), (P30, 32, 16, 149)])
def test_cluster_sizes_ragged_batches(ntt, p, bits, ell, batch):
    """The 2-CTA cluster kernel (k_splitk) over batches that are not whole waves of its 74 clusters (one
    transform; two waves plus one): first, middle and last transforms whole against the oracle (forward),
    every transform through inverse o forward = L x."""
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(batch * L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(4), batch, bound=p)
    xh = x.cpu().numpy().astype(np.uint64).reshape(batch, L)
    plan.forward(x)
    fh = x.cpu().numpy().astype(np.uint64).reshape(batch, L)
    picks = sorted({0, batch // 2, batch - 1})
    ref = oracle.ntt_forward(p, w, xh[picks], nthreads=NTHREADS)
    assert np.array_equal(fh[picks], ref)
    plan.inverse(x)
    got = x.cpu().numpy().astype(np.uint64).reshape(batch, L).astype(object)
    assert np.array_equal(got, (xh.astype(object) * L) % p)


@pytest.mark.parametrize("ell", [22, 24, 26])
def test_u32_long_transforms(ntt, ell):
    """beta = 2^32 up to the longest length its primes allow (p = 469762049 = 7*2^26+1, so 2^26): the
    three-pass schedules.  Sampled outputs by Horner evaluation, inverse o forward = L x exactly."""
    p = RNS[0]
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, 32)
    x = torch.empty(L, dtype=torch.uint32, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(3), 7, bound=p)
    xh = x.cpu().numpy().astype(np.uint64)
    plan.forward(x)
    fh = x.cpu().numpy().astype(np.uint64)
    rng = np.random.default_rng(ell)
    for j in [0, 1, L // 2, L - 1] + [int(v) for v in rng.integers(0, L, 4)]:
        assert int(fh[j]) == oracle.ntt_output_at(p, w, xh, j), j
    plan.inverse(x)
    assert np.array_equal(x.cpu().numpy().astype(np.uint64), (xh * np.uint64(L)) % np.uint64(p))


@pytest.mark.parametrize("ell", [25, 27])
def test_u64_three_pass_lengths(ntt, ell):
    """beta = 2^64 lengths with three-pass schedules ([7,6,12], [8,7,12]): Horner-sampled outputs and
    inverse o forward = L x on a 2^17-position sample."""
    p = P62
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, 64)
    info = plan.info()
    assert info.n_passes == 3
    x = torch.empty(L, dtype=torch.uint64, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(4), 9, bound=p)
    xh = x.cpu().numpy()
    plan.forward(x)
    fh = x.cpu().numpy()
    rng = np.random.default_rng(ell)
    for j in [0, 1, L - 1] + [int(v) for v in rng.integers(0, L, 3)]:
        assert int(fh[j]) == oracle.ntt_output_at(p, w, xh, j), j
    plan.inverse(x)
    ih = x.cpu().numpy()
    idx = rng.integers(0, L, 1 << 17)
    assert all(int(ih[i]) == int(xh[i]) * L % p for i in idx)


def test_range_checking_mode(ntt):
    """ntt_set_range_checks: inputs outside Algorithm 3's [0,2p) / Algorithm 4's [0,4p)
    are refused with NTT_ERR_RANGE and left untouched; the tops of the ranges are accepted."""
    p, ell = P62, 12
    plan = ntt.Plan(p, root(p, 1 << ell), ell, 64)
    prev = ntt.set_range_checks(True)
    try:
        x = np.full((2, 1 << ell), 2 * p - 1, dtype=np.uint64)
        d = to_dev(x, 64)
        plan.forward(d)  # 2p - 1 is legal
        x[1, 77] = 2 * p
        d = to_dev(x, 64)
        with pytest.raises(ntt.NttError) as ei:
            plan.forward(d)
        assert ei.value.status == -9
        assert np.array_equal(to_host(d), x)  # untouched
        y = np.full((1, 1 << ell), 4 * p - 1, dtype=np.uint64)
        dy = to_dev(y, 64)
        plan.inverse(dy)  # 4p - 1 is legal for Algorithm 4
        y[0, 5] = 4 * p
        dy = to_dev(y, 64)
        with pytest.raises(ntt.NttError):
            plan.inverse(dy)
    finally:
        ntt.set_range_checks(prev)


@pytest.mark.parametrize("bits,p,ell,batch,buf_transforms", [
    (64, P62, 12, 4096, 2048), (64, P62, 12, 37, 1), (32, P30, 10, 1000, 7), (64, P62, 18, 3, 1), (32, RNS[0], 16, 5, 2),
])
def test_execute_host_pipeline(ntt, bits, p, ell, batch, buf_transforms):
    """ntt_execute_host (host buffers in and out, H2D / transforms / D2H pipelined over a device ring):
    forward, inverse and both, bit-exact with the device-resident calls, for ragged chunkings down to
    a one-transform device buffer."""
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits)
    dt = torch.uint64 if bits == 64 else torch.uint32
    x = torch.empty(batch * L, dtype=dt, device="cuda")
    ntt.synth_uniform(x, synth.config_seed(2), 11, bound=p)
    h_in = x.cpu().pin_memory()
    dbuf = torch.empty(buf_transforms * L, dtype=dt, device="cuda")
    ref_f = x.clone()
    plan.forward(ref_f)
    ref_fi = ref_f.clone()
    plan.inverse(ref_fi)
    ref_i = x.clone()
    plan.inverse(ref_i)
    for ops, ref in ((ntt.NTT_OP_FORWARD, ref_f), (ntt.NTT_OP_INVERSE, ref_i),
                     (ntt.NTT_OP_FORWARD | ntt.NTT_OP_INVERSE, ref_fi)):
        h_out = torch.empty_like(h_in).pin_memory()
        plan.execute_host(ops, h_in, h_out, dbuf)
        torch.cuda.synchronize()
        assert torch.equal(h_out.view(torch.int64 if bits == 64 else torch.int32),
                           ref.cpu().view(torch.int64 if bits == 64 else torch.int32)), ops


@pytest.mark.parametrize("bits,p,ell,batch", [(64, P62, 12, 9), (64, P62, 17, 2), (32, P30, 11, 5),
                                               (64, P62, 15, 77), (64, P62G, 15, 3), (32, RNS[1], 16, 75)])
def test_cyclic_convolution_other_shapes(ntt, bits, p, ell, batch):
    """ntt_cyclic_convolve beyond C3's shape (single-pass u64, multi-pass with separate pointwise): each
    pair against the oracle's per-coefficient definition on sampled k and the oracle NTT route."""
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits)
    rng = np.random.default_rng(ell + bits)
    a = rand_residues(rng, p, (batch, L))
    b = rand_residues(rng, p, (batch, L))
    da, db = to_dev(a, bits), to_dev(b, bits)
    plan.cyclic_convolve(da, db)
    got = to_host(da)
    for i in (0, batch - 1):
        ref = oracle.ntt_inverse(p, w, oracle.pointwise(p, oracle.ntt_forward(p, w, a[i]), oracle.ntt_forward(p, w, b[i]),
                                                        scale_L=L))
        assert np.array_equal(got[i], ref)
        for k in (0, 1, L // 2, L - 1):
            assert int(got[i, k]) == oracle.cyclic_conv_coeff(p, a[i], b[i], k)


# ---------------------------------------------------------------- pass-by-pass entry point
@pytest.mark.parametrize("p,bits,ell,batch", [(P62, 64, 12, 5), (P62, 64, 20, 2), (P30, 32, 22, 1),
                                              (P62, 64, 25, 1)])
def test_transform_pass_sequence_equals_transform(ntt, p, bits, ell, batch):
    """ntt_transform_pass over the schedule (forward 0..n-1, inverse n-1..0) = ntt_forward / ntt_inverse,
    and the forward equals the oracle (bench.py times multi-pass configs pass by pass)."""
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits)
    n = plan.info().n_passes
    x = rand_residues(np.random.default_rng(ell), p, (batch, L))
    a, b = to_dev(x, bits), to_dev(x, bits)
    plan.forward(a)
    for j in range(n):
        plan.transform_pass(b, j)
    fa = to_host(a)
    assert np.array_equal(fa, to_host(b))
    if L <= 1 << 20:
        assert np.array_equal(fa, oracle.ntt_forward(p, w, x, nthreads=NTHREADS))
    else:
        for j in (0, 1, L - 1, 12345):
            assert int(fa[0, j]) == oracle.ntt_output_at(p, w, x[0], j)
    plan.inverse(a)
    for j in reversed(range(n)):
        plan.transform_pass(b, j, inverse=True)
    assert np.array_equal(to_host(a), to_host(b))
    with pytest.raises(ntt.NttError):
        plan.transform_pass(b, n)


def _check_pairs(pairs, want_w, p, beta, idx):
    """(W, W') pairs at sampled indices: W = want_w(i), W' p <= W beta < (W'+1) p."""
    for i in idx:
        We, Wpe = int(pairs[i, 0]), int(pairs[i, 1])
        assert We == want_w(i), i
        assert Wpe * p <= We * beta < (Wpe + 1) * p, i


@pytest.mark.parametrize("p,bits,ell", [(P62, 64, 24), (P62, 64, 28), (P30, 32, 20), (P62, 64, 15)])
def test_device_resident_tables(ntt, p, bits, ell):
    """A1 on the tables the kernels actually read (ntt_plan_table): every pass's per-stage table
    (stage i: zeta_i^k for k <= N >> i, the extra entry -1 included), the four-step factors and the
    twiddle matrix of every column pass, checked entry by entry (sampled for the 2^20+ ones)."""
    import random
    L = 1 << ell
    w = root(p, L)
    beta = 1 << bits
    plan = ntt.Plan(p, w, ell, bits)
    info = plan.info()
    sched = [info.pass_log2[i] for i in range(info.n_passes)]
    rng = random.Random(ell)
    outer = 0
    for j, n in enumerate(sched):
        N = 1 << n
        rootN = pow(w, L // N, p)
        t = plan.table(0, j)
        assert t.shape[0] == N - 1 + n
        for i in range(1, n + 1):
            off = N - (N >> (i - 1)) + (i - 1)
            zeta = pow(rootN, 1 << (i - 1), p)
            m = N >> i
            ks = range(m + 1) if m < 4096 else [0, 1, m - 1, m] + rng.sample(range(m), 500)
            _check_pairs(t, lambda e, off=off, zeta=zeta: pow(zeta, e - off, p), p, beta, [off + k for k in ks])
            assert int(t[off + m, 0]) == p - 1  # zeta_i^{m_i} = -1: the inverse's negated entries rely on it
        if j + 1 < len(sched):
            lb = ell - outer
            B = 1 << lb
            wB = pow(w, L >> lb, p)
            fa, fb = plan.table(1, j), plan.table(2, j)
            H = int(fb.shape[0]).bit_length() - 1
            if fa.shape[0] == B and fb.shape[0] == B:
                H = 0  # direct table
            if H:
                _check_pairs(fb, lambda e: pow(wB, e, p), p, beta, range(fb.shape[0]))
                _check_pairs(fa, lambda e: pow(wB, e << H, p), p, beta,
                             rng.sample(range(fa.shape[0]), min(2000, fa.shape[0])))
            else:
                _check_pairs(fa, lambda e: pow(wB, e, p), p, beta, rng.sample(range(B), min(4000, B)))
            try:
                M = plan.table(3, j)
            except ntt.NttError:
                M = None
            if M is not None:
                S = B >> n
                assert M.shape[0] == N * S
                idx = rng.sample(range(N * S), 3000) + [0, S - 1, (N - 1) * S, N * S - 1]
                _check_pairs(M, lambda e: pow(wB, (e % S) * bitrev(e // S, n), p), p, beta, idx)
            outer += n


def test_device_resident_tables_alg5(ntt):
    """F2 tables hold one word W'_mont = beta W mod p per entry: per-stage, factors, matrix."""
    import random
    p, bits, ell = P62, 64, 24
    L = 1 << ell
    w = root(p, L)
    plan = ntt.Plan(p, w, ell, bits, butterfly=5)
    beta = 1 << bits
    n0, n1 = plan.info().pass_log2[0], plan.info().pass_log2[1]
    t = plan.table(0, 1)  # the row pass's per-stage table (one word per entry)
    N = 1 << n1
    rootN = pow(w, L // N, p)
    assert t.shape[0] == N - 1 + n1
    for k in range(0, N // 2 + 1, 97):
        assert int(t[k]) == pow(rootN, k, p) * beta % p
    M = plan.table(3, 0)
    S = L >> n0
    for e in random.Random(3).sample(range(M.shape[0]), 2000):
        assert int(M[e]) == pow(w, (e % S) * bitrev(e // S, n0), p) * beta % p


def test_execute_host_threads_share_a_plan(ntt):
    """ntt_execute_host from several host threads on one plan (the header's thread-safety contract):
    each call enqueues its whole pipeline under the plan's lock, on its own stream and device buffer,
    and every result equals the device-resident transform."""
    import threading
    p, bits, ell, batch = P62, 64, 12, 300
    L = 1 << ell
    plan = ntt.Plan(p, root(p, L), ell, bits)
    nthr = 4
    xs, refs, outs, errs = [], [], [], []
    for i in range(nthr):
        x = torch.empty(batch * L, dtype=torch.uint64, device="cuda")
        ntt.synth_uniform(x, synth.config_seed(2), 40 + i, bound=p)
        r = x.clone()
        plan.forward(r)
        xs.append(x.cpu().pin_memory())
        refs.append(r.cpu())
        outs.append(torch.empty_like(xs[-1]).pin_memory())
    torch.cuda.synchronize()

    def work(i):
        try:
            s = torch.cuda.Stream()
            dbuf = torch.empty(16 * L, dtype=torch.uint64, device="cuda")
            for _ in range(3):
                plan.execute_host(ntt.NTT_OP_FORWARD, xs[i], outs[i], dbuf, stream=s)
            s.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(nthr)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(nthr):
        assert torch.equal(outs[i].view(torch.int64), refs[i].view(torch.int64)), i
