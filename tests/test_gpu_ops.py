"""GPU parity of the individual sm_100a operators against the oracle / numpy (fp64)."""

import numpy as np
import pytest
import torch

from conftest import golden_cores, load_golden, rel
from oracle import tenring_oracle as O

pytestmark = pytest.mark.gpu

SMALL = ["spec_n3_i30_r3", "nonuni_n4", "n5_i6", "n2_mat", "odd_n3"]


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


@pytest.mark.parametrize("P,M,K,N,ak", [
    (1, 128, 64, 64, True), (1, 300, 77, 50, True), (1, 1000, 1000, 400, True), (1, 37, 5000, 25, True),
    (3, 70, 33, 100, False), (1, 513, 129, 8, False), (2, 64, 4096, 24, True), (1, 257, 31, 1, True),
    (1, 100, 100, 112, False), (1, 5, 3, 7, True),
])
def test_gemm_engine(P, M, K, N, ak):
    import device_ops as ops
    rng = np.random.default_rng(P * 1000 + M + K + N)
    if ak:
        a = rng.standard_normal((P, M, K))
        sAp, sAm, sAk = M * K, K, 1
    else:
        a = rng.standard_normal((P, K, M))
        sAp, sAm, sAk = M * K, 1, M
    b = rng.standard_normal((K, N))
    ref = np.einsum("pmk,kn->pmn", a if ak else a.transpose(0, 2, 1), b)
    C = torch.zeros(P * M * N, dtype=torch.float64, device="cuda")
    ops.gemm(cuda(a), sAp, sAm, sAk, P, M, K, N, cuda(b), N, C, [M * N, 1 << 30, 0, N, 1 << 30, 0, 1])
    got = C.cpu().numpy().reshape(P, M, N)
    assert rel(got, ref) < 1e-14


def test_gemm_cmap_scatter_and_beta():
    import device_ops as ops
    rng = np.random.default_rng(3)
    M, K, N = 12, 9, 6  # m = (m1, m2) with M2 = 4; n = (n1, n2) with N2 = 3
    a, b = rng.standard_normal((M, K)), rng.standard_normal((K, N))
    ref = (a @ b).reshape(3, 4, 2, 3)  # [m1][m2][n1][n2]
    out = np.zeros((2, 4, 3, 3))       # dst [n1][m2][n2][m1]
    cm = [0, 4, 1, 3 * 3, 3, 4 * 3 * 3, 3]
    C = cuda(out)
    ops.gemm(cuda(a), 0, K, 1, 1, M, K, N, cuda(b), N, C, cm)
    ops.gemm(cuda(a), 0, K, 1, 1, M, K, N, cuda(b), N, C, cm, beta=1)
    np.testing.assert_allclose(C.cpu().numpy(), 2 * ref.transpose(2, 1, 3, 0), rtol=1e-14, atol=1e-13)


@pytest.mark.parametrize("name", SMALL)
def test_mttsp_every_mode(name):
    import device_ops as ops
    g = load_golden(name)
    dims = tuple(int(d) for d in g["dims"])
    N = len(dims)
    init = golden_cores(g, "init", N)
    x = cuda(g["x"])
    cores = [cuda(c) for c in init]
    for n in range(N):
        got = ops.mttsp(x, cores, n).cpu().numpy()
        assert rel(got, g[f"mttsp_{n}"]) < 1e-13, n


@pytest.mark.parametrize("dims,ranks", [((40, 30, 50), (5, 4, 6)), ((12, 10, 9, 11), (3, 4, 2, 5)),
                                        ((6, 5, 7, 4, 6), (2, 3, 2, 2, 3)), ((64, 64, 64, 64), (8, 8, 8, 8))])
def test_mttsp_random_shapes(dims, ranks):
    import device_ops as ops
    rng = np.random.default_rng(len(dims))
    x = rng.standard_normal(dims)
    cores = O.gaussian_ring(dims, ranks, O.philox(1))
    xt, ct = cuda(x), [cuda(c) for c in cores]
    for n in range(len(dims)):
        assert rel(ops.mttsp(xt, ct, n).cpu().numpy(), O.mttsp(x, cores, n)) < 1e-13


@pytest.mark.parametrize("name", SMALL)
def test_coefficient_gram(name):
    import device_ops as ops
    g = load_golden(name)
    N = len(g["dims"])
    cores = [cuda(c) for c in golden_cores(g, "init", N)]
    for n in range(N):
        assert rel(ops.coefficient_gram(cores, n).cpu().numpy(), g[f"S_{n}"]) < 1e-13


@pytest.mark.parametrize("m,rows", [(4, 7), (25, 100), (64, 64), (100, 500), (400, 160), (9, 3), (130, 33),
                                    (152, 20), (153, 41), (200, 7), (257, 300), (625, 64)])
def test_cholesky_solve(m, rows):
    import device_ops as ops
    rng = np.random.default_rng(m)
    a = rng.standard_normal((3 * m, m))
    s = a.T @ a
    rhs = rng.standard_normal((rows, m))
    f = ops.cholesky(cuda(s))
    assert f.info.cpu().numpy().tolist() == [0] * 6
    ref_u = np.linalg.cholesky(s).T
    assert rel(f.U.cpu().numpy(), ref_u) < 1e-12
    if m <= 112:
        assert rel(f.L.cpu().numpy(), np.linalg.inv(ref_u)) < 1e-10  # F = U^{-1}
    else:
        assert rel(f.L.cpu().numpy(), ref_u.T) < 1e-12               # F = U^T
    z = ops.chol_solve(f, cuda(rhs)).cpu().numpy()
    zref, _ = O.solve_spd_right(s, rhs)
    assert rel(z, zref) < 1e-11


@pytest.mark.parametrize("m", [4, 300])
def test_cholesky_flags(m):
    import device_ops as ops
    d = np.ones(m)
    d[2] = -1.0
    _, _, info = ops.cholesky(cuda(np.diag(d)))
    assert info.cpu().numpy()[0] == 3  # first non-positive pivot, 1-based
    s = np.eye(m)
    s[0, 2] = 1e-3
    _, _, info = ops.cholesky(cuda(s))
    assert info.cpu().numpy()[1] == 1  # asymmetric beyond 1e-8
    d = np.ones(m)
    d[1] = 1e-30
    _, _, info = ops.cholesky(cuda(np.diag(d)), check_degen=True)
    assert info.cpu().numpy()[2] == 2  # below the 1e-13 floor


def test_sumsq_and_error_terms():
    import device_ops as ops
    rng = np.random.default_rng(5)
    x = rng.standard_normal(1_000_003)
    out = ops.sumsq(cuda(x)).cpu().numpy()
    assert abs(out[0] - np.dot(x, x)) < 1e-10 * np.dot(x, x) and out[1] == 0
    x[[5, 77, 1_000_002]] = [np.nan, np.inf, -np.inf]
    assert ops.sumsq(cuda(x)).cpu().numpy()[1] == 3
    m, rows = 36, 50
    a = rng.standard_normal((90, m))
    s = a.T @ a
    z = rng.standard_normal((rows, m))
    M = z @ s + 1e-3 * rng.standard_normal((rows, m))
    x2 = torch.tensor([1e4], dtype=torch.float64, device="cuda")
    out = ops.error_terms(cuda(M), cuda(z), cuda(s), x2).cpu().numpy()
    cross, model = float(np.vdot(M, z)), float(np.vdot(s, z.T @ z))
    assert abs(out[1] - cross) < 1e-10 * abs(cross)
    assert abs(out[2] - model) < 1e-10 * abs(model)
    assert abs(out[0] - O.residual_from_sweep(100.0, cross, model)) < 1e-12


@pytest.mark.parametrize("dims,ranks", [((9, 8, 7), (2, 3, 4)), ((6, 5, 4, 7), (3, 2, 2, 3)),
                                        ((5, 4, 3, 4, 3), (2, 2, 3, 2, 2)), ((30, 40), (3, 2))])
def test_reconstruct_and_exact_residual(dims, ranks):
    from paper_2210_11362_b200 import _lib as L
    from paper_2210_11362_b200.synthetic import reconstruct_device
    cores = O.gaussian_ring(dims, ranks, O.philox(4))
    ref = O.dense_from_ring(cores)
    got = reconstruct_device(cores).cpu().numpy()
    assert rel(got, ref) < 1e-13
    # exact error through the fused residual == ||x - dense|| / ||x||
    x = ref + 0.05 * np.random.default_rng(1).standard_normal(dims)
    from engine_driver import run_engine
    N = len(dims)
    _, errs, eng = run_engine(x, list(ranks), "ne", cores, 1, device="cuda", lib=None, exact=True)
    # after one sweep the cores changed: compare with the oracle's exact error for those cores
    ocores, orep = O.solve(x, "ne", O.Config(ranks=ranks, max_iters=1, init_cores=cores, error_mode="exact"))
    assert abs(errs[0] - orep.errors[0]) < 1e-12


@pytest.mark.parametrize("pre,post,side,r_lo,r_hi,leaf", [
    (300, 77, 0, 3, 5, 0), (77, 300, 1, 4, 4, 0), (5, 13, 0, 2, 2, 1), (13, 5, 1, 2, 3, 1),
    (129, 1000, 1, 20, 20, 0), (1000, 129, 0, 11, 9, 0), (1600, 4000, 0, 8, 8, 0), (4000, 1600, 1, 8, 8, 1),
    (200, 70000, 0, 8, 8, 0), (70000, 150, 1, 6, 8, 0),
])
def test_env_oz_matches_f64(pre, post, side, r_lo, r_hi, leaf):
    """fp32 variant product path: the int8-tensor-core digit-sliced environment product
    (tcgen05 kind::i8, exact int32 accumulation) against the fp64 one on the same fp32 X:
    tails in every dimension, N tiles, split-K incl. the forced K > 32768 split, leaf CMap.
    Slicing keeps 28 bits below each row max (truncated digits: random ~2^-28 x max/|x|
    per element), so the product is good to a few 1e-8, below fp32 rounding itself (6e-8)."""
    from paper_2210_11362_b200 import _lib as L
    from fake_trals import oz_offsets
    lib = L.lib()
    rng = np.random.default_rng(pre + post + r_lo)
    x32 = torch.from_numpy(rng.standard_normal((pre, post)).astype(np.float32)).cuda()
    K = post if side == 0 else pre
    rows = pre if side == 0 else post
    H = cuda(rng.standard_normal((K, r_lo * r_hi)))
    digits = torch.empty(lib.trals_oz_digits_bytes(rows, K), dtype=torch.int8, device="cuda")
    exps = torch.empty(rows, dtype=torch.int32, device="cuda")
    s = int(torch.cuda.current_stream().cuda_stream)
    sws = torch.empty(lib.trals_oz_split_ws_elems(pre, post, side), dtype=torch.float64, device="cuda")
    L.check(lib.trals_oz_split_f32(x32.data_ptr(), pre, post, side, digits.data_ptr(), exps.data_ptr(),
                                   sws.data_ptr(), sws.numel(), s), "oz_split")
    n_out = rows * r_lo * r_hi
    ref = torch.empty(n_out, dtype=torch.float64, device="cuda")
    got = torch.empty(n_out, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(lib.trals_gemm_ws_elems(1, rows, K, r_lo * r_hi), 1 << 22), dtype=torch.float64, device="cuda")
    x64 = x32.double()
    L.check(lib.trals_env_f64(x64.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi, ref.data_ptr(), leaf,
                              ws.data_ptr(), ws.numel(), s), "env_f64")
    wso = torch.empty(lib.trals_env_oz_ws_elems(pre, post, side, r_lo, r_hi), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_oz(digits.data_ptr(), exps.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi,
                             got.data_ptr(), leaf, wso.data_ptr(), wso.numel(), s), "env_oz")
    torch.cuda.synchronize()
    # the tiled, swizzled digits rebuild X to 28 bits below each row's max
    if rows * K <= 4_000_000:
        buf = digits.cpu().numpy()
        a = sum(buf[oz_offsets(rows, K, j)].astype(np.float64) * 2.0 ** (-7 * (j + 1)) for j in range(4))
        a = np.ldexp(a, exps.cpu().numpy().astype(np.int64)[:, None])
        xs = x64.cpu().numpy() if side == 0 else x64.cpu().numpy().T
        assert np.max(np.abs(a - xs) / np.abs(xs).max(axis=1, keepdims=True)) < 2.0 ** -27
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) < 5e-8


def _oz64_env(lib, x64, pre, post, side, H, r_lo, r_hi, leaf, s):
    from paper_2210_11362_b200 import _lib as L
    K = post if side == 0 else pre
    rows = pre if side == 0 else post
    digits = torch.empty(lib.trals_oz64_digits_bytes(rows, K), dtype=torch.int8, device="cuda")
    exps = torch.empty(rows, dtype=torch.int32, device="cuda")
    sws = torch.empty(lib.trals_oz_split_ws_elems(pre, post, side), dtype=torch.float64, device="cuda")
    L.check(lib.trals_oz64_split_f64(x64.data_ptr(), pre, post, side, digits.data_ptr(), exps.data_ptr(),
                                     sws.data_ptr(), sws.numel(), s), "oz64_split")
    got = torch.empty(rows * r_lo * r_hi, dtype=torch.float64, device="cuda")
    wso = torch.empty(lib.trals_env_oz64_ws_elems(pre, post, side, r_lo, r_hi), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_oz64(digits.data_ptr(), exps.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi,
                               got.data_ptr(), leaf, wso.data_ptr(), wso.numel(), s), "env_oz64")
    return got, digits, exps


@pytest.mark.gpu
@pytest.mark.parametrize("pre,post,side,r_lo,r_hi,leaf", [
    (300, 77, 0, 3, 5, 0), (77, 300, 1, 4, 4, 0), (5, 13, 0, 2, 2, 1), (13, 5, 1, 2, 3, 1),
    (129, 1000, 1, 20, 20, 0), (1000, 129, 0, 11, 9, 0), (1600, 4000, 0, 8, 8, 0), (4000, 1600, 1, 8, 8, 1),
    (200, 70000, 0, 8, 8, 0), (70000, 150, 1, 6, 8, 0), (640, 640, 0, 20, 20, 1),
    (160000, 200, 0, 8, 8, 0),  # short K with many tiles: 64-wide n-tiles, permuted columns
])
def test_env_oz64_matches_f64(pre, post, side, r_lo, r_hi, leaf):
    """fp64 environment product on the int8 tensor cores (7 balanced radix-254 digits, levels
    0..6) against the DMMA one on the same X: tails in every dimension, all N tiles, split-K
    incl. the forced K > 18944 splits (fix-up pair and multi-split), leaf CMap.  The digits
    rebuild X to 2^-55.9 of each row's 2^e (< 2 x its max); the products agree to the fp64
    rounding level."""
    from paper_2210_11362_b200 import _lib as L
    from fake_trals import oz_offsets
    lib = L.lib()
    rng = np.random.default_rng(pre + post + r_lo + 1)
    x64 = cuda(rng.standard_normal((pre, post)) * np.exp(rng.standard_normal((pre, post))))
    K = post if side == 0 else pre
    rows = pre if side == 0 else post
    H = cuda(rng.standard_normal((K, r_lo * r_hi)))
    s = int(torch.cuda.current_stream().cuda_stream)
    ref = torch.empty(rows * r_lo * r_hi, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(lib.trals_gemm_ws_elems(1, rows, K, r_lo * r_hi), 1 << 22), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_f64(x64.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi, ref.data_ptr(), leaf,
                              ws.data_ptr(), ws.numel(), s), "env_f64")
    got, digits, exps = _oz64_env(lib, x64, pre, post, side, H, r_lo, r_hi, leaf, s)
    torch.cuda.synchronize()
    if rows * K <= 4_000_000:
        buf = digits.cpu().numpy()
        d = [buf[oz_offsets(rows, K, j, digits=7, bk=32)].astype(np.longdouble) for j in range(7)]
        assert max(np.abs(v).max() for v in d) <= 127
        # rebuilt in x87 extended precision: x = 2^e (d_0 + (d_1 + ...) / 254) / 127
        a = d[6]
        for j in range(5, -1, -1):
            a = d[j] + a / np.longdouble(254)
        a = a / np.longdouble(127) * np.longdouble(2.0) ** exps.cpu().numpy().astype(np.int64)[:, None]
        xs = (x64.cpu().numpy() if side == 0 else x64.cpu().numpy().T).astype(np.longdouble)
        # remainder <= 2^-55.9 2^e and 2^e < 2 max|x|
        assert float(np.max(np.abs(a - xs) / np.abs(xs).max(axis=1, keepdims=True))) <= 2.0 ** -54.5
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("heavy", [False, True])
def test_env_oz64_accuracy(heavy):
    """The Ozaki product is as accurate as the DMMA one: both against an extended-precision
    (x87 80-bit) product of the same operands, at the c5 contraction length K = 25600 and
    R^2 = 400 columns (relative Frobenius error; fp64 rounding gives ~7e-16 here)."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(11 + heavy)
    pre, post, r = 64, 25600, 20
    x = rng.standard_normal((pre, post))
    if heavy:
        x *= np.exp(0.5 * rng.standard_normal((pre, post)))
    h = rng.standard_normal((post, r * r))
    exact = (x.astype(np.longdouble) @ h.astype(np.longdouble))  # [pre][r_lo r_hi] rows
    x64, H = cuda(x), cuda(h)
    s = int(torch.cuda.current_stream().cuda_stream)
    ref = torch.empty(pre * r * r, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(lib.trals_gemm_ws_elems(1, pre, post, r * r), 1 << 22), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_f64(x64.data_ptr(), pre, post, 0, H.data_ptr(), r, r, ref.data_ptr(), 0,
                              ws.data_ptr(), ws.numel(), s), "env_f64")
    got, _, _ = _oz64_env(lib, x64, pre, post, 0, H, r, r, 0, s)
    torch.cuda.synchronize()
    # non-leaf side-0 env layout (CMap of env()): [r_hi][pre][r_lo], H column a r_hi + b
    def unperm(v):
        return v.cpu().numpy().reshape(r, pre, r).transpose(1, 2, 0).reshape(pre, r * r)
    e_dmma = np.linalg.norm((unperm(ref) - exact).astype(np.float64)) / np.linalg.norm(exact.astype(np.float64))
    e_oz = np.linalg.norm((unperm(got) - exact).astype(np.float64)) / np.linalg.norm(exact.astype(np.float64))
    print(f"heavy={heavy}: dmma {e_dmma:.3e}  ozaki {e_oz:.3e}")
    assert e_dmma < 2e-15
    assert e_oz < max(2.0 * e_dmma, 1e-15)


@pytest.mark.gpu
def test_env_oz64_deterministic():
    """Two launches of the split-K (fix-up) int8 environment product give bitwise-identical
    results: the two K halves are added in whichever order they finish, and fp addition
    commutes; the k-block rotation only reorders exact int32 sums."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(5)
    pre, post, r = 2560, 25600, 20
    x64 = cuda(rng.standard_normal((pre, post)))
    H = cuda(rng.standard_normal((post, r * r)))
    s = int(torch.cuda.current_stream().cuda_stream)
    a, _, _ = _oz64_env(lib, x64, pre, post, 0, H, r, r, 0, s)
    b, _, _ = _oz64_env(lib, x64, pre, post, 0, H, r, r, 0, s)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("K", [18944, 18945, 37888, 37889])
def test_env_oz64_kmax_boundaries(K):
    """Contraction lengths at the int32 level-sum bound of the 7-digit scheme (KMAX = 18944
    k per CTA: 7 pairs x 127^2 x 18944 < 2^31) and one past it, for one and two forced
    splits: the product stays at the fp64 rounding level of the DMMA one, so no level sum
    wrapped around."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(K)
    pre, r = 130, 6
    # worst case for the level sums: every digit of every row near the int8 bound
    x = np.where(rng.random((pre, K)) < 0.5, -1.0, 1.0) * (1.0 - 2.0 ** -40 * rng.random((pre, K)))
    x64, H = cuda(x), cuda(np.where(rng.random((K, r * r)) < 0.5, -1.0, 1.0))
    s = int(torch.cuda.current_stream().cuda_stream)
    ref = torch.empty(pre * r * r, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(lib.trals_gemm_ws_elems(1, pre, K, r * r), 1 << 22), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_f64(x64.data_ptr(), pre, K, 0, H.data_ptr(), r, r, ref.data_ptr(), 1,
                              ws.data_ptr(), ws.numel(), s), "env_f64")
    got, _, _ = _oz64_env(lib, x64, pre, K, 0, H, r, r, 1, s)
    torch.cuda.synchronize()
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) < 1e-14


@pytest.mark.gpu
def test_env_oz64_extreme_rows():
    """Rows of zeros, of tiny (1e-300), subnormal (1e-309) and huge (1e300) values, and a
    single nonzero per row: per-row power-of-two scaling keeps every row at full relative accuracy
    (and zero rows exactly zero)."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(3)
    pre, post, r = 64, 300, 5
    x = rng.standard_normal((pre, post))
    x[0] = 0.0
    x[1] *= 1e-300
    x[2] *= 1e300 / 8
    x[3] = 0.0
    x[3, 17] = 3.0
    x[4, ::2] *= 1e-200  # mixed magnitudes within a row: the small half sits below the row's 2^-56
    x[7] *= 1e-309       # subnormal inputs (the slicing scale 2^-e is applied in two exact halves)
    h = rng.standard_normal((post, r * r))
    x64, H = cuda(x), cuda(h)
    s = int(torch.cuda.current_stream().cuda_stream)
    got, _, _ = _oz64_env(lib, x64, pre, post, 0, H, r, r, 1, s)
    torch.cuda.synchronize()
    g = got.cpu().numpy().reshape(pre, r * r)
    exact = (x.astype(np.longdouble) @ h.astype(np.longdouble)).astype(np.float64)
    assert np.all(g[0] == 0.0)
    for i in (1, 2, 3, 5, 6):
        assert np.abs(g[i] - exact[i]).max() <= 1e-14 * np.abs(exact[i]).max(), i
    assert np.abs(g[7] - exact[7]).max() <= 1e-14 * np.abs(exact[7]).max() + 1e-320
    # row 4: accurate relative to its row maximum (the tiny entries are below the digit window)
    assert np.abs(g[4] - exact[4]).max() <= 1e-13 * np.abs(x[4]).max() * np.abs(h).sum(axis=0).max()


# ---------------------------------------------------------------------------
# R0 without V (TR-ALS-QR solvers.py:422-424, Alg. 1 :337-339): double-double Gram chain + Cholesky
# ---------------------------------------------------------------------------
def _r0_gpu(rts, ranks, n):
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    N = len(rts)
    s = int(torch.cuda.current_stream().cuda_stream)
    bufs = [cuda(np.ascontiguousarray(t)) for t in rts]
    E = []
    for j, t in enumerate(rts):
        ra, k, rb = t.shape
        eh = torch.empty(ra * ra * rb * rb, dtype=torch.float64, device="cuda")
        el = torch.empty_like(eh)
        L.check(lib.trals_dd_transfer_f64(bufs[j].data_ptr(), ra, k, rb, eh.data_ptr(), el.data_ptr(), s), "dd_tr")
        E.append((eh, el))
    ra = L.i32_array(ranks)
    m = ranks[n] * ranks[(n + 1) % N]
    out = torch.full((m, m), float("nan"), dtype=torch.float64, device="cuda")
    S = torch.empty((m, m), dtype=torch.float64, device="cuda")
    ws = torch.empty(max(1, lib.trals_dd_r0_ws_elems(N, ra)), dtype=torch.float64, device="cuda")
    L.check(lib.trals_dd_r0_f64(N, n, ra, L.ptr_array([e[0].data_ptr() for e in E]),
                                L.ptr_array([e[1].data_ptr() for e in E]), S.data_ptr(), out.data_ptr(),
                                ws.data_ptr(), ws.numel(), s), "dd_r0")
    return out.cpu().numpy(), S.cpu().numpy()


def _degenerate(r):
    d = np.abs(np.diagonal(r))
    return d.size < r.shape[1] or d.min() <= 1e-13 * np.abs(r).max()


@pytest.mark.parametrize("name", ["spec_n3_i30_r3", "nonuni_n4", "n5_i6", "n2_mat", "odd_n3", "rankdef_n3"])
@pytest.mark.parametrize("variant", ["qr", "als"])
def test_r0_matches_reference(name, variant):
    """The reference's per-mode R0 (qr_economy of V_[2], signs included): to 1e-13 of max|R0| where it
    is full rank; for a rank-deficient V (the reference's R0 is then non-square or has a diagonal below
    the 1e-13 floor, its trailing rows rounding noise) R0^T R0 to 1e-13 and the same degeneracy verdict."""
    g = load_golden(name)
    r0g = load_golden("r0_modes")
    N = len(g["dims"])
    ranks = [int(r) for r in g["ranks"]]
    rts = [r0g[f"{name}_rt_{j}"] if variant == "qr" else g[f"init_{j}"] for j in range(N)]
    for n in range(N):
        want = r0g[f"{name}_{variant}_r0_{n}"]
        got, S = _r0_gpu(rts, ranks, n)
        scale = max(1.0, np.abs(want).max())
        if not _degenerate(want):
            assert np.abs(got - want).max() <= 1e-13 * scale, n
        else:
            gram = want.T @ want
            assert np.abs(got.T @ got - gram).max() <= 1e-13 * max(1.0, np.abs(gram).max()), n
            assert _degenerate(got), n
        assert np.abs(S - want.T @ want).max() <= 1e-13 * max(1.0, np.abs(S).max())


@pytest.mark.parametrize("dims,R", [((40, 40, 40, 40), 20), ((30, 30, 30), 12), ((12, 10, 9, 8, 7), 6)])
def test_r0_large_vs_explicit_qr(dims, R):
    """A c5-shaped R0 (k = 40 < R^2 = 400) against a Householder QR of the explicitly assembled V_[2]
    (the reference's operation), every mode."""
    N = len(dims)
    rng = np.random.default_rng(sum(dims) + R)
    cores = [rng.standard_normal((R, d, R)) for d in dims]
    rts = [O.lateral_qr(c).r_tensor for c in cores]
    for n in range(N):
        _, want = O.qr_signed(O.unfold_cyclic(O.chain_without(rts, n), 1))
        got, _ = _r0_gpu(rts, [R] * N, n)
        assert rel(got, want) < 1e-12, n


def test_r0_resolves_ill_conditioned_v():
    """cond(V) ~ 1e11 (congruent cores): chol(S) in fp64 cannot resolve sigma_min (S squares the
    condition number past 1/eps); the double-double R0 reproduces V's singular values (from an SVD of
    the explicit V_[2]) to the accuracy that SVD itself has, eps sigma_max absolute."""
    rng = np.random.default_rng(9)
    dims, R = (20, 20, 20), 3
    cores = []
    for d in dims:
        base = rng.standard_normal((d, R * R))
        # right-bond columns r_b = 1 nearly equal to r_b = 0 (column r_a + R r_b): the subchain ending in
        # this core gets two nearly equal columns r_n = 0, 1, whatever mode it skips
        base[:, R:2 * R] = base[:, :R] + 1e-11 * base[:, R:2 * R]
        cores.append(O.fold_classical(base, 1, (R, d, R)))
    for n in range(3):
        v = O.unfold_cyclic(O.chain_without(cores, n), 1)
        sv = np.linalg.svd(v, compute_uv=False)
        assert sv[-1] / sv[0] < 1e-9  # genuinely ill-conditioned
        got, _ = _r0_gpu(cores, [R] * 3, n)
        sg = np.linalg.svd(got, compute_uv=False)
        assert np.abs(sg - sv).max() <= 1e-14 * sv[0]
        assert abs(sg[-1] - sv[-1]) <= 1e-3 * sv[-1] + 1e-15 * sv[0]


@pytest.mark.parametrize("m,rows", [(25, 100), (64, 64), (100, 500), (400, 160), (113, 40)])
def test_tri_prepare_and_solve(m, rows):
    """Z R0^T = M R0^{-1} ... i.e. Z = M R0^{-1} R0^{-T} through trals_tri_prepare_f64 + trals_chol_solve_f64."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(m + rows)
    _, r0 = O.qr_signed(rng.standard_normal((2 * m, m)))
    M = rng.standard_normal((rows, m))
    want = M @ np.linalg.inv(r0.T @ r0)
    s = int(torch.cuda.current_stream().cuda_stream)
    U = cuda(r0 + np.tril(rng.standard_normal((m, m)), -1))  # the lower triangle must be ignored
    F = torch.empty((m, m), dtype=torch.float64, device="cuda")
    aux = torch.empty(lib.trals_cholesky_aux_elems(m), dtype=torch.float64, device="cuda")
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    L.check(lib.trals_tri_prepare_f64(U.data_ptr(), m, F.data_ptr(), aux.data_ptr(), 1, info.data_ptr(), s), "tri")
    Md = cuda(M)
    Z = torch.empty((rows, m), dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.trals_chol_solve_ws_elems(rows, m), dtype=torch.float64, device="cuda")
    L.check(lib.trals_chol_solve_f64(U.data_ptr(), F.data_ptr(), aux.data_ptr(), m, Md.data_ptr(), rows,
                                     Z.data_ptr(), ws.data_ptr(), ws.numel(), s), "solve")
    assert rel(Z.cpu().numpy(), want) < 1e-11
    assert int(info[2].item()) == 0
    np.testing.assert_array_equal(np.tril(U.cpu().numpy(), -1), 0.0)


def test_tri_prepare_degeneracy_floor():
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    m = 30
    rng = np.random.default_rng(3)
    _, r0 = O.qr_signed(rng.standard_normal((40, m)))
    r0[17, 17] = 1e-14 * np.abs(r0).max()  # below the 1e-13 floor (linalg.py:96-99)
    U = cuda(r0)
    F = torch.empty((m, m), dtype=torch.float64, device="cuda")
    aux = torch.empty(lib.trals_cholesky_aux_elems(m), dtype=torch.float64, device="cuda")
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    L.check(lib.trals_tri_prepare_f64(U.data_ptr(), m, F.data_ptr(), aux.data_ptr(), 1, info.data_ptr(),
                                      int(torch.cuda.current_stream().cuda_stream)), "tri")
    assert int(info[2].item()) == 18


@pytest.mark.parametrize("Lr,m,mode", [(30, 30, 1), (12, 30, 2), (400, 400, 1)])
def test_tri_fallback_min_norm(Lr, m, mode):
    """linalg.py:104-112 on R0: Z = W pinv(R0)^T with W = M R0^{-1}, i.e. M V Sigma^-2 V^T, cut rcond."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(Lr + m)
    a = rng.standard_normal((max(Lr, 2 * m), m))
    if mode == 1:
        a[:, 5] = a[:, 3]  # rank deficient
    _, r0 = O.qr_signed(a)
    r0 = r0[:Lr]
    rows = 17
    W = rng.standard_normal((rows, Lr))
    M = W @ r0  # M = W R0
    want = W @ np.linalg.pinv(r0, rcond=1e-12).T
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    if mode == 1:
        info[2] = 6
    Z = torch.zeros((rows, m), dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.trals_spd_fallback_ws_elems(rows, m), dtype=torch.float64, device="cuda")
    R0 = cuda(np.ascontiguousarray(r0))
    Md = cuda(M)
    L.check(lib.trals_tri_fallback_f64(R0.data_ptr(), Lr, m, Md.data_ptr(), rows, Z.data_ptr(), info.data_ptr(), mode,
                                       1e-12, ws.data_ptr(), ws.numel(), int(torch.cuda.current_stream().cuda_stream)),
            "tri_fallback")
    assert rel(Z.cpu().numpy(), want) < 1e-9
    inf = info.cpu().numpy()
    assert inf[2] == 0 and inf[3] == (1 if mode == 1 else 0)


# ---------------------------------------------------------------------------
# accuracy guard of the int8 fp64 engine (include/trals.h: trals_oz_range_f64, fp64_gemm="auto")
# ---------------------------------------------------------------------------
def _rho_np(x, side):
    a = np.abs(x if side == 0 else x.T)
    s = a.sum(axis=1)
    return float(np.max(np.where(s > 0, a.max(axis=1) * a.shape[1] / np.where(s > 0, s, 1), 0.0)))


@pytest.mark.parametrize("rows,cols", [(300, 77), (7, 5000), (2000, 33)])
@pytest.mark.parametrize("side", [0, 1])
def test_oz_range_statistic(rows, cols, side):
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(rows + cols + side)
    x = rng.standard_normal((rows, cols))
    x[3] = 0.0
    x[5, 2] = 1e9  # one outlier: rho of that row ~ K
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.trals_oz_range_ws_elems(rows, cols, side), dtype=torch.float64, device="cuda")
    xd = cuda(x)
    L.check(lib.trals_oz_range_f64(xd.data_ptr(), rows, cols, side, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                   int(torch.cuda.current_stream().cuda_stream)), "oz_range")
    assert abs(out.item() - _rho_np(x, side)) <= 1e-12 * _rho_np(x, side)


def test_oz64_guard_adversarial():
    """Small-X x large-H terms dominate: rows of X with a 1e-12 dynamic range multiplied by an H that
    is zero where X is large.  The int8 product (exact to 2^-56.9 of each row's maximum) loses those
    terms; the DMMA product keeps them; the guard statistic flags X, so fp64_gemm="auto" runs it on
    DMMA (solver-level check in tests/test_gpu_solvers.py::test_auto_engine_guard)."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(11)
    pre, post, r = 256, 8192, 4
    x = rng.standard_normal((pre, post)) * 1e-12
    x[:, 0] = 1.0                              # one large entry per row ...
    h = rng.standard_normal((post, r * r))
    h[0] = 0.0                                 # ... that H ignores: the output is made of the small terms
    exact = (x.astype(np.longdouble) @ h.astype(np.longdouble)).astype(np.float64)
    x64, H = cuda(x), cuda(h)
    s = int(torch.cuda.current_stream().cuda_stream)
    got, _, _ = _oz64_env(lib, x64, pre, post, 0, H, r, r, 1, s)
    ref = torch.empty(pre * r * r, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(lib.trals_gemm_ws_elems(1, pre, post, r * r), 1 << 20), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_f64(x64.data_ptr(), pre, post, 0, H.data_ptr(), r, r, ref.data_ptr(), 1,
                              ws.data_ptr(), ws.numel(), s), "env_f64")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    rws = torch.empty(pre, dtype=torch.float64, device="cuda")
    L.check(lib.trals_oz_range_f64(x64.data_ptr(), pre, post, 0, out.data_ptr(), rws.data_ptr(), rws.numel(), s),
            "oz_range")
    torch.cuda.synchronize()
    e_dmma = rel(ref.cpu().numpy().reshape(pre, -1), exact)
    e_oz = rel(got.cpu().numpy().reshape(pre, -1), exact)
    assert e_dmma < 1e-14
    assert e_oz > 1e3 * e_dmma            # the failure mode the guard exists for
    assert out.item() > 2.0 ** 12         # ... and the guard sees it


def test_solve_refinement_on_ill_conditioned_s():
    """m <= 112, cond(S) ~ 1e11 (BASELINE c4's regime): the explicit-inverse solve alone is accurate only to
    ~eps cond(S); the gated refinement step (raised by the factorisation) brings the backward error of
    Z S = M to the level of scipy's cho_solve.  A well-conditioned S leaves the gate closed."""
    import scipy.linalg as sla

    import device_ops as ops
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(4)
    m, rows = 64, 40
    q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    s = (q * np.logspace(0, -11, m)) @ q.T
    s = 0.5 * (s + s.T)
    rhs = rng.standard_normal((rows, m)) @ s  # a consistent right-hand side
    sd, md = cuda(s), cuda(rhs)  # keep the device copies alive while the kernels use them
    f = ops.cholesky(sd)
    assert int(f.info[L.INFO_REFINE].item()) == 1
    z0 = ops.chol_solve(f, md)
    z = z0.clone()
    L.check(lib.trals_solve_refine_f64(f.L.data_ptr(), f.aux.data_ptr(), sd.data_ptr(), m, md.data_ptr(),
                                       rows, z.data_ptr(), f.info.data_ptr(),
                                       int(torch.cuda.current_stream().cuda_stream)), "refine")
    zr = sla.cho_solve(sla.cho_factor(s), rhs.T).T

    def backward(zz):
        return np.linalg.norm(zz @ s - rhs) / (np.linalg.norm(s) * np.linalg.norm(zz))
    assert backward(z.cpu().numpy()) <= 10 * backward(zr) + 1e-16
    assert backward(z.cpu().numpy()) < backward(z0.cpu().numpy())
    # well conditioned: gate closed, Z untouched
    s2 = rng.standard_normal((3 * m, m))
    s2 = s2.T @ s2
    s2d = cuda(s2)
    f2 = ops.cholesky(s2d)
    assert int(f2.info[L.INFO_REFINE].item()) == 0
    z2 = ops.chol_solve(f2, md)
    before = z2.clone()
    L.check(lib.trals_solve_refine_f64(f2.L.data_ptr(), f2.aux.data_ptr(), s2d.data_ptr(), m,
                                       md.data_ptr(), rows, z2.data_ptr(), f2.info.data_ptr(),
                                       int(torch.cuda.current_stream().cuda_stream)), "refine")
    assert torch.equal(z2, before)
