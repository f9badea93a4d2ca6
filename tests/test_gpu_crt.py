"""GPU parity of the CRT form of the int8 engine (csrc/crt_int8_gemm.cuh; fp64 MTTSP
solvers.py:379 as 16 modular int8 GEMMs + an exact 128-bit reconstruction) through the C-ABI."""

import numpy as np
import pytest
import torch

from conftest import rel

pytestmark = pytest.mark.gpu

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _stream():
    return int(torch.cuda.current_stream().cuda_stream)


def _crt_split(lib, x64, pre, post, side):
    from paper_2210_11362_b200 import _lib as L
    K = post if side == 0 else pre
    rows = pre if side == 0 else post
    planes = torch.empty(lib.trals_crt_planes_bytes(rows, K), dtype=torch.int8, device="cuda")
    exps = torch.empty(rows, dtype=torch.int32, device="cuda")
    sws = torch.empty(max(1, lib.trals_crt_split_ws_elems(pre, post, side)), dtype=torch.float64, device="cuda")
    L.check(lib.trals_crt_split_f64(x64.data_ptr(), pre, post, side, planes.data_ptr(), exps.data_ptr(),
                                    sws.data_ptr(), sws.numel(), _stream()), "crt_split")
    return planes, exps


def _crt_env(lib, x64, pre, post, side, H, r_lo, r_hi, leaf):
    from paper_2210_11362_b200 import _lib as L
    rows = pre if side == 0 else post
    planes, exps = _crt_split(lib, x64, pre, post, side)
    got = torch.full((rows * r_lo * r_hi,), float("nan"), dtype=torch.float64, device="cuda")
    need = lib.trals_env_crt_ws_elems(pre, post, side, r_lo, r_hi)
    assert need > 0
    wso = torch.empty(need, dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_crt(planes.data_ptr(), exps.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi,
                              got.data_ptr(), leaf, wso.data_ptr(), wso.numel(), _stream()), "env_crt")
    return got, planes, exps


def _dmma_env(lib, x64, pre, post, side, H, r_lo, r_hi, leaf):
    from paper_2210_11362_b200 import _lib as L
    K = post if side == 0 else pre
    rows = pre if side == 0 else post
    ref = torch.empty(rows * r_lo * r_hi, dtype=torch.float64, device="cuda")
    ws = torch.empty(max(lib.trals_gemm_ws_elems(1, rows, K, r_lo * r_hi), 1 << 22), dtype=torch.float64, device="cuda")
    L.check(lib.trals_env_f64(x64.data_ptr(), pre, post, side, H.data_ptr(), r_lo, r_hi, ref.data_ptr(), leaf,
                              ws.data_ptr(), ws.numel(), _stream()), "env_f64")
    return ref


def _plane_offsets(rows, k):
    """Byte offsets [rows, k] inside one residue plane: [128-row tile][64-k block][128 x 64 B], SWIZZLE_64B."""
    r = np.arange(rows, dtype=np.int64)[:, None]
    kk = np.arange(k, dtype=np.int64)[None, :]
    kblocks = -(-k // 64)
    t, rr, kb, c = r // 128, r % 128, kk // 64, kk % 64
    return (t * kblocks + kb) * (128 * 64) + rr * 64 + (((c >> 4) ^ ((rr >> 1) & 3)) << 4) + (c & 15)


def _crt_rebuild(res):
    """Exact integers from their residues res[i] in [0, p_i) (object arrays of Python ints)."""
    nm = len(res)
    P = 1
    for p in MODULI[:nm]:
        P *= p
    acc = np.zeros(res[0].shape, dtype=object)
    for i, p in enumerate(MODULI[:nm]):
        W = P // p
        q = pow(W % p, -1, p)
        acc = acc + (res[i] % p) * ((W * q) % P)
    acc = acc % P
    return np.where(acc > P // 2, acc - P, acc), P


@pytest.mark.parametrize("pre,post,side,r_lo,r_hi,leaf", [
    (300, 77, 0, 3, 5, 0), (77, 300, 1, 4, 4, 0), (5, 13, 0, 2, 2, 1), (13, 5, 1, 2, 3, 1),
    (129, 1000, 1, 20, 20, 0), (1000, 129, 0, 11, 9, 0), (1600, 4000, 0, 8, 8, 0), (4000, 1600, 1, 8, 8, 1),
    (200, 70000, 0, 8, 8, 0), (70000, 150, 1, 6, 8, 0), (640, 640, 0, 20, 20, 1), (260, 5000, 0, 16, 32, 0),
    (131, 4100, 0, 17, 16, 1),
    (2560, 8192, 0, 20, 20, 0), (6000, 2600, 1, 8, 8, 1),  # more than one wave of work units: tail K split
])
def test_env_crt_matches_f64(pre, post, side, r_lo, r_hi, leaf):
    """CRT environment product against the DMMA one on the same X: tails in every dimension, one and
    two MMA column chunks (R^2 <= 256 / > 256, up to 512 columns), K splits (incl. the forced one for
    K > 33024) and the tail K split of the last partial wave, both sides, both CMaps.  The residue planes rebuild rint(2^s x) exactly, with the
    scaled rows inside the 2^58 norm bound (15 moduli); the products agree to the fp64 rounding level."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    nm = lib.trals_crt_moduli()
    assert 12 <= nm <= 16
    rng = np.random.default_rng(pre + post + r_lo + 1)
    x = rng.standard_normal((pre, post)) * np.exp(rng.standard_normal((pre, post)))
    x64 = cuda(x)
    K = post if side == 0 else pre
    rows = pre if side == 0 else post
    assert lib.trals_crt_supported(rows, K, r_lo * r_hi) == 1
    H = cuda(rng.standard_normal((K, r_lo * r_hi)))
    ref = _dmma_env(lib, x64, pre, post, side, H, r_lo, r_hi, leaf)
    got, planes, exps = _crt_env(lib, x64, pre, post, side, H, r_lo, r_hi, leaf)
    torch.cuda.synchronize()
    if rows * K <= 400_000:
        buf = planes.cpu().numpy().view(np.uint8)
        psize = buf.size // nm
        off = _plane_offsets(rows, K)
        res = [buf[i * psize:(i + 1) * psize][off].astype(np.int64).astype(object) for i in range(nm)]
        for i, p in enumerate(MODULI[:nm]):
            assert max(int(v) for v in res[i].ravel()) < p
        val, _ = _crt_rebuild(res)
        xs = x if side == 0 else x.T
        s = exps.cpu().numpy().astype(np.int64)
        want = np.rint(np.ldexp(xs, s[:, None]))
        assert np.all(np.abs(want) < 2.0 ** 63)
        assert np.array_equal(val, np.vectorize(int, otypes=[object])(want))
        nrm = np.sqrt((want.astype(np.longdouble) ** 2).sum(axis=1)).astype(np.float64)
        bits = lib.trals_crt_row_bits(0)
        assert bits == {15: 58, 16: 62}.get(nm, bits)
        assert np.all(nrm <= 2.0 ** bits) and np.all(nrm[nrm > 0] > 2.0 ** (bits - 2))
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) < 1e-14


@pytest.mark.parametrize("heavy", [False, True])
def test_env_crt_accuracy(heavy):
    """As accurate as the DMMA product: both against an extended-precision (x87 80-bit) product of
    the same operands at the c5 contraction length K = 25600, R^2 = 400."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(11 + heavy)
    pre, post, r = 64, 25600, 20
    x = rng.standard_normal((pre, post))
    if heavy:
        x *= np.exp(0.5 * rng.standard_normal((pre, post)))
    h = rng.standard_normal((post, r * r))
    exact = (x.astype(np.longdouble) @ h.astype(np.longdouble))
    x64, H = cuda(x), cuda(h)
    ref = _dmma_env(lib, x64, pre, post, 0, H, r, r, 0)
    got, _, _ = _crt_env(lib, x64, pre, post, 0, H, r, r, 0)
    torch.cuda.synchronize()

    def unperm(v):  # non-leaf side-0 env layout [r_hi][pre][r_lo], H column a r_hi + b
        return v.cpu().numpy().reshape(r, pre, r).transpose(1, 2, 0).reshape(pre, r * r)
    nx = np.linalg.norm(exact.astype(np.float64))
    e_dmma = np.linalg.norm((unperm(ref) - exact).astype(np.float64)) / nx
    e_crt = np.linalg.norm((unperm(got) - exact).astype(np.float64)) / nx
    print(f"heavy={heavy}: dmma {e_dmma:.3e}  crt {e_crt:.3e}")
    assert e_dmma < 2e-15
    assert e_crt < max(2.0 * e_dmma, 1e-15)


def test_env_crt_exact_on_integers():
    """Integer operands small enough to need no rounding: the CRT product is the exact integer
    product (every output an integer below 2^53), bit for bit."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(2)
    pre, post, r = 200, 4096, 6
    x = rng.integers(-2 ** 18, 2 ** 18, size=(pre, post)).astype(np.float64)
    h = rng.integers(-2 ** 18, 2 ** 18, size=(post, r * r)).astype(np.float64)
    exact = (x.astype(np.int64) @ h.astype(np.int64)).astype(np.float64)  # |.| < 2^48
    got, _, _ = _crt_env(lib, cuda(x), pre, post, 0, cuda(h), r, r, 1)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy().reshape(pre, r * r), exact)


def test_env_crt_deterministic():
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(5)
    pre, post, r = 2560, 25600, 20
    x64 = cuda(rng.standard_normal((pre, post)))
    H = cuda(rng.standard_normal((post, r * r)))
    a, _, _ = _crt_env(lib, x64, pre, post, 0, H, r, r, 0)
    b, _, _ = _crt_env(lib, x64, pre, post, 0, H, r, r, 0)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("K", [33024, 33025])
def test_env_crt_kmax_boundaries(K):
    """Contraction lengths at the int32 bound of one K split (255^2 x 33024 < 2^31) and one past
    it (two splits, residues added mod p before the reconstruction), on rows of +-(1 - tiny): the
    product stays at the fp64 rounding level of the DMMA one, so no int32 sum wrapped around."""
    from paper_2210_11362_b200 import _lib as L
    lib = L.lib()
    rng = np.random.default_rng(K)
    pre, r = 130, 6
    x = np.where(rng.random((pre, K)) < 0.5, -1.0, 1.0) * (1.0 - 2.0 ** -40 * rng.random((pre, K)))
    x64, H = cuda(x), cuda(np.where(rng.random((K, r * r)) < 0.5, -1.0, 1.0))
    ref = _dmma_env(lib, x64, pre, K, 0, H, r, r, 1)
    got, _, _ = _crt_env(lib, x64, pre, K, 0, H, r, r, 1)
    torch.cuda.synchronize()
    assert rel(got.cpu().numpy(), ref.cpu().numpy()) < 1e-14


def test_env_crt_extreme_rows():
    """Rows of zeros, of tiny (1e-300), subnormal (1e-309) and huge (1e300) values, a single
    nonzero per row, and mixed magnitudes inside a row."""
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
    x[4, ::2] *= 1e-200
    x[7] *= 1e-309
    h = rng.standard_normal((post, r * r))
    got, _, _ = _crt_env(lib, cuda(x), pre, post, 0, cuda(h), r, r, 1)
    torch.cuda.synchronize()
    g = got.cpu().numpy().reshape(pre, r * r)
    exact = (x.astype(np.longdouble) @ h.astype(np.longdouble)).astype(np.float64)
    assert np.all(g[0] == 0.0)
    for i in (1, 2, 3, 5, 6):
        assert np.abs(g[i] - exact[i]).max() <= 1e-14 * np.abs(exact[i]).max(), i
    assert np.abs(g[7] - exact[7]).max() <= 1e-14 * np.abs(exact[7]).max() + 1e-320
    # row 4: accurate relative to the row's norm (the tiny entries are below the integer grid)
    assert np.abs(g[4] - exact[4]).max() <= 1e-13 * np.abs(x[4]).max() * np.abs(h).sum(axis=0).max()


@pytest.mark.parametrize("variant", ["ne", "qrne"])
def test_solver_crt_matches_dmma(variant):
    """decompose on the CRT engine (forced: fp64_gemm="crt") against the DMMA engine on a ring large
    enough to exercise the environment tree: errors to 1e-12, cores to 1e-9."""
    from paper_2210_11362_b200 import AlsConfig, decompose
    rng = np.random.default_rng(4)
    dims, ranks = (24, 20, 22, 18), (3, 4, 3, 2)
    cores = [rng.standard_normal((ranks[j], dims[j], ranks[(j + 1) % 4])) for j in range(4)]
    x = np.einsum("aib,bjc,ckd,dla->ijkl", *cores)
    x = cuda(x + 1e-3 * np.linalg.norm(x) / np.sqrt(x.size) * rng.standard_normal(x.shape))
    cfg = dict(ranks=ranks, max_iters=6, seed=1, error_mode="exact")
    cc, rc = decompose(x, variant, AlsConfig(fp64_gemm="crt", **cfg))
    cd, rd = decompose(x, variant, AlsConfig(fp64_gemm="dmma", **cfg))
    np.testing.assert_allclose(rc.errors, rd.errors, rtol=0, atol=1e-12)
    for a, b in zip(cc, cd):
        assert rel(np.asarray(a), np.asarray(b)) < 1e-9
