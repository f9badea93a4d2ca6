"""CPU model of the CRT form of the int8 engine (csrc/crt_int8_gemm.cuh): the integer identities the
kernels rely on, checked with numpy / Python integers.  No GPU, no library call.

  * the moduli are pairwise coprime and the scaled rows' product stays inside (-P/2, P/2);
  * residues from the two's-complement limb form (three 21-bit limbs + sign bit);
  * the epilogue's division-free remainder n - p * ((magic * n) >> 39) for every n < 2^31;
  * the reconstruction C' = sum_i t_i W_i - P rint(sum_i t_i q_i / p_i) with W_i = (P / p_i) q_i mod P,
    limb by limb modulo 2^128 as the kernel does it, and its fixed-point quotient estimate;
  * end to end: scale -> round -> residues -> per-modulus u8 x u8 products (int64) -> mod p -> CRT
    equals the exact product of the rounded operands, which is within the documented bound of
    the real product.
"""

import math

import numpy as np
import pytest

MODULI = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def tables(nm):
    P = math.prod(MODULI[:nm])
    gtot = int(math.floor(math.log2(P) - 1.0 - 0.01))
    ga, gb = (gtot + 1) // 2, gtot // 2
    q = [pow((P // p) % p, -1, p) for p in MODULI[:nm]]
    W = [(P // p) * qi for p, qi in zip(MODULI[:nm], q)]
    return P, ga, gb, q, W


@pytest.mark.parametrize("nm", [12, 14, 15, 16])
def test_moduli_and_bound(nm):
    P, ga, gb, q, W = tables(nm)
    for i, a in enumerate(MODULI[:nm]):
        for b in MODULI[i + 1:nm]:
            assert math.gcd(a, b) == 1
    assert 2 ** (ga + gb + 1) < P          # ||a'|| ||b'|| <= 2^(ga+gb) < P / 2
    assert max(ga, gb) <= 62               # rows fit int64
    assert all(w < P for w in W)           # (P / p) q < P: no reduction needed
    if nm == 15:
        assert (ga, gb) == (58, 58)
    if nm == 16:
        assert (ga, gb) == (62, 62)
    assert P < 2 ** 126                    # four 32-bit limbs
    assert sum(255 * round(2 ** 19 * qi / p) for qi, p in zip(q, MODULI)) < 2 ** 32  # fixed-point quotient sum


def residues_limb_form(v):
    """crt_residues: v (Python int, |v| <= 2^62) in two's complement, three 21-bit limbs + sign bit."""
    u = v & (2 ** 64 - 1)
    x0, x1, x2, x3 = u & 0x1FFFFF, (u >> 21) & 0x1FFFFF, (u >> 42) & 0x1FFFFF, u >> 63
    out = []
    for p in MODULI:
        c1, c2, c3 = (1 << 21) % p, (1 << 42) % p, (p - (1 << 63) % p) % p
        val = x2 * c2 + x1 * c1 + x3 * c3 + x0
        assert val < 2 ** 31
        out.append(val % p)
    return out


def test_residues_of_signed_values():
    rng = np.random.default_rng(0)
    vals = [0, 1, -1, 2 ** 62, -(2 ** 62), 2 ** 53 + 1, -(2 ** 53) - 1, 255, -256]
    vals += [int(x) for x in rng.integers(-2 ** 62, 2 ** 62, size=2000, dtype=np.int64)]
    for v in vals:
        assert residues_limb_form(v) == [v % p for p in MODULI]


def test_epilogue_remainder_is_exact():
    rng = np.random.default_rng(1)
    n = np.concatenate([rng.integers(0, 2 ** 31, size=200000, dtype=np.int64),
                        np.array([0, 1, 2 ** 31 - 1, 255 * 255 * 33024], dtype=np.int64)])
    assert 255 * 255 * 33024 < 2 ** 31     # kCrtKmax: int32 sums of u8 x u8 products
    for p in MODULI:
        magic = ((1 << 39) + p - 1) // p
        assert magic < 2 ** 32
        qn = (magic * n) >> 39             # umulhi(magic, n) >> 7
        assert np.array_equal(qn, n // p)
        # multiples of p and their neighbours
        k = rng.integers(0, (2 ** 31 - 1) // p, size=20000, dtype=np.int64) * p
        for d in (-1, 0, 1):
            m = np.clip(k + d, 0, 2 ** 31 - 1)
            assert np.array_equal((magic * m) >> 39, m // p)


def crt_value_limbs(t, nm):
    """crt_value: four 32-bit limbs without carries, fixed-point quotient, modulo 2^128."""
    P, _, _, q, W = tables(nm)
    w = [[(Wi >> (32 * j)) & 0xFFFFFFFF for j in range(4)] for Wi in W]
    Pl = [(P >> (32 * j)) & 0xFFFFFFFF for j in range(4)]
    fqt = [round(2 ** 19 * qi / p) for qi, p in zip(q, MODULI)]
    s = [sum(ti * w[i][j] for i, ti in enumerate(t)) for j in range(4)]
    assert all(x < 2 ** 45 for x in s)
    fq = sum(ti * f for ti, f in zip(t, fqt))
    qq = (fq + (1 << 18)) >> 19
    d = [s[j] - qq * Pl[j] for j in range(4)]
    for j in range(3):
        d[j + 1] += d[j] >> 32             # arithmetic shift: signed carry
    r = sum((d[j] & 0xFFFFFFFF) << (32 * j) for j in range(4))
    return r - (1 << 128) if r >> 127 else r


@pytest.mark.parametrize("nm", [15, 16])
def test_reconstruction_limbs(nm):
    P, ga, gb, _, _ = tables(nm)
    rng = np.random.default_rng(2)
    bound = 2 ** (ga + gb)
    vals = [0, 1, -1, bound, -bound, bound - 1, 12345678901234567890123, -(2 ** 100) - 7]
    vals += [int(rng.integers(-2 ** 62, 2 ** 62)) * int(rng.integers(1, 2 ** 54)) for _ in range(2000)]
    for c in vals:
        assert abs(c) <= bound
        t = [c % p for p in MODULI[:nm]]
        assert crt_value_limbs(t, nm) == c


def scale_exp(row, gamma):
    """crt_scale_exp: s with ||rint(2^s x)||_2 <= 2^gamma from max |x| and sum x^2."""
    mx = np.max(np.abs(row))
    if not mx > 0:
        return 0
    nb = max(math.sqrt(float(np.dot(row, row))), mx) * (1.0 + 2.0 ** -20)
    return gamma - (math.frexp(nb)[1])     # ilogb(nb) + 1 == frexp exponent


@pytest.mark.parametrize("nm", [15, 16])
def test_end_to_end_model(nm):
    P, ga, gb, _, _ = tables(nm)
    rng = np.random.default_rng(3)
    M, K, N = 6, 700, 5
    a = rng.standard_normal((M, K)) * np.exp(rng.standard_normal((M, K)))
    b = rng.standard_normal((K, N))
    sa = [scale_exp(a[i], ga) for i in range(M)]
    sb = [scale_exp(b[:, j], gb) for j in range(N)]
    ai = [[int(np.rint(np.ldexp(a[i, k], sa[i]))) for k in range(K)] for i in range(M)]
    bi = [[int(np.rint(np.ldexp(b[k, j], sb[j]))) for k in range(K)] for j in range(N)]
    for i in range(M):
        nrm2 = sum(v * v for v in ai[i])
        assert nrm2 <= 2 ** (2 * ga) and nrm2 > 2 ** (2 * ga - 4)
    exact = (a.astype(np.longdouble) @ b.astype(np.longdouble))
    for i in range(M):
        for j in range(N):
            c = sum(x * y for x, y in zip(ai[i], bi[j]))            # exact product of the rounded operands
            assert abs(c) < P // 2
            t = []
            for p in MODULI[:nm]:
                ra = np.array([v % p for v in ai[i]], dtype=np.int64)  # u8 residues
                rb = np.array([v % p for v in bi[j]], dtype=np.int64)
                s = int(np.dot(ra, rb))                                 # the int32 sum of one modular GEMM
                assert s < 2 ** 31
                t.append(s % p)
            assert crt_value_limbs(t, nm) == c
            got = np.ldexp(np.longdouble(c), -(sa[i] + sb[j]))  # (x87: 64-bit mantissa)
            # rounding each operand at 2^-(gamma+1) of its norm: |error| <= 2^-gamma ||a|| ||b|| (1 + ...)
            tol = 2.0 ** -(min(ga, gb) - 1) * np.linalg.norm(a[i]) * np.linalg.norm(b[:, j])
            assert abs(float(got - exact[i, j])) <= tol + 2.0 ** -60 * abs(float(exact[i, j]))
