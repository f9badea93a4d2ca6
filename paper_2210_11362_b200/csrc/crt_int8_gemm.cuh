// fp64 environment products on the int8 tcgen05 tensor cores by the Chinese remainder
// theorem (integer modular emulation, "Ozaki scheme II"): 16 int8 GEMMs per fp64 GEMM
// instead of the 28 digit-pair products of the radix-254 slicing (tc_int8_gemm.cuh).
//
//   C(m, n) = sum_k A[m][k] B[k][n]        A = X (K-major rows), B = the fp64 half chain
//
// 1. Scaling.  Every K-major row of A (column of B) gets a power-of-two scale 2^sa[m]
//    (2^sb[n]) from its 2-norm such that the integer rows a' = rint(2^sa a),
//    b' = rint(2^sb b) satisfy ||a'||_2 <= 2^ga, ||b'||_2 <= 2^gb with
//    2^(ga+gb) < P / 2, P the product of the moduli below (Cauchy-Schwarz: the exact
//    integer product C' = a'.b' then lies in (-P/2, P/2)).  With 16 moduli P = 2^125.38,
//    ga = gb = 62: a Gaussian row of 25600 entries keeps 2^-55 of its rms (entries above
//    2^53 of the scaled row are not rounded at all).
// 2. Residues.  For each modulus p_i (pairwise coprime, <= 256) the symmetric residues
//    a' mod p_i, (b' q_i) mod p_i fit int8 (q_i = (P/p_i)^-1 mod p_i folded into B).
//    X's residues are made once per X (16 planes in the MMA's shared-memory image), the
//    half chain's per call.
// 3. One int8 GEMM per modulus (exact int32 accumulation, K <= 65472 per split), whose
//    epilogue reduces the sums mod p_i to one byte per output: t_i = (C' q_i) mod p_i.
// 4. CRT.  C' = sum_i t_i (P/p_i) - P rint(sum_i t_i / p_i), evaluated exactly in 128-bit
//    integer arithmetic, rounded once to fp64 and scaled by 2^-(sa+sb).
// So the result is the correctly rounded exact product of the rounded operands: the only
// error is the rint() of step 1.
//
// Kernel (crt8_kernel): persistent, one CTA per SM; a work item is (K split, modulus,
// 128-row m-tile) x all N <= 512 columns: the whole N lives in TMEM (N int32 columns), so
// every A byte is read from HBM once per launch and the MMAs are 128 x {<= 256} x 32
// (two per 32 k for N = 400: 208 + 192).  Items are ordered modulus-major, so the CTAs
// share one B plane (K x N bytes, L2 resident) at a time.  Roles as in oz8_kernel: bulk-copy
// producer warp, single-thread MMA issuer, four epilogue warps.
#pragma once
#include "tc_int8_gemm.cuh"

namespace trals {

constexpr int kCrtMaxMod = 16;
constexpr int kCrtBK = 64;            // int8 k per stage row (SWIZZLE_64B)
constexpr int kCrtBM = 128;
constexpr int64_t kCrtKmax = 65472;   // 128^2 K < 2^30 - 256 (31-bit unsigned epilogue operand), multiple of 64
constexpr int kCrtMaxN = 512;         // TMEM columns

// the 16 largest pairwise coprime integers <= 256 (255 = 3 5 17, 253 = 11 23, 247 = 13 19, 217 = 7 31, primes)
#define TRALS_CRT_MODULI(F) \
  F(0, 256) F(1, 255) F(2, 253) F(3, 251) F(4, 247) F(5, 241) F(6, 239) F(7, 233) \
  F(8, 229) F(9, 227) F(10, 223) F(11, 217) F(12, 211) F(13, 199) F(14, 197) F(15, 193)

struct CrtTables {
  uint32_t p[kCrtMaxMod];
  uint32_t magic[kCrtMaxMod];  // ceil(2^39 / p): floor(n / p) = umulhi(magic, n) >> 7 for n < 2^31
  uint32_t offs[kCrtMaxMod];   // p floor(2^30 / p): makes the int32 sums non-negative
  uint32_t qinv[kCrtMaxMod];   // (P / p)^-1 mod p
  float invp[kCrtMaxMod];
  uint64_t w0[kCrtMaxMod], w1[kCrtMaxMod];  // P / p_i = w1 2^64 + w0
  uint64_t P0, P1;                          // P = P1 2^64 + P0
  int nm, ga, gb;
};
__constant__ CrtTables crt_tab;

// ---------------------------------------------------------------------------
// scaling exponents
// ---------------------------------------------------------------------------
// s with ||rint(2^s x)||_2 <= 2^gamma for a row of K entries with max |x| = mx, sum x^2 = ss
// (ss is trusted only when mx^2 K can neither overflow nor lose entries to underflow)
__device__ __forceinline__ int crt_scale_exp(double mx, double ss, int64_t K, int gamma) {
  if (!(mx > 0.0) || !isfinite(mx)) return 0;
  int ex;
  if (mx >= 1e-100 && mx <= 1e100) {
    const double nb = fmax(sqrt(ss), mx) * (1.0 + 0x1p-20);  // covers the rounding of ss and of rint()
    ex = ilogb(nb) + 1;
  } else {
    const int lk = ilogb(static_cast<double>(K)) + 1;  // K < 2^lk
    ex = ilogb(mx) + 2 + (lk + 1) / 2;                 // sqrt(K) mx (1 + 2^-20) < 2^ex
  }
  return gamma - ex;
}

// rows of a row-major [rows][ld] matrix (K = cols contiguous): one warp per row, fixed order
__global__ void __launch_bounds__(256) crt_row_scale_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                                            int64_t ld, int gamma, int32_t* __restrict__ sexp) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += nw) {
    double m = 0.0, ss = 0.0;
    for (int64_t c = lane; c < cols; c += 32) {
      const double v = x[r * ld + c];
      m = fmax(m, fabs(v));
      ss = fma(v, v, ss);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if (lane == 0) sexp[r] = crt_scale_exp(m, ss, cols, gamma);
  }
}

// columns of a row-major [rows][ld] matrix (K = rows): block = 32 columns x a slab of rows,
// 8 warps over the slab's rows combined in warp order -> part[slab][2][cols]
__global__ void __launch_bounds__(256) crt_col_stats_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                                            int64_t ld, int64_t rows_per_slab,
                                                            double* __restrict__ part) {
  __shared__ double sm[8][32], sq[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + lane;
  const int64_t r0 = blockIdx.y * rows_per_slab;
  const int64_t r1 = (r0 + rows_per_slab < rows) ? r0 + rows_per_slab : rows;
  double m = 0.0, ss = 0.0;
  if (c < cols)
    for (int64_t r = r0 + warp; r < r1; r += 8) {
      const double v = x[r * ld + c];
      m = fmax(m, fabs(v));
      ss = fma(v, v, ss);
    }
  sm[warp][lane] = m;
  sq[warp][lane] = ss;
  __syncthreads();
  if (warp == 0 && c < cols) {
    for (int w = 1; w < 8; ++w) {
      m = fmax(m, sm[w][lane]);
      ss += sq[w][lane];
    }
    part[(static_cast<int64_t>(blockIdx.y) * 2 + 0) * cols + c] = m;
    part[(static_cast<int64_t>(blockIdx.y) * 2 + 1) * cols + c] = ss;
  }
}

__global__ void __launch_bounds__(256) crt_col_scale_kernel(const double* __restrict__ part, int slabs, int64_t cols,
                                                            int64_t K, int gamma, int32_t* __restrict__ sexp) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  double m = 0.0, ss = 0.0;
  for (int s = 0; s < slabs; ++s) {
    m = fmax(m, part[(static_cast<int64_t>(s) * 2 + 0) * cols + c]);
    ss += part[(static_cast<int64_t>(s) * 2 + 1) * cols + c];
  }
  sexp[c] = crt_scale_exp(m, ss, K, gamma);
}

// ---------------------------------------------------------------------------
// residues
// ---------------------------------------------------------------------------
// symmetric int8 residues of the integer a (|a| <= 2^62, already rounded) modulo the 16 moduli;
// FOLD: of a q_i.  |a| is split into three 21-bit limbs, so each residue is a 32-bit
// remainder by a compile-time constant.
template <bool FOLD>
__device__ __forceinline__ void crt_residues(double a, int8_t (&r)[kCrtMaxMod]) {
  const long long v = __double2ll_rn(a);
  const bool neg = v < 0;
  const unsigned long long u = neg ? static_cast<unsigned long long>(-v) : static_cast<unsigned long long>(v);
  const uint32_t x0 = static_cast<uint32_t>(u) & 0x1FFFFFu, x1 = static_cast<uint32_t>(u >> 21) & 0x1FFFFFu,
                 x2 = static_cast<uint32_t>(u >> 42);
#define TRALS_CRT_RES(i, pp)                                                                  \
  {                                                                                           \
    constexpr uint32_t c1 = (1u << 21) % pp, c2 = static_cast<uint32_t>((1ull << 42) % pp);   \
    uint32_t t = (x2 * c2 + x1 * c1 + x0) % pp;                                               \
    if (FOLD) t = (t * crt_tab.qinv[i]) % pp;                                                 \
    int s = t > (pp - 1) / 2 ? static_cast<int>(t) - pp : static_cast<int>(t);                \
    r[i] = static_cast<int8_t>(neg ? -s : s);                                                 \
  }
  TRALS_CRT_MODULI(TRALS_CRT_RES)
#undef TRALS_CRT_RES
}

// x (row-major [rows][ld]) -> residue planes of its K-major rows (its rows, or its columns when
// transposed), plane i = modulus i, each plane tiled [row tile of tile_w][64-k block][tile_w x 64 B]
// in the UMMA K-major SWIZZLE_64B pattern, zero padded to rows_pad x ceil(K / 64) 64.
// A CTA owns a 64-row x 64-k block (read coalesced along the contiguous axis into shared
// memory); each group of 4 threads writes one row's 64 residue bytes per plane.
template <bool FOLD>
__global__ void __launch_bounds__(256) crt_slice_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld, int transpose,
                                                        const int32_t* __restrict__ sexp, int8_t* __restrict__ out,
                                                        int64_t rows_pad, int tile_w, int nm, int64_t plane_bytes) {
  __shared__ double tile[64][65];
  const int64_t out_rows = transpose ? cols : rows, K = transpose ? rows : cols;
  const int64_t kblocks = (K + kCrtBK - 1) / kCrtBK;
  const int64_t kb = blockIdx.x % kblocks, rb = blockIdx.x / kblocks;
  const int64_t r0 = rb * 64, k0 = kb * 64;
  const int tid = threadIdx.x;
  for (int e = tid; e < 64 * 64; e += 256) {
    int kk, rr;
    if (transpose) {
      rr = e & 63;
      kk = e >> 6;
    } else {
      kk = e & 63;
      rr = e >> 6;
    }
    const int64_t k = k0 + kk, r = r0 + rr;
    double v = 0.0;
    if (k < K && r < out_rows) v = transpose ? x[k * ld + r] : x[r * ld + k];
    tile[kk][rr] = v;
  }
  __syncthreads();
  const int rl = tid >> 2, ch = tid & 3;
  const int64_t orow = r0 + rl;
  if (orow >= rows_pad) return;
  const int s = orow < out_rows ? sexp[orow] : 0;
  uint32_t w[kCrtMaxMod][4];
#pragma unroll
  for (int i = 0; i < kCrtMaxMod; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[i][q] = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    int8_t rs[kCrtMaxMod];
    crt_residues<FOLD>(scalbn(tile[ch * 16 + j][rl], s), rs);
#pragma unroll
    for (int i = 0; i < kCrtMaxMod; ++i)
      w[i][j >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(rs[i])) << (8 * (j & 3));
  }
  const int64_t t = orow / tile_w;
  const int rr = static_cast<int>(orow - t * tile_w);
  const int64_t off = (t * kblocks + kb) * (static_cast<int64_t>(tile_w) * kCrtBK) + rr * kCrtBK +
                      ((ch ^ ((rr >> 1) & 3)) << 4);
#pragma unroll
  for (int i = 0; i < kCrtMaxMod; ++i)
    if (i < nm) *reinterpret_cast<uint4*>(out + i * plane_bytes + off) = make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
}

// ---------------------------------------------------------------------------
// the modular GEMMs
// ---------------------------------------------------------------------------
struct CrtArgs {
  int64_t M, K;
  int n16, nc0, nc1, nm;      // N padded to 16; MMA column chunks nc0 + nc1 = n16 (each <= 256)
  int mtiles, splits, stages;
  int64_t kblocks, kb_split;  // 64-k blocks in total / per K split
  int64_t a_plane, b_plane;   // bytes per residue plane
  const int8_t* ad;           // [nm][mtiles][kblocks][128 x 64 B]
  const int8_t* bd;           // [nm][kblocks][n16 x 64 B]
  uint8_t* out;               // [splits][nm][M][n16]: (C' q_i) mod p_i
};

// instruction descriptor: D s32, A/B signed int8, K-major, M = 128
__device__ __forceinline__ uint32_t crt_idesc(int n) { return i8_idesc(n); }

template <class F>
__device__ __forceinline__ void crt_for_items(const CrtArgs& g, F&& body) {
  const int per_split = g.nm * g.mtiles, total = per_split * g.splits;
  for (int u = blockIdx.x; u < total; u += gridDim.x) {
    const int rem = u % per_split;
    body(u / per_split, rem / g.mtiles, rem % g.mtiles);
  }
}

__global__ void __launch_bounds__(192, 1) crt8_kernel(const __grid_constant__ CrtArgs g) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int S = g.stages;
  const uint32_t bstage = static_cast<uint32_t>(g.n16) * kCrtBK;
  const uint32_t astage = kCrtBM * kCrtBK;
  const uint32_t stage = astage + bstage;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(S) * stage);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  auto item_k = [&](int split, int64_t& kb0, int& nkb) {
    kb0 = static_cast<int64_t>(split) * g.kb_split;
    const int64_t rest = g.kblocks - kb0;
    nkb = static_cast<int>(rest < g.kb_split ? (rest > 0 ? rest : 0) : g.kb_split);
  };

  if (warp == 0) {
    // ------------------------------ bulk-copy producer ------------------------------
    if (lane == 0) {
      uint32_t gk = 0;
      crt_for_items(g, [&](int split, int mod, int mt) {
        int64_t kb0;
        int nkb;
        item_k(split, kb0, nkb);
        const int8_t* asrc = g.ad + mod * g.a_plane + (static_cast<int64_t>(mt) * g.kblocks + kb0) * astage;
        const int8_t* bsrc = g.bd + mod * g.b_plane + kb0 * bstage;
        for (int kt = 0; kt < nkb; ++kt, ++gk) {
          const uint32_t s = gk % S;
          if (gk >= static_cast<uint32_t>(S)) mbar_wait(empty + s, ((gk / S) - 1) & 1);
          uint8_t* st = sm + static_cast<size_t>(s) * stage;
          mbar_expect_tx(full + s, stage);
          bulk_load(st, asrc + static_cast<int64_t>(kt) * astage, astage, full + s);
          bulk_load(st + astage, bsrc + static_cast<int64_t>(kt) * bstage, bstage, full + s);
        }
      });
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (whole warp, one elected lane) ------------------------------
    const uint64_t dA0 = oz_desc<kCrtBK>(smem_u32(sm)), dB0 = oz_desc<kCrtBK>(smem_u32(sm) + astage);
    const uint32_t id0 = crt_idesc(g.nc0), id1 = crt_idesc(g.nc1 > 0 ? g.nc1 : 16);
    const uint32_t b1off = (static_cast<uint32_t>(g.nc0) * kCrtBK) >> 4;
    uint32_t gk = 0, it = 0;
    crt_for_items(g, [&](int split, int, int) {
      int64_t kb0;
      int nkb;
      item_k(split, kb0, nkb);
      mbar_wait(acc_empty, it & 1);  // drained by the epilogue
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      for (int kt = 0; kt < nkb; ++kt, ++gk) {
        const uint32_t s = gk % S;
        mbar_wait(full + s, (gk / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t da = dA0 + ((s * stage) >> 4), db = dB0 + ((s * stage) >> 4);
#pragma unroll
        for (int k = 0; k < kCrtBK / 32; ++k) {
          const uint32_t acc = (kt > 0 || k > 0) ? 1u : 0u;
          umma_i8_warp(tmem, da + ((k * 32) >> 4), db + ((k * 32) >> 4), id0, acc);
          if (g.nc1 > 0) umma_i8_warp(tmem + g.nc0, da + ((k * 32) >> 4), db + b1off + ((k * 32) >> 4), id1, acc);
        }
        oz_commit_warp(empty + s);
        __syncwarp();
      }
      if (nkb > 0) oz_commit_warp(acc_full);
      else if (lane == 0) mbar_arrive(acc_full);
      __syncwarp();
      ++it;
    });
  } else {
    // ------------------------------ epilogue: int32 sums -> residues mod p (one byte each) ------------------------------
    const int quad = warp & 3;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    if (lane == 0) mbar_arrive(acc_empty);
    uint32_t it = 0;
    crt_for_items(g, [&](int split, int mod, int mt) {
      int64_t kb0;
      int nkb;
      item_k(split, kb0, nkb);
      const uint32_t p = crt_tab.p[mod], magic = crt_tab.magic[mod], offs = crt_tab.offs[mod];
      const int64_t m = static_cast<int64_t>(mt) * kCrtBM + quad * 32 + lane;
      uint8_t* orow = g.out + ((static_cast<int64_t>(split) * g.nm + mod) * g.M + m) * g.n16;
      mbar_wait(acc_full, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
      for (int c0 = 0; c0 < g.n16; c0 += 32) {
        uint32_t v[2][16];
        const bool two = c0 + 16 < g.n16;
        tmem_ld16(tlane + c0, v[0]);
        if (two) tmem_ld16(tlane + c0 + 16, v[1]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const uint32_t n = nkb > 0 ? v[h][q] + offs : 0u;  // in (0, 2^31)
            const uint32_t t = n - (__umulhi(magic, n) >> 7) * p;
            w[q >> 2] |= t << (8 * (q & 3));
          }
          if (m < g.M && (h == 0 || two)) *reinterpret_cast<uint4*>(orow + c0 + 16 * h) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      ++it;
    });
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// CRT reconstruction
// ---------------------------------------------------------------------------
// C' from its residues t_i = (C' q_i) mod p_i (|C'| < 0.39 P): exact 128-bit arithmetic
// modulo 2^128, one rounding to fp64; returns C' 2^e2
__device__ __forceinline__ double crt_value(const uint32_t (&t)[kCrtMaxMod], int nm, int e2) {
  uint64_t a0 = 0, a1 = 0;
  float f = 0.f;
#pragma unroll
  for (int i = 0; i < kCrtMaxMod; ++i)
    if (i < nm) {
      const uint64_t ti = t[i];
      const uint64_t lo = ti * crt_tab.w0[i], hi = __umul64hi(ti, crt_tab.w0[i]);
      a0 += lo;
      a1 += hi + (a0 < lo ? 1u : 0u) + ti * crt_tab.w1[i];
      f = fmaf(static_cast<float>(t[i]), crt_tab.invp[i], f);
    }
  // sum = C' + q P with q = rint(sum / P) = rint(sum_i t_i / p_i): |C' / P| < 0.39, float error ~1e-5
  const uint64_t q = static_cast<uint64_t>(__float2uint_rn(f));
  const uint64_t qp0 = q * crt_tab.P0;
  const uint64_t r0 = a0 - qp0;
  const uint64_t r1 = a1 - __umul64hi(q, crt_tab.P0) - q * crt_tab.P1 - (a0 < qp0 ? 1u : 0u);
  const bool neg = static_cast<int64_t>(r1) < 0;
  uint64_t m0 = r0, m1 = r1;
  if (neg) {
    m0 = ~r0 + 1;
    m1 = ~r1 + (m0 == 0 ? 1u : 0u);
  }
  double d;
  int sh = 0;
  if (m1 == 0) {
    d = __ull2double_rn(m0);
  } else {
    // top 64 bits + sticky, correctly rounded by the conversion
    const int z = __clzll(static_cast<long long>(m1));
    uint64_t top = z ? (m1 << z) | (m0 >> (64 - z)) : m1;
    const uint64_t rest = z ? (m0 << z) : m0;
    top |= rest != 0 ? 1u : 0u;
    d = __ull2double_rn(top);
    sh = 64 - z;
  }
  d = scalbn(d, sh + e2);
  return neg ? -d : d;
}

struct CrtOutArgs {
  const uint8_t* res;  // [splits][nm][M][n16]
  int64_t M;
  int n16, N, nm, splits;
  const int32_t* sa;   // [M]
  const int32_t* sb;   // [N]
  double* C;
  CMap cmap;
  int perm;            // > 0: store order n = (j % perm) N2 + j / perm (N = perm N2): contiguous runs of C
};

constexpr int kCrtRB = 8;  // rows per block of the reconstruction

__global__ void __launch_bounds__(256) crt_combine_kernel(const CrtOutArgs g) {
  extern __shared__ double vals[];  // [kCrtRB][n16 + 1]
  const int ldv = g.n16 + 1;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kCrtRB;
  const int groups = g.n16 / 4;
  const int64_t plane = g.M * g.n16;
  for (int e = threadIdx.x; e < kCrtRB * groups; e += blockDim.x) {
    const int rl = e / groups, gq = e % groups;
    const int64_t m = m0 + rl;
    if (m >= g.M) continue;
    uint32_t t[4][kCrtMaxMod];
#pragma unroll
    for (int i = 0; i < kCrtMaxMod; ++i) {
      uint32_t b[4] = {0, 0, 0, 0};
      if (i < g.nm) {
        for (int sp = 0; sp < g.splits; ++sp) {
          const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(
              g.res + (static_cast<int64_t>(sp) * g.nm + i) * plane + m * g.n16 + 4 * gq));
#pragma unroll
          for (int q = 0; q < 4; ++q) b[q] += (w >> (8 * q)) & 0xFFu;
        }
        if (g.splits > 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) b[q] %= crt_tab.p[i];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q][i] = b[q];
    }
    const int sa = g.sa[m];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int n = 4 * gq + q;
      vals[rl * ldv + n] = n < g.N ? crt_value(t[q], g.nm, -(sa + g.sb[n])) : 0.0;
    }
  }
  __syncthreads();
  const int rows = static_cast<int>((g.M - m0) < kCrtRB ? (g.M - m0) : kCrtRB);
  const uint32_t M2 = static_cast<uint32_t>(g.cmap.M2), N2 = static_cast<uint32_t>(g.cmap.N2);
  if (g.perm > 0) {
    // j -> (n2, row, n1): for Env[r_hi][m][r_lo] each n2 plane gets one contiguous rows x r_lo block
    const int q1 = g.perm, total = rows * g.N;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int n1 = e % q1, rl = (e / q1) % rows, n2 = e / (q1 * rows);
      const uint32_t mm = static_cast<uint32_t>(m0 + rl);
      const int64_t off = static_cast<int64_t>(mm / M2) * g.cmap.sm1 + static_cast<int64_t>(mm % M2) * g.cmap.sm2 +
                          static_cast<int64_t>(n1) * g.cmap.sn1 + static_cast<int64_t>(n2) * g.cmap.sn2;
      g.C[off] = vals[rl * ldv + n1 * static_cast<int>(N2) + n2];
    }
  } else {
    const int total = rows * g.N;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int n = e % g.N, rl = e / g.N;
      const uint32_t mm = static_cast<uint32_t>(m0 + rl), un = static_cast<uint32_t>(n);
      const int64_t off = static_cast<int64_t>(mm / M2) * g.cmap.sm1 + static_cast<int64_t>(mm % M2) * g.cmap.sm2 +
                          static_cast<int64_t>(un / N2) * g.cmap.sn1 + static_cast<int64_t>(un % N2) * g.cmap.sn2;
      g.C[off] = vals[rl * ldv + n];
    }
  }
}

}  // namespace trals
