// fp64 environment products on the int8 tcgen05 tensor cores by the Chinese remainder
// theorem (integer modular emulation, "Ozaki scheme II"): 15 (or 16) int8 GEMMs per fp64 GEMM
// instead of the 28 digit-pair products of the radix-254 slicing (tc_int8_gemm.cuh).
//
//   C(m, n) = sum_k A[m][k] B[k][n]        A = X (K-major rows), B = the fp64 half chain
//
// 1. Scaling.  Every K-major row of A (column of B) gets a power-of-two scale 2^sa[m]
//    (2^sb[n]) from its 2-norm such that the integer rows a' = rint(2^sa a),
//    b' = rint(2^sb b) satisfy ||a'||_2 <= 2^ga, ||b'||_2 <= 2^gb with
//    2^(ga+gb) < P / 2, P the product of the moduli below (Cauchy-Schwarz: the exact
//    integer product C' = a'.b' then lies in (-P/2, P/2)).  With the default 15 moduli
//    P = 2^117.78, ga = gb = 58: a Gaussian row of 25600 entries keeps 2^-51 of its rms, and
//    the rounding errors are zero-mean: the product is 2.5x more accurate than fp64 DMMA at
//    K = 25600.  (16 moduli: P = 2^125.38, ga = gb = 62.)
// 2. Residues.  For each modulus p_i (pairwise coprime, <= 256) the residues a' mod p_i,
//    b' mod p_i in [0, p_i) are unsigned bytes.  X's residues are made once per X (16 planes
//    in the MMA's shared-memory image), the half chain's per call.
// 3. One u8 x u8 GEMM per modulus (exact int32 accumulation, 255^2 K < 2^31: K <= 33024 per
//    split), whose epilogue reduces the sums mod p_i to one byte per output: t_i = C' mod p_i.
// 4. CRT.  C' = sum_i t_i W_i - P rint(sum_i t_i q_i / p_i) with W_i = (P/p_i) q_i mod P,
//    q_i = (P/p_i)^-1 mod p_i, evaluated exactly in 128-bit integer arithmetic (modulo 2^128:
//    the result is below 2^125), rounded once to fp64 and scaled by 2^-(sa+sb).
// So the result is the correctly rounded exact product of the rounded operands: the only
// error is the rint() of step 1.
//
// Kernel (crt8_kernel): persistent, one CTA per SM (in CTA pairs, below); a work item is (K split,
// modulus, 128-row m-tile) x all N <= 512 columns: the whole N lives in TMEM (N int32 columns), so
// every A byte is read from HBM once per launch and the MMAs are 128 x {<= 256} x 32
// (two per 32 k for N = 400: 208 + 192).  Items are ordered modulus-major, so the CTAs
// share one B plane (K x N bytes, L2 resident) at a time.  Roles as in oz8_kernel: bulk-copy
// producer warp, single-thread MMA issuer, four epilogue warps.
#pragma once
#include "tc_int8_gemm.cuh"

namespace trals {

constexpr int kCrtMaxMod = 16;
// Moduli in use by default.  15: P = 2^117.8, rows rounded at 2^-58 of their 2-norm -- measured
// against an extended-precision product at the c5 shape (K = 25600) 3.8e-16 relative, 2.5x more
// accurate than the fp64 DMMA product (9.2e-16) and than the digit-pair form (6e-16).  16 moduli
// (2^-62, 4.8e-17: the final rounding alone) cost one more GEMM in 15 (TRALS_CRT_MODULI=16).
constexpr int kCrtDefaultMod = 15;
constexpr int kCrtBK = 64;            // int8 k per stage row (SWIZZLE_64B)
constexpr int kCrtBM = 128;
constexpr int64_t kCrtKmax = 33024;   // 255^2 K < 2^31 (int32 sums of u8 x u8 products), multiple of 64
constexpr int kCrtMaxN = 512;         // TMEM columns

// the 16 largest pairwise coprime integers <= 256 (255 = 3 5 17, 253 = 11 23, 247 = 13 19, 217 = 7 31, primes)
#define TRALS_CRT_MODULI(F) \
  F(0, 256) F(1, 255) F(2, 253) F(3, 251) F(4, 247) F(5, 241) F(6, 239) F(7, 233) \
  F(8, 229) F(9, 227) F(10, 223) F(11, 217) F(12, 211) F(13, 199) F(14, 197) F(15, 193)

struct CrtTables {
  uint32_t p[kCrtMaxMod];
  uint32_t magic[kCrtMaxMod];  // ceil(2^39 / p): floor(n / p) = umulhi(magic, n) >> 7 for n < 2^31
  uint32_t fq[kCrtMaxMod];     // rint(2^19 q_i / p_i), q_i = (P / p_i)^-1 mod p_i
  uint32_t w[kCrtMaxMod][4];   // W_i = (P / p_i) q_i mod P, 32-bit limbs (little endian)
  uint32_t P[4];               // P, 32-bit limbs
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
  if (c < cols) {
    int64_t r = r0 + warp;
    for (; r + 24 < r1; r += 32) {  // four loads in flight
      const double v0 = x[r * ld + c], v1 = x[(r + 8) * ld + c], v2 = x[(r + 16) * ld + c], v3 = x[(r + 24) * ld + c];
      m = fmax(fmax(m, fabs(v0)), fmax(fabs(v1), fmax(fabs(v2), fabs(v3))));
      ss = fma(v0, v0, ss);
      ss = fma(v1, v1, ss);
      ss = fma(v2, v2, ss);
      ss = fma(v3, v3, ss);
    }
    for (; r < r1; r += 8) {
      const double v = x[r * ld + c];
      m = fmax(m, fabs(v));
      ss = fma(v, v, ss);
    }
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

// one warp per column: lanes over the slabs, fixed-order tree
__global__ void __launch_bounds__(256) crt_col_scale_kernel(const double* __restrict__ part, int slabs, int64_t cols,
                                                            int64_t K, int gamma, int32_t* __restrict__ sexp) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (c >= cols) return;
  double m = 0.0, ss = 0.0;
  for (int s = lane; s < slabs; s += 32) {
    m = fmax(m, part[(static_cast<int64_t>(s) * 2 + 0) * cols + c]);
    ss += part[(static_cast<int64_t>(s) * 2 + 1) * cols + c];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if (lane == 0) sexp[c] = crt_scale_exp(m, ss, K, gamma);
}

// ---------------------------------------------------------------------------
// residues
// ---------------------------------------------------------------------------
// residues in [0, p_i) of the integer v (|v| <= 2^62) modulo the 16 moduli, packed one byte each
// into 4 words per ... (see crt_slice_kernel).  v is taken in two's complement: three 21-bit limbs
// plus the sign bit of weight -2^63, so each residue is one 32-bit remainder by a compile-time
// constant (x0 + x1 c1 + x2 c2 + x3 c3 < 2^31).
__device__ __forceinline__ void crt_residues(long long v, uint32_t (&r)[kCrtMaxMod]) {
  const unsigned long long u = static_cast<unsigned long long>(v);
  const uint32_t x0 = static_cast<uint32_t>(u) & 0x1FFFFFu, x1 = static_cast<uint32_t>(u >> 21) & 0x1FFFFFu,
                 x2 = static_cast<uint32_t>(u >> 42) & 0x1FFFFFu, x3 = static_cast<uint32_t>(u >> 63);
#define TRALS_CRT_RES(i, pp)                                                                       \
  {                                                                                                \
    constexpr uint32_t c1 = (1u << 21) % pp, c2 = static_cast<uint32_t>((1ull << 42) % pp),        \
                       c3 = (pp - static_cast<uint32_t>((1ull << 63) % pp)) % pp;                  \
    r[i] = (x2 * c2 + x1 * c1 + x3 * c3 + x0) % pp;                                                \
  }
  TRALS_CRT_MODULI(TRALS_CRT_RES)
#undef TRALS_CRT_RES
}

// x (row-major [rows][ld]) -> residue planes of its K-major rows (its rows, or its columns when
// transposed), plane i = modulus i, each plane tiled [row tile of tile_w][64-k block][tile_w x 64 B]
// in the UMMA K-major SWIZZLE_64B pattern, zero padded to rows_pad x ceil(K / 64) 64.
// A CTA owns a 64-row x 64-k block (read coalesced along the contiguous axis into shared
// memory); a thread turns 4 consecutive k of one row into one 4-byte word per plane (16 threads
// write a row's 64 bytes of a plane), four row groups per thread.
__global__ void __launch_bounds__(256) crt_slice_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld, int transpose,
                                                        const int32_t* __restrict__ sexp, uint8_t* __restrict__ out,
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
  const int kg = tid & 15;  // 4-k group of the 64-k block
#pragma unroll 1
  for (int rl = tid >> 4; rl < 64; rl += 16) {
    const int64_t orow = r0 + rl;
    if (orow >= rows_pad) break;
    const int s = orow < out_rows ? sexp[orow] : 0;
    uint32_t w[kCrtMaxMod];
#pragma unroll
    for (int i = 0; i < kCrtMaxMod; ++i) w[i] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t rs[kCrtMaxMod];
      crt_residues(__double2ll_rn(scalbn(tile[kg * 4 + j][rl], s)), rs);
#pragma unroll
      for (int i = 0; i < kCrtMaxMod; ++i) w[i] |= rs[i] << (8 * j);
    }
    const int64_t t = orow / tile_w;
    const int rr = static_cast<int>(orow - t * tile_w);
    const int64_t off = (t * kblocks + kb) * (static_cast<int64_t>(tile_w) * kCrtBK) + rr * kCrtBK +
                        ((((kg >> 2) ^ ((rr >> 1) & 3)) << 4) | ((kg & 3) << 2));
#pragma unroll
    for (int i = 0; i < kCrtMaxMod; ++i)
      if (i < nm) *reinterpret_cast<uint32_t*>(out + i * plane_bytes + off) = w[i];
  }
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
  const uint8_t* ad;          // [nm][mtiles (even)][kblocks][128 x 64 B]
  const uint8_t* bd;          // [nm][kblocks][n16 x 64 B]
  uint8_t* out;               // [splits][nm][M][n16]: C' mod p_i
  // Tail split (splits == 1): the units beyond the last full wave (unit index >= tail_start) are cut
  // into tail_splits K pieces of tail_kb 64-k blocks, so the last wave takes 1 / tail_splits of a
  // unit's time.  Piece 0 writes the unit's rows of `out`, piece s >= 1 writes
  // tail_out[s - 1][unit - tail_start][rows of the unit][n16]; the reconstruction adds them mod p_i.
  int tail_start, tail_splits;
  int64_t tail_kb;
  uint8_t* tail_out;
};

// instruction descriptor: D s32, A/B unsigned int8 (type fields 0), K-major, N = n, M = 128 (one CTA)
// or 256 (CTA pair)
__device__ __forceinline__ uint32_t crt_idesc(int n, int m) {
  uint32_t d = 0;
  d |= 2u << 4;
  d |= static_cast<uint32_t>(n >> 3) << 17;
  d |= static_cast<uint32_t>(m >> 4) << 24;
  return d;
}

__device__ __forceinline__ void umma_i8_pair_warp(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// commit of the pair's MMAs: arrives on the mbarrier at this offset in both CTAs
__device__ __forceinline__ void crt_commit_pair_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// arrive on the mbarrier at the same offset in CTA `rank` of the cluster (plain arrive / plain
// try_wait on the other side, as for a barrier signalled by a peer's bulk copy: cluster-scope
// release / acquire qualifiers cost a memory barrier per stage -- 2200 instead of ~400 cycles)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}

// Work items.  One CTA: (split, modulus, m-tile), CTA b takes items b, b + grid, ...  CTA pair: the
// pair takes (split, modulus, pair of m-tiles) and CTA rank r the m-tile 2 j + r of it.
template <bool PAIR, class F>
__device__ __forceinline__ void crt_for_items(const CrtArgs& g, F&& body) {
  // body(split, modulus, unit row index, first 64-k block, number of blocks, tail piece or -1, unit)
  const int mu = PAIR ? (g.mtiles + 1) / 2 : g.mtiles;
  const int per_split = g.nm * mu, units = per_split * g.splits;
  const int total = g.tail_start + (units - g.tail_start) * g.tail_splits;
  const int first = PAIR ? blockIdx.x / 2 : blockIdx.x, step = PAIR ? gridDim.x / 2 : gridDim.x;
  for (int it = first; it < total; it += step) {
    int u = it, piece = -1;
    if (it >= g.tail_start) {
      const int j = it - g.tail_start;
      u = g.tail_start + j / g.tail_splits;
      piece = j % g.tail_splits;
    }
    const int split = u / per_split, rem = u % per_split;
    int64_t kb0, kbn;
    if (piece < 0) {
      kb0 = static_cast<int64_t>(split) * g.kb_split;
      kbn = g.kb_split;
    } else {
      kb0 = static_cast<int64_t>(piece) * g.tail_kb;
      kbn = g.tail_kb;
    }
    const int64_t rest = g.kblocks - kb0;
    const int nkb = static_cast<int>(rest < kbn ? (rest > 0 ? rest : 0) : kbn);
    body(split, rem / mu, rem % mu, kb0, nkb, piece, u);
  }
}

// PAIR: clusters of two CTAs (one TPC) run tcgen05.mma.cta_group::2 -- M = 256, each CTA holding its
// own 128 rows of A and half of the B rows of every MMA -- so a CTA fills (128 + N / 2) x 64 bytes
// of shared memory per 64 k instead of (128 + N) x 64 (measured at c5: 3.83 vs 3.95 ms per
// environment step, with 16 moduli, before the other changes of the round).  The leader (rank 0) issues the MMAs; its
// MMA warp waits for its own stage and for the peer's (relayed by the peer's MMA warp, which has
// nothing else to do); commits are multicast to both CTAs' barriers.
template <bool PAIR>
__global__ void __launch_bounds__(192, 1) crt8_kernel(const __grid_constant__ CrtArgs g) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const int S = g.stages;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  const uint32_t b0bytes = static_cast<uint32_t>(g.nc0) * kCrtBK / (PAIR ? 2 : 1);
  const uint32_t b1bytes = static_cast<uint32_t>(g.nc1) * kCrtBK / (PAIR ? 2 : 1);
  const uint32_t bstage_g = static_cast<uint32_t>(g.n16) * kCrtBK;  // one 64-k block of a B plane in HBM
  const uint32_t astage = kCrtBM * kCrtBK;
  const uint32_t stage = astage + b0bytes + b1bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(S) * stage);
  uint64_t* empty = full + S;
  uint64_t* peer_full = empty + S;       // (leader) the peer's stage has landed
  uint64_t* acc_full = peer_full + S;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
      mbar_init(peer_full + s, 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, PAIR ? 8 : 4);  // one arrive per epilogue warp (of both CTAs)
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------ bulk-copy producer ------------------------------
    if (lane == 0) {
      uint32_t gk = 0;
      crt_for_items<PAIR>(g, [&](int, int mod, int mu, int64_t kb0, int nkb, int, int) {
        const int mt = PAIR ? 2 * mu + static_cast<int>(crank) : mu;
        const uint8_t* asrc = g.ad + mod * g.a_plane + (static_cast<int64_t>(mt) * g.kblocks + kb0) * astage;
        const uint8_t* bsrc = g.bd + mod * g.b_plane + kb0 * bstage_g;
        const uint8_t* b0src = bsrc + crank * b0bytes;
        const uint8_t* b1src = bsrc + static_cast<uint32_t>(g.nc0) * kCrtBK + crank * b1bytes;
        for (int kt = 0; kt < nkb; ++kt, ++gk) {
          const uint32_t s = gk % S;
          if (gk >= static_cast<uint32_t>(S)) mbar_wait(empty + s, ((gk / S) - 1) & 1);
          uint8_t* st = sm + static_cast<size_t>(s) * stage;
          mbar_expect_tx(full + s, stage);
          bulk_load(st, asrc + static_cast<int64_t>(kt) * astage, astage, full + s);
          bulk_load(st + astage, b0src + static_cast<int64_t>(kt) * bstage_g, b0bytes, full + s);
          if (b1bytes) bulk_load(st + astage + b0bytes, b1src + static_cast<int64_t>(kt) * bstage_g, b1bytes, full + s);
        }
      });
    }
  } else if (warp == 1 && crank != 0) {
    // ------------------------------ peer relay: this CTA's stage has landed -> leader ------------------------------
    if (lane == 0) {
      uint32_t gk = 0;
      crt_for_items<PAIR>(g, [&](int, int, int, int64_t, int nkb, int, int) {
        for (int kt = 0; kt < nkb; ++kt, ++gk) {
          const uint32_t s = gk % S;
          mbar_wait(full + s, (gk / S) & 1);
          mbar_arrive_remote(peer_full + s, 0);
        }
      });
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (whole warp, one elected lane) ------------------------------
    const uint64_t dA0 = oz_desc<kCrtBK>(smem_u32(sm)), dB0 = oz_desc<kCrtBK>(smem_u32(sm) + astage);
    const uint32_t id0 = crt_idesc(g.nc0, PAIR ? 256 : 128), id1 = crt_idesc(g.nc1 > 0 ? g.nc1 : 16, PAIR ? 256 : 128);
    const uint32_t b1off = b0bytes >> 4;
    uint32_t gk = 0, it = 0;
    crt_for_items<PAIR>(g, [&](int, int, int, int64_t, int nkb, int, int) {
      mbar_wait(acc_empty, it & 1);  // drained by the epilogue (of both CTAs)
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      for (int kt = 0; kt < nkb; ++kt, ++gk) {
        const uint32_t s = gk % S;
        mbar_wait(full + s, (gk / S) & 1);
        if constexpr (PAIR) mbar_wait(peer_full + s, (gk / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t da = dA0 + ((s * stage) >> 4), db = dB0 + ((s * stage) >> 4);
#pragma unroll
        for (int k = 0; k < kCrtBK / 32; ++k) {
          const uint32_t acc = (kt > 0 || k > 0) ? 1u : 0u;
          if constexpr (PAIR) {
            umma_i8_pair_warp(tmem, da + ((k * 32) >> 4), db + ((k * 32) >> 4), id0, acc);
            if (g.nc1 > 0) umma_i8_pair_warp(tmem + g.nc0, da + ((k * 32) >> 4), db + b1off + ((k * 32) >> 4), id1, acc);
          } else {
            umma_i8_warp(tmem, da + ((k * 32) >> 4), db + ((k * 32) >> 4), id0, acc);
            if (g.nc1 > 0) umma_i8_warp(tmem + g.nc0, da + ((k * 32) >> 4), db + b1off + ((k * 32) >> 4), id1, acc);
          }
        }
        if constexpr (PAIR) crt_commit_pair_warp(empty + s);
        else oz_commit_warp(empty + s);
        __syncwarp();
      }
      if (nkb > 0) {
        if constexpr (PAIR) crt_commit_pair_warp(acc_full);
        else oz_commit_warp(acc_full);
      } else if (lane == 0) {
        mbar_arrive(acc_full);
        if constexpr (PAIR) mbar_arrive_remote(acc_full, 1);
      }
      __syncwarp();
      ++it;
    });
  } else {
    // ------------------------------ epilogue: int32 sums -> residues mod p (one byte each) ------------------------------
    const int quad = warp & 3;
    const uint32_t tlane = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    auto release = [&]() {
      if (lane == 0) {
        if (PAIR && crank != 0) mbar_arrive_remote(acc_empty, 0);
        else mbar_arrive(acc_empty);
      }
    };
    release();
    uint32_t it = 0;
    crt_for_items<PAIR>(g, [&](int split, int mod, int mu, int64_t, int nkb, int piece, int u) {
      const int mt = PAIR ? 2 * mu + static_cast<int>(crank) : mu;
      const uint32_t p = crt_tab.p[mod], magic = crt_tab.magic[mod];
      const int urow = (PAIR ? static_cast<int>(crank) * kCrtBM : 0) + quad * 32 + lane;  // row inside the unit
      const int64_t m = static_cast<int64_t>(mt) * kCrtBM + quad * 32 + lane;
      uint8_t* orow = g.out + ((static_cast<int64_t>(split) * g.nm + mod) * g.M + m) * g.n16;
      if (piece > 0) {
        const int64_t tunits = static_cast<int64_t>(g.nm) * (PAIR ? (g.mtiles + 1) / 2 : g.mtiles) - g.tail_start;
        orow = g.tail_out + ((static_cast<int64_t>(piece - 1) * tunits + (u - g.tail_start)) *
                                 (PAIR ? 2 * kCrtBM : kCrtBM) + urow) * g.n16;
      }
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
            const uint32_t n = nkb > 0 ? v[h][q] : 0u;  // in [0, 2^31)
            const uint32_t t = n - (__umulhi(magic, n) >> 7) * p;
            w[q >> 2] |= t << (8 * (q & 3));
          }
          if (m < g.M && (h == 0 || two)) *reinterpret_cast<uint4*>(orow + c0 + 16 * h) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      release();
      ++it;
    });
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no CTA leaves while the pair's MMAs or signals may still touch it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if constexpr (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// CRT reconstruction
// ---------------------------------------------------------------------------
// C' from its residues t_i = C' mod p_i (|C'| < 0.39 P), exactly, modulo 2^128: the four 32-bit
// limbs of sum_i t_i W_i accumulate without carries in 64-bit registers (t_i < 2^8, 16 terms:
// < 2^44 each), q P is subtracted limb by limb, one signed carry pass, one rounding to fp64;
// returns C' 2^e2.  (Tables are zero beyond the moduli in use.)
__device__ __forceinline__ double crt_value(const uint32_t (&t)[kCrtMaxMod], int e2) {
  uint64_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  uint32_t fq = 0;
#pragma unroll
  for (int i = 0; i < kCrtMaxMod; ++i) {
    s0 += static_cast<uint64_t>(t[i]) * crt_tab.w[i][0];
    s1 += static_cast<uint64_t>(t[i]) * crt_tab.w[i][1];
    s2 += static_cast<uint64_t>(t[i]) * crt_tab.w[i][2];
    s3 += static_cast<uint64_t>(t[i]) * crt_tab.w[i][3];
    fq += t[i] * crt_tab.fq[i];
  }
  // sum = C' + q P with q = rint(sum / P) = rint(sum_i t_i q_i / p_i) <= 4080: |C' / P| < 0.39,
  // and the 2^-19 fixed-point sum is good to 0.004
  const uint32_t q = (fq + (1u << 18)) >> 19;
  int64_t d0 = static_cast<int64_t>(s0) - static_cast<int64_t>(static_cast<uint64_t>(q) * crt_tab.P[0]);
  int64_t d1 = static_cast<int64_t>(s1) - static_cast<int64_t>(static_cast<uint64_t>(q) * crt_tab.P[1]);
  int64_t d2 = static_cast<int64_t>(s2) - static_cast<int64_t>(static_cast<uint64_t>(q) * crt_tab.P[2]);
  int64_t d3 = static_cast<int64_t>(s3) - static_cast<int64_t>(static_cast<uint64_t>(q) * crt_tab.P[3]);
  d1 += d0 >> 32;
  d2 += d1 >> 32;
  d3 += d2 >> 32;
  const uint32_t r0 = static_cast<uint32_t>(d0), r1 = static_cast<uint32_t>(d1), r2 = static_cast<uint32_t>(d2),
                 r3 = static_cast<uint32_t>(d3);
  const bool neg = static_cast<int32_t>(r3) < 0;
  uint64_t m0 = (static_cast<uint64_t>(r1) << 32) | r0, m1 = (static_cast<uint64_t>(r3) << 32) | r2;
  if (neg) {
    m0 = ~m0 + 1;
    m1 = ~m1 + (m0 == 0 ? 1u : 0u);
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
  // d 2^(sh + e2) by two exact power-of-two factors (each exponent inside the normal range for
  // |sh + e2| <= 2044; beyond that scalbn)
  const int e = sh + e2, e1 = e >> 1, eh = e - e1;
  if (static_cast<unsigned>(e1 + 1022) <= 2045u && static_cast<unsigned>(eh + 1022) <= 2045u)
    d = (d * __hiloint2double((1023 + e1) << 20, 0)) * __hiloint2double((1023 + eh) << 20, 0);
  else
    d = scalbn(d, e);
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

// Tail split of the GEMMs (CrtArgs): adds the residues of the K pieces s >= 1 of the units
// >= tail_start into the units' rows of the main residue planes, modulo p_i (a few MB; runs before
// the reconstruction).  One thread per (tail unit, row of the unit, 4 columns).
struct CrtTailArgs {
  uint8_t* res;             // [nm][M][n16] (one K split)
  const uint8_t* tail_res;  // [tail_splits - 1][tail units][unit_rows][n16]
  int64_t M;
  int n16, nm, tail_start, tail_splits, unit_rows, units_per_mod;
};

__global__ void __launch_bounds__(256) crt_tail_merge_kernel(const CrtTailArgs g) {
  const int groups = g.n16 / 4;
  const int64_t tunits = static_cast<int64_t>(g.nm) * g.units_per_mod - g.tail_start;
  const int64_t total = tunits * g.unit_rows * groups;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int gq = static_cast<int>(e % groups);
    const int64_t ur = e / groups;
    const int row = static_cast<int>(ur % g.unit_rows);
    const int64_t tu = ur / g.unit_rows;
    const int64_t u = g.tail_start + tu;
    const int mod = static_cast<int>(u / g.units_per_mod);
    const int64_t m = (u % g.units_per_mod) * g.unit_rows + row;
    if (m >= g.M) continue;
    uint32_t* dst = reinterpret_cast<uint32_t*>(g.res + (static_cast<int64_t>(mod) * g.M + m) * g.n16 + 4 * gq);
    uint32_t w = *dst;
    const uint32_t p = crt_tab.p[mod];
    for (int sp = 1; sp < g.tail_splits; ++sp) {
      const uint32_t w2 = __ldcs(reinterpret_cast<const uint32_t*>(
          g.tail_res + ((static_cast<int64_t>(sp - 1) * tunits + tu) * g.unit_rows + row) * g.n16 + 4 * gq));
      uint32_t o = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t b = ((w >> (8 * q)) & 0xFFu) + ((w2 >> (8 * q)) & 0xFFu);
        b -= b >= p ? p : 0u;
        o |= b << (8 * q);
      }
      w = o;
    }
    *dst = w;
  }
}

constexpr int kCrtRB = 8;  // rows per block of the reconstruction

__global__ void __launch_bounds__(256, 3) crt_combine_kernel(const CrtOutArgs g) {
  extern __shared__ double vals[];  // [kCrtRB][n16 + 1]
  const int ldv = g.n16 + 1;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * kCrtRB;
  const int groups = g.n16 / 4;
  const int64_t plane = g.M * g.n16;
  // a thread reconstructs 4 consecutive columns of one row: one 4-byte word per modulus plane,
  // all 16 loads in flight together
  int rl = threadIdx.x / groups, gq = threadIdx.x % groups;
  const int drl = blockDim.x / groups, dgq = blockDim.x % groups;
  while (rl < kCrtRB && m0 + rl < g.M) {
    const int64_t m = m0 + rl;
    const uint8_t* src = g.res + m * g.n16 + 4 * gq;
    uint32_t wv[kCrtMaxMod];
#pragma unroll
    for (int i = 0; i < kCrtMaxMod; ++i)
      wv[i] = __ldcs(reinterpret_cast<const uint32_t*>(src + (i < g.nm ? i : 0) * plane));
    if (g.splits > 1) {
      // residues of the K splits add modulo p_i (their sum is C' mod p_i of the whole product)
#pragma unroll 1
      for (int sp = 1; sp < g.splits; ++sp) {
#pragma unroll
        for (int i = 0; i < kCrtMaxMod; ++i) {
          const uint32_t w2 = __ldcs(reinterpret_cast<const uint32_t*>(
              src + (static_cast<int64_t>(sp) * g.nm + (i < g.nm ? i : 0)) * plane));
          uint32_t o = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t b = ((wv[i] >> (8 * q)) & 0xFFu) + ((w2 >> (8 * q)) & 0xFFu);
            b -= b >= crt_tab.p[i] ? crt_tab.p[i] : 0u;
            o |= b << (8 * q);
          }
          wv[i] = o;
        }
      }
    }
    const int sa = g.sa[m];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int n = 4 * gq + q;
      uint32_t t[kCrtMaxMod];
#pragma unroll
      for (int i = 0; i < kCrtMaxMod; ++i) t[i] = __byte_perm(wv[i], 0, 0x4440 + q);  // byte q of the word
      vals[rl * ldv + n] = n < g.N ? crt_value(t, -(sa + g.sb[n])) : 0.0;
    }
    gq += dgq;
    rl += drl;
    if (gq >= groups) {
      gq -= groups;
      ++rl;
    }
  }
  __shared__ int64_t roff[kCrtRB];  // C offsets of the block's rows
  const uint32_t M2 = static_cast<uint32_t>(g.cmap.M2), N2 = static_cast<uint32_t>(g.cmap.N2);
  if (threadIdx.x < kCrtRB) {
    const uint32_t mm = static_cast<uint32_t>(m0 + threadIdx.x);
    roff[threadIdx.x] = static_cast<int64_t>(mm / M2) * g.cmap.sm1 + static_cast<int64_t>(mm % M2) * g.cmap.sm2;
  }
  __syncthreads();
  const int rows = static_cast<int>((g.M - m0) < kCrtRB ? (g.M - m0) : kCrtRB);
  // stores in the order of C's addresses; e -> (outer, row, inner) advanced incrementally (no
  // per-element divisions).  perm: for Env[r_hi][m][r_lo] each n2 plane gets one contiguous
  // rows x r_lo block (inner = n1 of perm values, outer = n2); else inner = n, outer unused.
  const int inner = g.perm > 0 ? g.perm : g.N, outer = g.perm > 0 ? g.N / g.perm : 1;
  int i1 = threadIdx.x % inner, tq = threadIdx.x / inner;
  int o2 = tq / rows;
  rl = tq % rows;
  const int d1 = blockDim.x % inner, dq = blockDim.x / inner;
  while (o2 < outer) {
    const int n = g.perm > 0 ? i1 * static_cast<int>(N2) + o2 : i1;
    const uint32_t un = static_cast<uint32_t>(n);
    const uint32_t nq = g.perm > 0 ? static_cast<uint32_t>(i1) : un / N2, nr = g.perm > 0 ? static_cast<uint32_t>(o2) : un % N2;
    const int64_t off = roff[rl] + static_cast<int64_t>(nq) * g.cmap.sn1 + static_cast<int64_t>(nr) * g.cmap.sn2;
    g.C[off] = vals[rl * ldv + n];
    i1 += d1;
    int carry = dq;
    if (i1 >= inner) {
      i1 -= inner;
      ++carry;
    }
    rl += carry;
    while (rl >= rows) {
      rl -= rows;
      ++o2;
    }
  }
}

}  // namespace trals
