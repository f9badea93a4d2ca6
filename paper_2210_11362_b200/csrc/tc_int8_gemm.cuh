// Exact-integer GEMM on the int8 tcgen05 tensor cores (Ozaki-style digit slicing)
// for the environment products: the fp32 variant's (4 digits, below) and the fp64
// path's (7 balanced radix-254 digits, 28 pairs, fp64-accurate: see OzF64).
//
//   C(m, n) (fp64 out) = sum_k A[m][k] * B[n][k]      A from X, B from the fp64 half chain
//
// The description below is the fp32 scheme; the fp64 one differs only in the
// digit count, the kept levels, the balanced digits and the output staging.
//
// Why not 3xTF32: the tf32 MMA accumulates in truncated fp32, a ~1e-6 relative
// bias on M_n that the normal equations (cond(S) up to 5e11 on BASELINE c4) and
// the cheap error's cancellation amplify far past the 1e-4 fp32 contract.  The
// int8 MMA is exact (int32 accumulation), so the only error is the slicing:
//
//   A[m][k] = 2^ea[m] * sum_{s<4} a_s[m][k] 2^(-7(s+1)),   a_s int8 in [-127, 127]
//   B[n][k] = 2^eb[n] * sum_{t<4} b_t[n][k] 2^(-7(t+1))
//
// (per-row / per-column power-of-two scales with |x| < 2^e, truncated base-128
// digits: 28 bits below the row maximum, exact for fp32 values within 16x of
// it).  All 16 digit pairs are kept, in 4 MMAs per 32-k step: the B tile holds
// the 4 B planes stacked as one N = 4 BN operand, so the MMA of A plane s
// writes pair (s, t) into accumulator column block s + t -- i.e. issuing A plane
// s at TMEM column offset s BN makes every level L = s + t land in one int32
// block (7 x BN columns), each A plane is read from shared memory once per step
// (SS-mode operand reads, not the tensor pipe, bounded the 13-MMA pairwise
// form).  The epilogue zeroes the levels for the next tile and combines them
// exactly in fp64 (Horner in 2^-7):
//   C = 2^(ea+eb-14) * sum_L acc_L 2^(-7L).
// Measured on N(0,1) data: 1.2-1.9e-8 relative Frobenius against an fp64
// product of the same fp32 X, i.e. the digit truncation of the row / column
// maxima's 28-bit window.
// No overflow: a level sums at most 4 pairs of |a b| <= 127^2 over at most
// kOzKmax (32768) k per CTA, < 2^31; longer K is always split.
//
// Operand layout in HBM: the digits are stored as the exact shared-memory image
// of the MMA operand tiles -- blocks of [row tile][64-k block][digit plane]
// [rows x 64 B], each plane already in the UMMA K-major SWIZZLE_64B pattern
// (16-byte chunk c of row r at chunk c ^ ((r >> 1) & 3)), zero padded to whole
// tiles.  One pipeline stage is then two contiguous bulk copies (A: 32 KB, B:
// 16 KB, cp.async.bulk), so X streams from HBM strictly sequentially instead
// of as 64 B pieces of 128 different rows (which capped the tensor-map version
// at 2.8 TB/s).
//
// Structure (persistent, one CTA per SM over 128 x BN x kchunk tiles): warp 0 =
// bulk-copy producer (a STAGES-deep ring running across tiles), warp 1 = TMEM
// allocator + single-thread MMA issuer (tcgen05.mma.cta_group::1.kind::i8,
// K-major both, 32 k per MMA), warps 2-5 = epilogue (tcgen05.ld 32x32b; warp w
// owns TMEM lanes 32*(w%4)); acc_full / acc_empty mbarriers hand the
// accumulators over.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dmma_gemm.cuh"
#include "dmma_tma_gemm.cuh"

namespace trals {

constexpr int kOzBK = 64;        // int8 k per stage of the fp32 scheme (one 64 B swizzle row)
constexpr int kOzBM = 128;

// Digit schemes.  D digit planes per operand, the LV lowest pair levels L = s + t
// kept (pairs with s + t >= LV are dropped), BAL = balanced (round-to-nearest)
// digits instead of truncated ones, KMAX = longest k per CTA whose int32 level
// sums cannot overflow; C0 = scale of the first digit, RAD = radix of the rest:
//   x = 2^e (d_0 + (d_1 + (d_2 + ...) / RAD) / RAD) / C0,
// so a pair (s, t) weighs 2^(ea+eb) W0 RAD^-L with W0 = 1 / C0^2, and the epilogue
// combines the levels by Horner in 1 / RAD.
//   fp32 variant: 4 truncated base-128 digits (28 bits), all 16 pairs (7 levels):
//     C0 = RAD = 128, |d_s| <= 127, W0 = 2^-14 (every step exact).
//     A level sums <= 4 pairs of 127^2 per k -> KMAX 32768.
//   fp64 (emulated DMMA): 7 balanced digits, first d_0 = rint(127 v), then
//     d_s = rint(254 r), |d_s| <= 127 (|r| <= 1/2, 254 / 2 = 127: the int8 range is
//     used in full, 7.99 bits per digit); remainder <= 2^-55.9 2^e, the fp64 mantissa
//     of the row maximum plus 3 guard bits.  Levels 0..6 kept (28 pairs; the dropped
//     level-7 terms are 6 pairs of <= 254^-7 = 2^-55.9 per k, zero-mean -- the same
//     bound as 8 base-128 digits with 36 pairs, at 22 % fewer int8 MMAs and 7 instead of 8
//     digit bytes per element).  The slicing's products by 127 / 254 round at 2^-53
//     of the current remainder, i.e. below the truncation.  A level sums <= 7 pairs of
//     127^2 per k -> KMAX 18944 (7 x 127^2 x 18944 < 2^31).
//     Measured against an extended-precision product: the same error as fp64 DMMA
//     (tests/test_gpu_ops.py::test_env_oz64_accuracy).
// BK: int8 k per pipeline stage and digit row: 64 (SWIZZLE_64B rows) for the fp32 scheme,
// 32 (SWIZZLE_32B rows) for the fp64 one -- its 7-plane stages are larger, and at
// 32 k four of them fit in flight (the short-K shapes, c3/c4, were DRAM-latency bound
// with two 64-k stages: tensor pipe 33 % busy at c3)
template <int D_, int LV_, bool BAL_, int64_t KMAX_, int BK_, int C0_, int RAD_>
struct OzScheme {
  static constexpr int D = D_;
  static constexpr int LV = LV_;
  static constexpr bool BAL = BAL_;
  static constexpr int64_t KMAX = KMAX_;
  static constexpr int BK = BK_;
  static constexpr double C0 = C0_;
  static constexpr double RAD = RAD_;
  static constexpr double HR = 1.0 / RAD_;              // Horner factor
  static constexpr double W0 = 1.0 / (double(C0_) * C0_);  // weight of the level-0 pair
  static_assert(int64_t(BAL_ ? (LV_ < D_ ? LV_ : D_) : D_) * 127 * 127 * KMAX_ < (int64_t(1) << 31),
                "int32 level sums may overflow");
};
using OzF32 = OzScheme<4, 7, false, 32768, 64, 128, 128>;
using OzF64 = OzScheme<7, 7, true, 18944, 32, 127, 254>;
constexpr int kOzDigits = OzF32::D;  // (fp32 variant layout helpers)
constexpr int kOzLevels = OzF32::LV;
constexpr int64_t kOzKmax = OzF32::KMAX;

// RAD^-p (p >= 0) as the nearest double (exact for the power-of-two radix)
template <class SC>
__host__ __device__ constexpr double oz_rad_pow(int p) {
  double r = 1.0;  // RAD^p exactly (< 2^53 for the p used), then one rounding
  for (int i = 0; i < p; ++i) r *= SC::RAD;
  return 1.0 / r;
}

// ACC = 512 / (levels x BN) accumulator buffers in TMEM: with two (fp64 digits, n-tiles
// <= 32 wide) the epilogue drains tile i while the MMAs of tile i+1 run -- the short-K
// shapes (c3 phase R: K = 500) are otherwise epilogue-bound.
template <int BN, class SC>
struct OzTile {
  static constexpr int ACC = (512 / (SC::LV * BN)) >= 2 ? 2 : 1;
  static constexpr int A_PLANE = kOzBM * SC::BK;  // 8 KB (BK 64) / 4 KB (BK 32)
  static constexpr int B_PLANE = BN * SC::BK;
  static constexpr int STAGE = SC::D * (A_PLANE + B_PLANE);
  // fp64 output staging: the whole 128 x BN tile for the fp32 scheme (TMEM is released
  // before the global stores), 16-column chunks for the fp64 one (deeper stage ring; the
  // split-K fix-up and the residual epilogue live in the chunked path)
  static constexpr int FULL_OUT = kOzBM * (BN + 1) * 8;
  static constexpr bool CHUNKED = SC::BAL || (212 * 1024 - FULL_OUT) / STAGE < 3;
  // CW: columns per TMEM load step and staging chunk.  (CW = 8 for the 64-wide fp64 tiles,
  // whose 9 KB staging buffer leaves room for a fifth 42 KB stage, measured no faster at c5
  // -- 4.61 ms either way -- and 5 % slower at c3: 16 everywhere.)
  static constexpr bool WIDE64 = false;
  static constexpr int CW = WIDE64 ? 8 : 16;
  static constexpr int OUT_COLS = CHUNKED ? CW : BN;
  static constexpr int OUT_LD = OUT_COLS + 1;                 // odd: no bank conflicts
  static constexpr int OUT_BYTES = kOzBM * OUT_LD * 8;
  static constexpr int CAP = (WIDE64 ? 224 : 212) * 1024;   // dynamic smem for stages + staging
  static constexpr int STAGES = (CAP - OUT_BYTES) / STAGE < 6 ? (CAP - OUT_BYTES) / STAGE : 6;
  static constexpr int TMEM_COLS = 512;
  static constexpr int THREADS = 6 * 32;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE + OUT_BYTES + 1024 + 256;
  static_assert(SC::LV * BN <= TMEM_COLS, "levels x BN accumulator columns exceed TMEM");
  static constexpr int ACC_COLS = SC::LV * BN;  // one accumulator buffer
  static_assert(STAGES >= 2, "digit stage too large for shared memory");
};

// Row tiling of a digit operand: tiles [0, nbig) are wbig rows, the rest wsmall rows
// (A: all 128; B: N split into ceil(N / 64) tiles of widths 16 q or 16 (q + 1) <= 64,
// so R^2 = 400 is 4 x 64 + 3 x 48 -- no MMA work on padding columns).
struct OzRowTiles {
  int ntiles, nbig, wbig, wsmall;
  __host__ __device__ __forceinline__ int64_t start(int t) const {
    return t < nbig ? static_cast<int64_t>(t) * wbig
                    : static_cast<int64_t>(nbig) * wbig + static_cast<int64_t>(t - nbig) * wsmall;
  }
  __host__ __device__ __forceinline__ int width(int t) const { return t < nbig ? wbig : wsmall; }
  __host__ __device__ __forceinline__ int64_t rows_pad() const { return start(ntiles); }
  __host__ __device__ __forceinline__ void locate(int64_t r, int& t, int& rr) const {
    const int64_t nb = static_cast<int64_t>(nbig) * wbig;
    if (r < nb) {
      t = static_cast<int>(r / wbig);
      rr = static_cast<int>(r - static_cast<int64_t>(t) * wbig);
    } else if (r - nb < 0x7fffffff) {  // 32-bit division (the common case)
      const uint32_t q = static_cast<uint32_t>(r - nb);
      t = nbig + static_cast<int>(q / static_cast<uint32_t>(wsmall));
      rr = static_cast<int>(q % static_cast<uint32_t>(wsmall));
    } else {
      t = nbig + static_cast<int>((r - nb) / wsmall);
      rr = static_cast<int>((r - nb) % wsmall);
    }
  }
  static OzRowTiles fixed(int64_t rows, int w) {
    const int n = static_cast<int>((rows + w - 1) / w);
    return {n, 0, w, w};
  }
  // mult > 1: the tile count is rounded up to a multiple of mult (cluster groups of n-tiles);
  // returns ntiles = 0 when that leaves a tile without a 16-row unit
  static OzRowTiles balanced(int64_t rows, int wmax, int mult = 1) {
    int n = static_cast<int>((rows + wmax - 1) / wmax);
    n = (n + mult - 1) / mult * mult;
    const int units = static_cast<int>((rows + 15) / 16);
    const int q = units / n, big = units % n;
    if (q == 0) return {0, 0, 16, 16};
    return {n, big, 16 * (q + 1), 16 * q};
  }
};

struct OzArgs {
  int64_t M, K, N;
  int64_t kchunk;
  int splits;
  int mtiles, ntiles;  // tile t -> (split, m-tile, n-tile), n fastest
  OzRowTiles nt;       // widths of the n-tiles (<= BN)
  int rotate;          // rotate the k-block order by the m-tile index
  // two-way split-K fix-up (chunked epilogue): the first of a tile's two K halves to finish
  // leaves its partial in ws ([M][N]) and raises ready[tile]; the second adds it to its own
  // and stores the result (fp addition commutes: the sum is the same whichever is first)
  int fixup;
  int* tickets;        // [mtiles * ntiles], zero at launch
  int* ready;          // [mtiles * ntiles], zero at launch
  // residual mode (exact error, chunked epilogue, one K split): C is never stored; the
  // epilogue accumulates sum (X[m][n] - C[m][n])^2 (X row-major, pitch ldx) and every CTA
  // writes its fixed-order partial to rpart[blockIdx.x]
  const double* X;
  int64_t ldx;
  double* rpart;
  int64_t kblocks;     // 64-k blocks of the tiled digit layout (ceil(K / 64))
  const int8_t* ad;    // A digits, tiled: [mtiles][kblocks][D][128 x 64 B]
  const int8_t* bd;    // B digits, tiled: [n-tile][kblocks][D][width x 64 B]
  CMap cmap;
  const int32_t* ea;  // [M] row exponents of A
  const int32_t* eb;  // [N] row exponents of B
  double* C;
  double* ws;
};

// byte offset of (row r, k) inside the tiled digit layout of one plane block
// (rows_per_tile rows x 64 B, SWIZZLE_64B)
// byte offset of (row r, k) of one digit plane in the tiled layout: rows of bk bytes,
// SWIZZLE_64B (bk 64: 16-byte chunk c of row r at c ^ ((r >> 1) & 3)) or SWIZZLE_32B
// (bk 32: chunk c at c ^ ((r >> 2) & 1))
__host__ __device__ __forceinline__ int64_t oz_tiled_offset(int64_t r, int64_t k, int plane, const OzRowTiles& rt,
                                                            int64_t kblocks, int digits, int bk = 64) {
  int t, rr;
  rt.locate(r, t, rr);
  const int w = rt.width(t);
  const int64_t kb = k / bk, c = k % bk;
  const int64_t sw = bk == 64 ? ((c >> 4) ^ ((rr >> 1) & 3)) : ((c >> 4) ^ ((rr >> 2) & 1));
  return rt.start(t) * kblocks * bk * digits + (kb * digits + plane) * w * bk + rr * bk + (sw << 4) + (c & 15);
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor (K-major, SWIZZLE_64B, version 1): 64 B rows, 8-row groups 512 B apart
template <int BK = 64>
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  // K-major, version 1; BK 64: SWIZZLE_64B, 8-row groups 512 B apart; BK 32: SWIZZLE_32B, 256 B
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;                  // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>((8 * BK) >> 4) << 32;      // SBO
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(BK == 64 ? 4 : 6) << 61;   // SWIZZLE_64B / SWIZZLE_32B
  return d;
}

// instruction descriptor: D s32, A/B signed int8, K-major, N = bn, M = 128
__device__ __forceinline__ uint32_t i8_idesc(int bn) {
  uint32_t d = 0;
  d |= 2u << 4;                                  // D format: S32
  d |= 1u << 7;                                  // A: signed int8
  d |= 1u << 10;                                 // B: signed int8
  d |= static_cast<uint32_t>(bn >> 3) << 17;
  d |= static_cast<uint32_t>(kOzBM >> 4) << 24;
  return d;
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

// Warp-wide forms: all 32 lanes execute them with warp-uniform operands (so the
// descriptors live in uniform registers, no per-MMA R2UR), one elected lane issues.
__device__ __forceinline__ void umma_i8_warp(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void oz_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// cluster variants: the bulk copy lands at the same shared-memory offset in every CTA of
// `mask` and signals each one's mbarrier at the same offset; the commit arrives on the
// mbarrier of every CTA in `mask`
__device__ __forceinline__ void bulk_load_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                             uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
      "%4;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void oz_commit_mc_warp(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

// zero this warp's 32 TMEM lanes over the first COLS accumulator columns
template <int COLS>
__device__ __forceinline__ void tmem_zero(uint32_t tlane) {
#pragma unroll
  for (int c = 0; c < COLS; c += 16)
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
            tlane + c),
        "r"(0u)
        : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]);
template <int CW>
__device__ __forceinline__ void tmem_ldc(uint32_t taddr, uint32_t (&v)[CW]) {
  if constexpr (CW == 8) tmem_ld8(taddr, v);
  else tmem_ld16(taddr, v);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// One 64-k stage of MMAs for an n-tile of width W (<= BN): A plane s meets the B planes
// t < min(D, LV - s), stacked as one N = (#planes) W operand (at most 256 / W planes per
// MMA) issued at TMEM column (s + t0) W -- the level stride equals the plane stride of the
// stacked operand -- so pair (s, t) lands in level block s + t (W columns each).  The
// descriptors are linear in the smem address (start field = addr >> 4), so each MMA's
// pair is the stage base plus a compile-time offset.
template <int W, int BN, int D, int LV, int BK = 64>
__device__ __forceinline__ void oz_issue_stage(uint32_t tmem, uint64_t da, uint64_t db) {
  constexpr int CH = 256 / W;
  constexpr int A_PLANE = kOzBM * BK, B_PLANE = W * BK;
#pragma unroll
  for (int k = 0; k < BK / 32; ++k)
#pragma unroll
    for (int sa = 0; sa < D; ++sa) {
      const int nb = (D < LV - sa) ? D : LV - sa;
#pragma unroll
      for (int t0 = 0; t0 < nb; t0 += CH) {
        const int cnt = (CH < nb - t0) ? CH : nb - t0;
        umma_i8_warp(tmem + (sa + t0) * W, da + ((sa * A_PLANE + k * 32) >> 4), db + ((t0 * B_PLANE + k * 32) >> 4),
                     i8_idesc(cnt * W), 1u);
      }
    }
}

// Persistent tile schedule shared by the producer, MMA and epilogue roles: CTA b runs
// tiles b, b + gridDim.x, ...; tile t -> (split, m-tile, n-tile) with, inside a split,
// first every wide n-tile (nbig per m-tile) of every m-tile, then every narrow one, n
// fastest -- so the n-tiles of an m-tile run side by side in one round and read their
// shared A stages from L2 together.  (Measured at c5, ncu: widths mixed inside a round
// let the CTAs drift apart, 21 GB of DRAM reads per launch instead of 11; rounds cut to
// whole m-tile groups were slower still.)
// Cluster schedule (CN > 1): a cluster of CN CTAs runs the CN consecutive n-tiles of one
// (split, m-tile) together -- CTA rank r the n-tile group * CN + r -- sharing its A stages
// by multicast; clusters stride over the (split, m-tile, group) units.
template <int CN, class F>
__device__ __forceinline__ void oz_for_tiles_cl(const OzArgs& g, int crank, F&& body) {
  const int groups = g.ntiles / CN, per_split = g.mtiles * groups, total = per_split * g.splits;
  const int cid = blockIdx.x / CN, ncl = gridDim.x / CN;
  for (int u = cid; u < total; u += ncl) {
    const int rem = u % per_split;
    body(u / per_split, rem / groups, (rem % groups) * CN + crank);
  }
}

template <class F>
__device__ __forceinline__ void oz_for_tiles(const OzArgs& g, F&& body) {
  const int per_split = g.mtiles * g.ntiles, total = per_split * g.splits;
  const int nb = g.nt.nbig, ns = g.ntiles - g.nt.nbig;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int rem = t % per_split;
    int mt, nt;
    if (rem < g.mtiles * nb) {
      mt = rem / nb;
      nt = rem % nb;
    } else {
      const int r2 = rem - g.mtiles * nb;
      mt = r2 / ns;
      nt = nb + r2 % ns;
    }
    body(t / per_split, mt, nt);
  }
}

// RES: residual mode (exact error) compiled in only where used -- its per-element loads and
// branches cost the short-K tiles of the plain product ~10 % (c3) when merely predicated off
// CN > 1: launched in clusters of CN along the n-tiles; every CTA loads D / CN of each A stage
// and multicasts it to the cluster, its own B stage locally; a stage is free once all CN
// CTAs' MMAs have read it (empty barriers count CN commits).
// Residual mode runs 8 epilogue warps (two per TMEM lane quarter, alternating 16-column chunks)
// without the staging buffer: every thread owns one output row.
template <bool RES>
constexpr int oz_threads() { return (RES ? 10 : 6) * 32; }

// W8 (chunked storing epilogue): 8 epilogue warps as well -- the two warps of a lane quarter take
// alternate 16-column chunks, each half with its own staging buffer and named barrier.  For the
// short-K shapes (c3, c4), whose tiles spend longer in the epilogue than in their MMAs.
template <int BN, class SC, bool RES = false, int CN = 1, bool W8 = false>
__global__ void __launch_bounds__(oz_threads<RES || W8>(), 1)
oz8_kernel(const __grid_constant__ OzArgs g) {
  // Persistent: CTA b takes tiles b, b + gridDim.x, ...; the smem ring runs across
  // tile boundaries, so the producer prefetches the next tile while the
  // epilogue drains the accumulators of the current one.
  using T = OzTile<BN, SC>;
  constexpr int S = T::STAGES;
  constexpr int D = SC::D, LV = SC::LV;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  static_assert(!W8 || (T::CHUNKED && !RES), "W8 is the chunked storing epilogue on 8 warps");
  constexpr int OUTB = (W8 ? 2 : 1) * T::OUT_BYTES;            // one staging buffer per epilogue half
  double* otile = reinterpret_cast<double*>(sm + S * T::STAGE);  // [kOzBM][OUT_LD] epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * T::STAGE + OUTB);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;          // [ACC]
  uint64_t* acc_empty = acc_full + T::ACC;  // [ACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + T::ACC);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int crank = CN > 1 ? static_cast<int>(cluster_ctarank()) : 0;
  constexpr uint16_t kMask = static_cast<uint16_t>((1u << CN) - 1u);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CN);
    }
    for (int b = 0; b < T::ACC; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, (RES || W8) ? 8 : 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(T::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (CN > 1) cluster_sync_all();  // peers' barriers are initialised before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  auto for_tiles = [&](auto&& body) {
    if constexpr (CN > 1) oz_for_tiles_cl<CN>(g, crank, body);
    else oz_for_tiles(g, body);
  };

  auto tile_k = [&](int split, int64_t& kbeg, int& ktiles) {
    kbeg = static_cast<int64_t>(split) * g.kchunk;
    const int64_t kend = (g.K < kbeg + g.kchunk) ? g.K : kbeg + g.kchunk;
    ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + SC::BK - 1) / SC::BK) : 0;
  };

  if (warp == 0) {
    // ------------------------------ bulk-copy producer ------------------------------
    if (lane == 0) {
      uint32_t gk = 0;
      for_tiles([&](int split, int mt, int nt) {
        int64_t kbeg;
        int ktiles;
        tile_k(split, kbeg, ktiles);
        const int bw = g.nt.width(nt);
        const int64_t bstart = g.nt.start(nt) * g.kblocks * SC::BK * D;
        // k blocks in a rotated order (the int32 accumulation is exact, so the order is
        // free): the rotation follows the m-tile, so the CTAs that share an A tile (its
        // n-tiles run side by side) read it in step and hit L2, while different m-tiles
        // spread over different B blocks
        const int rot = (ktiles > 0 && g.rotate) ? mt % ktiles : 0;
        for (int kt = 0; kt < ktiles; ++kt, ++gk) {
          const uint32_t s = gk % S;
          if (gk >= S) mbar_wait(empty + s, ((gk / S) - 1) & 1);
          uint8_t* st = sm + s * T::STAGE;
          const uint32_t bbytes = static_cast<uint32_t>(D * bw * SC::BK);
          mbar_expect_tx(full + s, D * T::A_PLANE + bbytes);
          const int kr = kt + rot < ktiles ? kt + rot : kt + rot - ktiles;
          const int64_t kb = kbeg / SC::BK + kr;
          const int8_t* asrc = g.ad + (static_cast<int64_t>(mt) * g.kblocks + kb) * (D * T::A_PLANE);
          if constexpr (CN > 1) {
#pragma unroll
            for (int pl = crank * D / CN; pl < (crank + 1) * D / CN; ++pl)  // (uneven split when CN does not divide D)
              bulk_load_mc(st + pl * T::A_PLANE, asrc + pl * T::A_PLANE, T::A_PLANE, full + s, kMask);
          } else {
            bulk_load(st, asrc, D * T::A_PLANE, full + s);
          }
          bulk_load(st + D * T::A_PLANE, g.bd + bstart + kb * bbytes, bbytes, full + s);
        }
      });
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    // The whole warp runs this loop with warp-uniform values (oz_issue_stage).
    const uint64_t dA0 = oz_desc<SC::BK>(smem_u32(sm)), dB0 = oz_desc<SC::BK>(smem_u32(sm) + D * T::A_PLANE);
    uint32_t gk = 0, it = 0;
    for_tiles([&](int split, int, int nt) {
      int64_t kbeg;
      int ktiles;
      tile_k(split, kbeg, ktiles);
      const int bw = g.nt.width(nt);
      const int ab = static_cast<int>(it % T::ACC);
      const uint32_t tacc = tmem + ab * T::ACC_COLS;
      mbar_wait(acc_empty + ab, (it / T::ACC) & 1);  // this buffer drained and zeroed by the epilogue
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      for (int kt = 0; kt < ktiles; ++kt, ++gk) {
        const uint32_t s = gk % S;
        mbar_wait(full + s, (gk / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        {
          const uint64_t da = dA0 + ((s * T::STAGE) >> 4), db = dB0 + ((s * T::STAGE) >> 4);
          // warp-uniform: the n-tile width fixes the MMA shapes (widths <= BN)
          if constexpr (BN >= 64) {
            if (bw == 64) oz_issue_stage<64, BN, D, LV, SC::BK>(tacc, da, db);
            else if (bw == 48) oz_issue_stage<48, BN, D, LV, SC::BK>(tacc, da, db);
            else if (bw == 32) oz_issue_stage<32, BN, D, LV, SC::BK>(tacc, da, db);
            else oz_issue_stage<16, BN, D, LV, SC::BK>(tacc, da, db);
          } else {
            if (bw == 32) oz_issue_stage<32, BN, D, LV, SC::BK>(tacc, da, db);
            else oz_issue_stage<16, BN, D, LV, SC::BK>(tacc, da, db);
          }
          // the stage is free once these MMAs (and, in a cluster, every peer's) have read it
          if constexpr (CN > 1) oz_commit_mc_warp(empty + s, kMask);
          else oz_commit_warp(empty + s);
        }
        __syncwarp();
      }
      if (ktiles > 0) oz_commit_warp(acc_full + ab);
      else if (lane == 0) mbar_arrive(acc_full + ab);
      __syncwarp();
      ++it;
    });
  } else {
    // ------------------------------ epilogue ------------------------------
    // TMEM -> fp64 combination of the exact int32 levels (Horner in 1 / RAD) -> smem tile
    // (lane = row) -> global with lanes along n (contiguous for every CMap the
    // engine uses).  Whole-tile staging releases TMEM before the global stores;
    // chunked staging (large digit stages) stores 16 columns at a time.
    const int quad = warp & 3;
    constexpr int EH = (RES || W8) ? 2 : 1;              // epilogue warps per TMEM lane quarter
    const int half = (RES || W8) ? (warp - 2) >> 2 : 0;  // this warp's 16-column chunks are ci % EH == half
    const uint32_t tlane0 = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    __shared__ int64_t roff_all[W8 ? 2 : 1][kOzBM];  // chunked path: C offsets of the current tile's rows
    int64_t* roff_s = roff_all[W8 ? half : 0];
    double* otile_h = otile + (W8 ? half : 0) * (T::OUT_BYTES / 8);  // this half's staging buffer
    // named barriers: one per epilogue half (128 threads), one across both halves (fix-up ticket)
    auto bar_half = [&]() {
      if (W8 && half == 1) asm volatile("bar.sync 2, 128;\n" ::: "memory");
      else asm volatile("bar.sync 1, 128;\n" ::: "memory");
    };
    auto bar_all = [&]() {
      if constexpr (W8) asm volatile("bar.sync 3, 256;\n" ::: "memory");
      else asm volatile("bar.sync 1, 128;\n" ::: "memory");
    };
    if (half == 0)
      for (int b = 0; b < T::ACC; ++b) tmem_zero<LV * BN>(tlane0 + b * T::ACC_COLS);  // MMAs always accumulate
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0)
      for (int b = 0; b < T::ACC; ++b) mbar_arrive(acc_empty + b);
    uint32_t it = 0;
    double rsum = 0.0;  // residual mode: this thread's squared residuals, in tile order
    for_tiles([&](int split, int mt, int nt) {
      int64_t kbeg;
      int ktiles;
      tile_k(split, kbeg, ktiles);
      const int64_t m0 = static_cast<int64_t>(mt) * kOzBM, n0 = g.nt.start(nt);
      const int bw = g.nt.width(nt);
      const int64_t nend = (n0 + bw < g.N) ? n0 + bw : g.N;
      const int ab = static_cast<int>(it % T::ACC);
      const uint32_t tlane = tlane0 + ab * T::ACC_COLS;
      const int r = quad * 32 + lane;
      const int64_t m = m0 + r;
      if constexpr (RES) {
        // Residual mode: every thread owns one output row of the tile, so it reads its own X
        // entries (whole 128-byte lines per 16-column chunk) -- issued before the wait for the
        // accumulators, so the DRAM latency overlaps the tile's MMAs -- and needs neither the
        // staging buffer nor a CTA barrier.  Chunk ci of the tile belongs to the warp with
        // ci % EH == half of this lane quarter.
        constexpr int CWR = 16, NCH = BN / CWR / EH;  // chunk width, chunks per warp
        const bool rok = m < g.M;
        const double* xrow = g.X + (rok ? m : 0) * g.ldx + n0;
        const bool vec = ((g.ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(g.X) & 15u) == 0);
        double xres[NCH * CWR];
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c0 = (j * EH + half) * CWR;
#pragma unroll
          for (int q = 0; q < CWR; q += 2) {
            const bool ok0 = rok && c0 + q < bw && n0 + c0 + q < nend;
            const bool ok1 = rok && c0 + q + 1 < bw && n0 + c0 + q + 1 < nend;
            if (vec && ok1) {
              const double2 t = __ldcs(reinterpret_cast<const double2*>(xrow + c0 + q));
              xres[j * CWR + q] = t.x;
              xres[j * CWR + q + 1] = t.y;
            } else {
              xres[j * CWR + q] = ok0 ? __ldcs(xrow + c0 + q) : 0.0;
              xres[j * CWR + q + 1] = ok1 ? __ldcs(xrow + c0 + q + 1) : 0.0;
            }
          }
        }
        mbar_wait(acc_full + ab, (it / T::ACC) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const double sa = (rok && ktiles > 0) ? ldexp(1.0, g.ea[m]) : 0.0;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const int c0 = (j * EH + half) * CWR;
          if (c0 < bw) {
            uint32_t v[LV][CWR];
#pragma unroll
            for (int L = 0; L < LV; ++L) tmem_ld16(tlane + L * bw + c0, v[L]);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int q = 0; q < CWR; ++q) {
              constexpr int H = (LV + 1) / 2;
              int64_t hi = static_cast<int32_t>(v[0][q]), lo = static_cast<int32_t>(v[H][q]);
#pragma unroll
              for (int L = 1; L < H; ++L) hi = hi * static_cast<int64_t>(SC::RAD) + static_cast<int32_t>(v[L][q]);
#pragma unroll
              for (int L = H + 1; L < LV; ++L) lo = lo * static_cast<int64_t>(SC::RAD) + static_cast<int32_t>(v[L][q]);
              constexpr double CHI = SC::W0 * oz_rad_pow<SC>(H - 1), CLO = CHI * oz_rad_pow<SC>(LV - H);
              const double val = fma(static_cast<double>(lo), CLO, static_cast<double>(hi) * CHI);
              const int64_t n = n0 + c0 + q;
              if (rok && n < nend) {
                const int e = g.eb[n];  // (warp-uniform address: one broadcast load)
                const double sb = static_cast<unsigned>(e + 1022) <= 2045u ? __hiloint2double((e + 1023) << 20, 0)
                                                                            : ldexp(1.0, e);
                const double d = xres[j * CWR + q] - (val * sa) * sb;
                rsum = fma(d, d, rsum);
              }
            }
            // zero this chunk's level accumulators for the next tile (MMAs always accumulate)
#pragma unroll
            for (int L = 0; L < LV; ++L)
              asm volatile(
                  "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                      tlane + L * bw + c0),
                  "r"(0u)
                  : "memory");
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);
        ++it;
        return;
      }
      mbar_wait(acc_full + ab, (it / T::ACC) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const double sa = (m < g.M && ktiles > 0) ? ldexp(1.0, g.ea[m]) : 0.0;
      bool part = g.splits > 1;
      bool second = false;  // fix-up: this CTA finishes the tile (adds the other half's partial)
      const int tile = mt * g.ntiles + nt;
      if (T::CHUNKED && g.fixup) {
        __shared__ int ticket_s;
        if (half == 0 && quad == 0 && lane == 0) {
          const int tk = atomicAdd(g.tickets + tile, 1);
          if (tk == 1) {
            while (atomicAdd(g.ready + tile, 0) == 0) __nanosleep(200);
            __threadfence();
          }
          ticket_s = tk;
        }
        bar_all();
        second = ticket_s == 1;
        part = !second;
      }
      const bool fix = T::CHUNKED && g.fixup;
      const uint32_t M2 = part ? (1u << 30) : static_cast<uint32_t>(g.cmap.M2);
      const uint32_t N2 = part ? (1u << 30) : static_cast<uint32_t>(g.cmap.N2);
      const int64_t sm1 = part ? 0 : g.cmap.sm1, sm2 = part ? g.N : g.cmap.sm2;
      const int64_t sn1 = part ? 0 : g.cmap.sn1, sn2 = part ? 1 : g.cmap.sn2;
      double* base = part ? g.ws + (fix ? 0 : static_cast<int64_t>(split) * g.M * g.N) : g.C;
      const int rows = static_cast<int>((g.M - m0) < kOzBM ? (g.M - m0) : kOzBM);
      if constexpr (T::CHUNKED) {
        // row offsets of this tile in C, once per tile (read after the first chunk's barrier;
        // the previous tile's readers are past its last barrier)
        const uint32_t mm = static_cast<uint32_t>(m0 + r);
        roff_s[r] = r < rows ? static_cast<int64_t>(mm / M2) * sm1 + static_cast<int64_t>(mm % M2) * sm2 : 0;
      }
      constexpr int CW = T::CW;
      constexpr int RPW = 32 / CW;              // chunk rows per warp store instruction
      constexpr int NIT = kOzBM / (4 * RPW);    // store iterations per chunk
      const int cl = lane % CW, rsub = lane / CW;
#pragma unroll 1
      for (int c0 = half * CW; c0 < bw; c0 += EH * CW) {
        uint32_t v[LV][CW];
#pragma unroll
        for (int L = 0; L < LV; ++L) tmem_ldc<CW>(tlane + L * bw + c0, v[L]);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int oc = T::CHUNKED ? 0 : c0;
#pragma unroll
        for (int q = 0; q < CW; ++q) {
          // levels 0..H-1 and H..LV-1 combined exactly in int64 (Horner in RAD, < 2^55), two
          // conversions and one fma instead of LV conversions and LV - 1 dependent fmas
          constexpr int H = (LV + 1) / 2;
          int64_t hi = static_cast<int32_t>(v[0][q]), lo = static_cast<int32_t>(v[H][q]);
#pragma unroll
          for (int L = 1; L < H; ++L) hi = hi * static_cast<int64_t>(SC::RAD) + static_cast<int32_t>(v[L][q]);
#pragma unroll
          for (int L = H + 1; L < LV; ++L) lo = lo * static_cast<int64_t>(SC::RAD) + static_cast<int32_t>(v[L][q]);
          // the pair weight W0 RAD^-(H-1) (~2^-38) is applied here, not folded into the row
          // scale: 2^ea stays an exact power of two, so rows near the bottom of the exponent
          // range do not lose bits to a subnormal scale factor
          constexpr double CHI = SC::W0 * oz_rad_pow<SC>(H - 1), CLO = CHI * oz_rad_pow<SC>(LV - H);
          const double val = fma(static_cast<double>(lo), CLO, static_cast<double>(hi) * CHI);
          otile_h[r * T::OUT_LD + oc + q] = val * sa;
        }
        if constexpr (T::CHUNKED) {
          // store this CW-column chunk: lane -> (row rsub, column cl), warp -> rows quad*RPW + ...
          bar_half();
          const int64_t n = n0 + c0 + cl;
          const bool nok = n < nend;
          const uint32_t un = static_cast<uint32_t>(n);
          const int64_t coff = nok ? static_cast<int64_t>(un / N2) * sn1 + static_cast<int64_t>(un % N2) * sn2 : 0;
          const double sb = nok ? ldexp(1.0, g.eb[n]) : 0.0;
          // the other K half's partial (fix-up) or X (residual mode) for this chunk: all 16
          // loads issued before any use (one memory latency per chunk, not one per row)
          double pv[NIT], xv[NIT];
          if (second || RES) {
#pragma unroll
            for (int k = 0; k < NIT; ++k) {
              const int rr = quad * RPW + rsub + 4 * RPW * k;
              pv[k] = (second && nok && rr < rows) ? __ldcg(g.ws + static_cast<int64_t>(m0 + rr) * g.N + n) : 0.0;
              xv[k] = (RES && nok && rr < rows) ? __ldcs(g.X + static_cast<int64_t>(m0 + rr) * g.ldx + n) : 0.0;
            }
          } else {
#pragma unroll
            for (int k = 0; k < NIT; ++k) pv[k] = xv[k] = 0.0;
          }
#pragma unroll
          for (int k = 0; k < NIT; ++k) {
            const int rr = quad * RPW + rsub + 4 * RPW * k;
            if (rr >= rows) break;
            const int64_t roff = roff_s[rr];
            const double o = otile_h[rr * T::OUT_LD + cl] * sb + pv[k];
            if constexpr (RES) {
              if (nok) {
                const double d = xv[k] - o;
                rsum = fma(d, d, rsum);
              }
            } else {
              if (nok) base[roff + coff] = o;
            }
          }
          bar_half();
        }
      }
      if (T::CHUNKED && g.fixup && part) {  // publish this half's partial
        __threadfence();
        bar_all();
        if (half == 0 && quad == 0 && lane == 0) atomicExch(g.ready + tile, 1);
      }
      if constexpr (W8) {
        // each half zeroes the level accumulators of its own chunks
        for (int c0 = half * CW; c0 < bw; c0 += EH * CW) {
#pragma unroll
          for (int L = 0; L < LV; ++L)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                    tlane + L * bw + c0),
                "r"(0u)
                : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      } else {
        tmem_zero<LV * BN>(tlane);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + ab);  // the MMA warp may reuse this buffer
      if constexpr (!T::CHUNKED) {
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        // coalesced stores: lane -> column n (BN / 32 per lane), warp -> rows quad, quad + 4, ...
        int64_t coff[BN / 32];
        double sb[BN / 32];
        bool nok[BN / 32];
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) {
          const int64_t n = n0 + lane + 32 * j;
          nok[j] = n < nend;
          const uint32_t un = static_cast<uint32_t>(n);
          coff[j] = nok[j] ? static_cast<int64_t>(un / N2) * sn1 + static_cast<int64_t>(un % N2) * sn2 : 0;
          sb[j] = nok[j] ? ldexp(1.0, g.eb[n]) : 0.0;
        }
        for (int rr = quad; rr < rows; rr += 4) {
          const uint32_t mm = static_cast<uint32_t>(m0 + rr);
          const int64_t roff = static_cast<int64_t>(mm / M2) * sm1 + static_cast<int64_t>(mm % M2) * sm2;
#pragma unroll
          for (int j = 0; j < BN / 32; ++j)
            if (nok[j]) base[roff + coff[j]] = otile[rr * T::OUT_LD + lane + 32 * j] * sb[j];
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");  // otile reused by the next tile
      }
      ++it;
    });
    if constexpr (RES) {  // fixed-order CTA partial: warp shuffles, then the 8 warps in order
      for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
      double* red = otile;  // (unused in residual mode)
      if (lane == 0) red[warp - 2] = rsum;
      asm volatile("bar.sync 1, 256;\n" ::: "memory");
      if (warp == 2 && lane == 0) {
        double t = red[0];
        for (int w = 1; w < 8; ++w) t += red[w];
        g.rpart[blockIdx.x] = t;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (CN > 1) cluster_sync_all();  // no CTA leaves while peers may still signal it
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// slicing: per-output-row max |x| -> exponent -> D int8 digit planes
// ---------------------------------------------------------------------------
// row max of a row-major [rows][ld] matrix (one warp per row); out[r] = max_c |x[r][c]|
template <typename Tin>
__global__ void __launch_bounds__(256) oz_rowmax_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += nw) {
    double m = 0.0;
    for (int64_t c = lane; c < cols; c += 32) m = fmax(m, fabs(static_cast<double>(x[r * ld + c])));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) out[r] = m;
  }
}

// column max of a row-major [rows][ld] matrix; out[c] must be zeroed (atomicMax on the
// bit pattern of non-negative doubles).  A block covers min(cols, 256) columns x
// (256 / that) row phases of a rows_per_block slab, so narrow matrices (the half
// chain's 64 columns) still use every thread.
template <typename Tin>
__global__ void __launch_bounds__(256) oz_colmax_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld, int64_t rows_per_block, double* __restrict__ out) {
  const int cw = cols < 256 ? static_cast<int>(cols) : 256;
  const int phases = 256 / cw;
  const int tc = threadIdx.x % cw, tr = threadIdx.x / cw;
  const int64_t c = blockIdx.x * static_cast<int64_t>(cw) + tc;
  if (tr >= phases || c >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per_block;
  const int64_t r1 = (r0 + rows_per_block < rows) ? r0 + rows_per_block : rows;
  double m = 0.0;
  for (int64_t r = r0 + tr; r < r1; r += phases) m = fmax(m, fabs(static_cast<double>(x[r * ld + c])));
  atomicMax(reinterpret_cast<unsigned long long*>(out) + c, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// exponent with |x| < 2^e for every |x| <= mx (mx == 0 -> 0); non-finite mx -> 0 (caught upstream)
__device__ __forceinline__ int oz_exponent(double mx) {
  if (!(mx > 0.0) || !isfinite(mx)) return 0;
  return ilogb(mx) + 1;
}

// v = x 2^-e, |v| < 1 -> the scheme's digits.  Truncated (fp32 scheme): every step
// exact (power-of-two scalings, subtraction of an integer within 1 of its operand).
// Balanced: d_0 = rint(C0 v), then d_s = rint(RAD r), the remainder r = m r_prev - d
// taken by one fma (exact whenever it fits 53 bits -- always for |v| >= 1/2 -- else
// rounded at 2^-54 of the digit unit).  q comes from the rounded product m r_prev, so when
// that sat within an ulp of a half-integer |r| may exceed 1/2 by ~2^-53: the next digit is
// still rint(<= 127 + 2^-45) <= 127, and d_0 = rint(127 v) <= 127 since |v| < 1.
template <class SC>
__device__ __forceinline__ void oz_digits(double v, int8_t (&d)[SC::D]) {
  if constexpr (SC::BAL) {
    double r = v;
#pragma unroll
    for (int s = 0; s < SC::D; ++s) {
      const double m = s == 0 ? SC::C0 : SC::RAD;
      const double q = rint(r * m);
      r = fma(r, m, -q);
      d[s] = static_cast<int8_t>(static_cast<int>(q));
    }
  } else {
#pragma unroll
    for (int s = 0; s < SC::D; ++s) {
      const double t = v * 128.0;
      const double q = trunc(t);
      d[s] = static_cast<int8_t>(static_cast<int>(q));
      v = t - q;
    }
  }
}

// x [rows][ld_in] -> tiled digit planes of the output rows (rows, or cols when
// transposed; K = the other extent), covering the whole padded layout (zero
// digits in the tile padding, so no memset is needed); mx[out_rows] = max |x| of
// each output row, exps[out_rows] its exponent.  One thread per (output row,
// 16-k chunk): 16 values -> D planes x one 16 B store.
template <typename Tin, class SC>
__global__ void __launch_bounds__(256) oz_digits_tiled_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                              int64_t ld_in, int transpose,
                                                              const double* __restrict__ mx, int8_t* __restrict__ out,
                                                              OzRowTiles rt, int32_t* __restrict__ exps) {
  constexpr int D = SC::D, BK = SC::BK;
  const int64_t out_rows = transpose ? cols : rows, K = transpose ? rows : cols;
  const int64_t kblocks = (K + BK - 1) / BK, kchunks = kblocks * (BK / 16);
  const int64_t rows_pad = rt.rows_pad();
  const int64_t total = rows_pad * kchunks;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // coalesced reads: consecutive threads walk k within a row (row-major input)
    // or rows at a fixed k (transposed input)
    const int64_t orow = transpose ? idx % rows_pad : idx / kchunks;
    const int64_t ch = transpose ? idx / rows_pad : idx % kchunks;
    const bool rok = orow < out_rows;
    const int e = rok ? oz_exponent(mx[orow]) : 0;
    const double sc = ldexp(1.0, -(e / 2)), sc2 = ldexp(1.0, e / 2 - e);  // (finite for subnormal rows)
    uint32_t w[D][4];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int q = 0; q < 4; ++q) w[d][q] = 0;
    if (rok && ch * 16 < K) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t k = ch * 16 + j;
        double v = 0.0;
        if (k < K) v = static_cast<double>(transpose ? x[k * ld_in + orow] : x[orow * ld_in + k]);
        int8_t dg[D];
        oz_digits<SC>(v * sc * sc2, dg);
#pragma unroll
        for (int d = 0; d < D; ++d)
          w[d][j >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(dg[d])) << (8 * (j & 3));
      }
    }
    // plane d of a row sits width x 64 bytes after plane d - 1
    int tt, rr_;
    rt.locate(orow, tt, rr_);
    const int64_t pstride = static_cast<int64_t>(rt.width(tt)) * BK;
    const int64_t off0 = oz_tiled_offset(orow, ch * 16, 0, rt, kblocks, D, BK);
#pragma unroll
    for (int d = 0; d < D; ++d)
      *reinterpret_cast<uint4*>(out + off0 + d * pstride) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
    if (rok && ch == 0) exps[orow] = e;
  }
}

// Transposed slicing (out rows = columns of x, K = rows of x): a CTA owns a 64 k x 64 n
// block, reads it coalesced along n into shared memory, and each group of 4 threads
// writes one output row's full 64-byte digit row per plane (4 x 16 B, contiguous), so
// the tiled digit layout is written in whole sectors.  256 threads; grid (ceil(rows/64)
// k blocks, ceil(padded out rows / 64)) covers the layout's padding too (zero digits there).
template <typename Tin, class SC>
__global__ void __launch_bounds__(256) oz_digits_tiled_t_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                                int64_t ld_in, const double* __restrict__ mx,
                                                                int8_t* __restrict__ out, OzRowTiles rt,
                                                                int32_t* __restrict__ exps, int plo = 0,
                                                                int phi = 0) {
  // plo > 0: output row n' takes column (n' % plo) phi + n' / plo of x (and its maximum
  // mx[]) -- the column order that makes the environment's output tiles contiguous
  constexpr int D = SC::D, BK = SC::BK;
  __shared__ double tile[64][65];
  const int64_t K = rows, out_rows = cols;
  const int64_t kblocks = (K + BK - 1) / BK;
  const int64_t n0 = static_cast<int64_t>(blockIdx.y) * 64, k0 = static_cast<int64_t>(blockIdx.x) * 64;
  const int tid = threadIdx.x;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int kk = e >> 6, nn = e & 63;
    const int64_t k = k0 + kk, n = n0 + nn;
    const int64_t nc = plo > 0 ? (n % plo) * phi + n / plo : n;
    tile[kk][nn] = (k < K && n < out_rows) ? static_cast<double>(x[k * ld_in + nc]) : 0.0;
  }
  __syncthreads();
  const int nl = tid >> 2, ch = tid & 3;
  const int64_t orow = n0 + nl;
  if (orow >= rt.rows_pad() || k0 + ch * 16 >= kblocks * BK) return;  // (BK 32: a 64-k tile may pass the layout)
  const bool rok = orow < out_rows;
  const int e = rok ? oz_exponent(mx[plo > 0 ? (orow % plo) * phi + orow / plo : orow]) : 0;
  const double sc = ldexp(1.0, -(e / 2)), sc2 = ldexp(1.0, e / 2 - e);  // (finite for subnormal rows)
  uint32_t w[D][4];
#pragma unroll
  for (int d = 0; d < D; ++d)
#pragma unroll
    for (int q = 0; q < 4; ++q) w[d][q] = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    int8_t dg[D];
    oz_digits<SC>(tile[ch * 16 + j][nl] * sc * sc2, dg);
#pragma unroll
    for (int d = 0; d < D; ++d) w[d][j >> 2] |= static_cast<uint32_t>(static_cast<uint8_t>(dg[d])) << (8 * (j & 3));
  }
  int tt, rr_;
  rt.locate(orow, tt, rr_);
  const int64_t pstride = static_cast<int64_t>(rt.width(tt)) * BK;
  const int64_t off0 = oz_tiled_offset(orow, k0 + ch * 16, 0, rt, kblocks, D, BK);
#pragma unroll
  for (int d = 0; d < D; ++d)
    *reinterpret_cast<uint4*>(out + off0 + d * pstride) = make_uint4(w[d][0], w[d][1], w[d][2], w[d][3]);
  if (rok && blockIdx.x == 0 && ch == 0) exps[orow] = e;
}

}  // namespace trals
