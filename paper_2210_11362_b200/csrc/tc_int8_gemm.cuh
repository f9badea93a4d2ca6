// fp32-accurate GEMM on the int8 tcgen05 tensor cores (Ozaki-style digit slicing)
// for the fp32 variant's environment products.
//
//   C(m, n) (fp64 out) = sum_k A[m][k] * B[n][k]      A from fp32 X, B from the fp64 half chain
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
// it), and the product keeps every digit pair with s + t <= 4 (13 int8 MMAs per
// k-step).  Measured on N(0,1) data: 1.2-1.9e-8 relative Frobenius against an
// fp64 product of the same fp32 X, dominated by the digit truncation of the
// row/column maxima's 28-bit window (keeping only s + t <= 3 gave 6e-8).
// Pairs of equal level L = s + t share one int32 TMEM accumulator (5 x BN
// columns); the epilogue combines them exactly in fp64 (Horner in 2^-7):
//   C = 2^(ea+eb-14) * sum_L acc_L 2^(-7L).
// No overflow: a level sums at most 4 pairs of |a b| <= 127^2 over at most
// kOzKmax (32768) k per CTA, < 2^31; longer K is always split.
//
// Structure (one 128 x BN tile per CTA, split-K): warp 0 = TMA producer (4 A
// digit planes + 4 B digit planes per stage, {128 k, rows} boxes, 128B
// swizzle), warp 1 = TMEM allocator + single-thread MMA issuer
// (tcgen05.mma.cta_group::1.kind::i8, K-major both, 32 k per MMA),
// warps 2-5 = epilogue (tcgen05.ld 32x32b; warp w owns TMEM lanes 32*(w%4)).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dmma_gemm.cuh"
#include "dmma_tma_gemm.cuh"

namespace trals {

constexpr int kOzBK = 128;       // int8 k per stage (one 128 B swizzle row)
constexpr int kOzBM = 128;
constexpr int kOzDigits = 4;
constexpr int kOzLevels = 5;     // digit-pair levels L = s + t kept (0..4)
constexpr int64_t kOzKmax = 32768;

template <int BN>
struct OzTile {
  static constexpr int A_PLANE = kOzBM * kOzBK;  // 16 KB
  static constexpr int B_PLANE = BN * kOzBK;
  static constexpr int STAGE = kOzDigits * (A_PLANE + B_PLANE);
  static constexpr int STAGES = (200 * 1024) / STAGE < 4 ? (200 * 1024) / STAGE : 4;
  static constexpr int TMEM_COLS = kOzLevels * BN <= 256 ? 256 : 512;
  static constexpr int THREADS = 6 * 32;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE + 1024 + 256;
};

struct OzArgs {
  int64_t M, K, N;
  int64_t kchunk;
  int splits;
  CMap cmap;
  const int32_t* ea;  // [M] row exponents of A
  const int32_t* eb;  // [N] row exponents of B
  double* C;
  double* ws;
};

// UMMA shared-memory descriptor (K-major, SWIZZLE_128B, version 1): 8-row groups 1 KB apart
__device__ __forceinline__ uint64_t oz_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
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

__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

// A maps: 4 digit planes of A, B maps: 4 digit planes of B (each a 2-D int8 tensor map)
struct OzMaps {
  CUtensorMap a[kOzDigits];
  CUtensorMap b[kOzDigits];
};

template <int BN>
__global__ void __launch_bounds__(OzTile<BN>::THREADS, 1)
oz8_kernel(const __grid_constant__ OzMaps maps, const OzArgs g) {
  using T = OzTile<BN>;
  constexpr int S = T::STAGES;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * T::STAGE);
  uint64_t* empty = full + S;
  uint64_t* accum = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kOzBM;
  const int split = blockIdx.z;
  const int64_t kbeg = static_cast<int64_t>(split) * g.kchunk;
  const int64_t kend = (g.K < kbeg + g.kchunk) ? g.K : kbeg + g.kchunk;
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kOzBK - 1) / kOzBK) : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(T::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % S;
        if (kt >= S) mbar_wait(empty + s, ((kt / S) - 1) & 1);
        uint8_t* st = sm + s * T::STAGE;
        mbar_expect_tx(full + s, T::STAGE);
        const int k0 = static_cast<int>(kbeg + static_cast<int64_t>(kt) * kOzBK);
#pragma unroll
        for (int d = 0; d < kOzDigits; ++d) {
          tma_load_2d(st + d * T::A_PLANE, &maps.a[d], full + s, k0, static_cast<int>(m0));
          tma_load_2d(st + kOzDigits * T::A_PLANE + d * T::B_PLANE, &maps.b[d], full + s, k0, static_cast<int>(n0));
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    const uint32_t idesc = i8_idesc(BN);
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % S;
      mbar_wait(full + s, (kt / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sm + s * T::STAGE), b0 = a0 + kOzDigits * T::A_PLANE;
#pragma unroll
        for (int k = 0; k < kOzBK / 32; ++k) {
          const uint32_t first = (kt > 0 || k > 0) ? 1u : 0u;
#pragma unroll
          for (int L = 0; L < kOzLevels; ++L) {
            const int s_lo = L < kOzDigits ? 0 : L - (kOzDigits - 1);
            const int s_hi = L < kOzDigits ? L : kOzDigits - 1;
#pragma unroll
            for (int sa = s_lo; sa <= s_hi; ++sa) {
              const int tb = L - sa;
              umma_i8(tmem + L * BN, oz_desc(a0 + sa * T::A_PLANE + k * 32), oz_desc(b0 + tb * T::B_PLANE + k * 32),
                      idesc, sa == s_lo ? first : 1u);
            }
          }
        }
        oz_commit(empty + s);
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (ktiles > 0) oz_commit(accum);
      else mbar_arrive(accum);
    }
    __syncwarp();
  } else {
    // ------------------------------ epilogue ------------------------------
    mbar_wait(accum, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int quad = warp & 3;
    const int64_t m = m0 + quad * 32 + lane;
    const bool mok = m < g.M;
    const bool have = ktiles > 0;
    const uint32_t m2 = static_cast<uint32_t>(g.cmap.M2), n2 = static_cast<uint32_t>(g.cmap.N2);
    const int ea = mok ? g.ea[m] : 0;
    const int64_t row_off = !mok ? 0
                                 : (g.splits > 1 ? (static_cast<int64_t>(split) * g.M + m) * g.N
                                                 : static_cast<int64_t>(static_cast<uint32_t>(m) / m2) * g.cmap.sm1 +
                                                       static_cast<int64_t>(static_cast<uint32_t>(m) % m2) * g.cmap.sm2);
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (n0 + c0 >= g.N) break;  // warp-uniform
      uint32_t v0[16], v1[16], v2[16], v3[16], v4[16];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0;
      tmem_ld16(taddr, v0);
      tmem_ld16(taddr + BN, v1);
      tmem_ld16(taddr + 2 * BN, v2);
      tmem_ld16(taddr + 3 * BN, v3);
      tmem_ld16(taddr + 4 * BN, v4);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (mok) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t n = n0 + c0 + q;
          if (n >= g.N) continue;
          double val = 0.0;
          if (have) {
            val = static_cast<double>(static_cast<int32_t>(v4[q]));
            val = fma(val, 0.0078125, static_cast<double>(static_cast<int32_t>(v3[q])));
            val = fma(val, 0.0078125, static_cast<double>(static_cast<int32_t>(v2[q])));
            val = fma(val, 0.0078125, static_cast<double>(static_cast<int32_t>(v1[q])));
            val = fma(val, 0.0078125, static_cast<double>(static_cast<int32_t>(v0[q])));
            val = ldexp(val, ea + g.eb[n] - 14);
          }
          if (g.splits > 1) {
            g.ws[row_off + n] = val;
          } else {
            const uint32_t un = static_cast<uint32_t>(n);
            g.C[row_off + static_cast<int64_t>(un / n2) * g.cmap.sn1 + static_cast<int64_t>(un % n2) * g.cmap.sn2] =
                val;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// slicing: per-output-row max |x| -> exponent -> 4 int8 base-128 digit planes
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

// column max of a row-major [rows][ld] matrix; out[c] must be zeroed (atomicMax on the bit pattern)
template <typename Tin>
__global__ void __launch_bounds__(256) oz_colmax_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld, int64_t rows_per_block, double* __restrict__ out) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per_block;
  const int64_t r1 = (r0 + rows_per_block < rows) ? r0 + rows_per_block : rows;
  double m = 0.0;
  for (int64_t r = r0; r < r1; ++r) m = fmax(m, fabs(static_cast<double>(x[r * ld + c])));
  atomicMax(reinterpret_cast<unsigned long long*>(out) + c, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// exponent with |x| < 2^e for every |x| <= mx (mx == 0 -> 0); non-finite mx -> 0 (caught upstream)
__device__ __forceinline__ int oz_exponent(double mx) {
  if (!(mx > 0.0) || !isfinite(mx)) return 0;
  return ilogb(mx) + 1;
}

__device__ __forceinline__ void oz_digits(double v, int8_t (&d)[kOzDigits]) {
#pragma unroll
  for (int s = 0; s < kOzDigits; ++s) {
    const double t = v * 128.0;
    const double q = trunc(t);
    d[s] = static_cast<int8_t>(static_cast<int>(q));
    v = t - q;  // exact
  }
}

// x [rows][ld_in] -> digit planes of the output rows (rows, or cols when transposed),
// planes [4][out_rows][ld_out] int8 (plane stride out_rows * ld_out), exps[out_rows];
// mx[out_rows] = max |x| of each output row.
template <typename Tin>
__global__ void __launch_bounds__(256) oz_digits_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ld_in, int transpose, const double* __restrict__ mx,
                                                        int8_t* __restrict__ planes, int64_t ld_out,
                                                        int32_t* __restrict__ exps) {
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t out_rows = transpose ? cols : rows;
  const int64_t pstride = out_rows * ld_out;
  const int64_t tiles_c = (cols + 31) / 32, tiles = ((rows + 31) / 32) * tiles_c;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = (t / tiles_c) * 32, c0 = (t % tiles_c) * 32;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t r = r0 + ty + j, c = c0 + tx;
      tile[ty + j][tx] = (r < rows && c < cols) ? static_cast<double>(x[r * ld_in + c]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      // output element (orow, ocol): orow = r (or c), ocol = c (or r)
      const int64_t orow = transpose ? c0 + ty + j : r0 + ty + j;
      const int64_t ocol = transpose ? r0 + tx : c0 + tx;
      const bool ok = transpose ? (orow < cols && ocol < rows) : (orow < rows && ocol < cols);
      if (ok) {
        const int e = oz_exponent(mx[orow]);
        const double v = transpose ? tile[tx][ty + j] : tile[ty + j][tx];
        int8_t d[kOzDigits];
        oz_digits(ldexp(v, -e), d);
#pragma unroll
        for (int s = 0; s < kOzDigits; ++s) planes[s * pstride + orow * ld_out + ocol] = d[s];
        if (ocol == 0) exps[orow] = e;
      }
    }
    __syncthreads();
  }
}

}  // namespace trals
