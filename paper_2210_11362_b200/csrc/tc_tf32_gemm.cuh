// tcgen05 (5th-gen tensor core) 3xTF32 GEMM for the fp32 variant's environment products.
//
//   C(m, n) (fp64 out) = sum_k A[m][k] * B[n][k]      A, B fp32, both K-contiguous
//
// Every operand is stored pre-split as hi = tf32(x) (low 13 mantissa bits
// cleared) and lo = x - hi (exact in fp32), and each k-step issues three UMMAs
// into the same fp32 TMEM accumulator: hi*hi + hi*lo + lo*hi.  Dropping lo*lo
// and truncating lo to tf32 costs ~2^-22 relative per product, i.e. fp32-level
// accuracy on the tensor-core path (kind::tf32) that 1xTF32 (2^-11) would not
// give.  Split-K partials are reduced in fp64.
//
// Structure (one 128 x BN output tile per CTA, optional split-K):
//   warp 0   : TMA producer -- A_hi, A_lo, B_hi, B_lo boxes into a STAGES-deep
//              ring (128B swizzle, mbarrier transaction counts);
//   warp 1   : TMEM allocator + MMA issuer (one thread issues
//              tcgen05.mma.cta_group::1.kind::tf32; tcgen05.commit releases
//              each smem stage and finally signals the accumulator);
//   warps 2-5: epilogue -- tcgen05.ld 32x32b from TMEM (warp w owns TMEM lanes
//              32*(w%4)..+31 = tile rows), fp32 -> fp64, stored through the
//              same CMap as the fp64 engine (or as split-K partials).
// Operand layout (UMMA canonical K-major, SWIZZLE_128B): one TMA box of
// {32 k, rows} per operand, rows of 128 B, 8-row groups 1 KB apart (SBO), the
// k-th UMMA_K=8 slice starting 32 B further along the swizzled row.
// Only K-major operands are used: the MN-major (transposed) descriptor form
// produced all-zero accumulators for kind::tf32 on this stack (see
// tools/tc/tc_test.cu), so the engine stores the phase-R copy of X transposed.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dmma_gemm.cuh"
#include "dmma_tma_gemm.cuh"

namespace trals {

constexpr int kTcBK = 32;  // fp32 elements of K per stage (one 128 B swizzle row)
constexpr int kTcBM = 128;

template <int BN>
struct TcTile {
  static constexpr int A_BYTES = kTcBM * kTcBK * 4;  // 16 KB
  static constexpr int B_BYTES = kTcBK * BN * 4;
  static constexpr int STAGE = 2 * (A_BYTES + B_BYTES);  // hi + lo
  static constexpr int STAGES = (200 * 1024 / STAGE) < 6 ? (200 * 1024 / STAGE) : 6;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  static constexpr int THREADS = 6 * 32;
  static constexpr size_t SMEM = static_cast<size_t>(STAGES) * STAGE + 1024 + 256;
};

struct TcArgs {
  int64_t M, K, N;
  int64_t kchunk;
  int splits;
  CMap cmap;
  double* C;
  double* ws;
};

// UMMA shared-memory descriptor: start, leading / stride byte offsets (16 B units),
// version 1 (sm_100), SWIZZLE_128B.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = bn, M = 128
__device__ __forceinline__ uint32_t tf32_idesc(int bn) {
  uint32_t d = 0;
  d |= 1u << 4;                                  // D format: F32
  d |= 2u << 7;                                  // A format: TF32
  d |= 2u << 10;                                 // B format: TF32
  d |= static_cast<uint32_t>(bn >> 3) << 17;     // N >> 3
  d |= static_cast<uint32_t>(kTcBM >> 4) << 24;  // M >> 4
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}

template <int BN>
__global__ void __launch_bounds__(TcTile<BN>::THREADS, 1)
tc_tf32_kernel(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
               const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, const TcArgs g) {
  using T = TcTile<BN>;
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
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kTcBM;
  const int split = blockIdx.z;
  const int64_t kbeg = static_cast<int64_t>(split) * g.kchunk;
  const int64_t kend = (g.K < kbeg + g.kchunk) ? g.K : kbeg + g.kchunk;
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kTcBK - 1) / kTcBK) : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmAh)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmAl)) : "memory");
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
        const int k0 = static_cast<int>(kbeg + static_cast<int64_t>(kt) * kTcBK);
        tma_load_2d(st, &tmAh, full + s, k0, static_cast<int>(m0));
        tma_load_2d(st + T::A_BYTES, &tmAl, full + s, k0, static_cast<int>(m0));
        tma_load_2d(st + 2 * T::A_BYTES, &tmBh, full + s, k0, static_cast<int>(n0));
        tma_load_2d(st + 2 * T::A_BYTES + T::B_BYTES, &tmBl, full + s, k0, static_cast<int>(n0));
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    const uint32_t idesc = tf32_idesc(BN);
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % S;
      mbar_wait(full + s, (kt / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (lane == 0) {
        const uint32_t ah = smem_u32(sm + s * T::STAGE), al = ah + T::A_BYTES;
        const uint32_t bh = ah + 2 * T::A_BYTES, bl = bh + T::B_BYTES;
#pragma unroll
        for (int k = 0; k < kTcBK / 8; ++k) {
          const uint64_t dah = umma_desc(ah + k * 32, 16, 1024), dal = umma_desc(al + k * 32, 16, 1024);
          const uint64_t dbh = umma_desc(bh + k * 32, 16, 1024), dbl = umma_desc(bl + k * 32, 16, 1024);
          umma_tf32(tmem, dah, dbh, idesc, (kt > 0 || k > 0) ? 1u : 0u);
          umma_tf32(tmem, dah, dbl, idesc, 1u);
          umma_tf32(tmem, dal, dbh, idesc, 1u);
        }
        umma_commit(empty + s);  // the stage is free once these MMAs have read it
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (ktiles > 0) umma_commit(accum);
      else mbar_arrive(accum);
    }
    __syncwarp();
  } else {
    // ------------------------------ epilogue ------------------------------
    mbar_wait(accum, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const int quad = warp & 3;
    const int64_t m = m0 + quad * 32 + lane;
    const uint32_t m2 = static_cast<uint32_t>(g.cmap.M2), n2 = static_cast<uint32_t>(g.cmap.N2);
    const bool mok = ktiles > 0;
    const int64_t row_off = m >= g.M ? 0
                                 : (g.splits > 1 ? (static_cast<int64_t>(split) * g.M + m) * g.N
                                                 : static_cast<int64_t>(static_cast<uint32_t>(m) / m2) * g.cmap.sm1 +
                                                       static_cast<int64_t>(static_cast<uint32_t>(m) % m2) * g.cmap.sm2);
#pragma unroll
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (n0 + c0 >= g.N) break;  // warp-uniform
      uint32_t v[16];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quad * 32) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (m < g.M) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int64_t n = n0 + c0 + q;
          if (n >= g.N) continue;
          // an empty K range (ktiles == 0) contributes exact zeros
          const double val = mok ? static_cast<double>(__uint_as_float(v[q])) : 0.0;
          if (g.splits > 1) {
            g.ws[(static_cast<int64_t>(split) * g.M + m) * g.N + n] = val;
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

// hi = tf32(x) (low 13 mantissa bits cleared), lo = x - hi (fp32), optionally transposed:
//   in  [rows][ld_in] row-major (cols valid);
//   out [rows][ld_out] (transpose = 0) or [cols][ld_out] (transpose = 1); padding untouched.
// 32 x 32 tiles through shared memory so the transposed write stays coalesced.
template <typename Tin>
__global__ void __launch_bounds__(256) tf32_split_kernel(const Tin* __restrict__ x, int64_t rows, int64_t cols,
                                                         int64_t ld_in, int transpose, float* __restrict__ hi,
                                                         float* __restrict__ lo, int64_t ld_out) {
  __shared__ float th[32][33], tl[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t tiles_c = (cols + 31) / 32, tiles = ((rows + 31) / 32) * tiles_c;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t r0 = (t / tiles_c) * 32, c0 = (t % tiles_c) * 32;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t r = r0 + ty + j, c = c0 + tx;
      const bool ok = r < rows && c < cols;
      const float f = ok ? static_cast<float>(x[r * ld_in + c]) : 0.f;
      const float h = __uint_as_float(__float_as_uint(f) & 0xFFFFE000u);
      if (!transpose) {
        if (ok) {
          hi[r * ld_out + c] = h;
          lo[r * ld_out + c] = f - h;
        }
      } else {
        th[ty + j][tx] = h;
        tl[ty + j][tx] = f - h;
      }
    }
    if (transpose) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        const int64_t c = c0 + ty + j, r = r0 + tx;  // out row = c, out col = r
        if (c < cols && r < rows) {
          hi[c * ld_out + r] = th[tx][ty + j];
          lo[c * ld_out + r] = tl[tx][ty + j];
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace trals
