// Warp-specialised DMMA GEMM with a TMA producer, for the X-streaming
// environment products (the dominant kernel of the sweep).
//
//   C[m][n] = sum_k A(m, k) B[k][n]     (P = 1; same contract as dmma_gemm.cuh)
//
// One producer warp issues cp.async.bulk.tensor (TMA) loads of the A (X) and B
// (half-chain) tiles into a 6-stage shared-memory ring, signalling per-stage
// "full" mbarriers with transaction bytes; eight consumer warps wait on those
// barriers, run the m8n8k4 f64 MMAs (SASS DMMA.8x8x4) and release each stage
// through an "empty" mbarrier.  No CTA-wide barrier in the main loop, no
// address arithmetic for loads in the math warps, and TMA zero-fills the M/N/K
// tails.  Tile layouts are chosen so the DMMA fragment reads are bank-conflict
// free:
//   * A, K-contiguous (X rows, phase L): one {16 k x 128 m} box, 128B swizzle;
//   * A, M-contiguous (X columns, phase R): {8 m x 16 k} boxes, no swizzle --
//     a fragment's 4 k-rows x 8 m are 256 contiguous bytes;
//   * B ([K][N] row-major): {8 n x 16 k} boxes, no swizzle, same argument.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "dmma_gemm.cuh"

namespace trals {

constexpr int kTmaBK = 16;
constexpr int kTmaStages = 6;

template <int TN>
struct TmaTile {
  static constexpr int WM = 4, WN = 2, TM = 4;
  static constexpr int BM = WM * TM * 8;  // 128
  static constexpr int BN = WN * TN * 8;  // 16 * TN
  static constexpr int A_BYTES = BM * kTmaBK * 8;
  static constexpr int B_BYTES = kTmaBK * BN * 8;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int CONSUMERS = WM * WN;
  static constexpr int THREADS = (CONSUMERS + 1) * 32;
  static constexpr size_t SMEM = static_cast<size_t>(kTmaStages) * STAGE + 1024 + 2 * kTmaStages * 8;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// double offset of A(m, k) inside a stage's A tile
template <bool AK>
__device__ __forceinline__ int a_off(int m, int k) {
  if constexpr (AK) {
    // rows of 16 doubles (128 B), 128B swizzle: 16-byte chunk index ^= row % 8
    return m * 16 + ((((k >> 1) ^ (m & 7))) << 1) + (k & 1);
  } else {
    // {8 m x 16 k} boxes back to back: box (m / 8), row k, column m % 8
    return (m >> 3) * (8 * kTmaBK) + k * 8 + (m & 7);
  }
}

__device__ __forceinline__ int b_off(int k, int n) { return (n >> 3) * (8 * kTmaBK) + k * 8 + (n & 7); }

template <int TN, bool AK>
__global__ void __launch_bounds__(TmaTile<TN>::THREADS, 1)
dmma_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
  using T = TmaTile<TN>;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kTmaStages * T::STAGE);
  uint64_t* empty = full + kTmaStages;

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * T::BN;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * T::BM;
  const int split = blockIdx.z;
  const int64_t kbeg = static_cast<int64_t>(split) * g.kchunk;
  const int64_t kend = (g.K < kbeg + g.kchunk) ? g.K : kbeg + g.kchunk;
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kTmaBK - 1) / kTmaBK) : 0;

  if (tid == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, T::CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  __syncthreads();

  if (warp == T::CONSUMERS) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % kTmaStages;
        if (kt >= kTmaStages) mbar_wait(empty + s, ((kt / kTmaStages) - 1) & 1);
        uint8_t* st = sm + s * T::STAGE;
        double* As = reinterpret_cast<double*>(st);
        double* Bs = reinterpret_cast<double*>(st + T::A_BYTES);
        mbar_expect_tx(full + s, T::STAGE);
        const int k0 = static_cast<int>(kbeg + static_cast<int64_t>(kt) * kTmaBK);
        if constexpr (AK) {
          tma_load_2d(As, &tmA, full + s, k0, static_cast<int>(m0));
        } else {
#pragma unroll
          for (int b = 0; b < T::BM / 8; ++b) tma_load_2d(As + b * 8 * kTmaBK, &tmA, full + s, static_cast<int>(m0) + 8 * b, k0);
        }
#pragma unroll
        for (int b = 0; b < T::BN / 8; ++b) tma_load_2d(Bs + b * 8 * kTmaBK, &tmB, full + s, static_cast<int>(n0) + 8 * b, k0);
      }
    }
    return;
  }

  // ------------------------------ consumers ------------------------------
  const int wm = warp % T::WM, wn = warp / T::WM;
  const int fr = lane >> 2, fk = lane & 3;
  const int wm0 = wm * T::TM * 8, wn0 = wn * TN * 8;
  double acc[T::TM][TN][2];
#pragma unroll
  for (int i = 0; i < T::TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % kTmaStages;
    mbar_wait(full + s, (kt / kTmaStages) & 1);
    const double* As = reinterpret_cast<const double*>(sm + s * T::STAGE);
    const double* Bs = reinterpret_cast<const double*>(sm + s * T::STAGE + T::A_BYTES);
#pragma unroll
    for (int kk = 0; kk < kTmaBK / 4; ++kk) {
      double a[T::TM], b[TN];
#pragma unroll
      for (int i = 0; i < T::TM; ++i) a[i] = As[a_off<AK>(wm0 + i * 8 + fr, kk * 4 + fk)];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[b_off(kk * 4 + fk, wn0 + j * 8 + fr)];
#pragma unroll
      for (int i = 0; i < T::TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  // epilogue (identical contract to dmma_gemm_kernel)
  int64_t row_off[T::TM];
#pragma unroll
  for (int i = 0; i < T::TM; ++i) {
    const int64_t m = m0 + wm0 + i * 8 + fr;
    const uint32_t um = static_cast<uint32_t>(m), m2 = static_cast<uint32_t>(g.cmap.M2);
    row_off[i] = m < g.M ? (g.splits > 1 ? (static_cast<int64_t>(split) * g.M + m) * g.N
                                         : static_cast<int64_t>(um / m2) * g.cmap.sm1 +
                                               static_cast<int64_t>(um % m2) * g.cmap.sm2)
                         : int64_t(-1);
  }
#pragma unroll
  for (int j = 0; j < TN; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t n = n0 + wn0 + j * 8 + 2 * fk + e;
      if (n >= g.N) continue;
      const uint32_t un = static_cast<uint32_t>(n), n2 = static_cast<uint32_t>(g.cmap.N2);
      const int64_t col = g.splits > 1 ? n
                                       : static_cast<int64_t>(un / n2) * g.cmap.sn1 +
                                             static_cast<int64_t>(un % n2) * g.cmap.sn2;
#pragma unroll
      for (int i = 0; i < T::TM; ++i) {
        if (row_off[i] < 0) continue;
        if (g.splits > 1) {
          g.ws[row_off[i] + col] = acc[i][j][e];
        } else {
          double* dst = g.C + row_off[i] + col;
          const double v = g.alpha * acc[i][j][e];
          *dst = g.beta ? *dst + v : v;
        }
      }
    }
  }
}

}  // namespace trals
