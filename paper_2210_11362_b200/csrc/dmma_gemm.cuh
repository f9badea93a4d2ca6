// fp64 contraction engine for the TR-ALS hot path on sm_100a.
//
// Every contraction on the path (the X-times-half-chain environment product,
// the bond absorptions that walk an environment down to M_n, the half-chain
// build, the per-core Gram and the Gram-chain products) is expressed as one
// strided, optionally batched, GEMM
//
//     C[p][m][n] = sum_k A(p, m, k) * B[k][n]
//
// with A read through (sAp, sAm, sAk) where either sAk == 1 ("K-contiguous",
// e.g. X rows) or sAm == 1 ("M-contiguous", e.g. X columns), B row-major with
// leading dimension ldb, and C written through a two-level index map (see
// CMap) so that the epilogue lands results directly in the layout the next
// step wants (environment, M_n, transfer matrix, S_n).
//
// fp64 has no tcgen05/UMMA kind on sm_100a, so the math runs on the legacy
// warp-level DMMA pipe (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), measured at
// 37.1 TFLOP/s on B200 (DFMA tops out at 33.8; profiles/r01_fp64_pipes.md).
// Operand tiles are staged HBM/L2 -> shared memory with 16-byte cp.async in
// a 3-stage ring; fragments are read from padded shared memory
// (bank-conflict-free for both operand orientations).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace trals {

constexpr int kBK = 16;      // K depth per pipeline stage (4 DMMA k-steps)
constexpr int kStages = 3;   // cp.async ring depth

struct CMap {
  // address of C(p, m, n) = p*sp + (m / M2)*sm1 + (m % M2)*sm2
  //                               + (n / N2)*sn1 + (n % N2)*sn2
  int64_t sp, M2, sm1, sm2, N2, sn1, sn2;
};

struct GemmArgs {
  const double* A;
  int64_t sAp, sAm, sAk;
  const double* B;
  int64_t ldb;
  double* C;
  CMap cmap;
  int64_t P, M, K, N;
  int beta;           // 0: C = alpha*acc, 1: C += alpha*acc
  double alpha;
  int64_t kchunk;     // K range per split (multiple of kBK)
  int splits;         // > 1: write raw partials to ws[split][p][m][n]
  double* ws;
  const double* X;    // residual mode: X[m * ldx + n]
  int64_t ldx;
};

__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, int bytes_valid, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  if (bytes == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes_valid));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes_valid));
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int64_t clamp_valid(int64_t rem, int vec) {
  return rem <= 0 ? 0 : (rem < vec ? rem : vec);
}

__device__ __forceinline__ int64_t cmap_addr(const CMap& c, int64_t p, int64_t m, int64_t n) {
  return p * c.sp + (m / c.M2) * c.sm1 + (m % c.M2) * c.sm2 + (n / c.N2) * c.sn1 + (n % c.N2) * c.sn2;
}

// WM x WN warps; each warp owns a (TM*8) x (TN*8) tile of m8n8 DMMA blocks.
// AK: A is K-contiguous (sAk == 1); otherwise M-contiguous (sAm == 1).
// VEC: doubles per cp.async (2 -> 16 B, 1 -> 8 B) for both operands.
template <int WM, int WN, int TM, int TN, bool AK, int VEC>
struct Tile {
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int BM = WM * TM * 8;
  static constexpr int BN = WN * TN * 8;
  static constexpr int LDA = AK ? (kBK + 4) : (BM + 4);   // padded smem pitch (doubles)
  static constexpr int LDB = BN + 4;
  static constexpr int A_STAGE = AK ? BM * LDA : kBK * LDA;
  static constexpr int B_STAGE = kBK * LDB;
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr size_t kSmemBytes = sizeof(double) * STAGE * kStages;
};

// RES: instead of storing C, accumulate sum((X - C)^2) over the tile and write
// one partial per CTA to ws[blockIdx.y * gridDim.x + blockIdx.x] (the fused
// residual of the exact error, solvers.py:164-174; no split-K).
template <int WM, int WN, int TM, int TN, bool AK, int VEC, bool RES = false>
__global__ void __launch_bounds__(WM * WN * 32, 2)
dmma_gemm_kernel(const GemmArgs g) {
  using T = Tile<WM, WN, TM, TN, AK, VEC>;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp % WM, wn = warp / WM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * T::BN;
  const int64_t mtiles = (g.M + T::BM - 1) / T::BM;
  const int64_t p = blockIdx.y / mtiles;
  const int64_t m0 = (blockIdx.y % mtiles) * T::BM;
  const int split = blockIdx.z;
  const int64_t kbeg = static_cast<int64_t>(split) * g.kchunk;
  const int64_t kend = (g.K < kbeg + g.kchunk) ? g.K : kbeg + g.kchunk;
  const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kBK - 1) / kBK) : 0;

  const double* Ab = g.A + p * g.sAp;

  auto load_stage = [&](int slot, int kt) {
    double* As = smem + slot * T::STAGE;
    double* Bs = As + T::A_STAGE;
    const int64_t k0 = kbeg + static_cast<int64_t>(kt) * kBK;
    if constexpr (AK) {
      constexpr int CPR = kBK / VEC;  // chunks per A row
      for (int c = tid; c < T::BM * CPR; c += T::kThreads) {
        const int r = c / CPR, kc = (c % CPR) * VEC;
        const int64_t gm = m0 + r, gk = k0 + kc;
        int valid = 0;
        if (gm < g.M) valid = static_cast<int>(clamp_valid(kend - gk, VEC));
        const double* src = valid ? Ab + gm * g.sAm + gk : g.A;
        cp_async_zfill(As + r * T::LDA + kc, src, valid * 8, VEC * 8);
      }
    } else {
      constexpr int CPR = T::BM / VEC;
      for (int c = tid; c < kBK * CPR; c += T::kThreads) {
        const int r = c / CPR, mc = (c % CPR) * VEC;
        const int64_t gk = k0 + r, gm = m0 + mc;
        int valid = 0;
        if (gk < kend) valid = static_cast<int>(clamp_valid(g.M - gm, VEC));
        const double* src = valid ? Ab + gk * g.sAk + gm : g.A;
        cp_async_zfill(As + r * T::LDA + mc, src, valid * 8, VEC * 8);
      }
    }
    {
      constexpr int CPR = T::BN / VEC;
      for (int c = tid; c < kBK * CPR; c += T::kThreads) {
        const int r = c / CPR, nc = (c % CPR) * VEC;
        const int64_t gk = k0 + r, gn = n0 + nc;
        int valid = 0;
        if (gk < kend) valid = static_cast<int>(clamp_valid(g.N - gn, VEC));
        const double* src = valid ? g.B + gk * g.ldb + gn : g.B;
        cp_async_zfill(Bs + r * T::LDB + nc, src, valid * 8, VEC * 8);
      }
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2;  // fragment row (A) / column (B)
  const int fk = lane & 3;   // fragment k
  const int wm0 = wm * TM * 8, wn0 = wn * TN * 8;

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nxt = kt + kStages - 1;
      if (nxt < ktiles) load_stage(nxt % kStages, nxt);
      cp_async_commit();
    }
    const double* As = smem + (kt % kStages) * T::STAGE;
    const double* Bs = As + T::A_STAGE;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int mm = wm0 + i * 8 + fr, k = kk * 4 + fk;
        a[i] = AK ? As[mm * T::LDA + k] : As[k * T::LDA + mm];
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[(kk * 4 + fk) * T::LDB + wn0 + j * 8 + fr];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  if constexpr (RES) {
    double local = 0.0;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int64_t m = m0 + wm0 + i * 8 + fr;
      if (m >= g.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int64_t n = n0 + wn0 + j * 8 + 2 * fk;
        if (VEC == 2 && n + 1 < g.N) {
          const double2 xv = *reinterpret_cast<const double2*>(g.X + m * g.ldx + n);
          const double d0 = xv.x - acc[i][j][0], d1 = xv.y - acc[i][j][1];
          local = fma(d0, d0, local);
          local = fma(d1, d1, local);
        } else {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (n + e >= g.N) continue;
            const double d = g.X[m * g.ldx + n + e] - acc[i][j][e];
            local = fma(d, d, local);
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    __syncthreads();  // smem ring is free now: reuse it for the warp partials
    if (lane == 0) smem[warp] = local;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < WM * WN; ++w) t += smem[w];
      g.ws[static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
    return;
  }
  // epilogue: C fragment (row fr, cols 2*fk, 2*fk+1) of every m8n8 block.
  // Address parts are computed once per row / column (32-bit div/mod).
  int64_t row_off[TM];
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + wm0 + i * 8 + fr;
    const uint32_t um = static_cast<uint32_t>(m), m2 = static_cast<uint32_t>(g.cmap.M2);
    row_off[i] = m < g.M ? (g.splits > 1 ? ((static_cast<int64_t>(split) * g.P + p) * g.M + m) * g.N
                                         : p * g.cmap.sp + static_cast<int64_t>(um / m2) * g.cmap.sm1 +
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
      for (int i = 0; i < TM; ++i) {
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

// Deterministic split-K reduction: partials summed in split order.
__global__ void splitk_reduce_kernel(const GemmArgs g) {
  const int64_t plane = g.P * g.M * g.N;
  const uint32_t N = static_cast<uint32_t>(g.N), M = static_cast<uint32_t>(g.M);
  const uint32_t M2 = static_cast<uint32_t>(g.cmap.M2), N2 = static_cast<uint32_t>(g.cmap.N2);
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < plane;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < g.splits; ++z) s += g.ws[z * plane + idx];
    s *= g.alpha;
    const int64_t pm = idx / N;  // (p, m) row index
    const uint32_t n = static_cast<uint32_t>(idx - pm * N);
    const uint32_t m = static_cast<uint32_t>(pm % M);
    const int64_t p = pm / M;
    double* dst = g.C + p * g.cmap.sp + static_cast<int64_t>(m / M2) * g.cmap.sm1 +
                  static_cast<int64_t>(m % M2) * g.cmap.sm2 + static_cast<int64_t>(n / N2) * g.cmap.sn1 +
                  static_cast<int64_t>(n % N2) * g.cmap.sn2;
    *dst = g.beta ? *dst + s : s;
  }
}

}  // namespace trals
