// clock64 phases of the resident Cholesky + inverse (m <= 112) and of one 64 x 64
// augmented factorisation (chol8_aug_smem), one CTA of 512 threads.
#include <cstdio>
#include "../../paper_2210_11362_b200/csrc/trals.cu"
__device__ int chol8_timed(double* a, int ld, int n, int aug, double* scratch, long long* ck) {
  long long tA = 0, tB = 0, tW = 0, tS = 0;
  const int tid = threadIdx.x, lane = tid & 31, nwarps = blockDim.x >> 5;
  // warp index through a shuffle from lane 0: provably warp-uniform, so the warp-0
  // branches below keep the fast (non-collective) shuffle path
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int fr = lane >> 2, fk = lane & 3;
  __shared__ int fail_at;
  if (tid == 0) fail_at = 0;
  if (warp == 0) {
    const int bad = chol8_factor_block(a, ld, 0, min(8, n), scratch, scratch + 64);
    if (bad && lane == 0) fail_at = bad;
  }
  __syncthreads();
  if (fail_at) return fail_at;
  for (int p = 0, it = 0; p < n; p += 8, ++it) {
    const int pb = min(8, n - p);
    const double* Ud = scratch + (it & 1) * 128;
    const double* Xd = Ud + 64;
    long long c0 = clock64();
    // (A) panel rows <- Xd * panel rows: A part columns [p, n), augmented columns [0, p + pb)
    {
      const int wa = n - p, wt = wa + p + pb;
      for (int cc = tid; cc < wt; cc += blockDim.x) {
        const int col = cc < wa ? p + cc : aug + (cc - wa);
        double old[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) old[t] = t < pb ? a[(p + t) * ld + col] : 0.0;
        const bool diag = cc < pb;  // inside the diagonal block: write Ud (exact zeros below)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= pb) break;
          double v = 0.0;
#pragma unroll
          for (int t = 0; t <= i; ++t) v = fma(Xd[i * 8 + t], old[t], v);
          a[(p + i) * ld + col] = diag ? Ud[i * 8 + cc] : v;
        }
      }
    }
    long long c1 = clock64();
    __syncthreads();
    long long c2 = clock64();
    // (B) trailing rows r >= p + 8: a[r][c] -= sum_t P[t][r] P[t][c]  (A part c >= r, augmented c < p + 8)
    const int r0 = p + 8;
    if (r0 < n) {
      const int nbr = (n - r0 + 7) / 8;                 // trailing row blocks
      const int nba = (p + 8) / 8;                      // augmented column blocks
      const int nupper = nbr * (nbr + 1) / 2;
      const int ntiles = nupper + nbr * nba;
      auto update_tile = [&](int rb, int cbase) {
        double* c = a + (rb + fr) * ld + cbase + 2 * fk;
        double c0 = c[0], c1 = c[1];
#pragma unroll
        for (int k0 = 0; k0 < 8; k0 += 4) {
          const double av = -a[(p + k0 + fk) * ld + rb + fr];
          const double bv = a[(p + k0 + fk) * ld + cbase + fr];
          trals::dmma884(c0, c1, av, bv);
        }
        c[0] = c0;
        c[1] = c1;
      };
      if (warp == 0) {
        // look-ahead: next diagonal block first, then factor it into the other scratch half
        update_tile(r0, r0);
        __syncwarp();
        double* nUd = scratch + ((it + 1) & 1) * 128;
        long long w0 = clock64();
        const int bad = chol8_factor_block(a, ld, r0, min(8, n - r0), nUd, nUd + 64);
        if (bad && lane == 0) fail_at = r0 + bad;
        if (lane == 0) tW += clock64() - w0;
      } else {
        auto tile_base = [&](int tile, int& rb, int& cbase) -> bool {
          if (tile < nupper) {  // upper-triangular tile grid of the trailing A part
            int bi = 0, rem = tile;
            while (rem >= nbr - bi) { rem -= nbr - bi; ++bi; }
            if (bi == 0 && rem == 0) return false;  // next diagonal block: warp 0 owns it
            rb = r0 + bi * 8;
            cbase = r0 + (bi + rem) * 8;
          } else {
            const int q = tile - nupper;
            rb = r0 + (q / nba) * 8;
            cbase = aug + (q % nba) * 8;
          }
          return true;
        };
        const int stride = nwarps - 1;
        for (int tile = warp - 1; tile < ntiles; tile += 2 * stride) {
          // two independent tiles per iteration: their load/DMMA/store chains overlap
          int rb0 = 0, cb0 = 0, rb1 = 0, cb1 = 0;
          const bool v0 = tile_base(tile, rb0, cb0);
          const bool v1 = tile + stride < ntiles && tile_base(tile + stride, rb1, cb1);
          double* c0p = a + (rb0 + fr) * ld + cb0 + 2 * fk;
          double* c1p = a + (rb1 + fr) * ld + cb1 + 2 * fk;
          double x0 = v0 ? c0p[0] : 0.0, x1 = v0 ? c0p[1] : 0.0;
          double y0 = v1 ? c1p[0] : 0.0, y1 = v1 ? c1p[1] : 0.0;
#pragma unroll
          for (int k0 = 0; k0 < 8; k0 += 4) {
            const double* prow = a + (p + k0 + fk) * ld;
            const double a0 = -prow[rb0 + fr], b0 = prow[cb0 + fr];
            const double a1 = -prow[rb1 + fr], b1 = prow[cb1 + fr];
            trals::dmma884(x0, x1, a0, b0);
            trals::dmma884(y0, y1, a1, b1);
          }
          if (v0) { c0p[0] = x0; c0p[1] = x1; }
          if (v1) { c1p[0] = y0; c1p[1] = y1; }
        }
      }
    }
    long long c3 = clock64();
    __syncthreads();
    long long c4 = clock64();
    tA += c1 - c0; tB += c3 - c2; tS += (c2 - c1) + (c4 - c3);
    if (fail_at) return fail_at;
  }
  if (threadIdx.x == 0) { ck[3] = tA; ck[4] = tB; ck[5] = tS; }
  if (threadIdx.x == 0) ck[6] = tW;
  return 0;
}


__global__ void __launch_bounds__(512) probe(const double* S, int m, long long* ck) {
  extern __shared__ __align__(16) double a[];
  __shared__ double scratch[256];
  const int npad = (m + 7) & ~7, ld = 2 * npad + 4;
  long long t0 = clock64();
  for (int t = threadIdx.x; t < npad * npad; t += blockDim.x) {
    const int i = t / npad, j = t - i * npad;
    a[i * ld + j] = (i < m && j < m) ? S[i * m + j] : 0.0;
    a[i * ld + npad + j] = (i == j && i < m) ? 1.0 : 0.0;
  }
  __syncthreads();
  long long t1 = clock64();
  const int f = chol8_timed(a, ld, m, npad, scratch, ck);
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { ck[0] = t1 - t0; ck[1] = t2 - t1; ck[2] = f; }
}

int main1() {
  for (int m : {64, 100}) {
    double* hs = new double[m * m];
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) hs[i * m + j] = (i == j ? m : 0.0) + 1.0 / (1 + i + j);
    double* S; long long* o; long long h[7];
    cudaMalloc(&S, sizeof(double) * m * m); cudaMalloc(&o, 56);
    cudaMemcpy(S, hs, sizeof(double) * m * m, cudaMemcpyHostToDevice);
    const int npad = (m + 7) & ~7;
    const size_t smem = sizeof(double) * npad * (2 * npad + 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 3; ++r) probe<<<1, 512, smem>>>(S, m, o);
    cudaMemcpy(h, o, 56, cudaMemcpyDeviceToHost);
    printf("{\"m\": %d, \"load\": %lld, \"factor\": %lld, \"A\": %lld, \"B\": %lld, \"syncs\": %lld, \"warp0_factor8\": %lld}\n", m, h[0], h[1], h[3], h[4], h[5], h[6]);
  }
  return 0;
}

// isolated 8x8 block factor (one warp, nothing else running on the SM)
__global__ void f8_alone(const double* S, long long* ck) {
  __shared__ double a[8 * 8], scr[128];
  for (int t = threadIdx.x; t < 64; t += 32) a[t] = S[(t / 8) * 8 + t % 8];
  __syncwarp();
  long long t0 = clock64();
  int bad = 0;
  for (int r = 0; r < 16; ++r) {
    bad |= chol8_factor_block(a, 8, 0, 8, scr, scr + 64);
    __syncwarp();
    if (threadIdx.x == 0) a[0] += scr[0] * 1e-300 + scr[127] * 1e-300;
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { ck[0] = (t1 - t0) / 16; ck[1] = bad; }
}

int main2() {
  double hs[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) hs[i * 8 + j] = (i == j ? 8.0 : 0.0) + 1.0 / (1 + i + j);
  double* S; long long* o; long long h[2];
  cudaMalloc(&S, sizeof(hs)); cudaMalloc(&o, 16);
  cudaMemcpy(S, hs, sizeof(hs), cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) f8_alone<<<1, 32>>>(S, o);
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("{\"factor8_alone_cycles\": %lld, \"bad\": %lld}\n", h[0], h[1]);
  return 0;
}

int main() { main1(); return main2(); }
