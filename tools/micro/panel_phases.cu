// Phase cycle counts (clock64) of one Householder panel factorisation (copy of hh_panel_warp
// with timers): load, column loop, store, V^T V, T.
#include <cstdio>
#include "../../paper_2210_11362_b200/csrc/trals.cu"
template <int RPL>
__device__ void hh_panel_timed(double* A, int ld, int mr, int p, int nb, double* tau, double* T, double* Tg, long long* ck) {
  long long c0 = clock64();
  const int lane = threadIdx.x & 31;
  double a[RPL][kHhNB];
#pragma unroll
  for (int i = 0; i < RPL; ++i)
#pragma unroll
    for (int c = 0; c < kHhNB; ++c) {
      const int r = p + lane + 32 * i;
      a[i][c] = (r < mr && c < nb) ? A[r * ld + p + c] : 0.0;
    }
  long long c1 = clock64();
  double taus[kHhNB];
#pragma unroll
  for (int jj = 0; jj < kHhNB; ++jj) {
    // one fused reduction per column: |x|^2 below the diagonal and x . a_c for every
    // panel column c > jj (v = scale x is applied afterwards: v . a_c = a_jj,c + scale x . a_c)
    double red[kHhNB];
#pragma unroll
    for (int c = jj; c < kHhNB; ++c) red[c] = 0.0;
#pragma unroll
    for (int i = 0; i < RPL; ++i)
      if (lane + 32 * i > jj) {
#pragma unroll
        for (int c = jj; c < kHhNB; ++c) red[c] = fma(a[i][jj], a[i][c], red[c]);
      }
    double top[kHhNB];  // row jj of the panel (lane jj), broadcast while the reduction runs
#pragma unroll
    for (int c = jj; c < kHhNB; ++c) top[c] = __shfl_sync(0xffffffffu, a[0][c], jj);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = jj; c < kHhNB; ++c) red[c] += __shfl_xor_sync(0xffffffffu, red[c], o);
    const double s = red[jj], alpha = top[jj];
    double t = 0.0, scale = 0.0, beta = alpha;
    if (s > 0.0) {
      const double nrm = sqrt(alpha * alpha + s);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
#pragma unroll
    for (int i = 0; i < RPL; ++i)
      if (lane + 32 * i > jj) a[i][jj] *= scale;
    if (lane == jj) a[0][jj] = beta;
    taus[jj] = t;
#pragma unroll
    for (int c = jj + 1; c < kHhNB; ++c) {
      const double w = t * fma(scale, red[c], top[c]);
      if (lane == jj) a[0][c] -= w;
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        if (lane + 32 * i > jj) a[i][c] = fma(-w, a[i][jj], a[i][c]);
    }
  }
  long long c2 = clock64();
#pragma unroll
  for (int i = 0; i < RPL; ++i)
#pragma unroll
    for (int c = 0; c < kHhNB; ++c) {
      const int r = p + lane + 32 * i;
      if (r < mr && c < nb) A[r * ld + p + c] = a[i][c];
    }
  long long c3 = clock64();
  // G = V^T V (strict upper part): v_c1 . v_c2 = v_c1[row c2] + sum_{rows > c2} v_c1 v_c2
  double g[kHhNB][kHhNB];
#pragma unroll
  for (int c1 = 0; c1 < kHhNB; ++c1)
#pragma unroll
    for (int c2 = c1 + 1; c2 < kHhNB; ++c2) {
      double v = (lane == c2) ? a[0][c1] : 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        if (lane + 32 * i > c2) v = fma(a[i][c1], a[i][c2], v);
      g[c1][c2] = v;
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c1 = 0; c1 < kHhNB; ++c1)
#pragma unroll
      for (int c2 = c1 + 1; c2 < kHhNB; ++c2) g[c1][c2] += __shfl_xor_sync(0xffffffffu, g[c1][c2], o);
  long long c4 = clock64();
  // T row by row in parallel: lane i < 8 owns row i, T[i][jj] = -tau_jj sum_{i<=l<jj} T[i][l] G[l][jj]
  // (every index compile-time; the lane's own row selected by predicates)
  {
    double trow[kHhNB];
#pragma unroll
    for (int jj = 0; jj < kHhNB; ++jj) {
      double acc = 0.0;
#pragma unroll
      for (int l = 0; l < jj; ++l) acc = (l >= lane) ? fma(trow[l], g[l][jj], acc) : acc;
      trow[jj] = (jj < lane) ? 0.0 : (jj == lane ? taus[jj] : -taus[jj] * acc);
    }
    if (lane < kHhNB) {
#pragma unroll
      for (int jj = 0; jj < kHhNB; ++jj) {
        T[lane * kHhNB + jj] = trow[jj];
        if (Tg) Tg[lane * kHhNB + jj] = trow[jj];
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < kHhNB; ++jj)
    if (lane == jj && jj < nb) tau[p + jj] = taus[jj];
  long long c5 = clock64();
  if (lane == 0) { ck[0]=c1-c0; ck[1]=c2-c1; ck[2]=c3-c2; ck[3]=c4-c3; ck[4]=c5-c4; }
}


__global__ void k(const double* G, int mr, int nc, long long* out) {
  extern __shared__ __align__(16) double A[];
  __shared__ double tau[512], Tbuf[128];
  const int ld = nc + 1;
  for (int t = threadIdx.x; t < mr * nc; t += blockDim.x) A[(t / nc) * ld + t % nc] = G[t];
  __syncthreads();
  if (threadIdx.x < 32) {
    if (mr <= 64) hh_panel_timed<2>(A, ld, mr, 0, 8, tau, Tbuf, nullptr, out);
    else hh_panel_timed<7>(A, ld, mr, 0, 8, tau, Tbuf, nullptr, out);
  }
}
int main() {
  for (int n : {64, 160}) {
    double* G; long long* o; long long h[5];
    cudaMalloc(&G, sizeof(double) * n * n); cudaMalloc(&o, 40);
    double* hg = new double[n * n];
    for (int i = 0; i < n * n; ++i) hg[i] = ((i * 2654435761u) % 1000) / 500.0 - 1.0;
    cudaMemcpy(G, hg, sizeof(double) * n * n, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(double) * n * (n + 1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 3; ++r) k<<<1, 32, smem>>>(G, n, n, o);
    cudaMemcpy(h, o, 40, cudaMemcpyDeviceToHost);
    printf("{\"n\": %d, \"load\": %lld, \"columns\": %lld, \"store\": %lld, \"vtv\": %lld, \"T\": %lld}\n", n, h[0], h[1], h[2], h[3], h[4]);
  }
}
