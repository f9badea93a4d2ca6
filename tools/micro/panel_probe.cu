// Cycle counts (clock64) of the Householder QR pieces: one panel factorisation by one
#include <cstdio>
// warp (hh_panel_warp) and a whole resident blocked QR (hh_factor_smem), 64 x 64 and 160 x 160.
#include "../../paper_2210_11362_b200/csrc/trals.cu"

__global__ void panel_probe(const double* G, int mr, int nc, long long* out) {
  extern __shared__ __align__(16) double A[];
  __shared__ double tau[512], red[32], Tbuf[128], scratch[64 * 8], xch[80];
  const int ld = nc + 1;
  for (int t = threadIdx.x; t < mr * nc; t += blockDim.x) A[(t / nc) * ld + t % nc] = G[t];
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    if (mr <= 64) hh_panel_team<2>(A, ld, mr, 0, 8, tau, Tbuf, nullptr, 1, xch, scratch);
    else hh_panel_team<8>(A, ld, mr, 0, 8, tau, Tbuf, nullptr, 1, xch, scratch);
  }
  __syncthreads();
  long long t1 = clock64();
  for (int t = threadIdx.x; t < mr * nc; t += blockDim.x) A[(t / nc) * ld + t % nc] = G[t];
  __syncthreads();
  long long t2 = clock64();
  hh_factor_smem(A, ld, mr, nc, tau, red, Tbuf, nullptr, scratch, xch);
  __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t3 - t2; }
}

int main() {
  for (int n : {64, 160}) {
    double* G; long long* o; long long h[2];
    cudaMalloc(&G, sizeof(double) * n * n); cudaMalloc(&o, 16);
    double* hg = new double[n * n];
    for (int i = 0; i < n * n; ++i) hg[i] = ((i * 2654435761u) % 1000) / 500.0 - 1.0 + (i % (n + 1) == 0 ? 3.0 : 0.0);
    cudaMemcpy(G, hg, sizeof(double) * n * n, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(double) * n * (n + 1);
    cudaFuncSetAttribute(panel_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) panel_probe<<<1, 256, smem>>>(G, n, n, o);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("{\"n\": %d, \"panel_cycles\": %lld, \"qr_cycles\": %lld, \"err\": \"%s\"}\n", n, h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
