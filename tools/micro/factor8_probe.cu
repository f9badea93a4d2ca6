// Cycle counts of the pieces of the resident Cholesky (one warp / one CTA), clock64-timed.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double warp_bcast(double v, int k) { return __shfl_sync(0xffffffffu, v, k); }

__global__ void probe(double* out, long long* cyc, int reps) {
  const int lane = threadIdx.x & 31;
  double d[8], x[8];
  for (int c = 0; c < 8; ++c) { d[c] = (c == lane) ? 10.0 + lane : 0.1 * (c + lane); x[c] = (c == lane); }
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double dk = warp_bcast(d[k], k);
      const bool ok = dk > 0.0;
      const double sk = rsqrt(ok ? dk : 1.0);
      if (ok && lane == k) {
#pragma unroll
        for (int c = 0; c < 8; ++c) { d[c] = c >= k ? d[c] * sk : 0.0; x[c] *= sk; }
      }
      double u[8], xk[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) { u[c] = warp_bcast(d[c], k); xk[c] = warp_bcast(x[c], k); }
      double uki = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) uki = (c == lane) ? u[c] : uki;
      if (ok && lane > k && lane < 8) {
#pragma unroll
        for (int c = 0; c < 8; ++c) { if (c >= lane) d[c] = fma(-uki, u[c], d[c]); x[c] = fma(-uki, xk[c], x[c]); }
      }
    }
    d[lane & 7] += 1.0;  // keep it alive / positive
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < 8; ++c) s += d[c] + x[c];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  // rsqrt chain alone
  double v = 2.0 + lane;
  t0 = clock64();
  for (int r = 0; r < reps; ++r) v = rsqrt(v) + 1.5;
  t1 = clock64();
  out[32 + threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / reps;
  // dfma chain
  v = 1.0 + lane;
  t0 = clock64();
  for (int r = 0; r < reps; ++r) v = fma(v, 0.999, 1e-3);
  t1 = clock64();
  out[64 + threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / reps;
  // shfl chain (double)
  v = 1.0 + lane;
  t0 = clock64();
  for (int r = 0; r < reps; ++r) v = warp_bcast(v, r & 7) + 1.0;
  t1 = clock64();
  out[96 + threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / reps;
  // syncthreads cost with 512 threads is measured by probe_bar
}

__global__ void probe_bar(long long* cyc, int reps) {
  __shared__ double s[512];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) { s[threadIdx.x] += 1.0; __syncthreads(); }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / reps;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
  probe<<<1, 32>>>(out, cyc, 1000);
  probe_bar<<<1, 512>>>(cyc, 1000);
  cudaDeviceSynchronize();
  printf("{\"factor8_cycles\": %lld, \"rsqrt_chain\": %lld, \"dfma_chain\": %lld, \"shfl_chain\": %lld, \"bar512\": %lld}\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[4]);
  return 0;
}
