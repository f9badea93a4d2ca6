// Dependent-chain latencies (clock64, one warp) of the fp64 operations on the small-solve
// critical paths: DFMA, DADD, rsqrt, 1/x, sqrt, x/y, SHFL of a double, LDS.64.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* ck, double seed) {
  __shared__ double sm[64];
  double x = seed + threadIdx.x * 1e-9, y = 1.0 + 1e-12 * threadIdx.x;
  sm[threadIdx.x] = x;
  __syncwarp();
  const int N = 256;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-300);
  long long t1 = clock64();
  for (int i = 0; i < N; ++i) x = x + y;
  long long t2 = clock64();
  for (int i = 0; i < N; ++i) x = rsqrt(x);
  long long t3 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / x;
  long long t4 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x);
  long long t5 = clock64();
  for (int i = 0; i < N; ++i) x = y / x;
  long long t6 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long t7 = clock64();
  int idx = threadIdx.x & 7;
  for (int i = 0; i < N; ++i) { x = sm[idx]; idx = (__double_as_longlong(x) & 1) + (threadIdx.x & 7); }
  long long t8 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) {
    ck[0] = t1 - t0; ck[1] = t2 - t1; ck[2] = t3 - t2; ck[3] = t4 - t3; ck[4] = t5 - t4; ck[5] = t6 - t5;
    ck[6] = t7 - t6; ck[7] = t8 - t7;
  }
}

int main() {
  double* o; long long* c; long long h[8];
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 64);
  for (int r = 0; r < 3; ++r) lat<<<1, 32>>>(o, c, 1.2345);
  cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* names[8] = {"dfma", "dadd", "rsqrt", "rcp", "sqrt", "div", "shfl_f64", "lds_f64"};
  printf("{");
  for (int i = 0; i < 8; ++i) printf("\"%s\": %.1f%s", names[i], h[i] / 256.0, i < 7 ? ", " : "");
  printf("}\n");
  return 0;
}
