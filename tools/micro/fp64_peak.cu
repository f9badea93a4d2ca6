// Microbenchmark: fp64 issue-rate ceilings on sm_100a (DFMA vs DMMA.8x8x4).
// Used once to pick the fp64 pipe for the MTTSP kernel; numbers go to profiles/.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
__global__ void dmma_loop(double* out, int iters, double a0, double b0) {
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) { c[i][0] = i; c[i][1] = threadIdx.x; }
  double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, p.multiProcessorCount, p.major, p.minor);
  double* out; cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int iters = 20000;
      dfma_loop<16><<<sms * bps, threads>>>(out, 100, 1.0000001, 1e-7);
      cudaEventRecord(e0);
      dfma_loop<16><<<sms * bps, threads>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 16 * iters * (double)threads * sms * bps;
      printf("{\"kind\": \"dfma\", \"threads\": %d, \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", threads, bps, fl / ms / 1e9);
      dmma_loop<8><<<sms * bps, threads>>>(out, 100, 1.0000001, 1e-7);
      cudaEventRecord(e0);
      dmma_loop<8><<<sms * bps, threads>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = 2.0 * 256 * 8 * iters * (double)(threads / 32) * sms * bps;
      printf("{\"kind\": \"dmma_m8n8k4\", \"threads\": %d, \"blocks_per_sm\": %d, \"tflops\": %.2f}\n", threads, bps, fl / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
