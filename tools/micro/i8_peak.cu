// Microbenchmark: int8 tcgen05 tensor-core ceiling on sm_100a (the denominator of the
// fp64-on-int8 environment GEMM's roofline).  One CTA per SM; one elected thread issues
// tcgen05.mma.cta_group::1.kind::i8 (M = 128, N = 256, K = 32, both operands K-major in
// shared memory, SWIZZLE_64B) back to back into two 256-column TMEM accumulators, with a
// commit + wait every 64 MMAs.  Reports TOPS = 2 * 128 * 256 * 32 * MMAs / time (CUDA events),
// burst (one ~50 ms launch) and sustained (launches back to back for ~3 s).
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2210_11362_b200/csrc/tc_int8_gemm.cuh"

using namespace trals;

__global__ void __launch_bounds__(128, 1) i8_loop(int iters, int* out) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 128 * 64 + 256 * 64);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 + 256) * 64 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * ((i * 2654435761u) >> 28) ^ 0x80402010u;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint64_t da = oz_desc(smem_u32(sm)), db = oz_desc(smem_u32(sm) + 128 * 64);
    const uint32_t idesc = i8_idesc(256);
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 64; ++j)
        umma_i8_warp(tmem + (j & 1) * 256, da + (((j >> 1) & 1) * 32 >> 4), db + (((j >> 1) & 1) * 32 >> 4), idesc,
                     j > 1 ? 1u : (it > 0));
      oz_commit_warp(bar);
      mbar_wait(bar, phase);
      phase ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t v[16];
    tmem_ld16(tmem, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (v[0] == 0x12345678u) out[0] = 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int* out;
  cudaMalloc(&out, 4);
  const int smem = 1024 + (128 + 256) * 64 + 64;
  cudaFuncSetAttribute(i8_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double ops_per_iter = 64.0 * 2 * 128 * 256 * 32;
  i8_loop<<<sms, 128, smem>>>(100, out);
  cudaDeviceSynchronize();
  int iters = 2000;
  cudaEventRecord(a);
  i8_loop<<<sms, 128, smem>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double burst = ops_per_iter * iters * sms / (ms * 1e-3) / 1e12;
  printf("{\"probe\": \"i8_mma_m128n256k32\", \"sms\": %d, \"iters\": %d, \"ms\": %.3f, \"tops_burst\": %.1f}\n", sms,
         iters, ms, burst);
  // sustained: back-to-back launches for ~3 s
  const int reps = static_cast<int>(3000.0 / ms) + 1;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) i8_loop<<<sms, 128, smem>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double sus = ops_per_iter * iters * sms * reps / (ms * 1e-3) / 1e12;
  printf("{\"probe\": \"i8_mma_m128n256k32_sustained\", \"reps\": %d, \"ms\": %.1f, \"tops_sustained\": %.1f, "
         "\"err\": \"%s\"}\n", reps, ms, sus, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
