// Microbenchmark: how many bytes per second one SM can take in from L2 with bulk copies
// (cp.async.bulk global -> shared, mbarrier completion), the path every operand stage of the int8
// environment / residual kernels uses.  One CTA per SM, one producer thread keeps `stages` copies
// of `chunk` bytes in flight into a shared-memory ring; nothing consumes the data.
//   mode 0: all CTAs read the same L2-resident region (like the B plane of crt8_kernel)
//   mode 1: every CTA reads its own L2-resident region (small private slices)
//   mode 2: every CTA streams its own slice of a buffer far larger than L2 (HBM)
// argv: chunk bytes, stages, 1 = poll with mbarrier.test_wait instead of try_wait.
// Prints GB/s per SM and in total.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o tools/micro/l2_ingest tools/micro/l2_ingest.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../paper_2210_11362_b200/csrc/tc_int8_gemm.cuh"

using namespace trals;

// non-blocking poll (mbarrier.test_wait) instead of the potentially suspending try_wait
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

template <bool SPIN>
__global__ void __launch_bounds__(64, 1) ingest_kernel(const uint8_t* __restrict__ src, size_t region, size_t stride,
                                                       int chunk, int stages, long iters, unsigned long long* sink) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(stages) * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint8_t* base = src + blockIdx.x * stride;
    const uint32_t nchunks = static_cast<uint32_t>(region / chunk);
    // (no divisions in the loop: a 64-bit modulo per copy costs more than the copy's issue)
    uint32_t s = 0, ph = 0, ci = 0;
    for (long i = 0; i < iters + stages; ++i) {
      if (i >= stages) {
        if (SPIN) mbar_spin(full + s, ph ^ 1);
        else mbar_wait(full + s, ph ^ 1);
      }
      if (i < iters) {
        mbar_expect_tx(full + s, chunk);
        bulk_load(sm + static_cast<size_t>(s) * chunk, base + static_cast<size_t>(ci) * chunk, chunk, full + s);
      }
      if (++ci == nchunks) ci = 0;
      if (++s == static_cast<uint32_t>(stages)) {
        s = 0;
        ph ^= 1;
      }
    }
    sink[blockIdx.x] = sm[0];
  }
}

int main(int argc, char** argv) {
  const int sms = 148;
  const int chunk = argc > 1 ? atoi(argv[1]) : 32768;
  const int stages = argc > 2 ? atoi(argv[2]) : 6;
  const size_t big = size_t(8) << 30;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  cudaMalloc(&sink, sms * sizeof(unsigned long long));
  const bool spin = argc > 3 && atoi(argv[3]) != 0;
  const size_t smem = static_cast<size_t>(stages) * chunk + stages * 8 + 1024 + 64;
  auto kern = spin ? ingest_kernel<true> : ingest_kernel<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  struct { const char* name; size_t region, stride; } modes[3] = {
      {"shared L2-resident 16 MB region", size_t(16) << 20, 0},
      {"private L2-resident 256 KB slices", size_t(256) << 10, size_t(256) << 10},
      {"private HBM slices (48 MB each, 7 GB in total)", size_t(48) << 20, size_t(48) << 20},
  };
  for (auto& m : modes) {
    const long iters = (size_t(1) << 30) / chunk;  // 1 GiB per SM
    kern<<<sms, 64, smem>>>(buf, m.region, m.stride, chunk, stages, 2000, sink);  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<sms, 64, smem>>>(buf, m.region, m.stride, chunk, stages, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = static_cast<double>(iters) * chunk;
    printf("{\"wait\": \"%s\", \"mode\": \"%s\", \"chunk\": %d, \"stages\": %d, \"gb_per_s_per_sm\": %.1f, \"tb_per_s_total\": %.2f, \"err\": \"%s\"}\n",
           spin ? "test_wait spin" : "try_wait", m.name, chunk, stages, bytes / (ms * 1e-3) / 1e9, bytes * sms / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
