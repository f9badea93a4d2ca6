// Standalone check of the tcgen05 3xTF32 GEMM (tc_tf32_gemm.cuh) against a CPU fp64 reference.
// Round-1 finding kept here: with the same TMA boxes, the MN-major operand form
// (idesc transpose bit + LBO/SBO swept over 16 B..8 KB) returned all-zero
// accumulators for kind::tf32, while K-major/K-major matched to 1.4e-6 -- so
// the kernel takes K-major operands only.
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2210_11362_b200/csrc/tc_tf32_gemm.cuh"

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static CUtensorMap map2d(const float* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t bi, uint32_t bo) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {bi, bo};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("tensor map error %d\n", (int)r);
  return m;
}

double run(int M, int K, int N) {
  constexpr bool AK = true, BK = true;
  std::vector<float> A((size_t)M * K), B((size_t)K * N);
  srand(7);
  for (auto& v : A) v = (float)(rand() / (double)RAND_MAX - 0.5);
  for (auto& v : B) v = (float)(rand() / (double)RAND_MAX - 0.5);
  // A stored K-major ([M][K]) when AK, else M-major ([K][M])
  std::vector<float> Ast((size_t)M * K);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) (AK ? Ast[(size_t)m * K + k] : Ast[(size_t)k * M + m]) = A[(size_t)m * K + k];
  float *dA, *dAh, *dAl, *dB, *dBh, *dBl;
  double *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dAh, A.size() * 4); cudaMalloc(&dAl, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dBh, B.size() * 4); cudaMalloc(&dBl, B.size() * 4);
  cudaMalloc(&dC, (size_t)M * N * 8);
  cudaMemset(dC, 0xFF, (size_t)M * N * 8);
  cudaMemcpy(dA, Ast.data(), A.size() * 4, cudaMemcpyHostToDevice);
  std::vector<float> Bst(B.size());
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) (BK ? Bst[(size_t)n * K + k] : Bst[(size_t)k * N + n]) = B[(size_t)k * N + n];
  cudaMemcpy(dB, Bst.data(), B.size() * 4, cudaMemcpyHostToDevice);
  trals::tf32_split_kernel<float><<<256, 256>>>(dA, M, K, K, 0, dAh, dAl, K);
  trals::tf32_split_kernel<float><<<256, 256>>>(dB, N, K, K, 0, dBh, dBl, K);
  constexpr int BN = 64;
  CUtensorMap mah, mal, mbh, mbl;
  mah = map2d(dAh, K, M, K, 32, 128); mal = map2d(dAl, K, M, K, 32, 128);
  mbh = map2d(dBh, K, N, K, 32, BN); mbl = map2d(dBl, K, N, K, 32, BN);
  trals::TcArgs g{};
  g.M = M; g.K = K; g.N = N; g.kchunk = ((K + 31) / 32) * 32; g.splits = 1;
  g.cmap = trals::CMap{0, 1 << 30, 0, N, 1 << 30, 0, 1};
  g.C = dC; g.ws = nullptr;
  auto kern = trals::tc_tf32_kernel<BN>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)trals::TcTile<BN>::SMEM);
  dim3 grid((N + BN - 1) / BN, (M + 127) / 128, 1);
  kern<<<grid, trals::TcTile<BN>::THREADS, trals::TcTile<BN>::SMEM>>>(mah, mal, mbh, mbl, g);
  cudaError_t e = cudaDeviceSynchronize();
  { std::vector<double> C0(8); cudaMemcpy(C0.data(), dC, 64, cudaMemcpyDeviceToHost);
    printf("first launch C[0..3] = %g %g %g %g\n", C0[0], C0[1], C0[2], C0[3]);
    std::vector<float> h(8); cudaMemcpy(h.data(), dAh, 32, cudaMemcpyDeviceToHost);
    printf("Ah[0..3] = %g %g %g %g\n", h[0], h[1], h[2], h[3]); }
  if (e != cudaSuccess) { printf("kernel error %s\n", cudaGetErrorString(e)); return -1; }
  // timing
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<grid, trals::TcTile<BN>::THREADS, trals::TcTile<BN>::SMEM>>>(mah, mal, mbh, mbl, g);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> C((size_t)M * N);
  cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
  printf("C[0..3] = %g %g %g %g  C[last]=%g\n", C[0], C[1], C[2], C[3], C[C.size()-1]);
  double num = 0, den = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)A[(size_t)m * K + k] * (double)B[(size_t)k * N + n];
      const double d = C[(size_t)m * N + n] - r;
      num += d * d; den += r * r;
    }
  printf("{ \"M\": %d, \"K\": %d, \"N\": %d, \"rel_fro_err\": %.3e, \"ms\": %.4f, \"tflops_3pass\": %.1f}\n",
         M, K, N, sqrt(num / den), ms / 5, 3.0 * 2.0 * M * K * N / (ms / 5) / 1e9);
  return sqrt(num / den);
}

int main() {
  run(4096, 32, 64);
  run(4096, 128, 64);
  run(256, 128, 64);
  run(1000, 1000, 64);
  run(4096, 2048, 64);
  run(64000, 1600, 64);
  return 0;
}
