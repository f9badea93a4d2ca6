// The QR variants' triangular factor R0 (solvers.py:262-273 with linalg.py:84-101): the operands of
// the two triangular solves Z = M R0^{-1} R0^{-T} and the 1e-13 degeneracy floor.  R0 itself comes
// from the double-double Gram chain of dd_r0.cuh.
namespace {

// Inverse of the upper-triangular diagonal block U[p0.., p0..] (pb x pb) of a row-major m x m
// factor: W = U_bb^{-1} (upper), WT = W^T, both with pitch ldw.  Row-oriented back substitution,
// one CTA, the block resident in shared memory; columns of W in parallel.
__global__ void __launch_bounds__(512) tri_inv_kernel(double* __restrict__ U, int m, int p0_stride, int nb_blk,
                                                      double* __restrict__ W0, double* __restrict__ WT0,
                                                      int64_t wstride, int ldw, int zero_lower) {
  extern __shared__ __align__(16) double sm[];
  const int b = blockIdx.x;
  const int p0 = b * p0_stride;
  const int pb = min(nb_blk, m - p0);
  double* u = sm;             // [pb][pb + 1]
  double* x = sm + pb * (pb + 1);  // [pb][pb + 1]: W
  const int ld = pb + 1;
  for (int t = threadIdx.x; t < pb * pb; t += blockDim.x) {
    const int r = t / pb, c = t - r * pb;
    u[r * ld + c] = c >= r ? U[static_cast<int64_t>(p0 + r) * m + p0 + c] : 0.0;
    x[r * ld + c] = 0.0;
  }
  __syncthreads();
  // W[i][j] = (delta_ij - sum_{i<l<=j} U[i][l] W[l][j]) / U[i][i], i from the bottom up
  for (int i = pb - 1; i >= 0; --i) {
    const double d = u[i * ld + i];
    for (int j = i + threadIdx.x; j < pb; j += blockDim.x) {
      double acc = (i == j) ? 1.0 : 0.0;
      for (int l = i + 1; l <= j; ++l) acc = fma(-u[i * ld + l], x[l * ld + j], acc);
      x[i * ld + j] = acc / d;
    }
    __syncthreads();
  }
  if (zero_lower)  // the diagonal block's strict lower triangle (the whole matrix when one block covers it)
    for (int t = threadIdx.x; t < pb * pb; t += blockDim.x) {
      const int r = t / pb, c = t - r * pb;
      if (c < r) U[static_cast<int64_t>(p0 + r) * m + p0 + c] = 0.0;
    }
  double* W = W0 + b * wstride;
  double* WT = WT0 + b * wstride;
  for (int t = threadIdx.x; t < ldw * ldw; t += blockDim.x) {
    const int r = t / ldw, c = t - r * ldw;
    const bool in = r < pb && c < pb;
    W[t] = (in && c >= r) ? x[r * ld + c] : 0.0;
    WT[t] = (in && c <= r) ? x[c * ld + r] : 0.0;
  }
}

int tri_prepare(double* U, int m, double* F, double* aux, int check_degen, int* info, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  if (m <= kInvMax) {
    // F = U^{-1}, aux = U^{-T} (the m <= 112 layout of trals_cholesky_f64)
    const size_t smem = sizeof(double) * 2 * m * (m + 1);
    tri_inv_kernel<<<1, 512, smem, s>>>(U, m, m, m, F, aux, 0, m, 1);
    if (int st = launch_status()) return st;
  } else {
    // F = U^T, aux = per 64-row block W_b, W_b^T (the blocked layout of trals_cholesky_f64)
    const int nblk = (m + kBlkNB - 1) / kBlkNB;
    const size_t smem = sizeof(double) * 2 * kBlkNB * (kBlkNB + 1);
    tri_inv_kernel<<<nblk, 512, smem, s>>>(U, m, kBlkNB, kBlkNB, aux, aux + kBlkNB * kBlkNB,
                                           2 * kBlkNB * kBlkNB, kBlkNB, 0);
    if (int st = launch_status()) return st;
    dim3 grid((m + 31) / 32, (m + 31) / 32);
    chol_finalize_kernel<<<grid, dim3(32, 8), 0, s>>>(U, F, m);
    if (int st = launch_status()) return st;
  }
  if (check_degen) {
    degen_kernel<<<1, 1024, 0, s>>>(U, m, info, sqrt(m * 2.220446049250313e-16));
    return launch_status();
  }
  return TRALS_OK;
}

}  // namespace
