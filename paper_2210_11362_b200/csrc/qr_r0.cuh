// R0 of the QR-stabilised variants without V (tr_als_qr, solvers.py:422-424; tr_als, :337-339).
//
// The reference forms V = R_{n+1} [x]_2 ... [x]_2 R_{n-1} (ring.py:138-152, the subchain of the
// per-core R-tensors; for Alg. 1 of the cores themselves), unfolds it (c5: 4.1M x 400 = 13 GB) and
// takes Q0, R0 = qr(V_[2]) (linalg.py:36-52).  Only R0 is needed here -- the right-hand side is
// the shared environment-tree M_n and W = M_n R0^{-1} (SURVEY 8a identity (iii)) -- and R0 is
// invariant under orthogonal transformations of V_[2]'s rows.  So V is merged one core at a time
// and compressed after every merge:
//
//   T <- R-tensor of core n+1 (layout C, (Ra, m, Rb))
//   for j = n+2, ..., n-1:
//     T'[a][mu + m i][c] = sum_b T[a][mu][b] R_j[b][i][c]          (one DMMA GEMM, batched over a)
//     written as the column-major (m k_j) x (Ra Rc) matrix of T''s lateral unfolding, columns in
//     the order c + Rc a (the cyclic 2-unfolding order of S_n, r_n + R_n r_{n+1});
//     if m k_j > Ra Rc: Householder QR of it (cuSOLVER dgeqrf, deterministic mode), T <- its R
//     (rows sign-normalised), i.e. T' = Q T_new with Q orthogonal;
//   R0 = the final R (nonnegative diagonal: qr_economy's convention).
//
// Every compression is an orthogonal transformation of V_[2]'s rows, so R0 equals the
// reference's R factor up to rounding (to ~eps cond(V)) -- including for ill-conditioned and
// rank-deficient V, where chol(S_n) cannot resolve singular values below sqrt(eps) sigma_max.
// Cost at c5: 25600 x 400 and 64000 x 400 QRs per mode (~29 GFLOP) instead of the reference's
// 4.1M x 400.
#include <cusolverDn.h>

namespace {

cusolverDnHandle_t solver_handle() {
  static cusolverDnHandle_t handles[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!handles[dev]) {
    cusolverDnHandle_t h = nullptr;
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) return nullptr;
    // replicas on several GPUs must stay bitwise identical (trals.h conventions)
    cusolverDnSetDeterministicMode(h, CUSOLVER_DETERMINISTIC_RESULTS);
    handles[dev] = h;
  }
  return handles[dev];
}

struct MergeStep {
  int j;         // core merged in
  int Ra, Rb, Rc;
  int64_t m;     // lateral rows of T before the merge
  int64_t k;     // lateral size of core j
  int64_t rows;  // m * k
  int64_t ncol;  // Ra * Rc
  bool qr;       // Householder QR of this step's matrix: rows > ncol (compress), or the final step
};

std::vector<MergeStep> r0_plan(int N, int n, const int32_t* ranks, const int32_t* ks) {
  std::vector<int> order;
  for (int j = n + 1; j < N; ++j) order.push_back(j);
  for (int j = 0; j < n; ++j) order.push_back(j);
  std::vector<MergeStep> st;
  const int Ra = ranks[(n + 1) % N];
  int64_t m = ks[order[0]];
  int Rb = ranks[(order[0] + 1) % N];
  if (order.size() == 1) {
    // N == 2: V is core n+1 itself -- one step that only lays it out and factors it
    MergeStep s{};
    s.j = -1;
    s.Ra = Ra;
    s.Rb = Rb;
    s.Rc = Rb;
    s.m = m;
    s.k = 1;
    s.rows = m;
    s.ncol = static_cast<int64_t>(Ra) * Rb;
    s.qr = true;
    st.push_back(s);
    return st;
  }
  for (size_t t = 1; t < order.size(); ++t) {
    const int j = order[t];
    MergeStep s{};
    s.j = j;
    s.Ra = Ra;
    s.Rb = Rb;
    s.Rc = ranks[(j + 1) % N];
    s.m = m;
    s.k = ks[j];
    s.rows = m * s.k;
    s.ncol = static_cast<int64_t>(Ra) * s.Rc;
    s.qr = s.rows > s.ncol || t + 1 == order.size();
    st.push_back(s);
    m = s.qr ? std::min(s.rows, s.ncol) : s.rows;
    Rb = s.Rc;
  }
  return st;
}

struct R0Ws {
  int64_t mat, tbuf, lwork, gemm, hh, rbuf, total;
};

// the own Householder kernels (hh_qr: one CTA / TSQR tree / wide) when the step's matrix is inside
// their envelope (R_a R_c <= ~115 for tall merges), cuSOLVER dgeqrf otherwise (c5: 400 columns)
inline bool r0_own_qr(const MergeStep& s) { return s.qr && hh_supported(static_cast<int>(s.rows), static_cast<int>(s.ncol)); }

R0Ws r0_ws(int N, int n, const int32_t* ranks, const int32_t* ks) {
  R0Ws w{};
  const auto plan = r0_plan(N, n, ranks, ks);
  cusolverDnHandle_t h = solver_handle();
  for (const auto& s : plan) {
    w.mat = std::max(w.mat, s.rows * s.ncol);
    const int64_t tnext = static_cast<int64_t>(s.Ra) * (s.qr ? std::min(s.rows, s.ncol) : s.rows) * s.Rc;
    w.tbuf = std::max(w.tbuf, tnext);
    if (s.j >= 0) w.gemm = std::max(w.gemm, gemm_ws(s.Ra, s.m, s.Rb, s.k * s.Rc));
    if (r0_own_qr(s)) {
      w.hh = std::max(w.hh, hh_plan(static_cast<int>(s.rows), static_cast<int>(s.ncol)).ws);
      w.rbuf = std::max(w.rbuf, std::min(s.rows, s.ncol) * s.ncol);
    } else if (s.qr && h) {
      int lw = 0;
      if (cusolverDnDgeqrf_bufferSize(h, static_cast<int>(s.rows), static_cast<int>(s.ncol), nullptr,
                                      static_cast<int>(s.rows), &lw) == CUSOLVER_STATUS_SUCCESS)
        w.lwork = std::max<int64_t>(w.lwork, lw);
    }
  }
  const int64_t ncol_max = 4096;
  // Mat | 2 T buffers | tau | lwork | devInfo (2 doubles) | gemm split-K | hh_qr workspace | R buffer
  w.total = w.mat + 2 * w.tbuf + ncol_max + w.lwork + 2 + w.gemm + w.hh + w.rbuf;
  return w;
}

// T_new from the column-major (rows x ncol) matrix after (optional) QR: rows [0, kk) of its upper
// triangle (qr) or all of it (no qr), rows negated where the diagonal is negative (qr only).
// tensor != 0: write T_new[a][mu][c] (layout C, (Ra, kk, Rc)); else the row-major kk x ncol R0.
__global__ void r0_extract_kernel(const double* __restrict__ mat, int64_t ld, int64_t kk, int64_t ncol, int Rc,
                                  int qr, int tensor, double* __restrict__ out) {
  const int64_t total = kk * ncol;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t col = t / kk, r = t - col * kk;  // consecutive threads: consecutive rows (coalesced read)
    double v = mat[col * ld + r];
    if (qr) {
      if (r > col) v = 0.0;
      else if (mat[r * ld + r] < 0.0) v = -v;
    }
    if (tensor) {
      const int64_t a = col / Rc, c = col - a * Rc;
      out[(a * kk + r) * Rc + c] = v;
    } else {
      out[r * ncol + col] = v;
    }
  }
}

// N == 2: the lateral unfolding of T (Ra, m, Rc), column c + Rc a: column-major mat[col * m + mu]
// (rowmajor = 0) or row-major mat[mu * Ra Rc + col] (rowmajor = 1)
__global__ void r0_layout_kernel(const double* __restrict__ T, int64_t m, int Ra, int Rc, int rowmajor,
                                 double* __restrict__ mat) {
  const int64_t ncol = static_cast<int64_t>(Ra) * Rc, total = m * ncol;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t col = t / m, mu = t - col * m;
    const int64_t a = col / Rc, c = col - a * Rc;
    mat[rowmajor ? mu * ncol + col : t] = T[(a * m + mu) * Rc + c];
  }
}

// T_new[a][r][c] = R[r][c + Rc a] (R row-major kk x Ra Rc, already sign-normalised by hh_qr)
__global__ void r0_tensor_from_rm_kernel(const double* __restrict__ R, int64_t kk, int Ra, int Rc,
                                         double* __restrict__ out) {
  const int64_t ncol = static_cast<int64_t>(Ra) * Rc, total = kk * ncol;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = t / ncol, col = t - r * ncol;
    const int64_t a = col / Rc, c = col - a * Rc;
    out[(a * kk + r) * Rc + c] = R[t];
  }
}

int r0_merge(int N, int n, const int32_t* ranks, const int32_t* ks, const double* const* rt, double* U, double* ws,
             int64_t ws_elems, cudaStream_t s) {
  const auto plan = r0_plan(N, n, ranks, ks);
  const R0Ws w = r0_ws(N, n, ranks, ks);
  if (ws_elems < w.total) return TRALS_ERR_WORKSPACE;
  cusolverDnHandle_t h = solver_handle();
  if (!h) return TRALS_ERR_CUDA;
  if (cusolverDnSetStream(h, s) != CUSOLVER_STATUS_SUCCESS) return TRALS_ERR_CUDA;
  double* mat = ws;
  double* tb[2] = {mat + w.mat, mat + w.mat + w.tbuf};
  double* tau = tb[1] + w.tbuf;
  double* work = tau + 4096;
  int* dinfo = reinterpret_cast<int*>(work + w.lwork);
  double* gws = work + w.lwork + 2;
  double* hws = gws + w.gemm;
  double* rbuf = hws + w.hh;
  constexpr int64_t kBig = int64_t(1) << 40;
  const double* T = rt[(n + 1) % N];  // layout C [a][mu][b]
  for (size_t t = 0; t < plan.size(); ++t) {
    const MergeStep& p = plan[t];
    if (p.ncol > 4096) return TRALS_ERR_UNSUPPORTED;
    const bool last = (t + 1 == plan.size());
    const bool own = r0_own_qr(p);
    double* out = last ? U : tb[t & 1];
    // T'[a][mu + m i][c] = sum_b T[a][mu][b] Rj[b][i][c]: a DMMA GEMM batched over a, A(a, mu, b) =
    // T[(a m + mu) Rb + b], B[b][i Rc + c] = Rj (layout C, ldb = k Rc); C(a, mu, n = i Rc + c) lands
    //   own QR:    row-major  mat[(mu + m i) ncol + c + Rc a]
    //   cuSOLVER:  col-major  mat[(c + Rc a) rows + mu + m i]
    //   no QR:     T_new      out[(a rows + mu + m i) Rc + c]   (layout C, nothing to compress)
    if (p.j >= 0) {
      const CMap cm = own ? CMap{p.Rc, kBig, 0, p.ncol, p.Rc, p.m * p.ncol, 1}
                          : p.qr ? CMap{static_cast<int64_t>(p.Rc) * p.rows, kBig, 0, 1, p.Rc, p.m, p.rows}
                                 : CMap{p.rows * p.Rc, kBig, 0, p.Rc, p.Rc, p.m * p.Rc, 1};
      int st = gemm(T, p.m * p.Rb, p.Rb, 1, p.Ra, p.m, p.Rb, p.k * p.Rc, rt[p.j], p.k * p.Rc, p.qr ? mat : out, cm,
                    0, gws, w.gemm, s);
      if (st) return st;
    } else {
      const int64_t total = p.rows * p.ncol;
      const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kSMs));
      r0_layout_kernel<<<blocks, 256, 0, s>>>(T, p.m, p.Ra, p.Rc, own ? 1 : 0, mat);
      if (int e = launch_status()) return e;
    }
    if (p.qr) {
      const int64_t kk = std::min(p.rows, p.ncol);
      const int64_t total = kk * p.ncol;
      const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kSMs));
      if (own) {
        int st = hh_qr(mat, static_cast<int>(p.rows), static_cast<int>(p.ncol), last ? U : rbuf, hws, w.hh, s);
        if (st) return st;
        if (!last) {
          r0_tensor_from_rm_kernel<<<blocks, 256, 0, s>>>(rbuf, kk, p.Ra, p.Rc, out);
          if (int e = launch_status()) return e;
        }
      } else {
        if (cusolverDnDgeqrf(h, static_cast<int>(p.rows), static_cast<int>(p.ncol), mat, static_cast<int>(p.rows),
                             tau, work, static_cast<int>(w.lwork), dinfo) != CUSOLVER_STATUS_SUCCESS)
          return TRALS_ERR_CUDA;
        ++g_launches;
        r0_extract_kernel<<<blocks, 256, 0, s>>>(mat, p.rows, kk, p.ncol, p.Rc, 1, last ? 0 : 1, out);
        if (int e = launch_status()) return e;
      }
    }
    T = out;
  }
  return TRALS_OK;
}

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
    degen_kernel<<<1, 1024, 0, s>>>(U, m, info);
    return launch_status();
  }
  return TRALS_OK;
}

}  // namespace
