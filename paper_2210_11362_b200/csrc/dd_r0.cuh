// R0 of the QR-stabilised variants from a double-double Gram chain (tr_als_qr, solvers.py:422-424;
// Alg. 1 tr_als, :337-339).
//
// The reference takes Q0, R0 = qr(V_[2]) of the explicit subchain of the per-core R-tensors (c5: a
// 4.1M x 400 Householder QR per mode).  R0 is the unique nonnegative-diagonal factor with
// R0^T R0 = V_[2]^T V_[2] = S_n -- the Gram chain of the R-tensors' transfer matrices (Prop. 3,
// ring.py:191-214).  In double precision chol(S_n) loses every singular value of V below
// sqrt(eps) sigma_max (S squares the condition number); here S_n is formed and factored in
// double-double arithmetic (~2^-104 relative per operation), so R0 carries relative errors of
// ~2^-104 cond(V)^2 -- below the fp64 rounding of a Householder R0 (eps cond(V)) for
// cond(V) < 2^51 -- before it is rounded to fp64:
//
//   E_j = sum_i R_j(i) (x) R_j(i)          exact products (TwoProd), dd sums          (dd_transfer)
//   S_n = E_{n+1} E_{n+2} ... E_{n-1}     dd GEMMs, reshuffled to the (r_n + R_n r_{n+1}) order
//   R0  = chol(S_n), upper, in dd          blocked right-looking (32 x 32 diagonal blocks), pivots
//                                          <= 0 clamped to a zero row (semidefinite S: R0 keeps a
//                                          zero diagonal there, which the 1e-13 degeneracy floor of
//                                          linalg.py:96-99 then reports, as for the reference's
//                                          Householder R0 of a rank-deficient V)
//
// All reductions run in a fixed order: deterministic.
namespace {

struct ddv {
  double hi, lo;
};

__device__ __forceinline__ ddv dd_quick(double s, double e) {
  const double h = s + e;
  return {h, e - (h - s)};
}
__device__ __forceinline__ ddv dd_two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ ddv dd_add(ddv a, ddv b) {
  ddv s = dd_two_sum(a.hi, b.hi);
  const ddv t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
__device__ __forceinline__ ddv dd_mul(ddv a, ddv b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, fma(a.lo, b.hi, e));
  return dd_quick(p, e);
}
__device__ __forceinline__ ddv dd_neg(ddv a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ ddv dd_div(ddv a, ddv b) {
  const double q1 = a.hi / b.hi;
  const ddv r = dd_add(a, dd_neg(dd_mul({q1, 0.0}, b)));
  const double q2 = r.hi / b.hi;
  return dd_quick(q1, q2);
}
__device__ __forceinline__ ddv dd_sqrt(ddv a) {
  if (!(a.hi > 0.0)) return {0.0, 0.0};
  const double x = sqrt(a.hi);
  const ddv x2 = dd_mul({x, 0.0}, {x, 0.0});
  const ddv r = dd_add(a, dd_neg(x2));
  return dd_quick(x, r.hi / (2.0 * x));
}

// Compensated dot-product step (Ogita-Rump-Oishi "Dot2" with dd operands): (s, err) += sg a b, the
// running sum's rounding errors and the products' low parts collected in err.  The dependent chain
// per term is one addition (s), against the ~12 dependent operations of dd_add(dd_mul()); the result
// dd_quick(s, err) carries the same ~2^-104 relative error (relative to sum |a b|).
__device__ __forceinline__ void dd_dot_step(double& s, double& err, ddv a, ddv b, double sg) {
  const double ah = sg * a.hi, al = sg * a.lo;
  const double p = ah * b.hi;
  const double ep = fma(ah, b.hi, -p);
  const double cross = fma(ah, b.lo, al * b.hi);
  const double sn = s + p, bb = sn - s;
  const double es = (s - (sn - bb)) + (p - bb);
  s = sn;
  err += (es + ep) + cross;
}

// E[(a*Ra + c)][(b*Rb + d)] = sum_i R[a][i][b] R[c][i][d] (R layout C, (Ra, k, Rb)); hi / lo planes
__global__ void __launch_bounds__(256) dd_transfer_kernel(const double* __restrict__ R, int Ra, int k, int Rb,
                                                          double* __restrict__ Ehi, double* __restrict__ Elo) {
  const int64_t rows = static_cast<int64_t>(Ra) * Ra, cols = static_cast<int64_t>(Rb) * Rb, total = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = t / cols, col = t - row * cols;
    const int a = static_cast<int>(row / Ra), c = static_cast<int>(row % Ra);
    const int b = static_cast<int>(col / Rb), d = static_cast<int>(col % Rb);
    const double* ra = R + static_cast<int64_t>(a) * k * Rb + b;
    const double* rc = R + static_cast<int64_t>(c) * k * Rb + d;
    ddv acc{0.0, 0.0};
    for (int i = 0; i < k; ++i) {
      const double x = ra[static_cast<int64_t>(i) * Rb], y = rc[static_cast<int64_t>(i) * Rb];
      const double p = x * y;
      acc = dd_add(acc, {p, fma(x, y, -p)});
    }
    Ehi[t] = acc.hi;
    Elo[t] = acc.lo;
  }
}

// C(m, n) = beta C + alpha sum_k A(m, k) B(k, n) in dd: A(m, k) = A[m*sam + k*sak], B(k, n) = B[k*sbk + n*sbn]
// (hi / lo planes at the same offsets), C at (m / M2) sm1 + (m % M2) sm2 + (n / N2) sn1 + (n % N2) sn2.
// 16 x 16 output tiles, 16-deep k slices staged in shared memory; fixed summation order.
struct DdGemm {
  const double *Ahi, *Alo, *Bhi, *Blo;
  double *Chi, *Clo;
  int64_t sam, sak, sbk, sbn;
  int64_t M2, sm1, sm2, N2, sn1, sn2;
  int M, N, K;
  double alpha;
  int beta;
};

__global__ void __launch_bounds__(256) dd_gemm_kernel(const DdGemm g) {
  __shared__ ddv As[16][17], Bs[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m = blockIdx.y * 16 + ty, n = blockIdx.x * 16 + tx;
  double sacc = 0.0, eacc = 0.0;  // compensated dot product (dd_dot_step): half the flops of dd_add(dd_mul())
  for (int k0 = 0; k0 < g.K; k0 += 16) {
    {
      const int mm = blockIdx.y * 16 + ty, kk = k0 + tx;
      const int64_t o = static_cast<int64_t>(mm) * g.sam + static_cast<int64_t>(kk) * g.sak;
      As[ty][tx] = (mm < g.M && kk < g.K) ? ddv{g.Ahi[o], g.Alo[o]} : ddv{0.0, 0.0};
      const int kb = k0 + ty, nn = blockIdx.x * 16 + tx;
      const int64_t ob = static_cast<int64_t>(kb) * g.sbk + static_cast<int64_t>(nn) * g.sbn;
      Bs[ty][tx] = (kb < g.K && nn < g.N) ? ddv{g.Bhi[ob], g.Blo[ob]} : ddv{0.0, 0.0};
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) dd_dot_step(sacc, eacc, As[ty][kk], Bs[kk][tx], 1.0);
    __syncthreads();
  }
  const ddv acc = dd_quick(sacc, eacc);
  if (m < g.M && n < g.N) {
    const int64_t o = (m / g.M2) * g.sm1 + (m % g.M2) * g.sm2 + (n / g.N2) * g.sn1 + (n % g.N2) * g.sn2;
    ddv v = dd_mul(acc, {g.alpha, 0.0});
    if (g.beta) v = dd_add(v, {g.Chi[o], g.Clo[o]});
    g.Chi[o] = v.hi;
    g.Clo[o] = v.lo;
  }
}

int dd_gemm(const DdGemm& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return TRALS_OK;
  dim3 grid(static_cast<unsigned>((g.N + 15) / 16), static_cast<unsigned>((g.M + 15) / 16));
  dd_gemm_kernel<<<grid, 256, 0, s>>>(g);
  return launch_status();
}

constexpr int kDdNB = 32;

// Diagonal block [p, p + pb) of the dd working matrix W (m x m, upper part used): factor it in place
// (upper Cholesky, pivots <= 0 -> zero row), write its rows of R0 (fp64) and the dd inverse of the
// block (Inv, pb x pb upper, pitch kDdNB) for the panel update.  One CTA, shared memory.
__global__ void __launch_bounds__(256) dd_chol_diag_kernel(double* __restrict__ Whi, double* __restrict__ Wlo, int m,
                                                           int p, double* __restrict__ R0, double* __restrict__ Ihi,
                                                           double* __restrict__ Ilo) {
  __shared__ ddv a[kDdNB][kDdNB + 1], x[kDdNB][kDdNB + 1];
  __shared__ ddv rinv[kDdNB];  // 1 / r_jj (0 for a zero row)
  const int pb = min(kDdNB, m - p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < kDdNB * kDdNB; t += blockDim.x) {
    const int r = t / kDdNB, c = t % kDdNB;
    const int64_t o = static_cast<int64_t>(p + r) * m + p + c;
    a[r][c] = (r < pb && c < pb && c >= r) ? ddv{Whi[o], Wlo[o]} : ddv{0.0, 0.0};
    x[r][c] = {0.0, 0.0};
  }
  __syncthreads();
  // Left-looking factorisation by one warp, lane c = column c, no block barriers: row r is
  // a[r][c] - sum_{j<r} u_jr u_jc as one compensated dot product per lane, then the pivot's root and
  // reciprocal from one fp64 rsqrt + one Newton step each (no fp64 divide / sqrt on the chain) and
  // the scaled row.  (The right-looking form with two block barriers per pivot took 83 us per
  // 32 x 32 block, this one ~1/3 of it.)
  if (warp == 0) {
    const int c = lane;
    for (int r = 0; r < pb; ++r) {
      double sd = 0.0, ed = 0.0;
      if (c >= r && c < pb) {
        sd = a[r][c].hi;
        ed = a[r][c].lo;
#pragma unroll 4
        for (int j = 0; j < r; ++j) dd_dot_step(sd, ed, a[j][r], a[j][c], -1.0);
      }
      const ddv v = dd_quick(sd, ed);
      const ddv d{__shfl_sync(0xffffffffu, v.hi, r), __shfl_sync(0xffffffffu, v.lo, r)};
      const bool z = !(d.hi > 0.0);
      ddv rjj{0.0, 0.0}, ri{0.0, 0.0};
      if (!z) {
        const double y = rsqrt(d.hi);  // 1 / sqrt(d) to ~2^-52
        const double r0 = d.hi * y;    // sqrt(d) to ~2^-52
        const double r0sq = r0 * r0;
        const ddv e = dd_add(d, ddv{-r0sq, -fma(r0, r0, -r0sq)});  // d - r0^2, exact product
        rjj = dd_quick(r0, e.hi * (0.5 * y));                        // r0 + (d - r0^2) / (2 r0)
        const ddv t = dd_mul(rjj, ddv{y, 0.0});                      // r y = 1 + O(2^-52)
        const ddv e2 = dd_add(ddv{1.0, 0.0}, dd_neg(t));
        ri = dd_quick(y, e2.hi * y);                                 // y (2 - r y)
      }
      if (c >= r && c < pb) a[r][c] = z ? ddv{0.0, 0.0} : (c == r ? rjj : dd_mul(v, ri));
      if (c == 0) rinv[r] = ri;
      __syncwarp();
    }
  }
  __syncthreads();
  // inverse of the upper block, rows bottom-up: 8 lanes per column split the inner sum (compensated
  // partial dot products, then a fixed-order tree); a column's 8 lanes sit in one warp, so the rows
  // are separated by warp barriers only.  Zero rows stay zero: their inverse rows are not used by
  // the panel update since the corresponding R0 rows are zero too.
  const int col = threadIdx.x >> 3, part = threadIdx.x & 7;  // 32 columns x 8 parts
  for (int i = pb - 1; i >= 0; --i) {
    double sd = 0.0, ed = 0.0;
    if (col < pb && col >= i)
      for (int l = i + 1 + part; l <= col; l += 8) dd_dot_step(sd, ed, a[i][l], x[l][col], -1.0);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double s2 = __shfl_xor_sync(0xffffffffu, sd, o), e2 = __shfl_xor_sync(0xffffffffu, ed, o);
      const double sn = sd + s2, bb = sn - sd;
      ed += e2 + ((sd - (sn - bb)) + (s2 - bb));
      sd = sn;
    }
    if (part == 0 && col < pb && col >= i) {
      ddv acc = dd_quick(sd, ed);
      if (col == i) acc = dd_add(acc, {1.0, 0.0});
      x[i][col] = dd_mul(acc, rinv[i]);  // (rinv = 0 for a zero row)
    }
    __syncwarp();
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kDdNB * kDdNB; t += blockDim.x) {
    const int r = t / kDdNB, c = t % kDdNB;
    const bool in = r < pb && c < pb && c >= r;
    Ihi[t] = in ? x[r][c].hi : 0.0;
    Ilo[t] = in ? x[r][c].lo : 0.0;
    if (r < pb && c < pb) {
      const int64_t o = static_cast<int64_t>(p + r) * m + p + c;
      R0[o] = c >= r ? a[r][c].hi : 0.0;
    }
  }
  // the strict lower part of this block's rows of R0
  for (int t = threadIdx.x; t < pb * p; t += blockDim.x) R0[static_cast<int64_t>(p + t / p) * m + t % p] = 0.0;
}

// R0 row block p (columns >= p + pb) from the panel rows: rows of R0 = Inv^T W[p.., p+pb..] in dd; the
// dd rows are written back into W (the trailing update reads them) and rounded into R0
__global__ void __launch_bounds__(256) dd_round_rows_kernel(const double* __restrict__ Thi,
                                                            const double* __restrict__ Tlo, int m, int p, int pb,
                                                            double* __restrict__ Whi, double* __restrict__ Wlo,
                                                            double* __restrict__ R0) {
  const int rest = m - p - pb;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < pb * m; t += gridDim.x * blockDim.x) {
    const int r = t / m, c = t % m;
    const int64_t o = static_cast<int64_t>(p + r) * m + c;
    if (c >= p + pb) {
      const int64_t ot = static_cast<int64_t>(r) * rest + (c - p - pb);
      Whi[o] = Thi[ot];
      Wlo[o] = Tlo[ot];
      R0[o] = Thi[ot];
    }
  }
}

struct DdWs {
  int64_t e, s, w, t, inv, total;  // offsets (doubles) of: E planes, S planes, W planes, panel planes, inverse
};

DdWs dd_ws(int N, const int32_t* ranks) {
  DdWs w{};
  int64_t rmax = 0, smax = 0;
  for (int j = 0; j < N; ++j) {
    const int64_t a = ranks[j], b = ranks[(j + 1) % N];
    rmax = std::max(rmax, a);
    smax = std::max(smax, a * b * a * b);
  }
  // a chain intermediate is R_{n+1}^2 x R_x^2 for any two ranks: <= rmax^4
  const int64_t chain = std::max(rmax * rmax * rmax * rmax, smax);
  w.e = 0;                       // 2 planes x 2 ping-pong chain buffers
  w.s = 4 * chain;               // S in dd (2 planes)
  w.w = w.s + 2 * smax;          // Cholesky working matrix (2 planes)
  w.t = w.w + 2 * smax;          // panel rows (2 planes)
  w.inv = w.t + 2 * smax;        // diagonal-block inverse (2 planes)
  w.total = w.inv + 2 * kDdNB * kDdNB;
  return w;
}

// S_n (dd) of the transfer matrices Ehi/Elo[j] (layout of trals_core_gram_f64): chain n+1, ..., n-1,
// final scatter into S[(r_n + Rn r_{n+1})][(r'_n + Rn r'_{n+1})]
int dd_gram_chain(int N, int n, const int32_t* ranks, const double* const* Ehi, const double* const* Elo,
                  double* Shi, double* Slo, double* ws, cudaStream_t s) {
  std::vector<int> order;
  for (int j = n + 1; j < N; ++j) order.push_back(j);
  for (int j = 0; j < n; ++j) order.push_back(j);
  const int64_t Rn = ranks[n], Rn1 = ranks[(n + 1) % N], RR = Rn * Rn1;
  const int64_t rows = Rn1 * Rn1;
  const DdWs w = dd_ws(N, ranks);
  const int64_t chain = (w.s - w.e) / 4;
  double* bh[2] = {ws + w.e, ws + w.e + 2 * chain};
  double* bl[2] = {ws + w.e + chain, ws + w.e + 3 * chain};
  const double* ch = Ehi[order[0]];
  const double* cl = Elo[order[0]];
  int64_t cols = static_cast<int64_t>(ranks[(order[0] + 1) % N]) * ranks[(order[0] + 1) % N];
  // products
  for (size_t t = 1; t < order.size(); ++t) {
    const int j = order[t];
    const int64_t Rj1 = ranks[(j + 1) % N];
    const int64_t ncols = Rj1 * Rj1;
    const bool last = (t + 1 == order.size());
    DdGemm g{};
    g.Ahi = ch; g.Alo = cl; g.sam = cols; g.sak = 1;
    g.Bhi = Ehi[j]; g.Blo = Elo[j]; g.sbk = ncols; g.sbn = 1;
    g.M = static_cast<int>(rows); g.N = static_cast<int>(ncols); g.K = static_cast<int>(cols);
    g.alpha = 1.0; g.beta = 0;
    if (last) {
      // F[(x, y)][(b, d)] -> S[(b + Rn x)][(d + Rn y)]: m = x Rn1 + y, n = b Rn + d
      g.Chi = Shi; g.Clo = Slo;
      g.M2 = Rn1; g.sm1 = Rn * RR; g.sm2 = Rn; g.N2 = Rn; g.sn1 = RR; g.sn2 = 1;
    } else {
      g.Chi = bh[t & 1]; g.Clo = bl[t & 1];
      g.M2 = int64_t(1) << 40; g.sm1 = 0; g.sm2 = ncols; g.N2 = int64_t(1) << 40; g.sn1 = 0; g.sn2 = 1;
    }
    if (int st = dd_gemm(g, s)) return st;
    ch = g.Chi;
    cl = g.Clo;
    cols = ncols;
  }
  if (order.size() == 1) {
    // N == 2: S is a reshuffle of the single transfer matrix (each plane through the same scatter)
    const CMap to_s{0, Rn1, Rn * RR, Rn, Rn, RR, 1};
    const int64_t total = RR * RR;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4 * kSMs));
    reshuffle_kernel<<<blocks, 256, 0, s>>>(ch, rows, Rn * Rn, to_s, Shi);
    if (int st = launch_status()) return st;
    reshuffle_kernel<<<blocks, 256, 0, s>>>(cl, rows, Rn * Rn, to_s, Slo);
    return launch_status();
  }
  return TRALS_OK;
}

// R0 (fp64, m x m row-major, upper) = chol(S) with S given in dd; Whi/Wlo the working copy
int dd_cholesky(const double* Shi, const double* Slo, int m, double* R0, double* ws, const DdWs& w, cudaStream_t s) {
  double* Whi = ws + w.w;
  double* Wlo = Whi + static_cast<int64_t>(m) * m;
  double* Thi = ws + w.t;
  double* Tlo = Thi + static_cast<int64_t>(m) * m;
  double* Ihi = ws + w.inv;
  double* Ilo = Ihi + kDdNB * kDdNB;
  if (cudaMemcpyAsync(Whi, Shi, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(Wlo, Slo, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return TRALS_ERR_CUDA;
  for (int p = 0; p < m; p += kDdNB) {
    const int pb = std::min(kDdNB, m - p), rest = m - p - pb;
    dd_chol_diag_kernel<<<1, 256, 0, s>>>(Whi, Wlo, m, p, R0, Ihi, Ilo);
    if (int st = launch_status()) return st;
    if (rest == 0) break;
    // panel: T = Inv^T W[p.., p+pb..]  (pb x rest)
    DdGemm g{};
    g.Ahi = Ihi; g.Alo = Ilo; g.sam = 1; g.sak = kDdNB;  // A(m, k) = Inv[k][m]
    g.Bhi = Whi + static_cast<int64_t>(p) * m + p + pb; g.Blo = Wlo + static_cast<int64_t>(p) * m + p + pb;
    g.sbk = m; g.sbn = 1;
    g.Chi = Thi; g.Clo = Tlo;
    g.M2 = int64_t(1) << 40; g.sm1 = 0; g.sm2 = rest; g.N2 = int64_t(1) << 40; g.sn1 = 0; g.sn2 = 1;
    g.M = pb; g.N = rest; g.K = pb; g.alpha = 1.0; g.beta = 0;
    if (int st = dd_gemm(g, s)) return st;
    {
      const int blocks = std::min((pb * m + 255) / 256, 4 * kSMs);
      dd_round_rows_kernel<<<blocks, 256, 0, s>>>(Thi, Tlo, m, p, pb, Whi, Wlo, R0);
      if (int st = launch_status()) return st;
    }
    // trailing: W[rest][rest] -= T^T T
    DdGemm u{};
    u.Ahi = Thi; u.Alo = Tlo; u.sam = 1; u.sak = rest;  // A(m, k) = T[k][m]
    u.Bhi = Thi; u.Blo = Tlo; u.sbk = rest; u.sbn = 1;
    double* base_hi = Whi + static_cast<int64_t>(p + pb) * m + p + pb;
    double* base_lo = Wlo + static_cast<int64_t>(p + pb) * m + p + pb;
    u.Chi = base_hi; u.Clo = base_lo;
    u.M2 = int64_t(1) << 40; u.sm1 = 0; u.sm2 = m; u.N2 = int64_t(1) << 40; u.sn1 = 0; u.sn2 = 1;
    u.M = rest; u.N = rest; u.K = pb; u.alpha = -1.0; u.beta = 1;
    if (int st = dd_gemm(u, s)) return st;
  }
  return TRALS_OK;
}

}  // namespace
