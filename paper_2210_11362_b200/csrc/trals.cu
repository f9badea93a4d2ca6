// libtrals: B200-native kernels + C-ABI for the TR-ALS NE / QR / QRNE sweep.
// See include/trals.h for the contract and DESIGN.md for the data layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "../../include/trals.h"
#include "dmma_gemm.cuh"
#include "dmma_tma_gemm.cuh"
#include "tc_int8_gemm.cuh"
#include "crt_int8_gemm.cuh"

using trals::CMap;
using trals::GemmArgs;
using trals::kTmaBK;

namespace {

constexpr int kSMs = 148;

long long g_launches = 0;  // kernels launched through this library (reported by trals_launch_count)

inline int launch_status() {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TRALS_OK : TRALS_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// GEMM dispatch
// ---------------------------------------------------------------------------
struct Cfg {
  int BM, BN;
  int id;
};
// (WM, WN, TM, TN): 128x64, 128x80, 128x32, 128x24, 128x16, 128x8, 64x112, and the
// 64-row tiles 64x8, 64x16, 64x32, 64x64 that spread small products over more SMs
constexpr Cfg kCfgs[] = {{128, 64, 0}, {128, 80, 1}, {128, 32, 2}, {128, 24, 3}, {128, 16, 4}, {128, 8, 5},
                         {64, 112, 6}, {64, 8, 7},   {64, 16, 8},  {64, 32, 9},  {64, 64, 10}};

struct SplitPlan {
  int splits;
  int64_t kchunk;
  double cost = 0.0;  // modelled seconds (plan_split only)
};

// Split-K choice: model the time of s splits as
//   waves(s)/s * t_tile  +  [s > 1] * (3 us + (s+1) * M*N*8 B / 6 TB/s)
// with waves(s) = ceil(tiles*s / slots) and t_tile the DMMA time of one full-K
// tile on one CTA slot (37 TFLOP/s over 296 slots).  Small outputs get enough
// splits to fill the GPU; large ones avoid a ragged last wave (c5: 1000
// tiles -> 3.38 waves unsplit, 3.4/5 per unit with s = 5).  Every
// configuration runs 2 CTAs/SM; splits keep >= 4 K-tiles; partials are
// reduced in a fixed order (deterministic).
SplitPlan plan_split(const Cfg& c, int64_t P, int64_t M, int64_t K, int64_t N) {
  const int64_t tiles = P * ((M + c.BM - 1) / c.BM) * ((N + c.BN - 1) / c.BN);
  const int64_t slots = 2 * kSMs;
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, K / (4 * trals::kBK)));
  const double out_bytes = 8.0 * static_cast<double>(P) * M * N;
  int64_t best_s = 1;
  double best = 1e300;
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t waves = (tiles * sp + slots - 1) / slots;
    // a CTA's K chunk: DMMA time at a slot's share of the peak, but never below the
    // pipeline's per-K-tile latency (small tiles are latency-, not flop-bound)
    const double kc = std::ceil(static_cast<double>(K) / sp);
    const double t_unit = std::max(2.0 * c.BM * c.BN * kc / (37.0e12 / slots),
                                   std::ceil(kc / trals::kBK) * 0.25e-6);
    double cost = static_cast<double>(waves) * t_unit;
    if (sp > 1) cost += 3e-6 + (sp + 1) * out_bytes / 6.0e12;
    if (cost < best * (1 - 1e-9)) {
      best = cost;
      best_s = sp;
    }
  }
  int64_t kchunk = (K + best_s - 1) / best_s;
  kchunk = ((kchunk + trals::kBK - 1) / trals::kBK) * trals::kBK;
  if (kchunk <= 0) kchunk = trals::kBK;
  const int64_t splits = std::max<int64_t>(1, (K + kchunk - 1) / kchunk);
  return {static_cast<int>(splits), kchunk, best};
}

// Tile shape for one product: the modelled time of every configuration (with its own
// split-K plan), ties within 3 % going to the larger tile (fewer operand re-reads).
Cfg pick_cfg_for(int64_t P, int64_t M, int64_t K, int64_t N) {
  double cost[sizeof(kCfgs) / sizeof(kCfgs[0])];
  double best = 1e300;
  for (size_t i = 0; i < sizeof(kCfgs) / sizeof(kCfgs[0]); ++i) {
    cost[i] = plan_split(kCfgs[i], P, M, K, N).cost;
    best = std::min(best, cost[i]);
  }
  Cfg pick = kCfgs[0];
  int area = -1;
  for (size_t i = 0; i < sizeof(kCfgs) / sizeof(kCfgs[0]); ++i)
    if (cost[i] <= best * 1.03 && kCfgs[i].BM * kCfgs[i].BN > area) {
      pick = kCfgs[i];
      area = kCfgs[i].BM * kCfgs[i].BN;
    }
  return pick;
}

template <int WM, int WN, int TM, int TN, bool AK, int VEC>
int launch_tile(const GemmArgs& g, cudaStream_t s) {
  using T = trals::Tile<WM, WN, TM, TN, AK, VEC>;
  auto kern = trals::dmma_gemm_kernel<WM, WN, TM, TN, AK, VEC>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(T::kSmemBytes));
    attr_done = true;
  }
  const int64_t mtiles = (g.M + T::BM - 1) / T::BM;
  dim3 grid(static_cast<unsigned>((g.N + T::BN - 1) / T::BN), static_cast<unsigned>(g.P * mtiles),
            static_cast<unsigned>(g.splits));
  if (grid.y > 65535u || grid.x > 65535u) return TRALS_ERR_UNSUPPORTED;
  kern<<<grid, T::kThreads, T::kSmemBytes, s>>>(g);
  return launch_status();
}

template <bool AK, int VEC>
int launch_cfg(int id, const GemmArgs& g, cudaStream_t s) {
  switch (id) {
    case 0: return launch_tile<4, 2, 4, 4, AK, VEC>(g, s);
    case 1: return launch_tile<4, 2, 4, 5, AK, VEC>(g, s);
    case 2: return launch_tile<8, 1, 2, 4, AK, VEC>(g, s);
    case 3: return launch_tile<8, 1, 2, 3, AK, VEC>(g, s);
    case 4: return launch_tile<8, 1, 2, 2, AK, VEC>(g, s);
    case 5: return launch_tile<8, 1, 2, 1, AK, VEC>(g, s);
    case 6: return launch_tile<4, 2, 2, 7, AK, VEC>(g, s);
    case 7: return launch_tile<8, 1, 1, 1, AK, VEC>(g, s);
    case 8: return launch_tile<8, 1, 1, 2, AK, VEC>(g, s);
    case 9: return launch_tile<4, 2, 2, 2, AK, VEC>(g, s);
    case 10: return launch_tile<4, 2, 2, 4, AK, VEC>(g, s);
  }
  return TRALS_ERR_ARG;
}

// fused residual sum((X - A B)^2): A = HL [M x K] row-major, B = HRt [K x N] row-major
int64_t residual_blocks(int64_t M, int64_t N) { return ((M + 127) / 128) * ((N + 63) / 64); }

int residual(const double* A, int64_t M, int64_t K, const double* B, int64_t N, const double* X, double* part,
             cudaStream_t s) {
  GemmArgs g{};
  g.A = A; g.sAp = 0; g.sAm = K; g.sAk = 1;
  g.B = B; g.ldb = N; g.C = nullptr;
  g.P = 1; g.M = M; g.K = K; g.N = N; g.beta = 0; g.alpha = 1.0;
  g.kchunk = ((K + trals::kBK - 1) / trals::kBK) * trals::kBK; g.splits = 1; g.ws = part;
  g.X = X; g.ldx = N;
  const bool vec2 = (reinterpret_cast<uintptr_t>(A) % 16 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                    (reinterpret_cast<uintptr_t>(X) % 16 == 0) && K % 2 == 0 && N % 2 == 0;
  using T = trals::Tile<4, 2, 4, 4, true, 2>;
  dim3 grid(static_cast<unsigned>((N + T::BN - 1) / T::BN), static_cast<unsigned>((M + T::BM - 1) / T::BM), 1);
  if (grid.y > 65535u || grid.x > 65535u) return TRALS_ERR_UNSUPPORTED;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(trals::dmma_gemm_kernel<4, 2, 4, 4, true, 2, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(T::kSmemBytes));
    cudaFuncSetAttribute(trals::dmma_gemm_kernel<4, 2, 4, 4, true, 1, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(T::kSmemBytes));
    attr = true;
  }
  if (vec2) trals::dmma_gemm_kernel<4, 2, 4, 4, true, 2, true><<<grid, T::kThreads, T::kSmemBytes, s>>>(g);
  else trals::dmma_gemm_kernel<4, 2, 4, 4, true, 1, true><<<grid, T::kThreads, T::kSmemBytes, s>>>(g);
  return launch_status();
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int gemm(const double* A, int64_t sAp, int64_t sAm, int64_t sAk, int64_t P, int64_t M, int64_t K, int64_t N,
         const double* B, int64_t ldb, double* C, const CMap& cm, int beta, double* ws, int64_t ws_elems,
         cudaStream_t s, double alpha = 1.0) {
  if (P <= 0 || M <= 0 || N <= 0) return TRALS_OK;
  if (!A || !B || !C) return TRALS_ERR_ARG;
  const bool ak = (sAk == 1);
  if (!ak && sAm != 1) return TRALS_ERR_ARG;
  if (cm.M2 <= 0 || cm.N2 <= 0) return TRALS_ERR_ARG;
  if (K <= 0) {
    // empty contraction: C = 0 (or unchanged when accumulating)
    if (beta) return TRALS_OK;
    return TRALS_ERR_ARG;
  }
  const Cfg c = pick_cfg_for(P, M, K, N);
  SplitPlan sp = plan_split(c, P, M, K, N);
  if (sp.splits > 1) {
    const int64_t need = static_cast<int64_t>(sp.splits) * P * M * N;
    if (!ws || need > ws_elems) {
      // fall back to fewer splits that fit the workspace
      int64_t fit = ws ? ws_elems / (P * M * N) : 1;
      if (fit < 2) {
        sp.splits = 1;
        sp.kchunk = ((K + trals::kBK - 1) / trals::kBK) * trals::kBK;
      } else {
        int64_t kchunk = (K + fit - 1) / fit;
        kchunk = ((kchunk + trals::kBK - 1) / trals::kBK) * trals::kBK;
        sp.kchunk = kchunk;
        sp.splits = static_cast<int>((K + kchunk - 1) / kchunk);
      }
    }
  }
  GemmArgs g;
  g.A = A; g.sAp = sAp; g.sAm = sAm; g.sAk = sAk;
  g.B = B; g.ldb = ldb; g.C = C; g.cmap = cm;
  g.P = P; g.M = M; g.K = K; g.N = N; g.beta = beta; g.alpha = alpha;
  g.kchunk = sp.kchunk; g.splits = sp.splits; g.ws = ws;
  // 16-byte vector loads need every row start 16-byte aligned
  const int64_t sA_lead = ak ? sAm : sAk;
  const bool vec2 = aligned16(A) && aligned16(B) && (sA_lead % 2 == 0) && (P == 1 || sAp % 2 == 0) &&
                    (ldb % 2 == 0);
  int st;
  if (ak) st = vec2 ? launch_cfg<true, 2>(c.id, g, s) : launch_cfg<true, 1>(c.id, g, s);
  else st = vec2 ? launch_cfg<false, 2>(c.id, g, s) : launch_cfg<false, 1>(c.id, g, s);
  if (st != TRALS_OK) return st;
  if (sp.splits > 1) {
    const int64_t total = P * M * N;
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<int64_t>((total + threads - 1) / threads, 8 * kSMs));
    trals::splitk_reduce_kernel<<<blocks, threads, 0, s>>>(g);
    return launch_status();
  }
  return TRALS_OK;
}

int64_t gemm_ws(int64_t P, int64_t M, int64_t K, int64_t N) {
  const Cfg c = pick_cfg_for(P, M, K, N);
  const SplitPlan sp = plan_split(c, P, M, K, N);
  return sp.splits > 1 ? static_cast<int64_t>(sp.splits) * P * M * N : 0;
}

// ---------------------------------------------------------------------------
// TMA-fed, warp-specialised DMMA GEMM for the X-streaming environment products
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
              uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride_elems * sizeof(double)};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_disabled() {
  static int v = -1;
  if (v < 0) v = std::getenv("TRALS_NO_TMA") ? 1 : 0;
  return v == 1;
}

int tma_tn_for(int64_t N) {
  // BN = 16 * TN in {32, 64, 80, 112}; least padding, then widest
  const int tns[] = {2, 4, 5, 7};
  int best = 5;
  double bs = -1;
  for (int tn : tns) {
    const int64_t bn = 16 * tn, nt = (N + bn - 1) / bn;
    const double sc = static_cast<double>(N) / static_cast<double>(nt * bn) + 0.002 * bn;
    if (sc > bs + 1e-12) { bs = sc; best = tn; }
  }
  return best;
}

SplitPlan plan_split_tma(int tn, int64_t M, int64_t K, int64_t N) {
  const int64_t BM = 128, BN = 16 * tn;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int64_t slots = kSMs;  // one CTA per SM
  const int64_t smax = std::max<int64_t>(1, std::min<int64_t>(64, K / (4 * kTmaBK)));
  const double t_tile = 2.0 * BM * BN * static_cast<double>(K) / (37.0e12 / slots);
  const double out_bytes = 8.0 * static_cast<double>(M) * N;
  int64_t best_s = 1;
  double best = 1e300;
  for (int64_t sp = 1; sp <= smax; ++sp) {
    const int64_t waves = (tiles * sp + slots - 1) / slots;
    double cost = static_cast<double>(waves) / sp * t_tile;
    if (sp > 1) cost += 3e-6 + (sp + 1) * out_bytes / 6.0e12;
    if (cost < best * (1 - 1e-9)) { best = cost; best_s = sp; }
  }
  int64_t kchunk = (K + best_s - 1) / best_s;
  kchunk = ((kchunk + kTmaBK - 1) / kTmaBK) * kTmaBK;
  return {static_cast<int>(std::max<int64_t>(1, (K + kchunk - 1) / kchunk)), kchunk};
}

int64_t gemm_tma_ws(int64_t M, int64_t K, int64_t N) {
  const SplitPlan sp = plan_split_tma(tma_tn_for(N), M, K, N);
  return sp.splits > 1 ? static_cast<int64_t>(sp.splits) * M * N : 0;
}

template <int TN, bool AK>
int launch_tma(const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& g, cudaStream_t s) {
  using T = trals::TmaTile<TN>;
  auto kern = trals::dmma_tma_kernel<TN, AK>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(T::SMEM));
    attr = true;
  }
  dim3 grid(static_cast<unsigned>((g.N + T::BN - 1) / T::BN), static_cast<unsigned>((g.M + T::BM - 1) / T::BM),
            static_cast<unsigned>(g.splits));
  if (grid.x > 65535u || grid.y > 65535u) return TRALS_ERR_UNSUPPORTED;
  kern<<<grid, T::THREADS, T::SMEM, s>>>(a, b, g);
  return launch_status();
}

// Returns TRALS_ERR_UNSUPPORTED (nothing launched) when the TMA path does not apply.
int gemm_tma(const double* A, int64_t sAm, int64_t sAk, int64_t M, int64_t K, int64_t N, const double* B, int64_t ldb,
             double* C, const CMap& cm, double* ws, int64_t ws_elems, cudaStream_t s) {
  if (tma_disabled() || !tensor_map_encoder()) return TRALS_ERR_UNSUPPORTED;
  const bool ak = (sAk == 1);
  const int64_t lead = ak ? sAm : sAk;
  if ((reinterpret_cast<uintptr_t>(A) & 15u) || (reinterpret_cast<uintptr_t>(B) & 15u) || (lead & 1) || (ldb & 1))
    return TRALS_ERR_UNSUPPORTED;
  if (M > INT32_MAX || K > INT32_MAX || N > INT32_MAX || K < kTmaBK || M < 128) return TRALS_ERR_UNSUPPORTED;
  const int tn = tma_tn_for(N);
  SplitPlan sp = plan_split_tma(tn, M, K, N);
  if (sp.splits > 1 && (!ws || static_cast<int64_t>(sp.splits) * M * N > ws_elems)) return TRALS_ERR_UNSUPPORTED;
  CUtensorMap ma, mb;
  bool ok = ak ? make_map(&ma, A, K, M, sAm, kTmaBK, 128, true) : make_map(&ma, A, M, K, sAk, 8, kTmaBK, false);
  ok = ok && make_map(&mb, B, N, K, ldb, 8, kTmaBK, false);
  if (!ok) return TRALS_ERR_UNSUPPORTED;
  GemmArgs g{};
  g.A = A; g.sAp = 0; g.sAm = sAm; g.sAk = sAk;
  g.B = B; g.ldb = ldb; g.C = C; g.cmap = cm;
  g.P = 1; g.M = M; g.K = K; g.N = N; g.beta = 0; g.alpha = 1.0;
  g.kchunk = sp.kchunk; g.splits = sp.splits; g.ws = ws;
  int st;
  switch (tn * 2 + (ak ? 1 : 0)) {
    case 5: st = launch_tma<2, true>(ma, mb, g, s); break;
    case 4: st = launch_tma<2, false>(ma, mb, g, s); break;
    case 9: st = launch_tma<4, true>(ma, mb, g, s); break;
    case 8: st = launch_tma<4, false>(ma, mb, g, s); break;
    case 11: st = launch_tma<5, true>(ma, mb, g, s); break;
    case 10: st = launch_tma<5, false>(ma, mb, g, s); break;
    case 15: st = launch_tma<7, true>(ma, mb, g, s); break;
    default: st = launch_tma<7, false>(ma, mb, g, s); break;
  }
  if (st) return st;
  if (sp.splits > 1) {
    const int64_t total = M * N;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kSMs));
    trals::splitk_reduce_kernel<<<blocks, 256, 0, s>>>(g);
    return launch_status();
  }
  return TRALS_OK;
}


// ---------------------------------------------------------------------------
// int8 tcgen05 digit-sliced GEMM (tc_int8_gemm.cuh): the fp32 variant (OzF32) and
// the fp64 environment products (OzF64)
// ---------------------------------------------------------------------------
constexpr int kOzBN = 64;
// bytes of a tiled digit layout: D planes x rows padded to the tiling x K padded to the stage k
inline int64_t oz_digits_bytes(const trals::OzRowTiles& rt, int64_t k, int digits, int bk = 64) {
  return digits * rt.rows_pad() * ((k + bk - 1) / bk * bk);
}
inline trals::OzRowTiles oz_a_tiles(int64_t rows) { return trals::OzRowTiles::fixed(rows, trals::kOzBM); }
// n-tiles of at most 32 columns (two TMEM accumulator buffers with 7 digit levels) when the
// contraction is short and the 64-wide tiling leaves few tiles per SM: a tile's MMAs then
// last about as long as its epilogue, which the second buffer overlaps, and the finer tiles
// even out the last wave (c4: 64000 x 1600 x 64 -> 500 64-wide tiles on 148 SMs; 166 vs 185 us).
// With many tiles per SM the 64-wide ones win: the epilogue's TMEM loads slow down under the
// next tile's MMAs anyway, and A is read from shared memory half as often per output
// (c3: 250000 x 500 x 100, 448 vs 486 us).  fp64 scheme only; for the fp32 one -- staged
// epilogue, 4 digits -- the narrower tiles measured slower at c4: 1965 vs 2040 sweeps/s.
constexpr int64_t kOzShortK = 8192;
template <class SC>
inline int oz_bn(int64_t M, int64_t K, int64_t N) {
  static int64_t short_k = -1;  // TRALS_OZ_SHORT_K (experiments) overrides kOzShortK
  if (short_k < 0) short_k = std::getenv("TRALS_OZ_SHORT_K") ? std::atoll(std::getenv("TRALS_OZ_SHORT_K")) : kOzShortK;
  if (!SC::BAL || K >= short_k) return kOzBN;
  const int64_t tiles64 = ((M + trals::kOzBM - 1) / trals::kOzBM) * ((N + kOzBN - 1) / kOzBN);
  return tiles64 < 8 * kSMs ? 32 : kOzBN;
}
// TRALS_OZ_FIXED_TILES=1 (experiments): every n-tile kOzBN wide, the last one zero padded
inline trals::OzRowTiles oz_b_tiles(int64_t n, int bn = kOzBN, int cn = 1) {
  static int fixed = -1;
  if (fixed < 0) fixed = std::getenv("TRALS_OZ_FIXED_TILES") ? 1 : 0;
  return fixed ? trals::OzRowTiles::fixed(n, bn) : trals::OzRowTiles::balanced(n, bn, cn);
}
// cluster size of the fp64 int8 product (A stages multicast over CN n-tiles); 1 = no cluster.
// TRALS_OZ_CLUSTER (experiments) picks 2 or 4.
template <class SC>
inline int oz_cn(int64_t N, int bn) {
  static int env = -1;
  if (env < 0) env = std::getenv("TRALS_OZ_CLUSTER") ? std::atoi(std::getenv("TRALS_OZ_CLUSTER")) : 1;
  const int cn = (env == 2 || env == 4) ? env : 1;
  if (!SC::BAL || cn == 1) return 1;
  return oz_b_tiles(N, bn, cn).ntiles > 0 ? cn : 1;
}

// split-K over a per-tile time model and never more than SC::KMAX k per CTA (int32
// accumulator bound).  fp32: byte-bound (4 digit bytes per A element at the per-SM
// HBM share); fp64: tensor-bound (28 digit-pair MMAs at the int8 rate of one SM).
template <class SC>
SplitPlan plan_split_oz(int64_t M, int64_t K, int64_t N) {
  const int64_t BK = SC::BK;
  const int bn = oz_bn<SC>(M, K, N);
  const int cn = oz_cn<SC>(N, bn);
  const int64_t tiles = ((M + trals::kOzBM - 1) / trals::kOzBM) * oz_b_tiles(N, bn, cn).ntiles;
  const int64_t slots = kSMs;
  const int64_t smin = std::max<int64_t>(1, (K + SC::KMAX - 1) / SC::KMAX);
  const int64_t smax = std::max<int64_t>(smin, std::min<int64_t>(64, K / (4 * BK)));
  int pairs = 0;
  for (int a = 0; a < SC::D; ++a) pairs += std::min(SC::D, SC::LV - a);
  const double t_tile = SC::BAL ? static_cast<double>(pairs) * trals::kOzBM * N / oz_b_tiles(N, bn, cn).ntiles *
                                      static_cast<double>(K) /
                                      (8192.0 * 1.9e9)
                                : 4.0 * trals::kOzBM * static_cast<double>(K) / (6.5e12 / slots);
  const double out_bytes = 8.0 * static_cast<double>(M) * N;
  int64_t best_s = smin;
  double best = 1e300;
  for (int64_t sp = smin; sp <= smax; ++sp) {
    const int64_t waves = (tiles * sp + slots - 1) / slots;
    double cost = static_cast<double>(waves) / sp * t_tile;
    if (sp > 1) cost += 3e-6 + (sp + 1) * out_bytes / 6.0e12;
    if (cost < best * (1 - 1e-9)) { best = cost; best_s = sp; }
  }
  int64_t kchunk = (K + best_s - 1) / best_s;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  return {static_cast<int>(std::max<int64_t>(1, (K + kchunk - 1) / kchunk)), kchunk};
}

// workspace (doubles): B digit planes (D x N x ldk bytes), eb (N int32), B column max (N), partials
struct OzWs {
  int64_t planes, eb, mx, flags, part, total;
};
// in-kernel two-way split-K fix-up (no reduce launch) for the chunked-epilogue scheme
template <class SC>
bool oz_fixup(const SplitPlan& sp, int64_t K) {
  (void)K;  // (both tile widths of the fp64 scheme use the chunked epilogue; fp32: kOzBN only)
  return sp.splits == 2 && (SC::BAL || trals::OzTile<kOzBN, SC>::CHUNKED);
}

template <class SC>
OzWs oz_ws_layout(int64_t M, int64_t K, int64_t N) {
  const SplitPlan sp = plan_split_oz<SC>(M, K, N);
  OzWs w{};
  w.planes = 0;
  const int bn = oz_bn<SC>(M, K, N);
  const int cn = oz_cn<SC>(N, bn);
  w.eb = w.planes + (oz_digits_bytes(oz_b_tiles(N, bn, cn), K, SC::D, SC::BK) + 15) / 16 * 2;
  w.mx = w.eb + (N + 3) / 4 * 2;
  w.flags = w.mx + (N + 1) / 2 * 2;
  const int64_t tiles = ((M + trals::kOzBM - 1) / trals::kOzBM) * oz_b_tiles(N, bn, cn).ntiles;
  const bool fix = oz_fixup<SC>(sp, K);
  w.part = w.flags + (fix ? (2 * tiles + 1) / 2 + 1 : 0);
  w.total = w.part + (sp.splits > 1 ? (fix ? 1 : static_cast<int64_t>(sp.splits)) * M * N : 0);
  return w;
}

template <class SC>
int64_t gemm_oz_ws(int64_t M, int64_t K, int64_t N) { return oz_ws_layout<SC>(M, K, N).total; }

template <typename T>
int launch_colmax(const T* x, int64_t rows, int64_t cols, int64_t ld, double* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, cols * sizeof(double), s);
  const int64_t cw = std::min<int64_t>(cols, 256), cblocks = (cols + cw - 1) / cw;
  // about 4 blocks per SM in total, at least 64 rows per block
  const int64_t want = std::max<int64_t>(1, 4 * kSMs / cblocks);
  const int64_t rpb = std::max<int64_t>(64, (rows + want - 1) / want);
  dim3 grid(static_cast<unsigned>(cblocks), static_cast<unsigned>((rows + rpb - 1) / rpb));
  trals::oz_colmax_kernel<T><<<grid, 256, 0, s>>>(x, rows, cols, ld, rpb, out);
  return launch_status();
}

template <int BN, class SC, bool RES = false, int CN = 1, bool W8 = false>
int launch_oz(const trals::OzArgs& g, int grid, cudaStream_t s) {
  using T = trals::OzTile<BN, SC>;
  auto kern = trals::oz8_kernel<BN, SC, RES, CN, W8>;
  constexpr size_t kSmem = T::SMEM + (W8 ? T::OUT_BYTES : 0);  // W8: a staging buffer per epilogue half
  static_assert(kSmem <= 227 * 1024, "shared memory of the int8 kernel");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmem));
    attr = true;
  }
  if constexpr (CN == 1) {
    kern<<<grid, trals::oz_threads<RES || W8>(), kSmem, s>>>(g);
    return launch_status();
  } else {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CN;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(trals::oz_threads<RES || W8>());
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // as many whole clusters as the GPCs hold at once (persistent), no more than the work units
    static int max_clusters = 0;
    if (!max_clusters) {
      cfg.gridDim = dim3(kSMs / CN * CN);
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
        max_clusters = kSMs / CN;
    }
    const int units = (grid + CN - 1) / CN;
    cfg.gridDim = dim3(static_cast<unsigned>(std::min(units, max_clusters) * CN));
    if (cudaLaunchKernelEx(&cfg, kern, g) != cudaSuccess) return TRALS_ERR_CUDA;
    return launch_status();
  }
}

// C(m, n) = sum_k A[m][k] B[k][n]: A given as tiled digits [D x 128-row tiles] + row exponents ea[M],
// B fp64 [K][ldb] (sliced per call into the workspace), C fp64 through cm.
// plo > 0 (cm.N2 == phi): the columns are taken in the order n' = (n % phi) plo + n / phi --
// for the environment layout Env[r_hi][m][r_lo] (n = r_lo-index phi + r_hi-index) that makes
// each r_hi group of a tile's columns one contiguous block of rows x r_lo in C, instead of
// every column landing in a different r_hi plane (short-K shapes, where the epilogue's stores
// weigh: c3 environment 698 -> 685 us).
template <class SC>
int gemm_oz(const int8_t* ad, const int32_t* ea, int64_t M, int64_t K, int64_t N, const double* B, int64_t ldb,
            double* C, const CMap& cm0, double* ws, int64_t ws_elems, cudaStream_t s, int plo = 0, int phi = 0) {
  if (plo > 0 && (static_cast<int64_t>(plo) * phi != N || cm0.N2 != phi)) return TRALS_ERR_ARG;
  const CMap cm = plo > 0 ? CMap{cm0.sp, cm0.M2, cm0.sm1, cm0.sm2, plo, cm0.sn2, cm0.sn1} : cm0;
  if ((reinterpret_cast<uintptr_t>(ad) & 15u) || M > INT32_MAX || K > INT32_MAX || N > INT32_MAX) return TRALS_ERR_ARG;
  const OzWs w = oz_ws_layout<SC>(M, K, N);
  if (!ws || w.total > ws_elems) return TRALS_ERR_ARG;
  const SplitPlan sp = plan_split_oz<SC>(M, K, N);
  int8_t* bd = reinterpret_cast<int8_t*>(ws + w.planes);
  int32_t* eb = reinterpret_cast<int32_t*>(ws + w.eb);
  double* bmx = ws + w.mx;
  // B^T rows = columns of B: max over k, then tiled digits (transposed read)
  if (int st = launch_colmax<double>(B, K, N, ldb, bmx, s)) return st;
  const int bn = oz_bn<SC>(M, K, N);
  const int cn = oz_cn<SC>(N, bn);
  {
    const trals::OzRowTiles bt = oz_b_tiles(N, bn, cn);
    dim3 grid(static_cast<unsigned>((K + 63) / 64), static_cast<unsigned>((bt.rows_pad() + 63) / 64));
    trals::oz_digits_tiled_t_kernel<double, SC><<<grid, 256, 0, s>>>(B, K, N, ldb, bmx, bd, bt, eb, plo, phi);
    if (int st = launch_status()) return st;
  }
  trals::OzArgs g{};
  g.M = M; g.K = K; g.N = N; g.kchunk = sp.kchunk; g.splits = sp.splits;
  g.mtiles = static_cast<int>((M + trals::kOzBM - 1) / trals::kOzBM);
  g.nt = oz_b_tiles(N, bn, cn);
  g.ntiles = g.nt.ntiles;
  static int norot = -1;  // TRALS_OZ_NOROT=1 (experiments): k blocks in natural order
  if (norot < 0) norot = std::getenv("TRALS_OZ_NOROT") ? 1 : 0;
  g.rotate = norot ? 0 : 1;
  g.fixup = oz_fixup<SC>(sp, K) ? 1 : 0;
  if (g.fixup) {
    const int64_t tiles = static_cast<int64_t>(g.mtiles) * g.ntiles;
    g.tickets = reinterpret_cast<int*>(ws + w.flags);
    g.ready = g.tickets + tiles;
    if (cudaMemsetAsync(g.tickets, 0, 2 * tiles * sizeof(int), s) != cudaSuccess) return TRALS_ERR_CUDA;
  }
  g.kblocks = (K + SC::BK - 1) / SC::BK;
  g.ad = ad; g.bd = bd;
  g.cmap = cm; g.ea = ea; g.eb = eb; g.C = C; g.ws = ws + w.part;
  const int64_t tiles = static_cast<int64_t>(g.mtiles) * g.ntiles * sp.splits;
  if (tiles > INT32_MAX) return TRALS_ERR_UNSUPPORTED;
  const int grid = static_cast<int>(std::min<int64_t>(tiles, kSMs));
  int st = TRALS_ERR_UNSUPPORTED;
  if (cn == 4) st = bn == 32 ? launch_oz<32, SC, false, 4>(g, grid, s) : launch_oz<kOzBN, SC, false, 4>(g, grid, s);
  if (cn == 2) st = bn == 32 ? launch_oz<32, SC, false, 2>(g, grid, s) : launch_oz<kOzBN, SC, false, 2>(g, grid, s);
  // short K (c3, c4): the tiles spend longer in the epilogue than in their MMAs -> 8 epilogue warps
  // (TRALS_OZ_W8=0, experiments: the 4-warp form everywhere)
  static int w8 = -1;
  if (w8 < 0) w8 = (std::getenv("TRALS_OZ_W8") && std::atoi(std::getenv("TRALS_OZ_W8")) == 0) ? 0 : 1;
  bool done = false;
  if constexpr (SC::BAL) {
    if (cn == 1 && w8 && K < kOzShortK) {
      st = bn == 32 ? launch_oz<32, SC, false, 1, true>(g, grid, s) : launch_oz<kOzBN, SC, false, 1, true>(g, grid, s);
      done = true;
    }
  }
  if (cn == 1 && !done) st = bn == 32 ? launch_oz<32, SC>(g, grid, s) : launch_oz<kOzBN, SC>(g, grid, s);
  if (st) return st;
  if (sp.splits > 1 && !g.fixup) {
    GemmArgs r{};
    r.P = 1; r.M = M; r.N = N; r.splits = sp.splits; r.ws = ws + w.part; r.C = C; r.cmap = cm; r.alpha = 1.0;
    r.beta = 0;
    const int64_t total = M * N;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kSMs));
    trals::splitk_reduce_kernel<<<blocks, 256, 0, s>>>(r);
    return launch_status();
  }
  return TRALS_OK;
}

// ---------------------------------------------------------------------------
// fp64 environment products by CRT on the int8 tensor cores (crt_int8_gemm.cuh)
// ---------------------------------------------------------------------------
// moduli tables: computed once on the host (128-bit integers) and copied to constant memory.
// TRALS_CRT_MODULI = number of moduli, 12..16 (default kCrtDefaultMod = 15; every modulus is one
// more int8 GEMM and ~4 more bits per operand row).
struct CrtHost {
  trals::CrtTables t{};
  bool ok = false;
};
CrtHost crt_host_build() {
  CrtHost c;
  static const uint32_t moduli[trals::kCrtMaxMod] = {
#define TRALS_CRT_LIST(i, pp) pp,
      TRALS_CRT_MODULI(TRALS_CRT_LIST)
#undef TRALS_CRT_LIST
  };
  int nm = std::getenv("TRALS_CRT_MODULI") ? std::atoi(std::getenv("TRALS_CRT_MODULI")) : trals::kCrtDefaultMod;
  nm = std::max(12, std::min(nm, trals::kCrtMaxMod));
  using u128 = unsigned __int128;
  u128 P = 1;
  long double lg = 0;
  for (int i = 0; i < nm; ++i) {
    P *= moduli[i];
    lg += std::log2(static_cast<long double>(moduli[i]));
  }
  c.t.nm = nm;
  for (int j = 0; j < 4; ++j) c.t.P[j] = static_cast<uint32_t>(P >> (32 * j));
  for (int i = 0; i < trals::kCrtMaxMod; ++i) {
    const uint32_t p = moduli[i];
    c.t.p[i] = p;
    c.t.magic[i] = static_cast<uint32_t>(((1ull << 39) + p - 1) / p);
    if (i >= nm) continue;
    const u128 W = P / p;
    const uint32_t wr = static_cast<uint32_t>(W % p);
    uint32_t q = 0;
    for (uint32_t z = 1; z < p; ++z)
      if ((wr * z) % p == 1) { q = z; break; }
    if (!q) return c;  // (moduli not coprime: cannot happen)
    const u128 Wq = W * q;  // = (P / p) q < P: already reduced mod P
    for (int j = 0; j < 4; ++j) c.t.w[i][j] = static_cast<uint32_t>(Wq >> (32 * j));
    c.t.fq[i] = static_cast<uint32_t>(std::llround(std::ldexp(static_cast<double>(q) / p, 19)));
  }
  // ||a'|| ||b'|| <= 2^(ga+gb) < P / 2; rows are int64 -> each <= 62
  int gtot = static_cast<int>(std::floor(static_cast<double>(lg) - 1.0 - 0.01));
  gtot = std::min(gtot, 124);
  c.t.ga = (gtot + 1) / 2;
  c.t.gb = gtot / 2;
  if (!((static_cast<u128>(1) << (c.t.ga + c.t.gb + 1)) < P)) return c;
  if (cudaMemcpyToSymbol(trals::crt_tab, &c.t, sizeof(c.t)) != cudaSuccess) return c;
  c.ok = true;
  return c;
}

// one table set per device (constant memory is per device): built and uploaded on first use
const CrtHost& crt_host() {
  constexpr int kMaxDev = 64;
  static CrtHost tabs[kMaxDev];
  static bool done[kMaxDev] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) dev = 0;
  std::lock_guard<std::mutex> lock(mu);
  if (!done[dev]) {
    tabs[dev] = crt_host_build();
    done[dev] = true;
  }
  return tabs[dev];
}

inline int crt_n16(int64_t N) { return static_cast<int>((N + 15) / 16 * 16); }
inline bool crt_shape_ok(int64_t M, int64_t K, int64_t N) {
  return M >= 1 && K >= 1 && N >= 1 && N <= trals::kCrtMaxN && M <= INT32_MAX && K <= INT32_MAX &&
         (M + trals::kCrtBM - 1) / trals::kCrtBM * trals::kCrtMaxMod * 64 < INT32_MAX;
}
inline int64_t crt_kblocks(int64_t K) { return (K + trals::kCrtBK - 1) / trals::kCrtBK; }
inline int64_t crt_mtiles(int64_t M) { return (M + trals::kCrtBM - 1) / trals::kCrtBM; }
// rows of an A residue plane: whole pairs of m-tiles (the CTA-pair kernel loads both tiles of a pair)
inline int64_t crt_a_rows_pad(int64_t M) { return (M + 2 * trals::kCrtBM - 1) / (2 * trals::kCrtBM) * (2 * trals::kCrtBM); }
// TRALS_CRT_PAIR=0 (experiments): one-CTA MMAs (cta_group::1) instead of CTA pairs
inline bool crt_pair() {
  static int v = -1;
  if (v < 0) v = (std::getenv("TRALS_CRT_PAIR") && std::atoi(std::getenv("TRALS_CRT_PAIR")) == 0) ? 0 : 1;
  return v == 1;
}
// bytes of the residue planes of a [rows][K] operand tiled in row tiles of tile_w
inline int64_t crt_plane_bytes(int64_t rows_pad, int64_t K) { return rows_pad * crt_kblocks(K) * trals::kCrtBK; }

// column statistics slabs: about 4 blocks per SM in total, at least 64 rows per slab
inline void crt_col_slabs(int64_t rows, int64_t cols, int& slabs, int64_t& rows_per_slab) {
  const int64_t cblocks = (cols + 31) / 32;
  const int64_t want = std::max<int64_t>(1, 4 * kSMs / cblocks);
  rows_per_slab = std::max<int64_t>(64, (rows + want - 1) / want);
  slabs = static_cast<int>((rows + rows_per_slab - 1) / rows_per_slab);
}

// K splits: never more than kCrtKmax k per item (int32 sums), more when the items are too few
// to fill the SMs; cost model in k units (an item's epilogue ~ 1024 k of MMAs)
inline int crt_splits(int64_t M, int64_t K, int nm) {
  const int64_t items = crt_mtiles(M) * nm;
  const int64_t smin = std::max<int64_t>(1, (K + trals::kCrtKmax - 1) / trals::kCrtKmax);
  const int64_t smax = std::max<int64_t>(smin, std::min<int64_t>(16, K / 2048));
  int64_t best_s = smin;
  double best = 1e300;
  for (int64_t sp = smin; sp <= smax; ++sp) {
    const int64_t waves = (items * sp + kSMs - 1) / kSMs;
    const double cost = static_cast<double>(waves) * (static_cast<double>(K) / sp + 1024.0);
    if (cost < best * (1 - 1e-9)) { best = cost; best_s = sp; }
  }
  return static_cast<int>(best_s);
}

struct CrtWs {
  int64_t bplanes, sb, part, res, tail, total;  // offsets in doubles
  int splits;
  int64_t kb_split;
  int tail_start, tail_splits, unit_rows, units_per_mod;  // tail split of the last partial wave (CrtArgs)
  int64_t tail_kb;
};
CrtWs crt_ws_layout(int64_t M, int64_t K, int64_t N) {
  const int nm = crt_host().t.nm;
  const int n16 = crt_n16(N);
  CrtWs w{};
  const int64_t kblocks = crt_kblocks(K);
  int sp = crt_splits(M, K, nm);
  w.kb_split = (kblocks + sp - 1) / sp;
  w.splits = static_cast<int>((kblocks + w.kb_split - 1) / w.kb_split);
  // tail split: with one K split and at least one full wave, the units of the last partial wave
  // are cut into K pieces that fill the wave (TRALS_CRT_TAIL=0 disables)
  static int tail_on = -1;
  if (tail_on < 0) tail_on = (std::getenv("TRALS_CRT_TAIL") && std::atoi(std::getenv("TRALS_CRT_TAIL")) == 0) ? 0 : 1;
  const bool pair = crt_pair();
  const int slots = pair ? kSMs / 2 : kSMs;
  w.unit_rows = pair ? 2 * trals::kCrtBM : trals::kCrtBM;
  w.units_per_mod = static_cast<int>(pair ? (crt_mtiles(M) + 1) / 2 : crt_mtiles(M));
  const int64_t units = static_cast<int64_t>(nm) * w.units_per_mod * w.splits;
  w.tail_start = static_cast<int>(units);
  w.tail_splits = 1;
  w.tail_kb = kblocks;
  if (tail_on && w.splits == 1 && units > slots && units % slots != 0) {
    const int64_t tail = units % slots;
    int64_t st = std::min<int64_t>({slots / tail, 8, kblocks / 32});
    if (st >= 2) {
      w.tail_kb = (kblocks + st - 1) / st;
      w.tail_splits = static_cast<int>((kblocks + w.tail_kb - 1) / w.tail_kb);
      w.tail_start = static_cast<int>(units - tail);
    }
  }
  int slabs;
  int64_t rps;
  crt_col_slabs(K, N, slabs, rps);
  w.bplanes = 0;
  w.sb = w.bplanes + (static_cast<int64_t>(nm) * crt_plane_bytes(n16, K) + 15) / 16 * 2;
  w.part = w.sb + (N + 3) / 4 * 2;
  w.res = w.part + static_cast<int64_t>(slabs) * 2 * N;
  w.tail = w.res + (static_cast<int64_t>(w.splits) * nm * M * n16 + 15) / 16 * 2;
  const int64_t tail_bytes = static_cast<int64_t>(w.tail_splits - 1) * (units - w.tail_start) * w.unit_rows * n16;
  w.total = w.tail + (tail_bytes + 15) / 16 * 2;
  return w;
}

// scale exponents of the K-major rows of x (its rows, or its columns when transposed)
int crt_scales(const double* x, int64_t rows, int64_t cols, int64_t ld, int transpose, int gamma, int32_t* sexp,
               double* part, cudaStream_t s) {
  if (!transpose) {
    const int blocks = static_cast<int>(std::min<int64_t>((rows + 7) / 8, 64 * kSMs));
    trals::crt_row_scale_kernel<<<blocks, 256, 0, s>>>(x, rows, cols, ld, gamma, sexp);
    return launch_status();
  }
  int slabs;
  int64_t rps;
  crt_col_slabs(rows, cols, slabs, rps);
  dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>(slabs));
  trals::crt_col_stats_kernel<<<grid, 256, 0, s>>>(x, rows, cols, ld, rps, part);
  if (int st = launch_status()) return st;
  trals::crt_col_scale_kernel<<<static_cast<unsigned>((cols + 7) / 8), 256, 0, s>>>(part, slabs, cols, rows, gamma,
                                                                                      sexp);
  return launch_status();
}

int crt_slice(const double* x, int64_t rows, int64_t cols, int64_t ld, int transpose, const int32_t* sexp,
              uint8_t* planes, int64_t rows_pad, int tile_w, cudaStream_t s) {
  const int64_t K = transpose ? rows : cols;
  const int64_t blocks = crt_kblocks(K) * ((rows_pad + 63) / 64);
  if (blocks > INT32_MAX) return TRALS_ERR_UNSUPPORTED;
  trals::crt_slice_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      x, rows, cols, ld, transpose, sexp, planes, rows_pad, tile_w, crt_host().t.nm, crt_plane_bytes(rows_pad, K));
  return launch_status();
}

int64_t crt_split_ws(int64_t rows, int64_t cols, int transpose) {
  if (!transpose) return 1;
  int slabs;
  int64_t rps;
  crt_col_slabs(rows, cols, slabs, rps);
  return static_cast<int64_t>(slabs) * 2 * cols;
}

// X (row-major [rows][cols]) -> residue planes of its rows (transpose = 0) or columns (1) + scale exponents
int crt_split(const double* x, int64_t rows, int64_t cols, int transpose, int8_t* planes, int32_t* exps, double* ws,
              int64_t ws_elems, cudaStream_t s) {
  const int64_t out_rows = transpose ? cols : rows, K = transpose ? rows : cols;
  if (!x || !planes || !exps || !ws || rows < 1 || cols < 1 || (transpose != 0 && transpose != 1) ||
      ws_elems < crt_split_ws(rows, cols, transpose) || (reinterpret_cast<uintptr_t>(planes) & 15u))
    return TRALS_ERR_ARG;
  if (!crt_host().ok) return TRALS_ERR_CUDA;
  if (!crt_shape_ok(out_rows, K, 1)) return TRALS_ERR_UNSUPPORTED;
  if (int st = crt_scales(x, rows, cols, cols, transpose, crt_host().t.ga, exps, ws, s)) return st;
  return crt_slice(x, rows, cols, cols, transpose, exps, reinterpret_cast<uint8_t*>(planes), crt_a_rows_pad(out_rows),
                   trals::kCrtBM, s);
}

// C(m, n) = sum_k A[m][k] B[k][n]: A given as residue planes + row scale exponents, B fp64 [K][ldb]
// (sliced per call into the workspace), C fp64 through cm
// stages: 1 = slice B (scales + residue planes into ws), 2 = the modular GEMMs, 4 = CRT reconstruction;
// the three run in this order on ws, in one call or in separate ones
int gemm_crt(const int8_t* ad, const int32_t* ea, int64_t M, int64_t K, int64_t N, const double* B, int64_t ldb,
             double* C, const CMap& cm, double* ws, int64_t ws_elems, int stages, cudaStream_t s) {
  if (!crt_host().ok) return TRALS_ERR_CUDA;
  if (!crt_shape_ok(M, K, N)) return TRALS_ERR_UNSUPPORTED;
  if (reinterpret_cast<uintptr_t>(ad) & 15u) return TRALS_ERR_ARG;
  const CrtWs w = crt_ws_layout(M, K, N);
  if (!ws || w.total > ws_elems) return TRALS_ERR_ARG;
  const trals::CrtTables& t = crt_host().t;
  const int n16 = crt_n16(N);
  uint8_t* bd = reinterpret_cast<uint8_t*>(ws + w.bplanes);
  int32_t* sb = reinterpret_cast<int32_t*>(ws + w.sb);
  uint8_t* res = reinterpret_cast<uint8_t*>(ws + w.res);
  if (stages & 1) {
    if (int st = crt_scales(B, K, N, ldb, 1, t.gb, sb, ws + w.part, s)) return st;
    if (int st = crt_slice(B, K, N, ldb, 1, sb, bd, n16, n16, s)) return st;
  }
  trals::CrtArgs g{};
  g.M = M; g.K = K; g.n16 = n16; g.nm = t.nm;
  if (n16 <= 256) { g.nc0 = n16; g.nc1 = 0; }
  else { g.nc0 = (n16 / 2 + 15) / 16 * 16; g.nc1 = n16 - g.nc0; }
  g.mtiles = static_cast<int>(crt_mtiles(M));
  g.splits = w.splits;
  g.kblocks = crt_kblocks(K);
  g.kb_split = w.kb_split;
  g.a_plane = crt_plane_bytes(crt_a_rows_pad(M), K);
  g.b_plane = crt_plane_bytes(n16, K);
  g.ad = reinterpret_cast<const uint8_t*>(ad); g.bd = bd; g.out = res;
  g.tail_start = w.tail_start; g.tail_splits = w.tail_splits; g.tail_kb = w.tail_kb;
  g.tail_out = reinterpret_cast<uint8_t*>(ws + w.tail);
  if (stages & 2) {
  const bool pair = crt_pair();
  const int stage = trals::kCrtBM * trals::kCrtBK + n16 * trals::kCrtBK / (pair ? 2 : 1);
  g.stages = std::min(8, (212 * 1024) / stage);
  if (g.stages < 2) return TRALS_ERR_UNSUPPORTED;
  const size_t smem = static_cast<size_t>(g.stages) * stage + (3 * g.stages + 2) * 8 + 16 + 1024;
  auto kern = pair ? trals::crt8_kernel<true> : trals::crt8_kernel<false>;
  static size_t smem_set[2] = {0, 0};
  if (smem > smem_set[pair]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
      return TRALS_ERR_CUDA;
    smem_set[pair] = smem;
  }
  if (pair) {
    const int64_t units = (static_cast<int64_t>(g.mtiles) + 1) / 2 * g.nm * g.splits +
                          static_cast<int64_t>(w.tail_splits - 1) * ((static_cast<int64_t>(g.mtiles) + 1) / 2 * g.nm -
                                                                    w.tail_start);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static int max_clusters = 0;  // CTA pairs resident at once (persistent kernel)
    if (!max_clusters) {
      cfg.gridDim = dim3(kSMs / 2 * 2);
      if (cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg) != cudaSuccess || max_clusters < 1)
        max_clusters = kSMs / 2;
      if (std::getenv("TRALS_CRT_DEBUG")) std::fprintf(stderr, "crt pair: max active clusters %d\n", max_clusters);
      max_clusters = std::min(max_clusters, kSMs / 2);
    }
    static int force = -1;  // TRALS_CRT_CLUSTERS (experiments): number of CTA pairs launched
    if (force < 0) force = std::getenv("TRALS_CRT_CLUSTERS") ? std::atoi(std::getenv("TRALS_CRT_CLUSTERS")) : 0;
    const int ncl = force > 0 ? force : max_clusters;
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(units, ncl) * 2));
    if (cudaLaunchKernelEx(&cfg, kern, g) != cudaSuccess) return TRALS_ERR_CUDA;
  } else {
    const int64_t items = static_cast<int64_t>(g.mtiles) * g.nm * g.splits;
    const int grid = static_cast<int>(std::min<int64_t>(items, kSMs));
    kern<<<grid, 192, smem, s>>>(g);
  }
  if (int st = launch_status()) return st;
  }
  if (!(stages & 4)) return TRALS_OK;
  if (w.tail_splits > 1) {  // fold the tail units' K pieces into the main residue planes
    trals::CrtTailArgs ta{};
    ta.res = res; ta.tail_res = reinterpret_cast<const uint8_t*>(ws + w.tail); ta.M = M; ta.n16 = n16; ta.nm = t.nm;
    ta.tail_start = w.tail_start; ta.tail_splits = w.tail_splits; ta.unit_rows = w.unit_rows;
    ta.units_per_mod = w.units_per_mod;
    const int64_t work = (static_cast<int64_t>(t.nm) * w.units_per_mod - w.tail_start) * w.unit_rows * (n16 / 4);
    const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 8 * kSMs));
    trals::crt_tail_merge_kernel<<<blocks, 256, 0, s>>>(ta);
    if (int st = launch_status()) return st;
  }
  trals::CrtOutArgs o{};
  o.res = res; o.M = M; o.n16 = n16; o.N = static_cast<int>(N); o.nm = t.nm; o.splits = g.splits;
  o.sa = ea; o.sb = sb; o.C = C; o.cmap = cm;
  o.perm = (cm.N2 > 0 && cm.N2 < N && N % cm.N2 == 0 && cm.sn1 < cm.sn2) ? static_cast<int>(N / cm.N2) : 0;
  const int64_t cblocks = (M + trals::kCrtRB - 1) / trals::kCrtRB;
  if (cblocks > INT32_MAX) return TRALS_ERR_UNSUPPORTED;
  trals::crt_combine_kernel<<<static_cast<unsigned>(cblocks), 256, trals::kCrtRB * (n16 + 1) * sizeof(double), s>>>(o);
  return launch_status();
}

// env() on the CRT engine: X given as residue planes + scale exponents, K-major for this side
int env_crt(const int8_t* xd, const int32_t* xe, int64_t pre, int64_t post, int side, const double* H, int r_lo,
            int r_hi, double* E, int leaf, double* ws, int64_t ws_elems, int stages, cudaStream_t s) {
  const int64_t RR = static_cast<int64_t>(r_lo) * r_hi;
  const int64_t rows = side == 0 ? pre : post, K = side == 0 ? post : pre;
  CMap cm{0, rows, 0, r_lo, r_hi, 1, rows * r_lo};
  if (leaf) cm = CMap{0, rows, 0, RR, r_hi, r_hi, 1};
  return gemm_crt(xd, xe, rows, K, RR, H, RR, E, cm, ws, ws_elems, stages, s);
}

// Accuracy guard of the digit-sliced fp64 products (AlsConfig.fp64_gemm = "auto"): per K-major row
// of X (its rows for transpose = 0, its columns for transpose = 1) the dynamic-range statistic
// rho = max|x| * K / sum|x| (0 for an all-zero row); out = max over rows.  The product truncates
// each row at 2^-56.9 of its maximum, so its error per output is <= 2^-56.9 max|a| sum|h| =
// 2^-56.9 rho mean|a| sum|h|: rho bounds how far that is from a dgemm's eps sum|a||h| for a
// spread-out h.  Reductions in a fixed order (deterministic).
__global__ void __launch_bounds__(256) oz_range_rows_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                                            double* __restrict__ rho) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += nw) {
    double m = 0.0, sa = 0.0;
    for (int64_t c = lane; c < cols; c += 32) {
      const double v = fabs(x[r * cols + c]);
      m = fmax(m, v);
      sa += v;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      sa += __shfl_xor_sync(0xffffffffu, sa, o);
    }
    if (lane == 0) rho[r] = sa > 0.0 ? m * static_cast<double>(cols) / sa : 0.0;
  }
}

__global__ void __launch_bounds__(256) oz_range_cols_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                                            double* __restrict__ rho) {
  __shared__ double sm[8][32], ss[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x * 32 + lane;
  double m = 0.0, sa = 0.0;
  if (c < cols)
    for (int64_t r = warp; r < rows; r += 8) {
      const double v = fabs(x[r * cols + c]);
      m = fmax(m, v);
      sa += v;
    }
  sm[warp][lane] = m;
  ss[warp][lane] = sa;
  __syncthreads();
  if (warp == 0 && c < cols) {
    for (int w = 1; w < 8; ++w) {
      m = fmax(m, sm[w][lane]);
      sa += ss[w][lane];
    }
    rho[c] = sa > 0.0 ? m * static_cast<double>(rows) / sa : 0.0;
  }
}

__global__ void __launch_bounds__(1024) max_reduce_kernel(const double* __restrict__ v, int64_t n,
                                                          double* __restrict__ out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, v[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    *out = m;
  }
}

// X (fp32 or fp64, row-major [rows][cols]) -> tiled digit planes of its rows (transpose = 0)
// or columns (transpose = 1) + their exponents; ws = out_rows doubles (row / column maxima)
template <typename Tin, class SC>
int oz_split(const Tin* x, int64_t rows, int64_t cols, int transpose, int8_t* digits, int32_t* exps, double* ws,
             int64_t ws_elems, cudaStream_t s) {
  const int64_t out_rows = transpose ? cols : rows, K = transpose ? rows : cols;
  if (!x || !digits || !exps || !ws || rows < 1 || cols < 1 || (transpose != 0 && transpose != 1) ||
      ws_elems < out_rows || (reinterpret_cast<uintptr_t>(digits) & 15u))
    return TRALS_ERR_ARG;
  if (!transpose) {
    const int blocks = static_cast<int>(std::min<int64_t>((rows + 7) / 8, 64 * kSMs));
    trals::oz_rowmax_kernel<Tin><<<blocks, 256, 0, s>>>(x, rows, cols, cols, ws);
    if (int st = launch_status()) return st;
  } else {
    if (int st = launch_colmax<Tin>(x, rows, cols, cols, ws, s)) return st;
  }
  if (transpose) {
    const trals::OzRowTiles at = oz_a_tiles(out_rows);
    const int64_t gy = (at.rows_pad() + 63) / 64;
    if (gy > 65535 || (K + 63) / 64 > INT32_MAX) return TRALS_ERR_UNSUPPORTED;
    dim3 grid(static_cast<unsigned>((K + 63) / 64), static_cast<unsigned>(gy));
    trals::oz_digits_tiled_t_kernel<Tin, SC><<<grid, 256, 0, s>>>(x, rows, cols, cols, ws, digits, at, exps);
    return launch_status();
  }
  const int64_t work = oz_digits_bytes(oz_a_tiles(out_rows), K, SC::D, SC::BK) / (16 * SC::D);  // (padded row, 16-k chunk)
  const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 64 * kSMs));
  trals::oz_digits_tiled_kernel<Tin, SC><<<blocks, 256, 0, s>>>(x, rows, cols, cols, transpose, ws, digits,
                                                                oz_a_tiles(out_rows), exps);
  return launch_status();
}

inline CMap rowmajor(int64_t ldc) { return CMap{0, 1 << 30, 0, ldc, 1 << 30, 0, 1}; }

// ---------------------------------------------------------------------------
// Exact error on the int8 tensor cores: ssr = sum (X - HL HRt)^2 with the product formed
// tile by tile from 8-digit slices of HL (rows) and HRt (columns) -- the same fp64-accurate
// scheme as the environment products -- and never stored (residual epilogue)
// ---------------------------------------------------------------------------
struct ResOzWs {
  int64_t adig, aexp, amx, bdig, bexp, bmx, part, total;  // offsets in doubles
};
// 32-wide double-buffered n-tiles, 8 epilogue warps (c5, K = 400): 7.7 ms against 20 ms for the
// DMMA residual.  Per 128 x 32 output tile it moves 465 KB of digit tiles (80 GB per launch,
// 8.4 TB/s: less than half of what the L2 -> SM bulk-copy path delivers, tools/micro/l2_ingest.cu)
// and issues 7 MMAs per 32 k, 224 down to 32 columns wide; the tensor pipe is 34 % active (narrow
// MMAs + epilogue, not bandwidth).  Round-2 measurements on the way: the staged 4-warp epilogue 9.9 ms
// (9.0 with its level combine stubbed out); the same epilogue without staging or barriers, X
// loads issued before the accumulator wait, 10.2; with 8 epilogue warps 7.7; 64-wide
// single-buffered tiles (less to take in, but the epilogue no longer overlaps the MMAs) 7.8; A
// stages multicast over clusters of 2 / 4 n-tiles (2.5x fewer L2 reads) 10.9 / 11.6 on the 4-warp form.
constexpr int kResBN = 32;
ResOzWs residual_oz64_layout(int64_t pre, int64_t post, int64_t K) {
  using SC = trals::OzF64;
  const int bn = kResBN;
  ResOzWs w{};
  w.adig = 0;
  w.aexp = w.adig + (oz_digits_bytes(oz_a_tiles(pre), K, SC::D, SC::BK) + 15) / 16 * 2;
  w.amx = w.aexp + (pre + 3) / 4 * 2;
  w.bdig = w.amx + (pre + 1) / 2 * 2;
  w.bexp = w.bdig + (oz_digits_bytes(oz_b_tiles(post, bn), K, SC::D, SC::BK) + 15) / 16 * 2;
  w.bmx = w.bexp + (post + 3) / 4 * 2;
  w.part = w.bmx + (post + 1) / 2 * 2;
  w.total = w.part + kSMs;
  return w;
}


// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
// index of core element (a, i, b) in each layout
__device__ __forceinline__ int64_t core_index(int layout, int64_t a, int64_t i, int64_t b, int Ra, int64_t I,
                                              int Rb) {
  if (layout == TRALS_LAYOUT_C) return (a * I + i) * Rb + b;
  if (layout == TRALS_LAYOUT_SLICE) return (i * Ra + a) * Rb + b;
  if (layout == TRALS_LAYOUT_TT) return (b * Ra + a) * I + i;
  return (i * Rb + b) * Ra + a;  // ZT
}

__global__ void relayout_kernel(const double* __restrict__ src, int sl, int Ra, int64_t I, int Rb,
                                double* __restrict__ dst, int dl) {
  const int64_t total = static_cast<int64_t>(Ra) * I * Rb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // t enumerates the destination in its own order
    const uint32_t u = static_cast<uint32_t>(t), I32 = static_cast<uint32_t>(I);
    const uint32_t ra = static_cast<uint32_t>(Ra), rb = static_cast<uint32_t>(Rb);
    int64_t a, i, b;
    if (dl == TRALS_LAYOUT_C) { b = u % rb; i = (u / rb) % I32; a = u / (rb * I32); }
    else if (dl == TRALS_LAYOUT_SLICE) { b = u % rb; a = (u / rb) % ra; i = u / (rb * ra); }
    else if (dl == TRALS_LAYOUT_TT) { i = u % I32; a = (u / I32) % ra; b = u / (I32 * ra); }
    else { a = u % ra; b = (u / ra) % rb; i = u / (ra * rb); }
    dst[t] = src[core_index(sl, a, i, b, Ra, I, Rb)];
  }
}

constexpr int kSumsqBlocks = 4 * kSMs;  // fixed -> deterministic summation tree

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  // every warp reduces the partials (no shuffles under a warp-dependent branch)
  double r = (l < NT / 32) ? red[l] : 0.0;
  r = warp_sum(r);
  __syncthreads();
  return r;  // valid in every thread
}

// partial sums of squares and of non-finite entries (the check of validation.py:53-54)
template <typename T>
__global__ void __launch_bounds__(512) sumsq_partial_kernel(const T* __restrict__ x, int64_t n,
                                                            double* __restrict__ part) {
  __shared__ double red[16];
  double acc = 0.0, bad = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (sizeof(T) == 8 && (reinterpret_cast<uintptr_t>(x) & 15u) == 0) {
    const double* xd = reinterpret_cast<const double*>(x);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const int64_t n2 = n / 2;
    for (int64_t j = i; j < n2; j += stride) {
      const double2 v = __ldg(x2 + j);
      acc = fma(v.x, v.x, acc);
      acc = fma(v.y, v.y, acc);
      bad += (isfinite(v.x) ? 0.0 : 1.0) + (isfinite(v.y) ? 0.0 : 1.0);
    }
    if (i == 0 && (n & 1)) {
      acc = fma(xd[n - 1], xd[n - 1], acc);
      bad += isfinite(xd[n - 1]) ? 0.0 : 1.0;
    }
  } else {
    for (int64_t j = i; j < n; j += stride) {
      const double v = static_cast<double>(x[j]);
      acc = fma(v, v, acc);
      bad += isfinite(v) ? 0.0 : 1.0;
    }
  }
  const double s = block_sum<512>(acc, red);
  const double b = block_sum<512>(bad, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    part[gridDim.x + blockIdx.x] = b;
  }
}

__global__ void __launch_bounds__(1024) sum_final_kernel(const double* __restrict__ part, int np,
                                                         double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0, bad = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    acc += part[i];
    bad += part[np + i];
  }
  const double s = block_sum<1024>(acc, red);
  const double b = block_sum<1024>(bad, red);
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = b;
  }
}

// ---------------------------------------------------------------------------
// Cholesky S = U^T U (upper, like scipy cho_factor(lower=False), linalg.py:75)
// and Z = M S^{-1} (cho_solve, linalg.py:76)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void chol_reduce_flags(double amax, double asym, double* red, int* info) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
  }
  if (lane == 0) { red[warp] = amax; red[32 + warp] = asym; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a = fmax(a, red[w]); b = fmax(b, red[32 + w]); }
    if (a > 0 && b > 1e-8 * a) info[TRALS_INFO_ASYM] = 1;  // linalg.py:70-72
  }
  __syncthreads();
}

// Blocked in-place upper Cholesky of an n x n SPD block (n <= 112) held in shared
// memory, augmented with the identity (Gauss-Jordan on [A | I]): on return the
// A part holds U (upper) and the augmented part holds V = U^{-T} (lower).
// Rows are processed in panels of 8.  Warp 0 factors each 8x8 diagonal block in
// registers (rows of [D | I_8] in lanes, shuffles, one rsqrt per pivot, no
// divisions); with one panel of look-ahead it updates and factors the NEXT
// diagonal block while the other warps apply the rank-8 update of the current
// panel to the trailing rows on the DMMA pipe.  Two barriers per 8 pivots.
// Layout: row r at a + r*ld, A part columns [0, npad), augmented columns
// [aug, aug + npad); padding rows/columns are 0.  scratch >= 256 doubles.
// Returns the 1-based failing pivot (0 on success), uniform across the CTA.
__device__ __forceinline__ int chol8_factor_block(const double* a, int ld, int p, int pb, double* Ud, double* Xd) {
  // Every lane factors the whole 8 x 8 block redundantly in registers (no shuffles, no
  // shared-memory round trips on the pivot chain: the shuffle-broadcast form cost ~560
  // cycles per pivot, tools/micro/chol_probe.cu), then inverts U in place; lane i writes
  // row i of Ud = U and of Xd = U^{-T}.  Pivots beyond pb are identity padding; a
  // non-positive (or NaN) pivot is reported 1-based.
  const int lane = threadIdx.x & 31;
  double u[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = r; c < 8; ++c) {
      double v = (r < pb && c < pb) ? a[(p + r) * ld + p + c] : 0.0;
      if (r == c && r >= pb) v = 1.0;
      u[r][c] = v;
    }
  int bad = 0;
  double rks[8];  // rsqrt of the pivots = the diagonal of U^{-1}
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double dk = u[k][k];
    const bool ok = bad == 0 && dk > 0.0;
    if (bad == 0 && !ok) bad = k + 1;
    const double rk = rsqrt(ok ? dk : 1.0);
    rks[k] = rk;
    u[k][k] = dk * rk;
#pragma unroll
    for (int c = k + 1; c < 8; ++c) u[k][c] *= rk;
#pragma unroll
    for (int i = k + 1; i < 8; ++i)
#pragma unroll
      for (int c = i; c < 8; ++c) u[i][c] = fma(-u[k][i], u[k][c], u[i][c]);
  }
  if (bad) return bad;
  if (lane < 8) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r == lane) {
#pragma unroll
        for (int c = 0; c < 8; ++c) Ud[r * 8 + c] = (r < pb && c < pb && c >= r) ? u[r][c] : 0.0;
      }
  }
  // in-place W = U^{-1} (upper), column by column, rows top-down
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double wjj = rks[j];  // 1 / u_jj = 1 / sqrt(d_j)
#pragma unroll
    for (int i = 0; i < j; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int l = i; l < j; ++l) acc = fma(u[i][l], u[l][j], acc);  // u[i][l] is W already (l < j)
      u[i][j] = -wjj * acc;
    }
    u[j][j] = wjj;
  }
  if (lane < 8) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if (r == lane) {
#pragma unroll
        for (int c = 0; c < 8; ++c) Xd[r * 8 + c] = (r < pb && c < pb && c <= r) ? u[c][r] : 0.0;
      }
  }
  return 0;
}

__device__ int chol8_aug_smem(double* a, int ld, int n, int aug, double* scratch /* >= 256 doubles */) {
  const int tid = threadIdx.x, lane = tid & 31, nwarps = blockDim.x >> 5;
  // warp index through a shuffle from lane 0: provably warp-uniform, so the warp-0
  // branches below keep the fast (non-collective) shuffle path
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int fr = lane >> 2, fk = lane & 3;
  __shared__ int fail_at;
  if (tid == 0) fail_at = 0;
  if (warp == 0) {
    const int bad = chol8_factor_block(a, ld, 0, min(8, n), scratch, scratch + 64);
    if (bad && lane == 0) fail_at = bad;
  }
  __syncthreads();
  if (fail_at) return fail_at;
  for (int p = 0, it = 0; p < n; p += 8, ++it) {
    const int pb = min(8, n - p);
    const double* Ud = scratch + (it & 1) * 128;
    const double* Xd = Ud + 64;
    // (A) panel rows <- Xd * panel rows: A part columns [p, n), augmented columns [0, p + pb)
    {
      const int wa = n - p, wt = wa + p + pb;
      for (int cc = tid; cc < wt; cc += blockDim.x) {
        const int col = cc < wa ? p + cc : aug + (cc - wa);
        double old[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) old[t] = t < pb ? a[(p + t) * ld + col] : 0.0;
        const bool diag = cc < pb;  // inside the diagonal block: write Ud (exact zeros below)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i >= pb) break;
          double v = 0.0;
#pragma unroll
          for (int t = 0; t <= i; ++t) v = fma(Xd[i * 8 + t], old[t], v);
          a[(p + i) * ld + col] = diag ? Ud[i * 8 + cc] : v;
        }
      }
    }
    __syncthreads();
    // (B) trailing rows r >= p + 8: a[r][c] -= sum_t P[t][r] P[t][c]  (A part c >= r, augmented c < p + 8)
    const int r0 = p + 8;
    if (r0 < n) {
      const int nbr = (n - r0 + 7) / 8;                 // trailing row blocks
      const int nba = (p + 8) / 8;                      // augmented column blocks
      const int nupper = nbr * (nbr + 1) / 2;
      const int ntiles = nupper + nbr * nba;
      auto update_tile = [&](int rb, int cbase) {
        double* c = a + (rb + fr) * ld + cbase + 2 * fk;
        double c0 = c[0], c1 = c[1];
#pragma unroll
        for (int k0 = 0; k0 < 8; k0 += 4) {
          const double av = -a[(p + k0 + fk) * ld + rb + fr];
          const double bv = a[(p + k0 + fk) * ld + cbase + fr];
          trals::dmma884(c0, c1, av, bv);
        }
        c[0] = c0;
        c[1] = c1;
      };
      if (warp == 0) {
        // look-ahead: next diagonal block first, then factor it into the other scratch half
        update_tile(r0, r0);
        __syncwarp();
        double* nUd = scratch + ((it + 1) & 1) * 128;
        const int bad = chol8_factor_block(a, ld, r0, min(8, n - r0), nUd, nUd + 64);
        if (bad && lane == 0) fail_at = r0 + bad;
      } else {
        auto tile_base = [&](int tile, int& rb, int& cbase) -> bool {
          if (tile < nupper) {  // upper-triangular tile grid of the trailing A part
            int bi = 0, rem = tile;
            while (rem >= nbr - bi) { rem -= nbr - bi; ++bi; }
            if (bi == 0 && rem == 0) return false;  // next diagonal block: warp 0 owns it
            rb = r0 + bi * 8;
            cbase = r0 + (bi + rem) * 8;
          } else {
            const int q = tile - nupper;
            rb = r0 + (q / nba) * 8;
            cbase = aug + (q % nba) * 8;
          }
          return true;
        };
        const int stride = nwarps - 1;
        for (int tile = warp - 1; tile < ntiles; tile += 2 * stride) {
          // two independent tiles per iteration: their load/DMMA/store chains overlap
          int rb0 = 0, cb0 = 0, rb1 = 0, cb1 = 0;
          const bool v0 = tile_base(tile, rb0, cb0);
          const bool v1 = tile + stride < ntiles && tile_base(tile + stride, rb1, cb1);
          double* c0p = a + (rb0 + fr) * ld + cb0 + 2 * fk;
          double* c1p = a + (rb1 + fr) * ld + cb1 + 2 * fk;
          double x0 = v0 ? c0p[0] : 0.0, x1 = v0 ? c0p[1] : 0.0;
          double y0 = v1 ? c1p[0] : 0.0, y1 = v1 ? c1p[1] : 0.0;
#pragma unroll
          for (int k0 = 0; k0 < 8; k0 += 4) {
            const double* prow = a + (p + k0 + fk) * ld;
            const double a0 = -prow[rb0 + fr], b0 = prow[cb0 + fr];
            const double a1 = -prow[rb1 + fr], b1 = prow[cb1 + fr];
            trals::dmma884(x0, x1, a0, b0);
            trals::dmma884(y0, y1, a1, b1);
          }
          if (v0) { c0p[0] = x0; c0p[1] = x1; }
          if (v1) { c1p[0] = y0; c1p[1] = y1; }
        }
      }
    }
    __syncthreads();
    if (fail_at) return fail_at;
  }
  return 0;
}

// Resident factor + inverse for m <= kInvMax: U (upper), W = U^{-1} (upper), V = U^{-T} (lower).
constexpr int kInvMax = 112;
// max|U| / min diag(U) above this (cond(S) beyond ~1e8): the explicit-inverse solve is refined once
constexpr double kRefineRatio = 1e4;

__global__ void __launch_bounds__(512) chol_inv_kernel(const double* __restrict__ S, int m, double* __restrict__ U,
                                                       double* __restrict__ W, double* __restrict__ V,
                                                       int check_degen, int* __restrict__ info) {
  extern __shared__ __align__(16) double a[];
  __shared__ double red[64];
  __shared__ double scratch[256];
  const int npad = (m + 7) & ~7, ld = 2 * npad + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  // coalesced load of S, then symmetrise in shared memory (linalg.py:70-73)
  for (int t = tid; t < npad * npad; t += blockDim.x) {
    const int i = t / npad, j = t - i * npad;
    a[i * ld + j] = (i < m && j < m) ? S[i * m + j] : 0.0;
    a[i * ld + npad + j] = (i == j && i < m) ? 1.0 : 0.0;
  }
  __syncthreads();
  double amax = 0.0, asym = 0.0;
  for (int t = tid; t < m * m; t += blockDim.x) {
    const int i = t / m, j = t - i * m;
    if (j < i) continue;
    const double sij = a[i * ld + j], sji = a[j * ld + i];
    amax = fmax(amax, fmax(fabs(sij), fabs(sji)));
    asym = fmax(asym, fabs(sij - sji));
    const double v = 0.5 * (sij + sji);
    a[i * ld + j] = v;
    a[j * ld + i] = v;
  }
  __syncthreads();
  chol_reduce_flags(amax, asym, red, info);
  const int fail = chol8_aug_smem(a, ld, m, npad, scratch);
  if (fail) {
    if (tid == 0) info[TRALS_INFO_CHOL] = fail;
    return;
  }
  double umax = 0.0, dmin = INFINITY;
  int didx = 0;
  for (int i = warp; i < m; i += nwarps)
    for (int j = lane; j < m; j += 32) {
      const double u = j >= i ? a[i * ld + j] : 0.0;
      U[i * m + j] = u;
      V[i * m + j] = j <= i ? a[i * ld + npad + j] : 0.0;
      W[i * m + j] = j >= i ? a[j * ld + npad + i] : 0.0;
      umax = fmax(umax, fabs(u));
      if (i == j && fabs(u) < dmin) { dmin = fabs(u); didx = i; }
    }
  for (int o = 16; o > 0; o >>= 1) {
    umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    const double od = __shfl_xor_sync(0xffffffffu, dmin, o);
    const int oi = __shfl_xor_sync(0xffffffffu, didx, o);
    if (od < dmin || (od == dmin && oi < didx)) { dmin = od; didx = oi; }
  }
  __shared__ double sd[32];
  __shared__ int si[32];
  __syncthreads();
  if (lane == 0) { red[warp] = umax; sd[warp] = dmin; si[warp] = didx; }
  __syncthreads();
  if (tid == 0) {
    double mx = 0, dm = INFINITY;
    int di = 0;
    for (int w = 0; w < nwarps; ++w) {
      mx = fmax(mx, red[w]);
      if (sd[w] < dm || (sd[w] == dm && si[w] < di)) { dm = sd[w]; di = si[w]; }
    }
    if (check_degen && dm <= 1e-13 * mx) info[TRALS_INFO_DEGEN] = di + 1;  // linalg.py:96-99
    // ill-conditioned factor: the explicit-inverse solve gets one refinement step (trals_solve_refine_f64)
    info[TRALS_INFO_REFINE] = (dm > 0.0 && mx > kRefineRatio * dm) ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// Blocked Cholesky + triangular solves for m > kInvMax (R = 20: m = 400).
// Right-looking with 64-row panels: a one-CTA kernel factors the 64x64
// diagonal block in shared memory and inverts it; the panel row block and the
// trailing update are DMMA GEMMs over the whole GPU (the inverse turns the
// panel TRSM into a GEMM).  The same diagonal inverses drive the blocked
// forward/backward substitution of the solve.
// ---------------------------------------------------------------------------
constexpr int kBlkNB = 64;

// U = (S + S^T)/2 tile by tile (coalesced through a shared-memory transpose); the
// largest |S| and |S - S^T| go to flags[0..1] as atomicMax on the (non-negative)
// double bit patterns -- order-independent, so deterministic.
__global__ void chol_sym_kernel(const double* __restrict__ S, int m, double* __restrict__ U,
                                unsigned long long* __restrict__ flags) {
  __shared__ double t1[32][33], t2[32][33];
  const int bi = blockIdx.y * 32, bj = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    t1[r][tx] = (bi + r < m && bj + tx < m) ? S[(bi + r) * m + bj + tx] : 0.0;  // S[bi+r][bj+tx]
    t2[r][tx] = (bj + r < m && bi + tx < m) ? S[(bj + r) * m + bi + tx] : 0.0;  // S[bj+r][bi+tx]
  }
  __syncthreads();
  double amax = 0.0, asym = 0.0;
  for (int r = ty; r < 32; r += 8) {
    const int i = bi + r, j = bj + tx;
    if (i < m && j < m) {
      const double sij = t1[r][tx], sji = t2[tx][r];
      amax = fmax(amax, fabs(sij));
      asym = fmax(asym, fabs(sij - sji));
      U[i * m + j] = 0.5 * (sij + sji);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
  }
  if (tx == 0) {
    atomicMax(flags, static_cast<unsigned long long>(__double_as_longlong(amax)));
    atomicMax(flags + 1, static_cast<unsigned long long>(__double_as_longlong(asym)));
  }
}

// factor the pb x pb diagonal block at (p0, p0) of U in place; W = block^{-1}, WT = W^T (ld kBlkNB)
__global__ void __launch_bounds__(512) chol_diag_kernel(double* __restrict__ U, int m, int p0, int pb,
                                                       double* __restrict__ W, double* __restrict__ WT,
                                                       int* __restrict__ info,
                                                       const unsigned long long* __restrict__ flags) {
  extern __shared__ __align__(16) double a[];  // [kBlkNB][2*kBlkNB + 4]
  constexpr int ld = 2 * kBlkNB + 4;
  __shared__ double scratch[256];
  __shared__ int failed;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  if (tid == 0) {
    failed = info[TRALS_INFO_CHOL];
    if (p0 == 0) {  // symmetry check of linalg.py:70-72 from chol_sym_kernel's maxima
      const double amax = __longlong_as_double(static_cast<long long>(flags[0]));
      const double asym = __longlong_as_double(static_cast<long long>(flags[1]));
      if (amax > 0 && asym > 1e-8 * amax) info[TRALS_INFO_ASYM] = 1;
    }
  }
  for (int r = warp; r < kBlkNB; r += nwarps)
    for (int c = lane; c < kBlkNB; c += 32) {
      a[r * ld + c] = (r < pb && c < pb && c >= r) ? U[(p0 + r) * m + p0 + c] : 0.0;
      a[r * ld + kBlkNB + c] = (r == c && r < pb) ? 1.0 : 0.0;
    }
  __syncthreads();
  if (failed) return;
  const int f = chol8_aug_smem(a, ld, pb, kBlkNB, scratch);
  if (f) {
    if (tid == 0) info[TRALS_INFO_CHOL] = p0 + f;
    return;
  }
  for (int r = warp; r < pb; r += nwarps)
    for (int c = lane; c < pb; c += 32)
      if (c >= r) U[(p0 + r) * m + p0 + c] = a[r * ld + c];
  // V = U_bb^{-T} (lower) sits in the augmented half: W = V^T, WT = V
  for (int r = warp; r < kBlkNB; r += nwarps)
    for (int c = lane; c < kBlkNB; c += 32) {
      const bool in = r < pb && c < pb;
      WT[r * kBlkNB + c] = (in && c <= r) ? a[r * ld + kBlkNB + c] : 0.0;
      W[r * kBlkNB + c] = (in && c >= r) ? a[c * ld + kBlkNB + r] : 0.0;
    }
}

// zero the strict lower triangle of U and write L = U^T
__global__ void chol_finalize_kernel(double* __restrict__ U, double* __restrict__ L, int m) {
  __shared__ double tile[32][33];
  const int bi = blockIdx.y * 32, bj = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int i = bi + r, j = bj + tx;
    double v = 0.0;
    if (i < m && j < m) {
      v = j >= i ? U[i * m + j] : 0.0;
    }
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = bi + r, j = bj + tx;
    if (i < m && j < m && j < i) U[i * m + j] = 0.0;
    const int li = bj + r, lj = bi + tx;  // L[li][lj] = U[lj][li]
    if (li < m && lj < m) L[li * m + lj] = tile[tx][r];
  }
}

// ill_scale > 0 (the QR variants' merged R0): also raise d_info[TRALS_INFO_ILLCOND] when the smallest
// diagonal is within ill_scale of the largest entry -- the solve then goes through the R0 SVD (see
// trals_tri_fallback_f64); the reference's 1e-13 floor (TRALS_INFO_DEGEN) is unchanged
__global__ void __launch_bounds__(1024) degen_kernel(const double* __restrict__ U, int m, int* __restrict__ info,
                                                     double ill_scale = 0.0) {
  __shared__ double red[32], sd[32];
  __shared__ int si[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double umax = 0.0, dmin = INFINITY;
  int didx = 0;
  for (int i = warp; i < m; i += nwarps)
    for (int j = lane; j < m; j += 32) {
      if (j < i) continue;
      const double u = fabs(U[i * m + j]);
      umax = fmax(umax, u);
      if (i == j && u < dmin) { dmin = u; didx = i; }
    }
  for (int o = 16; o > 0; o >>= 1) {
    umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    const double od = __shfl_xor_sync(0xffffffffu, dmin, o);
    const int oi = __shfl_xor_sync(0xffffffffu, didx, o);
    if (od < dmin || (od == dmin && oi < didx)) { dmin = od; didx = oi; }
  }
  if (lane == 0) { red[warp] = umax; sd[warp] = dmin; si[warp] = didx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, d = INFINITY;
    int di = 0;
    for (int w = 0; w < nwarps; ++w) {
      a = fmax(a, red[w]);
      if (sd[w] < d || (sd[w] == d && si[w] < di)) { d = sd[w]; di = si[w]; }
    }
    if (d <= 1e-13 * a) info[TRALS_INFO_DEGEN] = di + 1;  // linalg.py:96-99
    if (ill_scale > 0.0 && d <= ill_scale * a) info[TRALS_INFO_ILLCOND] = 1;
    if (m <= kInvMax) info[TRALS_INFO_REFINE] = (d > 0.0 && a > kRefineRatio * d) ? 1 : 0;
  }
}

int64_t blocked_aux_elems(int m) {  // diagonal-block inverses + 2 flag words
  const int nblk = (m + kBlkNB - 1) / kBlkNB;
  return static_cast<int64_t>(nblk) * 2 * kBlkNB * kBlkNB + 2;
}

int blocked_cholesky(const double* S, int m, double* U, double* L, double* aux, double* gws, int64_t gws_elems,
                     int check_degen, int* info, cudaStream_t s) {
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(aux + blocked_aux_elems(m) - 2);
  if (cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess) return TRALS_ERR_CUDA;
  {
    dim3 grid((m + 31) / 32, (m + 31) / 32);
    chol_sym_kernel<<<grid, dim3(32, 8), 0, s>>>(S, m, U, flags);
    if (int st = launch_status()) return st;
  }
  const CMap rm = rowmajor(m);
  for (int p0 = 0, b = 0; p0 < m; p0 += kBlkNB, ++b) {
    const int pb = std::min(kBlkNB, m - p0);
    const int rest = m - p0 - pb;
    double* W = aux + static_cast<int64_t>(b) * 2 * kBlkNB * kBlkNB;
    double* WT = W + kBlkNB * kBlkNB;
    constexpr size_t kDiagSmem = sizeof(double) * kBlkNB * (2 * kBlkNB + 4);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagSmem);
      attr = true;
    }
    chol_diag_kernel<<<1, 512, kDiagSmem, s>>>(U, m, p0, pb, W, WT, info, flags);
    if (int st = launch_status()) return st;
    if (rest == 0) continue;
    double* U12 = U + static_cast<int64_t>(p0) * m + p0 + pb;
    // U12 <- W^T A12 (in place: one M tile, each CTA rewrites exactly the columns it read)
    int st = gemm(WT, 0, kBlkNB, 1, 1, pb, pb, rest, U12, m, U12, rm, 0, nullptr, 0, s);  // no split: in place
    if (st) return st;
    // A22 -= U12^T U12
    double* A22 = U + static_cast<int64_t>(p0 + pb) * m + p0 + pb;
    st = gemm(U12, 0, 1, m, 1, rest, pb, rest, U12, m, A22, rm, 1, gws, gws_elems, s, -1.0);
    if (st) return st;
  }
  dim3 grid((m + 31) / 32, (m + 31) / 32);
  chol_finalize_kernel<<<grid, dim3(32, 8), 0, s>>>(U, L, m);
  if (int st = launch_status()) return st;
  if (check_degen) {
    degen_kernel<<<1, 1024, 0, s>>>(U, m, info);
    return launch_status();
  }
  return TRALS_OK;
}


// Fused blocked substitution for m > kInvMax: one CTA per 8 right-hand-side
// rows (one DMMA m8 row tile), all 2*nblk block steps in one launch.
//   forward  (Y U = M):   R_b -= Y_{<b} U_{<b,b};  Y_b = R_b W_b
//   backward (Z U^T = Y): T_b = Y_b - Z_{>b} L_{>b,b};  Z_b = T_b W_b^T
// The RHS rows live in shared memory; U / L column blocks and the diagonal
// inverses stream through a cp.async double buffer; warp w owns columns
// [8w, 8w+8) of the current 64-column block.
constexpr int kFsRows = 8;

__global__ void __launch_bounds__(256) fused_solve_kernel(const double* __restrict__ U, const double* __restrict__ L,
                                                          const double* __restrict__ aux, int m,
                                                          const double* __restrict__ Mr, int64_t rows,
                                                          double* __restrict__ Z) {
  // Operand blocks are read straight from L2 as DMMA fragments (each warp its own 8
  // columns, all 16 loads of a 64-k chunk issued before the MMAs): no staging and no
  // CTA barrier per chunk, two per 64-column block (R_b complete; Y_b / Z_b published).
  extern __shared__ __align__(16) double fs[];
  const int mp = ((m + kBlkNB - 1) / kBlkNB) * kBlkNB;
  const int ldr = mp + 4;
  double* Rs = fs;                  // [8][ldr] running rhs, later Z
  double* Ys = Rs + kFsRows * ldr;  // [8][ldr] forward solution
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kFsRows;
  const int nblk = mp / kBlkNB;
  for (int t = tid; t < kFsRows * ldr; t += blockDim.x) {
    const int r = t / ldr, c = t - r * ldr;
    Rs[t] = (row0 + r < rows && c < m) ? Mr[(row0 + r) * m + c] : 0.0;
    Ys[t] = 0.0;
  }
  __syncthreads();
  // acc (+)= Xs[:, xoff .. xoff+64] * G[k0 .. k0+64][col] for this warp's column col (G row-major,
  // pitch ldg, zero outside [0, limk) x [0, limc)); two DMMA chains
  auto load = [&](double (&bv)[16], const double* G, int64_t ldg, int k0, int col, int limk, int limc) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int kk = k0 + 4 * q + fk;
      bv[q] = (kk < limk && col < limc) ? __ldg(G + static_cast<int64_t>(kk) * ldg + col) : 0.0;
    }
  };
  auto mma = [&](const double (&bv)[16], const double* Xs, int xoff, double& a0, double& a1, double& a2, double& a3) {
#pragma unroll
    for (int q = 0; q < 16; q += 2) {
      trals::dmma884(a0, a1, Xs[fr * ldr + xoff + 4 * q + fk], bv[q]);
      trals::dmma884(a2, a3, Xs[fr * ldr + xoff + 4 * q + 4 + fk], bv[q + 1]);
    }
  };
  auto chunk = [&](const double* Xs, int xoff, const double* G, int64_t ldg, int k0, int col, int limk, int limc,
                   double& a0, double& a1, double& a2, double& a3) {
    double bv[16];
    load(bv, G, ldg, k0, col, limk, limc);
    mma(bv, Xs, xoff, a0, a1, a2, a3);
  };
  // chunks c = c0, c0 + 1, ... < c1 of 64 k (operand offset = k offset = 64 c): the next
  // chunk's 16 L2 loads are in flight while this one's MMAs run (two named fragment
  // buffers, compile-time indexed)
  auto chunks = [&](const double* Xs, const double* G, int c0, int c1, int col, double& a0, double& a1, double& a2,
                    double& a3) {
    if (c0 >= c1) return;
    double bA[16], bB[16];
    load(bA, G, m, c0 * kBlkNB, col, m, m);
    for (int c = c0; c < c1; c += 2) {
      if (c + 1 < c1) load(bB, G, m, (c + 1) * kBlkNB, col, m, m);
      mma(bA, Xs, c * kBlkNB, a0, a1, a2, a3);
      if (c + 2 < c1) load(bA, G, m, (c + 2) * kBlkNB, col, m, m);
      if (c + 1 < c1) mma(bB, Xs, (c + 1) * kBlkNB, a0, a1, a2, a3);
    }
  };
  // ---------------- forward: Y_b = (R_b - Y_{<b} U_{<b,b}) W_b ----------------
  for (int b = 0; b < nblk; ++b) {
    const int j0 = b * kBlkNB;
    const int col = j0 + warp * 8 + fr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    chunks(Ys, U, 0, b, col, a0, a1, a2, a3);
    Rs[fr * ldr + j0 + warp * 8 + 2 * fk] -= a0 + a2;
    Rs[fr * ldr + j0 + warp * 8 + 2 * fk + 1] -= a1 + a3;
    __syncthreads();
    const double* Wb = aux + static_cast<int64_t>(b) * 2 * kBlkNB * kBlkNB;
    double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
    chunk(Rs, j0, Wb, kBlkNB, 0, warp * 8 + fr, kBlkNB, kBlkNB, y0, y1, y2, y3);
    Ys[fr * ldr + j0 + warp * 8 + 2 * fk] = y0 + y2;
    Ys[fr * ldr + j0 + warp * 8 + 2 * fk + 1] = y1 + y3;
    __syncthreads();
  }
  // ---------------- backward (Z overwrites Rs): Z_b = (Y_b - Z_{>b} L_{>b,b}) W_b^T ----------------
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * kBlkNB, j1 = j0 + kBlkNB;
    const int col = j0 + warp * 8 + fr;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    chunks(Rs, L, b + 1, nblk, col, a0, a1, a2, a3);
    Ys[fr * ldr + j0 + warp * 8 + 2 * fk] -= a0 + a2;
    Ys[fr * ldr + j0 + warp * 8 + 2 * fk + 1] -= a1 + a3;
    __syncthreads();
    const double* WTb = aux + static_cast<int64_t>(b) * 2 * kBlkNB * kBlkNB + kBlkNB * kBlkNB;
    double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
    chunk(Ys, j0, WTb, kBlkNB, 0, warp * 8 + fr, kBlkNB, kBlkNB, z0, z1, z2, z3);
    Rs[fr * ldr + j0 + warp * 8 + 2 * fk] = z0 + z2;
    Rs[fr * ldr + j0 + warp * 8 + 2 * fk + 1] = z1 + z3;
    __syncthreads();
  }
  for (int t = tid; t < kFsRows * m; t += blockDim.x) {
    const int r = t / m, c = t - r * m;
    if (row0 + r < rows) Z[(row0 + r) * m + c] = Rs[r * ldr + c];
  }
}

size_t fused_solve_smem(int m) {
  const int mp = ((m + kBlkNB - 1) / kBlkNB) * kBlkNB;
  return sizeof(double) * (2 * kFsRows * (mp + 4));
}

// Z S = M, S = U^T U:  Y U = M (forward), Z U^T = Y (backward), 64-column blocks
int blocked_solve(const double* U, const double* L, const double* aux, int m, const double* Mr, int64_t rows,
                  double* Z, double* ws, double* gws, int64_t gws_elems, cudaStream_t s) {
  const CMap rm = rowmajor(m);
  double* R = ws;   // running right-hand side
  double* Y = Z;    // forward result lives in Z's storage, then overwritten block by block
  const int nblk = (m + kBlkNB - 1) / kBlkNB;
  // forward: R = M; Y_b = (R_b - Y_{<b} U_{<b,b}) W_b
  if (cudaMemcpyAsync(R, Mr, sizeof(double) * rows * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return TRALS_ERR_CUDA;
  for (int b = 0; b < nblk; ++b) {
    const int j0 = b * kBlkNB, pb = std::min(kBlkNB, m - j0);
    const double* W = aux + static_cast<int64_t>(b) * 2 * kBlkNB * kBlkNB;
    if (j0 > 0) {
      int st = gemm(Y, 0, m, 1, 1, rows, j0, pb, U + j0, m, R + j0, rm, 1, gws, gws_elems, s, -1.0);
      if (st) return st;
    }
    int st = gemm(R + j0, 0, m, 1, 1, rows, pb, pb, W, kBlkNB, Y + j0, rm, 0, gws, gws_elems, s);
    if (st) return st;
  }
  // backward: R = Y; Z_b = (R_b - Z_{>b} L_{>b,b}) W_b^T, last block first (Z overwrites Y in place:
  // block b of Y is consumed into R before block b of Z is written)
  if (cudaMemcpyAsync(R, Y, sizeof(double) * rows * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return TRALS_ERR_CUDA;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * kBlkNB, pb = std::min(kBlkNB, m - j0);
    const int j1 = j0 + pb;
    const double* WT = aux + static_cast<int64_t>(b) * 2 * kBlkNB * kBlkNB + kBlkNB * kBlkNB;
    if (j1 < m) {
      int st = gemm(Z + j1, 0, m, 1, 1, rows, m - j1, pb, L + static_cast<int64_t>(j1) * m + j0, m, R + j0, rm, 1,
                    gws, gws_elems, s, -1.0);
      if (st) return st;
    }
    int st = gemm(R + j0, 0, m, 1, 1, rows, pb, pb, WT, kBlkNB, Z + j0, rm, 0, gws, gws_elems, s);
    if (st) return st;
  }
  return TRALS_OK;
}

// ---------------------------------------------------------------------------
// Numerical fallbacks (rare path, one CTA):
//   NE / QRNE (linalg.py:77-81): Cholesky failed -> least-squares solve of
//     Z sym = M with rank cut at eps * sigma_max (scipy lstsq gelsy, cond=eps);
//   QR (solvers.py:262-273, linalg.py:104-112): R0 = chol(S) degenerate (or
//     failed) and rank_deficient_fallback -> min-norm solve with singular values
//     of R0 cut at rcond * sigma_max(R0), i.e. eigenvalues of S at rcond^2.
// Both are Z = M pinv(S) with a relative cut; pinv(S) comes from a one-sided
// (Hestenes) Jacobi SVD of S with round-robin parallel rotations.  The kernel
// exits at once when its trigger flag is clear, so it sits in the sweep graph
// unconditionally; when it fires it overwrites Z, clears the flag and bumps
// d_info[TRALS_INFO_FALLBACKS] (report.fallback_count).
// ---------------------------------------------------------------------------
// tri != 0: S is instead the QR variants' triangular factor R0 (Lr x m row-major, Lr <= m; the
// merged R0 of qr_r0.cuh): the SVD is taken of R0 itself (R0 V = U Sigma), so singular values down
// to eps sigma_max survive, and Z = M V Sigma^{-2} V^T with the cut rcond * sigma_max(R0) --
// W pinv(R0)^T of the reference with W = M R0^{-1} (solvers.py:262-273, linalg.py:104-112).
__global__ void __launch_bounds__(1024) pinv_fallback_kernel(const double* __restrict__ S, int m,
                                                             const double* __restrict__ Mr, int64_t rows,
                                                             double* __restrict__ Z, int* __restrict__ info, int mode,
                                                             double rcond, double* __restrict__ ws, int Lr, int tri) {
  const int tid = threadIdx.x, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int trig_chol = info[TRALS_INFO_CHOL];
  const int trig_degen = info[TRALS_INFO_DEGEN];
  const int trig_ill = tri ? info[TRALS_INFO_ILLCOND] : 0;
  // mode 2: non-square R0 in the reference (prod_j k_j < R^2): always the SVD solve, not counted;
  // mode 3 (tri only, fallback disabled): only the ill-conditioning safety solve
  bool fire;
  if (mode == 0) fire = trig_chol != 0;
  else if (mode == 1) fire = trig_chol != 0 || trig_degen != 0 || trig_ill != 0;
  else if (mode == 2) fire = true;
  else fire = trig_ill != 0;
  if (!fire) return;
  const bool counted = (mode == 0) || (mode == 1 && (trig_chol != 0 || trig_degen != 0));
  const int m2 = (m + 1) & ~1;
  double* A = ws;                          // [m2][m] columns of S (column-major), zero column if padded
  double* V = A + static_cast<int64_t>(m2) * m;   // [m2][m2]
  double* sig = V + static_cast<int64_t>(m2) * m2;  // [m2]
  double* coef = sig + m2;                 // [rows][m2]
  const int L = tri ? Lr : m;  // column length of the Jacobi matrix
  for (int t = tid; t < m2 * m; t += blockDim.x) {
    const int c = t / m, r = t - c * m;
    if (tri) A[t] = (c < m && r < L) ? S[r * m + c] : 0.0;
    else A[t] = (c < m) ? 0.5 * (S[r * m + c] + S[c * m + r]) : 0.0;
  }
  for (int t = tid; t < m2 * m2; t += blockDim.x) V[t] = ((t / m2) == (t % m2)) ? 1.0 : 0.0;
  __syncthreads();
  __shared__ int rotated;
  const double eps = 2.220446049250313e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < m2 - 1; ++round) {
      for (int k = warp; k < m2 / 2; k += nwarps) {
        int i, j;
        if (k == 0) { i = round % (m2 - 1); j = m2 - 1; }
        else { i = (round + k) % (m2 - 1); j = (round - k + m2 - 1) % (m2 - 1); }
        double* ai = A + static_cast<int64_t>(i) * m;
        double* aj = A + static_cast<int64_t>(j) * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < L; r += 32) {
          const double x = ai[r], y = aj[r];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (fabs(ga) > eps * sqrt(al * be) && ga != 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int r = lane; r < L; r += 32) {
            const double x = ai[r], y = aj[r];
            ai[r] = c * x - s * y;
            aj[r] = s * x + c * y;
          }
          double* vi = V + static_cast<int64_t>(i) * m2;
          double* vj = V + static_cast<int64_t>(j) * m2;
          for (int r = lane; r < m2; r += 32) {
            const double x = vi[r], y = vj[r];
            vi[r] = c * x - s * y;
            vj[r] = s * x + c * y;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  // singular values (= eigenvalues of the PSD part), relative cut
  for (int c = warp; c < m2; c += nwarps) {
    double s2 = 0.0;
    for (int r = lane; r < L; r += 32) s2 = fma(A[c * m + r], A[c * m + r], s2);
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) sig[c] = sqrt(s2);
  }
  __syncthreads();
  __shared__ double smax;
  if (tid == 0) {
    double mx = 0.0;
    for (int c = 0; c < m2; ++c) mx = fmax(mx, sig[c]);
    smax = mx;
  }
  __syncthreads();
  // singular values of S below ~m eps sigma_max are rounding noise of the Jacobi SVD (and, for the
  // QR modes, squares of R0's), so the cut never goes below that noise floor: mode 0 (gelsy, cond = eps)
  // uses max(rcond, m eps), modes 1/2 map R0's rcond to max(rcond^2, m eps) on S
  const double floor_noise = m * eps;
  // tri: the right-hand side is M = W R0 (not W itself), so components are divided by sigma^2: the
  // cut never goes below sqrt(m eps) sigma_max (below it the M-based solve only amplifies rounding)
  const double cut = tri ? fmax(rcond, sqrt(floor_noise)) * smax
                         : (mode == 0 ? fmax(rcond, floor_noise) : fmax(rcond * rcond, floor_noise)) * smax;
  // S mode:   Z = M pinv(S) = sum_{sig_i > cut} (M a_i / sig_i^2) v_i^T   (a_i = S v_i = sig_i v_i)
  // tri mode: Z = M pinv(R0^T R0) = sum_{sig_i > cut} (M v_i / sig_i^2) v_i^T
  for (int t = tid; t < rows * m2; t += blockDim.x) {
    const int64_t r = t / m2;
    const int i = static_cast<int>(t - r * m2);
    double v = 0.0;
    if (sig[i] > cut) {
      const double* vec = tri ? V + static_cast<int64_t>(i) * m2 : A + static_cast<int64_t>(i) * m;
      for (int k = 0; k < m; ++k) v = fma(Mr[r * m + k], vec[k], v);
      v /= sig[i] * sig[i];
    }
    coef[t] = v;
  }
  __syncthreads();
  for (int64_t t = tid; t < rows * m; t += blockDim.x) {
    const int64_t r = t / m;
    const int c = static_cast<int>(t - r * m);
    double v = 0.0;
    for (int i = 0; i < m2; ++i) v = fma(coef[r * m2 + i], V[static_cast<int64_t>(i) * m2 + c], v);
    Z[t] = v;
  }
  __syncthreads();
  if (tid == 0 && mode != 2) {  // mode 2 replaces the factorisation outright: no flags, not counted
    if (mode != 3) {
      info[TRALS_INFO_CHOL] = 0;
      if (mode == 1) info[TRALS_INFO_DEGEN] = 0;
    }
    if (tri) info[TRALS_INFO_ILLCOND] = 0;
    if (counted) info[TRALS_INFO_FALLBACKS] += 1;
  }
}

// ---------------------------------------------------------------------------
// Per-core Householder QR of the classical 2-unfolding G_(2) (I x R R') for the
// QR / QRNE variants (mode2_qr, ring.py:236-249 + qr_economy, linalg.py:36-52):
// only R (k x RR, k = min(I, RR)) is needed -- the sweep never compresses X
// (one right-hand side serves all variants), the R-tensor feeds the R-Grams.
// LAPACK-style reflectors H = I - tau v v^T (v_0 = 1, beta = -sign(alpha)|x|),
// then rows of R with a negative diagonal are negated (nonnegative diag, the
// deterministic convention of qr_economy).
//  * whole matrix fits shared memory: one CTA;
//  * tall (I > RR) otherwise: TSQR -- row chunks factored by independent CTAs,
//    their R factors stacked pairwise and re-factored up a binary tree;
//  * wide (I < RR) otherwise: the I x I left block is factored in one CTA that
//    also stores its reflectors, then column chunks of the rest are multiplied
//    by Q^T in parallel CTAs.
// ---------------------------------------------------------------------------
constexpr int kHhThreads = 256;
constexpr size_t kHhSmemMax = 216 * 1024;
constexpr int kHhNB = 8;           // reflectors per panel (compact WY block)
constexpr int kHhPanelRows = 256;  // panel rows a team of up to 4 warps holds in registers (2 per lane)

// Unblocked fallback for matrices taller than kHhPanelRows (three barriers per reflector).
__device__ void hh_factor_unblocked(double* A, int ld, int mr, int nc, double* tau, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, nwarps = blockDim.x >> 5;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int k = min(mr, nc);
  for (int j = 0; j < k; ++j) {
    // |x|^2 of the sub-column below the diagonal (fixed-order block reduction)
    double s = 0.0;
    for (int r = j + 1 + tid; r < mr; r += blockDim.x) s = fma(A[r * ld + j], A[r * ld + j], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double sig = 0.0;
    for (int w = 0; w < nwarps; ++w) sig += red[w];
    const double alpha = A[j * ld + j];
    double t = 0.0, scale = 0.0, beta = alpha;
    if (sig > 0.0) {
      const double nrm = sqrt(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncthreads();  // everyone has alpha before it changes
    if (tid == 0) {
      tau[j] = t;
      A[j * ld + j] = beta;
    }
    for (int r = j + 1 + tid; r < mr; r += blockDim.x) A[r * ld + j] *= scale;  // v (v_0 = 1 implicit)
    __syncthreads();
    if (t != 0.0) {
      // columns c > j: w = v^T A[j:, c];  A[j:, c] -= t v w   (one warp per column)
      for (int c = j + 1 + warp; c < nc; c += nwarps) {
        double w = (lane == 0) ? A[j * ld + c] : 0.0;
        for (int r = j + 1 + lane; r < mr; r += 32) w = fma(A[r * ld + j], A[r * ld + c], w);
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        const double tw = t * w;
        if (lane == 0) A[j * ld + c] -= tw;
        for (int r = j + 1 + lane; r < mr; r += 32) A[r * ld + c] = fma(-tw, A[r * ld + j], A[r * ld + c]);
      }
    }
    __syncthreads();
  }
}


// V(r, t) of a staged panel: reflector t at absolute row r (1 at row p + t, 0 above or
// for padding reflectors t >= nb or rows >= mr, the stored entry below)
__device__ __forceinline__ double hh_v(const double* V, int vld, int p, int nb, int mr, int r, int t) {
  const int rel = r - p;
  if (t >= nb || r >= mr || rel < t) return 0.0;
  return rel == t ? 1.0 : V[r * vld + t];
}

// Q_panel^T applied to the columns [c_lo, c_hi) of A (rows [p, mr)) on the DMMA pipe
// (mma.sync m8n8k4 f64): per 8-column group, W = V^T A_c (8 x 8, k over the rows),
// W' = T^T W, A_c -= V W' (8-row tiles, k over the 8 reflectors).  V[r * vld + t] =
// reflector t at absolute row r.  Column groups go to warps wid, wid + nw, ...;
// scratch = 64 doubles per warp (W / W' handed from the accumulator to the operand
// layout).  Reductions run in a fixed order: deterministic.
__device__ void hh_panel_apply(const double* V, int vld, const double* T, int nb, double* A, int ld, int mr, int p,
                               int c_lo, int c_hi, int wid, int nw, double* scratch) {
  if (c_hi <= c_lo || wid >= nw) return;
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  const int groups = (c_hi - c_lo + 7) / 8;
  for (int gi = wid; gi < groups; gi += nw) {
    const int c0 = c_lo + 8 * gi;
    // W[t][c] = sum_r V(r, t) A[r][c0 + c]
    // two independent accumulation chains (even / odd 4-row steps), summed at the end
    double w0 = 0.0, w1 = 0.0, y0 = 0.0, y1 = 0.0;
    const int colb = c0 + fr;
    const bool cb = colb < c_hi;
    for (int r0 = p; r0 < mr; r0 += 8) {
      const int r = r0 + fk, r2 = r0 + 4 + fk;
      const double av = hh_v(V, vld, p, nb, mr, r, fr);
      const double bv = (cb && r < mr) ? A[r * ld + colb] : 0.0;
      const double av2 = hh_v(V, vld, p, nb, mr, r2, fr);
      const double bv2 = (cb && r2 < mr) ? A[r2 * ld + colb] : 0.0;
      trals::dmma884(w0, w1, av, bv);
      trals::dmma884(y0, y1, av2, bv2);
    }
    scratch[fr * 8 + 2 * fk] = w0 + y0;
    scratch[fr * 8 + 2 * fk + 1] = w1 + y1;
    __syncwarp();
    // W'[t][c] = sum_u T[u][t] W[u][c]
    double x0 = 0.0, x1 = 0.0;
#pragma unroll
    for (int u0 = 0; u0 < 8; u0 += 4) {
      const double av = T[(u0 + fk) * 8 + fr];
      const double bv = scratch[(u0 + fk) * 8 + fr];
      trals::dmma884(x0, x1, av, bv);
    }
    __syncwarp();
    scratch[fr * 8 + 2 * fk] = x0;
    scratch[fr * 8 + 2 * fk + 1] = x1;
    __syncwarp();
    // A[r][c0 + c] -= sum_t V(r, t) W'[t][c], 8-row tiles
    const double b0 = scratch[fk * 8 + fr], b1 = scratch[(4 + fk) * 8 + fr];
    const int cc = c0 + 2 * fk;
#pragma unroll 2
    for (int r8 = p; r8 < mr; r8 += 8) {
      const int r = r8 + fr;
      const bool rok = r < mr;
      double* row = A + r * ld;
      double d0 = (rok && cc < c_hi) ? row[cc] : 0.0;
      double d1 = (rok && cc + 1 < c_hi) ? row[cc + 1] : 0.0;
      trals::dmma884(d0, d1, -hh_v(V, vld, p, nb, mr, r, fk), b0);
      trals::dmma884(d0, d1, -hh_v(V, vld, p, nb, mr, r, 4 + fk), b1);
      if (rok && cc < c_hi) row[cc] = d0;
      if (rok && cc + 1 < c_hi) row[cc + 1] = d1;
    }
    __syncwarp();
  }
}

// Panel [p, p+nb) x rows [p, mr) factored by a team of NT warps (warps [0, NT)) in
// registers: row p + rel with rel = lane + 32 (wt + NT i), i < 2, lives in warp wt, so
// the diagonal rows p..p+7 are in warp 0.  Per column one fused reduction (|x|^2 below
// the diagonal and x . a_c for the later panel columns: v . a_c = a_jj,c + scale x . a_c),
// warp shuffles then, for NT > 1, a fixed-order sum of the warps' partials through
// shared memory (named barrier 1, double-buffered slots), and the LAPACK reflector
// (v_0 = 1, beta = -sign(alpha)|x|, tau = (beta - alpha)/beta).  Afterwards warp 0
// forms G = V^T V on the DMMA pipe and the compact-WY factor T (8 x 8 upper,
// H_1..H_nb = I - V T V^T, dlarft's forward recurrence, one row per lane) into T and,
// if Tg != nullptr, Tg.  Columns >= nb and rows >= mr are zero padding: every step runs
// unconditionally (tau = 0 there).  xch: 2 x (NT + 1) x 8 doubles; scratch: 64 doubles.
__device__ __forceinline__ void hh_team_sync(int nt) {
  if (nt > 1) asm volatile("bar.sync 1, %0;\n" ::"r"(nt * 32) : "memory");
  else __syncwarp();
}

template <int RW>
__device__ void hh_panel_team(double* A, int ld, int mr, int p, int nb, double* tau, double* T, double* Tg, int NT,
                              double* xch, double* scratch) {
  const int lane = threadIdx.x & 31;
  const int wt = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  // a[i][c] = panel column jj + c of this lane's rows: a window that rotates left as the
  // columns are finished, so every register index is a compile-time constant while the
  // column loop itself stays rolled (the fully unrolled form was ~300 KB of SASS per
  // kernel: single-warp code then ran at the instruction-fetch rate)
  double a[RW][kHhNB];
  int rel[RW];
#pragma unroll
  for (int i = 0; i < RW; ++i) {
    rel[i] = lane + 32 * (wt + NT * i);
#pragma unroll
    for (int c = 0; c < kHhNB; ++c) {
      const int r = p + rel[i];
      a[i][c] = (r < mr && c < nb) ? A[r * ld + p + c] : 0.0;
    }
  }
#pragma unroll 1
  for (int jj = 0; jj < kHhNB; ++jj) {
    double red[kHhNB];
#pragma unroll
    for (int c = 0; c < kHhNB; ++c) red[c] = 0.0;
#pragma unroll
    for (int i = 0; i < RW; ++i)
      if (rel[i] > jj) {
#pragma unroll
        for (int c = 0; c < kHhNB; ++c) red[c] = fma(a[i][0], a[i][c], red[c]);
      }
    double top[kHhNB];
#pragma unroll
    for (int c = 0; c < kHhNB; ++c) top[c] = __shfl_sync(0xffffffffu, a[0][c], jj);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < kHhNB; ++c) red[c] += __shfl_xor_sync(0xffffffffu, red[c], o);
    if (NT > 1) {
      double* slot = xch + (jj & 1) * (NT + 1) * kHhNB;
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < kHhNB; ++c) slot[wt * kHhNB + c] = red[c];
      }
      if (wt == 0 && lane == 0) {
#pragma unroll
        for (int c = 0; c < kHhNB; ++c) slot[NT * kHhNB + c] = top[c];
      }
      hh_team_sync(NT);
#pragma unroll
      for (int c = 0; c < kHhNB; ++c) {
        double v = 0.0;
        for (int w = 0; w < NT; ++w) v += slot[w * kHhNB + c];
        red[c] = v;
        top[c] = slot[NT * kHhNB + c];
      }
    }
    const double s = red[0], alpha = top[0];
    double t = 0.0, scale = 0.0, beta = alpha;
    if (s > 0.0) {
      // correctly rounded sqrt / divisions (LAPACK dlarfg's arithmetic): an rsqrt-based form
      // (-5 % QR time) moved the reflectors by an ulp, enough to flip the reference's 1e-13
      // degeneracy test on a rank-deficient golden (test_degenerate_without_fallback_raises)
      const double nrm = sqrt(alpha * alpha + s);
      beta = alpha >= 0.0 ? -nrm : nrm;
      t = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    const bool diag = (wt == 0 && lane == jj);
#pragma unroll
    for (int i = 0; i < RW; ++i)
      if (rel[i] > jj) a[i][0] *= scale;
    if (diag) a[0][0] = beta;
    // column jj is final: store it (reflector below the diagonal, R entries above)
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const int r = p + rel[i];
      if (r < mr && jj < nb) A[r * ld + p + jj] = a[i][0];
    }
    if (wt == 0 && lane == 0 && jj < nb) tau[p + jj] = t;
#pragma unroll
    for (int c = 1; c < kHhNB; ++c) {
      const double w = t * fma(scale, red[c], top[c]);
      if (diag) a[0][c] -= w;
#pragma unroll
      for (int i = 0; i < RW; ++i)
        if (rel[i] > jj) a[i][c] = fma(-w, a[i][0], a[i][c]);
    }
#pragma unroll
    for (int i = 0; i < RW; ++i) {
#pragma unroll
      for (int c = 0; c + 1 < kHhNB; ++c) a[i][c] = a[i][c + 1];
      a[i][kHhNB - 1] = 0.0;
    }
  }
  hh_team_sync(NT);
  if (wt != 0) return;
  // G = V^T V on the DMMA pipe (two accumulation chains), via scratch to every lane
  {
    const int fr = lane >> 2, fk = lane & 3;
    const double* V = A + p;
    double g0 = 0.0, g1 = 0.0, h0 = 0.0, h1 = 0.0;
    for (int r0 = p; r0 < mr; r0 += 8) {
      const int r = r0 + fk, r2 = r0 + 4 + fk;
      trals::dmma884(g0, g1, hh_v(V, ld, p, nb, mr, r, fr), hh_v(V, ld, p, nb, mr, r, fr));
      trals::dmma884(h0, h1, hh_v(V, ld, p, nb, mr, r2, fr), hh_v(V, ld, p, nb, mr, r2, fr));
    }
    scratch[fr * 8 + 2 * fk] = g0 + h0;
    scratch[fr * 8 + 2 * fk + 1] = g1 + h1;
    __syncwarp();
  }
  // T row by row in parallel: lane i < 8 owns row i, T[i][jj] = -tau_jj sum_{i<=l<jj} T[i][l] G[l][jj]
  double trow[kHhNB];
#pragma unroll
  for (int jj = 0; jj < kHhNB; ++jj) {
    const double tj = jj < nb ? tau[p + jj] : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < jj; ++l) acc = (l >= lane) ? fma(trow[l], scratch[l * 8 + jj], acc) : acc;
    trow[jj] = (jj < lane) ? 0.0 : (jj == lane ? tj : -tj * acc);
  }
  __syncwarp();
  if (lane < kHhNB) {
#pragma unroll
    for (int jj = 0; jj < kHhNB; ++jj) {
      T[lane * kHhNB + jj] = trow[jj];
      if (Tg) Tg[lane * kHhNB + jj] = trow[jj];
    }
  }
  __syncwarp();
}

// Blocked in-place Householder QR of A (mr x nc, pitch ld, mr <= kHhPanelRows) in shared
// memory: reflector j in A[j+1.., j], tau[j], R in the upper triangle; the T factor of
// panel b goes to Tg + 64 b when Tg != nullptr.  A team of NT = ceil(mr / 64) warps
// factors the panels; look-ahead: team warp 0 applies panel b to the columns of panel
// b+1, the team factors panel b+1, while the other warps apply panel b to everything
// right of it -- one CTA barrier per 8 reflectors.  xch: 2 x 5 x 8 doubles, scratch:
// 64 doubles per warp.
// Panel publication for the fused wide QR: after panel b is factored, its columns (rows
// p.., reflectors below the diagonal, R above) go to Vg (row-major, pitch ldv), then
// flags[b] is raised (release) for the CTAs applying the panels to the other columns.
struct HhPub {
  double* Vg;
  int ldv;
  int* flags;
};

__device__ __forceinline__ void hh_publish(const HhPub* pub, const double* A, int ld, int mr, int p, int nb, int b) {
  if (!pub) return;
  const int lane = threadIdx.x & 31;
  for (int t = lane; t < (mr - p) * kHhNB; t += 32) {
    const int r = p + t / kHhNB, c = t % kHhNB;
    if (c < nb) pub->Vg[static_cast<int64_t>(r) * pub->ldv + p + c] = A[r * ld + p + c];
  }
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicExch(pub->flags + b, 1);
}

template <int RW>
__device__ void hh_factor_blocked(double* A, int ld, int mr, int nc, double* tau, double* Tbuf, double* Tg,
                                  double* scratch, double* xch, const HhPub* pub) {
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  const int nwarps = blockDim.x >> 5;
  constexpr int NT = 1;  // one warp, RW rows per lane (measured: a multi-warp team paid ~2000
                         // cycles per column in the named-barrier exchange)
  const int k = min(mr, nc);
  if (warp < NT) {
    hh_panel_team<RW>(A, ld, mr, 0, min(kHhNB, k), tau, Tbuf, Tg, NT, xch, scratch);
    if (warp == 0) hh_publish(pub, A, ld, mr, 0, min(kHhNB, k), 0);
  }
  __syncthreads();
  int it = 0;
  for (int p = 0; p < k; p += kHhNB, ++it) {
    const int nb = min(kHhNB, k - p);
    const int nx = p + nb;
    const int nbx = min(kHhNB, k - nx);
    const double* T = Tbuf + (it & 1) * 64;
    double* Tn = Tbuf + ((it + 1) & 1) * 64;
    if (warp < NT) {
      if (nbx > 0) {
        if (warp == 0) hh_panel_apply(A + p, ld, T, nb, A, ld, mr, p, nx, nx + nbx, 0, 1, scratch);
        hh_team_sync(NT);
        hh_panel_team<RW>(A, ld, mr, nx, nbx, tau, Tn, Tg ? Tg + static_cast<int64_t>(it + 1) * 64 : nullptr, NT, xch,
                          scratch);
        if (warp == 0) hh_publish(pub, A, ld, mr, nx, nbx, it + 1);
      }
    } else {
      hh_panel_apply(A + p, ld, T, nb, A, ld, mr, p, nbx > 0 ? nx + nbx : nx, nc, warp - NT, nwarps - NT,
                     scratch + 64 * warp);
    }
    __syncthreads();
  }
}

// In-place QR of the smem matrix: blocked for mr <= kHhPanelRows, else unblocked.
// Tbuf: 128 doubles; Tg: optional per-panel T output (blocked path only).
__device__ void hh_factor_smem(double* A, int ld, int mr, int nc, double* tau, double* red, double* Tbuf,
                               double* Tg, double* scratch, double* xch, const HhPub* pub = nullptr) {
  // rows per lane = ceil(mr / 32) exactly: empty register rows still cost instructions
  switch ((mr + 31) / 32) {
    case 1: hh_factor_blocked<1>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 2: hh_factor_blocked<2>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 3: hh_factor_blocked<3>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 4: hh_factor_blocked<4>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 5: hh_factor_blocked<5>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 6: hh_factor_blocked<6>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 7: hh_factor_blocked<7>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    case 8: hh_factor_blocked<8>(A, ld, mr, nc, tau, Tbuf, Tg, scratch, xch, pub); break;
    default: hh_factor_unblocked(A, ld, mr, nc, tau, red); break;
  }
}

// load rows [r0, r0+mr) x cols [0, nc) of a row-major global matrix (pitch gld) into smem (pitch ld)
__device__ void hh_load(double* A, int ld, const double* G, int64_t gld, int r0, int mr, int nc) {
  for (int t = threadIdx.x; t < mr * nc; t += blockDim.x) {
    const int r = t / nc, c = t - r * nc;
    A[r * ld + c] = G[(static_cast<int64_t>(r0) + r) * gld + c];
  }
}

// write the upper part as R (row pitch nc, `rows_out` rows, zero below row min(mr, nc));
// sign-normalise rows if `sign`
__device__ void hh_store_r(const double* A, int ld, int mr, int nc, double* R, bool sign, int rows_out) {
  const int k = min(mr, nc);
  for (int t = threadIdx.x; t < rows_out * nc; t += blockDim.x) {
    const int r = t / nc, c = t - r * nc;
    if (r >= k) {
      R[static_cast<int64_t>(r) * nc + c] = 0.0;
      continue;
    }
    double v = c >= r ? A[r * ld + c] : 0.0;
    if (sign && A[r * ld + r] < 0.0) v = -v;
    R[static_cast<int64_t>(r) * nc + c] = v;
  }
}

// one CTA: QR of rows [r0, r0+mr) of G (or of two stacked R blocks when G2 != nullptr)
__global__ void __launch_bounds__(kHhThreads, 1) hh_block_kernel(const double* __restrict__ G, int64_t gld, int mr, int nc,
                                                              const double* __restrict__ G2, int mr2,
                                                              double* __restrict__ R, int64_t rstride, int sign) {
  extern __shared__ __align__(16) double A[];
  __shared__ double red[32];
  __shared__ double tau[512];
  __shared__ double Tbuf[128];
  __shared__ double scratch[64 * (kHhThreads / 32)];
  __shared__ double xch[2 * 5 * kHhNB];
  const int ld = nc + 1;
  const int b = blockIdx.x;
  int m_all;
  if (G2 == nullptr) {
    // chunk b of a tall matrix: rows [b*mr, min((b+1)*mr, total)) -- total passed through mr2
    const int total = mr2;
    const int r0 = b * mr, rows = min(mr, total - r0);
    hh_load(A, ld, G, gld, r0, rows, nc);
    m_all = rows;
  } else {
    // stack pair b: blocks 2b and 2b+1 of k x nc R factors (the last may be absent)
    const int k = min(mr, nc);
    const double* Ra = G + static_cast<int64_t>(2 * b) * rstride;
    hh_load(A, ld, Ra, nc, 0, k, nc);
    m_all = k;
    if (2 * b + 1 < mr2) {
      hh_load(A + k * ld, ld, Ra + rstride, nc, 0, k, nc);
      m_all = 2 * k;
    }
  }
  __syncthreads();
  hh_factor_smem(A, ld, m_all, nc, tau, red, Tbuf, nullptr, scratch, xch);
  // intermediate TSQR factors are zero-padded to nc rows so they stack uniformly
  const int rows_out = sign ? min(m_all, nc) : nc;
  hh_store_r(A, ld, m_all, nc, R + static_cast<int64_t>(b) * rstride, sign != 0, rows_out);
}

// Wide QR (I < nc) in one launch.  The first CTA to arrive factors the left I x I block (blocked, I <=
// kHhPanelRows) and publishes every panel (V columns to Vg, T to Tg, then flags[b]);
// the later ones each own a chunk of cw of the remaining columns and apply the panels in
// order as they appear (compact WY: W = V^T A, W' = T^T W, A -= V W' on DMMA), so the
// application runs behind the factorisation instead of after it.  R gets the rows
// sign-normalised by diag(R_left).  flags[0..panels] (panel flags + the role ticket) must be zero at launch.
__global__ void __launch_bounds__(kHhThreads, 1) hh_wide_kernel(const double* __restrict__ G, int I, int nc,
                                                             double* __restrict__ R, double* __restrict__ Vg,
                                                             double* __restrict__ Tg, int* __restrict__ flags,
                                                             int cw) {
  extern __shared__ __align__(16) double A[];
  __shared__ double red[32];
  __shared__ double tau[512];
  __shared__ double Tbuf[128];
  __shared__ double scratch[64 * (kHhThreads / 32)];
  __shared__ double xch[2 * 5 * kHhNB];
  const int tid = threadIdx.x;
  // roles by arrival (atomic ticket), not by blockIdx: the CTA that factors the left block is one that
  // is already running, so the spinning appliers can never wait on a CTA that has not been scheduled
  __shared__ int role;
  const int panels = (I + kHhNB - 1) / kHhNB;
  if (tid == 0) role = atomicAdd(flags + panels, 1);
  __syncthreads();
  if (role == 0) {
    const int ld = I + 1;
    for (int t = tid; t < I * I; t += blockDim.x) {
      const int r = t / I, c = t - r * I;
      A[r * ld + c] = G[static_cast<int64_t>(r) * nc + c];
    }
    __syncthreads();
    const HhPub pub{Vg, I, flags};
    hh_factor_smem(A, ld, I, I, tau, red, Tbuf, Tg, scratch, xch, &pub);
    __syncthreads();
    for (int t = tid; t < I * I; t += blockDim.x) {
      const int r = t / I, c = t - r * I;
      const double v = A[r * ld + c];
      const double sgn = A[r * ld + r] < 0.0 ? -1.0 : 1.0;
      R[static_cast<int64_t>(r) * nc + c] = c >= r ? sgn * v : 0.0;
    }
    return;
  }
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int c0 = I + (role - 1) * cw;
  const int w = min(cw, nc - c0);
  const int ld = cw + 1;
  double* buf = A + static_cast<int64_t>(I) * ld;  // V [I][8] + T [64] of the current panel
  for (int t = tid; t < I * w; t += blockDim.x) {
    const int r = t / w, c = t - r * w;
    A[r * ld + c] = G[static_cast<int64_t>(r) * nc + c0 + c];
  }
  for (int b = 0; b < panels; ++b) {
    if (tid == 0) {
      volatile int* f = flags + b;
      while (*f == 0) __nanosleep(100);
      __threadfence();
    }
    __syncthreads();
    const int p = b * kHhNB, nb = min(kHhNB, I - p);
    for (int t = tid; t < (I - p) * kHhNB; t += blockDim.x) {
      const int r = p + t / kHhNB, c = t % kHhNB;
      buf[r * kHhNB + c] = c < nb ? __ldcg(Vg + static_cast<int64_t>(r) * I + p + c) : 0.0;
    }
    for (int t = tid; t < 64; t += blockDim.x) buf[I * kHhNB + t] = __ldcg(Tg + static_cast<int64_t>(b) * 64 + t);
    __syncthreads();
    hh_panel_apply(buf, kHhNB, buf + I * kHhNB, nb, A, ld, I, p, 0, w, warp, blockDim.x >> 5, scratch + 64 * warp);
    __syncthreads();
  }
  for (int t = tid; t < I * w; t += blockDim.x) {
    const int r = t / w, c = t - r * w;
    const double sgn = __ldcg(Vg + static_cast<int64_t>(r) * I + r) < 0.0 ? -1.0 : 1.0;
    R[static_cast<int64_t>(r) * nc + c0 + c] = sgn * A[r * ld + c];
  }
}

struct HhPlan {
  int kind;     // 0 resident, 1 tsqr, 2 wide
  int chunk;    // tsqr rows per leaf / wide column chunk
  int leaves;
  int64_t ws;   // doubles
};

HhPlan hh_plan(int I, int nc) {
  HhPlan p{};
  const size_t whole = sizeof(double) * static_cast<size_t>(I) * (nc + 1);
  if (whole <= kHhSmemMax && I <= kHhPanelRows) {
    p.kind = 0;
    return p;
  }
  if (I > nc) {
    // rows per leaf: a leaf and a stacked pair (2 nc rows) both fit; the register-panel
    // (blocked) factorisation when both are <= kHhPanelRows rows
    int chunk = static_cast<int>(kHhSmemMax / (sizeof(double) * (nc + 1)));
    chunk = std::min(chunk, 2 * nc <= kHhPanelRows ? kHhPanelRows : 4096);
    p.kind = 1;
    p.chunk = chunk;
    p.leaves = (I + chunk - 1) / chunk;
    p.ws = 2 * static_cast<int64_t>(p.leaves) * nc * nc;  // ping-pong R stacks
    return p;
  }
  p.kind = 2;
  // column chunk: A [I][cw + 1] + the staged panel (V [I][8] + T [64])
  int cw = static_cast<int>((kHhSmemMax / sizeof(double) - (static_cast<size_t>(I) * kHhNB + 64)) / I) - 1;
  // narrow chunks: an apply CTA's time is the per-panel latency chain, not its columns,
  // so more CTAs finish sooner (one 8-column group per warp)
  cw = std::max(8, std::min(cw, 8 * (kHhThreads / 32)));
  p.chunk = cw;
  p.ws = static_cast<int64_t>(I) * I + 65 * ((I + kHhNB - 1) / kHhNB);  // Vg, T per panel, flags
  return p;
}

bool hh_supported(int I, int nc) {
  if (I > nc) return 2 * static_cast<size_t>(nc) * (nc + 1) * sizeof(double) <= kHhSmemMax && nc <= 512;
  return static_cast<size_t>(I) * (I + 1) * sizeof(double) <= kHhSmemMax && I <= kHhPanelRows;
}

int hh_qr(const double* G, int I, int nc, double* R, double* ws, int64_t ws_elems, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hh_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHhSmemMax);
    cudaFuncSetAttribute(hh_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kHhSmemMax);
    attr = true;
  }
  if (!hh_supported(I, nc)) return TRALS_ERR_UNSUPPORTED;
  const HhPlan p = hh_plan(I, nc);
  if (ws_elems < p.ws) return TRALS_ERR_WORKSPACE;
  if (p.kind == 0) {
    const size_t smem = sizeof(double) * static_cast<size_t>(I) * (nc + 1);
    hh_block_kernel<<<1, kHhThreads, smem, s>>>(G, nc, I, nc, nullptr, I, R, 0, 1);
    return launch_status();
  }
  if (p.kind == 1) {
    // leaves -> k x nc factors (k = nc), then pairwise stacking up the tree
    const int64_t rs = static_cast<int64_t>(nc) * nc;
    double* cur = ws;
    double* nxt = ws + static_cast<int64_t>(p.leaves) * rs;
    {
      const size_t smem = sizeof(double) * static_cast<size_t>(p.chunk) * (nc + 1);
      hh_block_kernel<<<p.leaves, kHhThreads, smem, s>>>(G, nc, p.chunk, nc, nullptr, I, p.leaves == 1 ? R : cur, rs,
                                                        p.leaves == 1 ? 1 : 0);
      if (int st = launch_status()) return st;
    }
    int n = p.leaves;
    while (n > 1) {
      const int pairs = (n + 1) / 2;
      const size_t smem = sizeof(double) * static_cast<size_t>(2 * nc) * (nc + 1);
      const bool last = (pairs == 1);
      hh_block_kernel<<<pairs, kHhThreads, smem, s>>>(cur, nc, nc, nc, cur, n, last ? R : nxt, rs, last ? 1 : 0);
      if (int st = launch_status()) return st;
      std::swap(cur, nxt);
      n = pairs;
    }
    return TRALS_OK;
  }
  // wide: one launch, CTA 0 factors the left block, CTAs 1.. apply its panels as they appear
  double* Vg = ws;
  double* Tg = ws + static_cast<int64_t>(I) * I;
  const int panels = (I + kHhNB - 1) / kHhNB;
  int* flags = reinterpret_cast<int*>(Tg + 64 * static_cast<int64_t>(panels));
  if (cudaMemsetAsync(flags, 0, sizeof(int) * (panels + 1), s) != cudaSuccess) return TRALS_ERR_CUDA;  // + ticket
  const int rest = nc - I;
  const int blocks = 1 + (rest > 0 ? (rest + p.chunk - 1) / p.chunk : 0);
  const size_t smem_left = sizeof(double) * static_cast<size_t>(I) * (I + 1);
  const size_t smem_apply = sizeof(double) * (static_cast<size_t>(I) * (p.chunk + 1) + static_cast<size_t>(I) * kHhNB + 64);
  hh_wide_kernel<<<blocks, kHhThreads, std::max(smem_left, smem_apply), s>>>(G, I, nc, R, Vg, Tg, flags, p.chunk);
  return launch_status();
}

// C(m, n) = F[m * ncols + n] scattered through a CMap
// Axis reversal of a dense N-d tensor: src first-index-fastest (Fortran, the .dten
// payload order, io.py:10-11) -> dst last-index-fastest (C, the engine's X).  The
// first and last axes are swapped through 32 x 32 shared-memory tiles (reads run
// along axis 0 of src, writes along axis N-1 of dst, both coalesced); the middle
// axes are reversed by index arithmetic, one tile column per middle index.
constexpr int kRevMaxN = 16;
struct RevDims {
  int N;
  int64_t d[kRevMaxN];
};

__global__ void __launch_bounds__(256) reverse_axes_kernel(const double* __restrict__ src, RevDims rd,
                                                           double* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int N = rd.N;
  const int64_t da = rd.d[0], dz = rd.d[N - 1];
  int64_t mid = 1;
  for (int j = 1; j < N - 1; ++j) mid *= rd.d[j];
  const int64_t ta = (da + 31) / 32, tz = (dz + 31) / 32, tiles = ta * tz * mid;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t q = t / (ta * tz), rem = t - q * (ta * tz);
    const int64_t a0 = (rem % ta) * 32, z0 = (rem / ta) * 32;
    // middle multi-index q = i_1 + d_1 (i_2 + ...) -> offsets in both layouts:
    // src (F) = sum_j i_j prod_{k<j} d_k, dst (C) = sum_j i_j prod_{k>j} d_k
    int64_t idx[kRevMaxN];
    int64_t soff = 0, sZ = da, qq = q;
    for (int j = 1; j < N - 1; ++j) {
      idx[j] = qq % rd.d[j];
      qq /= rd.d[j];
      soff += idx[j] * sZ;
      sZ *= rd.d[j];
    }
    int64_t doff = 0, dA = dz;
    for (int j = N - 2; j >= 1; --j) {
      doff += idx[j] * dA;
      dA *= rd.d[j];
    }
    // sZ = src stride of axis N-1, dA = dst stride of axis 0
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t a = a0 + tx, z = z0 + ty + j;
      tile[ty + j][tx] = (a < da && z < dz) ? src[soff + a + z * sZ] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      const int64_t z = z0 + tx, a = a0 + ty + j;
      if (a < da && z < dz) dst[doff + a * dA + z] = tile[tx][ty + j];
    }
    __syncthreads();
  }
}

__global__ void reshuffle_kernel(const double* __restrict__ F, int64_t rows, int64_t cols, CMap cm,
                                 double* __restrict__ C) {
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x)
    C[trals::cmap_addr(cm, 0, t / cols, t % cols)] = F[t];
}

// out[1] = sum of the per-CTA squared-residual partials (fixed order),
// out[0] = sqrt(out[1]) / |X| (solvers.py:164-174; zero input -> 0)
__global__ void __launch_bounds__(1024) residual_final_kernel(const double* __restrict__ part, int np,
                                                              const double* __restrict__ xnorm2,
                                                              double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += part[i];
  const double s = block_sum<1024>(acc, red);
  if (threadIdx.x == 0) {
    const double xn = sqrt(xnorm2 ? xnorm2[0] : 0.0);
    out[1] = s;
    out[0] = xn == 0.0 ? 0.0 : sqrt(s) / xn;
  }
}

// ---------------------------------------------------------------------------
// error terms: out[1] = <M,Z>, out[2] = <S, G> with G = Z^T Z (precomputed)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) error_terms_kernel(const double* __restrict__ M, const double* __restrict__ Z,
                                                           int64_t nz, const double* __restrict__ S,
                                                           const double* __restrict__ G, int64_t ns,
                                                           const double* __restrict__ xnorm2, double* __restrict__ out) {
  __shared__ double red[32];
  double a = 0.0;
  for (int64_t t = threadIdx.x; t < nz; t += blockDim.x) a = fma(M[t], Z[t], a);
  const double cross = block_sum<1024>(a, red);
  double b = 0.0;
  for (int64_t t = threadIdx.x; t < ns; t += blockDim.x) b = fma(S[t], G[t], b);
  const double model = block_sum<1024>(b, red);
  if (threadIdx.x == 0) {
    const double x2 = xnorm2[0];
    const double xn = sqrt(x2);
    double e = 0.0;
    if (xn != 0.0) {
      const double sq = xn * xn - 2.0 * cross + model;
      e = sqrt(fmax(0.0, sq)) / xn;
    }
    out[0] = e;
    out[1] = cross;
    out[2] = model;
  }
}

// ---------------------------------------------------------------------------
// composite host helpers (no allocation; stride bookkeeping only)
// ---------------------------------------------------------------------------
int half_chain(int nblk, const int64_t* dims, const int32_t* ranks, const double* first_slice,
               const double* const* cores_c, double* out, double* tmp, double* ws, int64_t ws_elems,
               cudaStream_t s, int transposed = 0) {
  // chain of cores u..u+nblk-1; dims[j], ranks[j] = left bond of core j, ranks[nblk] = right bond of last
  if (nblk < 1) return TRALS_ERR_ARG;
  const int64_t Ru = ranks[0];
  if (nblk == 1) {
    const int64_t n = dims[0] * Ru * ranks[1];
    if (transposed) {
      const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4 * kSMs));
      relayout_kernel<<<blocks, 256, 0, s>>>(first_slice, TRALS_LAYOUT_SLICE, static_cast<int>(Ru), dims[0],
                                             ranks[1], out, TRALS_LAYOUT_TT);
      return launch_status();
    }
    if (cudaMemcpyAsync(out, first_slice, n * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return TRALS_ERR_CUDA;
    return TRALS_OK;
  }
  // ping-pong so that the final product lands in `out`
  const double* cur = first_slice;
  int64_t pre = dims[0];
  for (int j = 1; j < nblk; ++j) {
    double* dst = ((nblk - 1 - j) % 2 == 0) ? out : tmp;
    const int64_t Rt = ranks[j], Ij = dims[j], Rn = ranks[j + 1];
    // A(m = (i_pre, r_u), k = t) = cur[m*Rt + t]; B[t][(i_j, r')] = core_c[j]
    // Out[i_pre][i_j][r_u][r'] : m1 = i_pre, m2 = r_u ; n1 = i_j, n2 = r'
    CMap cm{0, Ru, Ij * Ru * Rn, Rn, Rn, Ru * Rn, 1};
    if (transposed && j == nblk - 1) {
      // [r'][r_u][(i_pre, i_j)] : the K x post operand of the fused reconstruct
      const int64_t P = pre * Ij;
      cm = CMap{0, Ru, Ij, P, Rn, 1, Ru * P};
    }
    int st = gemm(cur, 0, Rt, 1, 1, pre * Ru, Rt, Ij * Rn, cores_c[j], Ij * Rn, dst, cm, 0, ws, ws_elems, s);
    if (st) return st;
    cur = dst;
    pre *= Ij;
  }
  return TRALS_OK;
}

int64_t half_chain_tmp(int nblk, const int64_t* dims, const int32_t* ranks) {
  int64_t pre = dims[0], best = 0;
  for (int j = 1; j < nblk; ++j) {
    pre *= dims[j];
    best = std::max<int64_t>(best, pre * ranks[0] * ranks[j + 1]);
  }
  return best;
}

int64_t half_chain_ws(int nblk, const int64_t* dims, const int32_t* ranks) {
  int64_t pre = dims[0], best = 0;
  for (int j = 1; j < nblk; ++j) {
    best = std::max(best, gemm_ws(1, pre * ranks[0], ranks[j], dims[j] * ranks[j + 1]));
    pre *= dims[j];
  }
  return best;
}

int env(const double* X, int64_t pre, int64_t post, int side, const double* H, int r_lo, int r_hi, double* E,
        int leaf, double* ws, int64_t ws_elems, cudaStream_t s) {
  const int64_t RR = static_cast<int64_t>(r_lo) * r_hi;
  if (side == 0) {
    // H over post modes (y..N-1): H[k][r_y][r_0], r_lo = r_y, r_hi = r_0
    // Env[r_0][m][r_y]; n = (r_y, r_0): n1 = r_y, n2 = r_0 (N2 = r_hi)
    CMap cm{0, pre, 0, r_lo, r_hi, 1, pre * r_lo};
    // single-mode segment [0]: write M_0[i_0][r_0 + R_0 r_1] (r_y = r_1)
    if (leaf) cm = CMap{0, pre, 0, RR, r_hi, r_hi, 1};
    const int st = gemm_tma(X, post, 1, pre, post, RR, H, RR, E, cm, ws, ws_elems, s);
    if (st != TRALS_ERR_UNSUPPORTED) return st;
    return gemm(X, 0, post, 1, 1, pre, post, RR, H, RR, E, cm, 0, ws, ws_elems, s);
  }
  // H over pre modes (0..x): H[k][r_0][r_{x+1}], r_lo = r_0, r_hi = r_{x+1}
  // Env[r_{x+1}][m][r_0]; n = (r_0, r_x1): n1 = r_0, n2 = r_x1
  CMap cm{0, post, 0, r_lo, r_hi, 1, post * r_lo};
  // single-mode segment [N-1]: M_{N-1}[i][r_{N-1} + R_{N-1} r_0] (r_{x+1} = r_{N-1})
  if (leaf) cm = CMap{0, post, 0, RR, r_hi, r_hi, 1};
  const int st = gemm_tma(X, 1, post, post, pre, RR, H, RR, E, cm, ws, ws_elems, s);
  if (st != TRALS_ERR_UNSUPPORTED) return st;
  return gemm(X, 0, 1, post, 1, post, pre, RR, H, RR, E, cm, 0, ws, ws_elems, s);
}


// TRALS_OZ_NOPERM=1 (experiments): keep the natural column order for the short-K env products
inline bool oz_noperm() {
  static int v = -1;
  if (v < 0) v = std::getenv("TRALS_OZ_NOPERM") ? 1 : 0;
  return v == 1;
}

// fp32 variant of env() on the int8 tensor cores: X given as digit planes + row exponents,
// K-major for this side (side 0: rows = pre, side 1: rows = post, the transposed copy).
template <class SC>
int env_oz(const int8_t* xd, const int32_t* xe, int64_t pre, int64_t post, int side, const double* H, int r_lo,
           int r_hi, double* E, int leaf, double* ws, int64_t ws_elems, cudaStream_t s) {
  const int64_t RR = static_cast<int64_t>(r_lo) * r_hi;
  if (side == 0) {
    CMap cm{0, pre, 0, r_lo, r_hi, 1, pre * r_lo};
    if (leaf) cm = CMap{0, pre, 0, RR, r_hi, r_hi, 1};
    const int plo = (!leaf && post < kOzShortK && !oz_noperm()) ? r_lo : 0;
    return gemm_oz<SC>(xd, xe, pre, post, RR, H, RR, E, cm, ws, ws_elems, s, plo, plo ? r_hi : 0);
  }
  CMap cm{0, post, 0, r_lo, r_hi, 1, post * r_lo};
  if (leaf) cm = CMap{0, post, 0, RR, r_hi, r_hi, 1};
  const int plo = (!leaf && pre < kOzShortK && !oz_noperm()) ? r_lo : 0;
  return gemm_oz<SC>(xd, xe, post, pre, RR, H, RR, E, cm, ws, ws_elems, s, plo, plo ? r_hi : 0);
}

int absorb_right(const double* E, int Ra, int64_t pre, int64_t Ib, int Rb, int Rb1, const double* core_zt,
                 double* out, int leaf, double* ws, int64_t ws_elems, cudaStream_t s) {
  const int64_t M = static_cast<int64_t>(Ra) * pre, K = Ib * Rb1;
  CMap cm = rowmajor(Rb);
  if (leaf) {
    // out = M_a[i_a][r_a + Ra r_b]: m = (r_a, i_a) -> m1 = r_a, m2 = i_a (M2 = pre)
    cm = CMap{0, pre, 1, static_cast<int64_t>(Ra) * Rb, 1 << 30, 0, Ra};
  }
  return gemm(E, 0, K, 1, 1, M, K, Rb, core_zt, Rb, out, cm, 0, ws, ws_elems, s);
}

int absorb_left(const double* E, int Ra, int64_t Ia, int64_t rest, int Ra1, int Rb1, const double* core_c,
                double* out, int leaf, double* ws, int64_t ws_elems, cudaStream_t s) {
  const int64_t M = rest * Rb1, K = static_cast<int64_t>(Ra) * Ia;
  // Out[r_{a+1}][m]: element (m, n) at n*M + m
  CMap cm{0, 1 << 30, 0, 1, 1 << 30, 0, M};
  if (leaf) {
    // out = M_b[i_b][r_b + R_b r_{b+1}] with r_b = n, (i_b, r_{b+1}) = m -> m1 = i_b, m2 = r_{b+1}
    cm = CMap{0, Rb1, static_cast<int64_t>(Ra1) * Rb1, Ra1, 1 << 30, 0, 1};
  }
  return gemm(E, 0, 1, M, 1, M, K, Ra1, core_c, Ra1, out, cm, 0, ws, ws_elems, s);
}


// ---------------------------------------------------------------------------
// stateless single-mode MTTSP plan (used by trals_mttsp_f64)
// ---------------------------------------------------------------------------
struct MttspPlan {
  int side;           // 0: half chain over suffix [y..N-1]; 1: over prefix [0..x]
  int lo, hi;         // chain block [lo..hi]
  int seg_a, seg_b;   // environment segment after the root product
  int64_t pre, post;  // X viewed as [pre][post]
  int64_t h_elems, tmp_elems, env_elems, ws_elems;
};

inline int64_t prod_dims(const int64_t* dims, int a, int b) {
  int64_t p = 1;
  for (int j = a; j <= b; ++j) p *= dims[j];
  return p;
}

MttspPlan plan_mttsp(int N, const int64_t* dims, const int32_t* ranks, int n) {
  MttspPlan best{};
  double best_cost = -1;
  const int64_t total = prod_dims(dims, 0, N - 1);
  auto consider = [&](int side, int lo, int hi) {
    const int64_t pc = prod_dims(dims, lo, hi);
    const double cost = static_cast<double>(std::max(pc, total / pc)) + 1e-9 * pc;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best.side = side; best.lo = lo; best.hi = hi;
    }
  };
  for (int y = n + 1; y <= N - 1; ++y) consider(0, y, N - 1);
  for (int x = 0; x <= n - 1; ++x) consider(1, 0, x);
  MttspPlan& p = best;
  if (p.side == 0) { p.seg_a = 0; p.seg_b = p.lo - 1; p.pre = prod_dims(dims, 0, p.lo - 1); p.post = prod_dims(dims, p.lo, N - 1); }
  else { p.seg_a = p.hi + 1; p.seg_b = N - 1; p.pre = prod_dims(dims, 0, p.hi); p.post = prod_dims(dims, p.hi + 1, N - 1); }
  const int nblk = p.hi - p.lo + 1;
  std::vector<int64_t> bd(dims + p.lo, dims + p.hi + 1);
  std::vector<int32_t> br;
  for (int j = p.lo; j <= p.hi + 1; ++j) br.push_back(ranks[j % N]);
  const int64_t r_lo = br.front(), r_hi = br.back();
  p.h_elems = prod_dims(dims, p.lo, p.hi) * r_lo * r_hi;
  p.tmp_elems = half_chain_tmp(nblk, bd.data(), br.data());
  int64_t ws = half_chain_ws(nblk, bd.data(), br.data());
  const int64_t seg_len = p.side == 0 ? p.pre : p.post;
  const int64_t RR = r_lo * r_hi;
  p.env_elems = seg_len * RR;
  const bool root_leaf = (p.seg_a == p.seg_b);
  ws = std::max(ws, p.side == 0 ? gemm_ws(1, p.pre, p.post, RR) : gemm_ws(1, p.post, p.pre, RR));
  (void)root_leaf;
  // walk the absorptions to size the gemm workspace
  int a = p.seg_a, b = p.seg_b;
  int64_t seg = seg_len;
  while (b > n) {
    const int64_t Ra = ranks[a], Rb = ranks[b], Rb1 = ranks[(b + 1) % N];
    ws = std::max(ws, gemm_ws(1, Ra * (seg / dims[b]), dims[b] * Rb1, Rb));
    seg /= dims[b];
    --b;
  }
  while (a < n) {
    const int64_t Ra = ranks[a], Ra1 = ranks[a + 1], Rb1 = ranks[(b + 1) % N];
    ws = std::max(ws, gemm_ws(1, (seg / dims[a]) * Rb1, Ra * dims[a], Ra1));
    seg /= dims[a];
    ++a;
  }
  p.ws_elems = ws;
  return p;
}

int64_t mttsp_total_ws(const MttspPlan& p) {
  // [H][tmp][env0][env1][gemm ws]
  return p.h_elems + p.tmp_elems + 2 * p.env_elems + p.ws_elems + 64;
}

int run_mttsp(const double* X, int N, const int64_t* dims, const int32_t* ranks, int n,
              const double* const* cc, const double* const* cs, const double* const* czt, double* M, double* ws,
              int64_t ws_elems, cudaStream_t s) {
  const MttspPlan p = plan_mttsp(N, dims, ranks, n);
  if (ws_elems < mttsp_total_ws(p)) return TRALS_ERR_WORKSPACE;
  auto al = [](int64_t v) { return (v + 7) & ~int64_t(7); };
  double* H = ws;
  double* tmp = H + al(p.h_elems);
  double* env0 = tmp + al(p.tmp_elems);
  double* env1 = env0 + al(p.env_elems);
  double* gws = env1 + al(p.env_elems);
  const int64_t gws_elems = ws_elems - (gws - ws);
  const int nblk = p.hi - p.lo + 1;
  std::vector<int64_t> bd(dims + p.lo, dims + p.hi + 1);
  std::vector<int32_t> br;
  for (int j = p.lo; j <= p.hi + 1; ++j) br.push_back(ranks[j % N]);
  std::vector<const double*> bc(cc + p.lo, cc + p.hi + 1);
  int st = half_chain(nblk, bd.data(), br.data(), cs[p.lo], bc.data(), H, tmp, gws, gws_elems, s);
  if (st) return st;
  const bool root_leaf = (p.seg_a == p.seg_b);
  st = env(X, p.pre, p.post, p.side, H, br.front(), br.back(), root_leaf ? M : env0, root_leaf, gws, gws_elems, s);
  if (st || root_leaf) return st;
  int a = p.seg_a, b = p.seg_b;
  int64_t seg = p.side == 0 ? p.pre : p.post;
  const double* cur = env0;
  double* nxt = env1;
  while (b > n) {
    const bool leaf = (a == n && b == n + 1);
    st = absorb_right(cur, ranks[a], seg / dims[b], dims[b], ranks[b], ranks[(b + 1) % N], czt[b],
                      leaf ? M : nxt, leaf, gws, gws_elems, s);
    if (st) return st;
    seg /= dims[b];
    --b;
    std::swap(const_cast<double*&>(cur), nxt);
    if (leaf) return TRALS_OK;
  }
  while (a < n) {
    const bool leaf = (a + 1 == n && b == n);
    st = absorb_left(cur, ranks[a], dims[a], seg / dims[a], ranks[a + 1], ranks[(b + 1) % N], cc[a],
                     leaf ? M : nxt, leaf, gws, gws_elems, s);
    if (st) return st;
    seg /= dims[a];
    ++a;
    std::swap(const_cast<double*&>(cur), nxt);
    if (leaf) return TRALS_OK;
  }
  return TRALS_ERR_ARG;  // unreachable for valid plans
}

// One step of iterative refinement of Z S = M for the explicit-inverse operands of the m <= 112
// factor (F = U^{-1}, aux = U^{-T}): R = M - Z S, Z += (R F) aux, one CTA per right-hand-side row,
// fixed summation order.  Runs only when the factorisation raised d_info[TRALS_INFO_REFINE]
// (max|U| / min diag(U) > 1e4, i.e. cond(S) beyond ~1e8 -- BASELINE c4's over-specified ranks);
// otherwise it returns at once, so it sits in the sweep graph unconditionally.
__global__ void __launch_bounds__(128) refine_kernel(const double* __restrict__ F, const double* __restrict__ aux,
                                                     const double* __restrict__ S, int m,
                                                     const double* __restrict__ Mr, int64_t rows,
                                                     double* __restrict__ Z, const int* __restrict__ info) {
  if (info[TRALS_INFO_REFINE] == 0) return;
  __shared__ double z[128], r[128], t[128];
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    for (int c = threadIdx.x; c < m; c += blockDim.x) z[c] = Z[row * m + c];
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      double acc = Mr[row * m + c];
      for (int k = 0; k < m; ++k) acc = fma(-z[k], S[k * m + c], acc);
      r[c] = acc;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc = fma(r[k], F[k * m + c], acc);
      t[c] = acc;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc = fma(t[k], aux[k * m + c], acc);
      Z[row * m + c] = z[c] + acc;
    }
    __syncthreads();
  }
}

}  // namespace

#include "dd_r0.cuh"
#include "qr_r0.cuh"

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* trals_strerror(int code) {
  switch (code) {
    case TRALS_OK: return "ok";
    case TRALS_ERR_ARG: return "invalid argument";
    case TRALS_ERR_CUDA: return "CUDA launch failure";
    case TRALS_ERR_WORKSPACE: return "workspace too small";
    case TRALS_ERR_UNSUPPORTED: return "size outside the supported envelope";
  }
  return "unknown error";
}

int trals_version(void) { return 1; }

long long trals_launch_count(void) { return g_launches; }

int64_t trals_gemm_ws_elems(int64_t P, int64_t M, int64_t K, int64_t N) {
  // P == 1 shapes may take the TMA kernel (environment products): size for either plan
  return P == 1 ? std::max(gemm_ws(P, M, K, N), gemm_tma_ws(M, K, N)) : gemm_ws(P, M, K, N);
}

int trals_gemm_f64(const double* A, int64_t sAp, int64_t sAm, int64_t sAk, int64_t P, int64_t M, int64_t K,
                   int64_t N, const double* B, int64_t ldb, double* C, const int64_t* h_cmap, int beta,
                   double* ws, int64_t ws_elems, void* stream) {
  if (!h_cmap) return TRALS_ERR_ARG;
  CMap cm{h_cmap[0], h_cmap[1], h_cmap[2], h_cmap[3], h_cmap[4], h_cmap[5], h_cmap[6]};
  return gemm(A, sAp, sAm, sAk, P, M, K, N, B, ldb, C, cm, beta, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

int trals_reverse_axes_f64(const double* src, int N, const int64_t* dims, double* dst, void* stream) {
  if (!src || !dst || !dims || N < 1 || N > kRevMaxN || src == dst) return TRALS_ERR_ARG;
  RevDims rd{};
  rd.N = N;
  int64_t total = 1;
  for (int j = 0; j < N; ++j) {
    if (dims[j] < 1) return TRALS_ERR_ARG;
    rd.d[j] = dims[j];
    total *= dims[j];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (N == 1) {
    if (cudaMemcpyAsync(dst, src, total * sizeof(double), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return TRALS_ERR_CUDA;
    return TRALS_OK;
  }
  const int64_t tiles = ((dims[0] + 31) / 32) * ((dims[N - 1] + 31) / 32) * (total / (dims[0] * dims[N - 1]));
  const int blocks = static_cast<int>(std::min<int64_t>(tiles, 32 * kSMs));
  reverse_axes_kernel<<<blocks, 256, 0, s>>>(src, rd, dst);
  return launch_status();
}

int trals_core_relayout_f64(const double* src, int sl, int Ra, int64_t I, int Rb, double* dst, int dl,
                            void* stream) {
  if (!src || !dst || Ra < 1 || Rb < 1 || I < 1 || sl < 0 || sl > 3 || dl < 0 || dl > 3) return TRALS_ERR_ARG;
  const int64_t total = static_cast<int64_t>(Ra) * I * Rb;
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<int64_t>((total + threads - 1) / threads, 4 * kSMs));
  relayout_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(src, sl, Ra, I, Rb, dst, dl);
  return launch_status();
}

int64_t trals_half_chain_tmp_elems(int nblk, const int64_t* dims, const int32_t* ranks) {
  return half_chain_tmp(nblk, dims, ranks);
}

int trals_half_chain_f64(int nblk, const int64_t* dims, const int32_t* ranks, const double* first_slice,
                         const double* const* cores_c, double* out, double* tmp, double* ws, int64_t ws_elems,
                         int transposed, void* stream) {
  if (!dims || !ranks || !first_slice || !out) return TRALS_ERR_ARG;
  if (nblk > 1 && (!cores_c || !tmp)) return TRALS_ERR_ARG;
  return half_chain(nblk, dims, ranks, first_slice, cores_c, out, tmp, ws, ws_elems,
                    static_cast<cudaStream_t>(stream), transposed);
}

int trals_env_f64(const double* X, int64_t pre, int64_t post, int side, const double* H, int r_lo, int r_hi,
                  double* E, int leaf, double* ws, int64_t ws_elems, void* stream) {
  if (!X || !H || !E || pre < 1 || post < 1 || r_lo < 1 || r_hi < 1 || (side != 0 && side != 1))
    return TRALS_ERR_ARG;
  return env(X, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

int64_t trals_oz_digits_bytes(int64_t rows, int64_t k) {
  return rows < 1 || k < 1 ? 0 : oz_digits_bytes(oz_a_tiles(rows), k, trals::OzF32::D, trals::OzF32::BK);
}

int64_t trals_oz_split_ws_elems(int64_t rows, int64_t cols, int transpose) { return transpose ? cols : rows; }

int trals_oz_split_f32(const float* x, int64_t rows, int64_t cols, int transpose, int8_t* digits, int32_t* exps,
                       double* ws, int64_t ws_elems, void* stream) {
  return oz_split<float, trals::OzF32>(x, rows, cols, transpose, digits, exps, ws, ws_elems,
                                       static_cast<cudaStream_t>(stream));
}

int64_t trals_env_oz_ws_elems(int64_t pre, int64_t post, int side, int r_lo, int r_hi) {
  const int64_t RR = static_cast<int64_t>(r_lo) * r_hi;
  return side == 0 ? gemm_oz_ws<trals::OzF32>(pre, post, RR) : gemm_oz_ws<trals::OzF32>(post, pre, RR);
}

int trals_env_oz(const int8_t* xd, const int32_t* xe, int64_t pre, int64_t post, int side, const double* H, int r_lo,
                 int r_hi, double* E, int leaf, double* ws, int64_t ws_elems, void* stream) {
  if (!xd || !xe || !H || !E || !ws || pre < 1 || post < 1 || r_lo < 1 || r_hi < 1 || (side != 0 && side != 1))
    return TRALS_ERR_ARG;
  return env_oz<trals::OzF32>(xd, xe, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems,
                              static_cast<cudaStream_t>(stream));
}

int64_t trals_oz64_digits_bytes(int64_t rows, int64_t k) {
  return rows < 1 || k < 1 ? 0 : oz_digits_bytes(oz_a_tiles(rows), k, trals::OzF64::D, trals::OzF64::BK);
}

int trals_oz64_split_f64(const double* x, int64_t rows, int64_t cols, int transpose, int8_t* digits, int32_t* exps,
                         double* ws, int64_t ws_elems, void* stream) {
  return oz_split<double, trals::OzF64>(x, rows, cols, transpose, digits, exps, ws, ws_elems,
                                        static_cast<cudaStream_t>(stream));
}

int64_t trals_env_oz64_ws_elems(int64_t pre, int64_t post, int side, int r_lo, int r_hi) {
  const int64_t RR = static_cast<int64_t>(r_lo) * r_hi;
  return side == 0 ? gemm_oz_ws<trals::OzF64>(pre, post, RR) : gemm_oz_ws<trals::OzF64>(post, pre, RR);
}

int trals_env_oz64(const int8_t* xd, const int32_t* xe, int64_t pre, int64_t post, int side, const double* H,
                   int r_lo, int r_hi, double* E, int leaf, double* ws, int64_t ws_elems, void* stream) {
  if (!xd || !xe || !H || !E || !ws || pre < 1 || post < 1 || r_lo < 1 || r_hi < 1 || (side != 0 && side != 1))
    return TRALS_ERR_ARG;
  return env_oz<trals::OzF64>(xd, xe, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems,
                              static_cast<cudaStream_t>(stream));
}


int trals_crt_supported(int64_t rows, int64_t k, int64_t n) {
  return crt_host().ok && crt_shape_ok(rows, k, n) ? 1 : 0;
}

int trals_crt_moduli(void) { return crt_host().ok ? crt_host().t.nm : 0; }

int trals_crt_row_bits(int operand) {
  if (!crt_host().ok) return 0;
  return operand == 0 ? crt_host().t.ga : crt_host().t.gb;
}

int64_t trals_crt_planes_bytes(int64_t rows, int64_t k) {
  if (rows < 1 || k < 1 || !crt_host().ok) return 0;
  return static_cast<int64_t>(crt_host().t.nm) * crt_plane_bytes(crt_a_rows_pad(rows), k);
}

int64_t trals_crt_split_ws_elems(int64_t rows, int64_t cols, int transpose) {
  return rows < 1 || cols < 1 ? 0 : crt_split_ws(rows, cols, transpose);
}

int trals_crt_split_f64(const double* x, int64_t rows, int64_t cols, int transpose, int8_t* planes, int32_t* exps,
                        double* ws, int64_t ws_elems, void* stream) {
  return crt_split(x, rows, cols, transpose, planes, exps, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

int64_t trals_env_crt_ws_elems(int64_t pre, int64_t post, int side, int r_lo, int r_hi) {
  const int64_t RR = static_cast<int64_t>(r_lo) * r_hi;
  const int64_t rows = side == 0 ? pre : post, K = side == 0 ? post : pre;
  if (!crt_host().ok || !crt_shape_ok(rows, K, RR)) return 0;
  return crt_ws_layout(rows, K, RR).total;
}

int trals_env_crt(const int8_t* xd, const int32_t* xe, int64_t pre, int64_t post, int side, const double* H,
                  int r_lo, int r_hi, double* E, int leaf, double* ws, int64_t ws_elems, void* stream) {
  if (!xd || !xe || !H || !E || !ws || pre < 1 || post < 1 || r_lo < 1 || r_hi < 1 || (side != 0 && side != 1))
    return TRALS_ERR_ARG;
  return env_crt(xd, xe, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems, 7, static_cast<cudaStream_t>(stream));
}

int trals_env_crt_stage(const int8_t* xd, const int32_t* xe, int64_t pre, int64_t post, int side, const double* H,
                        int r_lo, int r_hi, double* E, int leaf, double* ws, int64_t ws_elems, int stages,
                        void* stream) {
  if (!xd || !xe || !H || !E || !ws || pre < 1 || post < 1 || r_lo < 1 || r_hi < 1 || (side != 0 && side != 1) ||
      stages < 1 || stages > 7)
    return TRALS_ERR_ARG;
  return env_crt(xd, xe, pre, post, side, H, r_lo, r_hi, E, leaf, ws, ws_elems, stages,
                 static_cast<cudaStream_t>(stream));
}

int trals_absorb_right_f64(const double* E, int Ra, int64_t pre, int64_t Ib, int Rb, int Rb1, const double* core_zt,
                           double* out, int leaf, double* ws, int64_t ws_elems, void* stream) {
  if (!E || !core_zt || !out || Ra < 1 || pre < 1 || Ib < 1 || Rb < 1 || Rb1 < 1) return TRALS_ERR_ARG;
  return absorb_right(E, Ra, pre, Ib, Rb, Rb1, core_zt, out, leaf, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

int trals_absorb_left_f64(const double* E, int Ra, int64_t Ia, int64_t rest, int Ra1, int Rb1, const double* core_c,
                          double* out, int leaf, double* ws, int64_t ws_elems, void* stream) {
  if (!E || !core_c || !out || Ra < 1 || Ia < 1 || rest < 1 || Ra1 < 1 || Rb1 < 1) return TRALS_ERR_ARG;
  return absorb_left(E, Ra, Ia, rest, Ra1, Rb1, core_c, out, leaf, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

int trals_core_gram_f64(const double* Gs, int Ra, int64_t I, int Rb, double* E, double* ws, int64_t ws_elems,
                        void* stream) {
  if (!Gs || !E || Ra < 1 || Rb < 1 || I < 1) return TRALS_ERR_ARG;
  const int64_t RR = static_cast<int64_t>(Ra) * Rb;
  // C'[(a,b)][(c,d)] = sum_i Gs[i][a][b] Gs[i][c][d]; E[(a,c)][(b,d)] at (a*Ra + c)*Rb^2 + b*Rb + d
  CMap cm{0, Rb, static_cast<int64_t>(Ra) * Rb * Rb, Rb, Rb, static_cast<int64_t>(Rb) * Rb, 1};
  return gemm(Gs, 0, 1, RR, 1, RR, I, RR, Gs, RR, E, cm, 0, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

// part: 0 = the whole chain; 1 = every product but the last (the prefix stays in tmp); 2 = the last
// product from the prefix of an earlier part-1 call with the same arguments.  The last factor is the
// transfer matrix of core n-1 -- the core solved just before block n -- so the prefix can be formed
// while that core is still being solved.
static int gram_chain_part(int N, int n, const int32_t* ranks, const double* const* E, double* S, double* tmp,
                           double* ws, int64_t ws_elems, int part, cudaStream_t s) {
  // ring order n+1, ..., N-1, 0, ..., n-1 ; F = E_{n+1} E_{n+2} ... E_{n-1}
  std::vector<int> order;
  for (int j = n + 1; j < N; ++j) order.push_back(j);
  for (int j = 0; j < n; ++j) order.push_back(j);
  const int64_t Rn = ranks[n], Rn1 = ranks[(n + 1) % N];
  const int64_t RR = Rn * Rn1;
  // final scatter into S[(r_n + Rn r_{n+1})][(r'_n + Rn r'_{n+1})] from F[(r_{n+1}, r'_{n+1})][(r_n, r'_n)]
  const CMap to_s{0, Rn1, Rn * RR, Rn, Rn, RR, 1};
  const int64_t rows = Rn1 * Rn1;  // F rows
  if (order.size() == 1) {
    // N == 2: S is a reshuffle of the single transfer matrix
    if (part == 1) return TRALS_OK;
    const int64_t total = RR * RR;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4 * kSMs));
    reshuffle_kernel<<<blocks, 256, 0, s>>>(E[order[0]], rows, Rn * Rn, to_s, S);
    return launch_status();
  }
  // intermediate products: sized for the largest one, alternating halves of tmp
  int64_t maxc = 0;
  for (int j : order) maxc = std::max<int64_t>(maxc, static_cast<int64_t>(ranks[(j + 1) % N]) * ranks[(j + 1) % N]);
  double* bufs[2] = {tmp, tmp + rows * maxc};
  const double* cur = E[order[0]];
  int64_t cols = static_cast<int64_t>(ranks[(order[0] + 1) % N]) * ranks[(order[0] + 1) % N];
  for (size_t t = 1; t < order.size(); ++t) {
    const int j = order[t];
    const int64_t Rj1 = ranks[(j + 1) % N];
    const int64_t ncols = Rj1 * Rj1;
    const bool last = (t + 1 == order.size());
    double* dst = last ? S : bufs[t & 1];
    const CMap cm = last ? to_s : rowmajor(ncols);
    const bool run = part == 0 || (part == 1 && !last) || (part == 2 && last);
    if (run) {
      int st = gemm(cur, 0, cols, 1, 1, rows, cols, ncols, E[j], ncols, dst, cm, 0, ws, ws_elems, s);
      if (st) return st;
    }
    cur = dst;
    cols = ncols;
  }
  return TRALS_OK;
}

int trals_gram_chain_f64(int N, int n, const int32_t* ranks, const double* const* E, double* S, double* tmp,
                         double* ws, int64_t ws_elems, void* stream) {
  if (N < 2 || n < 0 || n >= N || !ranks || !E || !S) return TRALS_ERR_ARG;
  return gram_chain_part(N, n, ranks, E, S, tmp, ws, ws_elems, 0, static_cast<cudaStream_t>(stream));
}

int trals_gram_chain_part_f64(int N, int n, const int32_t* ranks, const double* const* E, double* S, double* tmp,
                              double* ws, int64_t ws_elems, int part, void* stream) {
  if (N < 2 || n < 0 || n >= N || !ranks || !E || !S || part < 0 || part > 2) return TRALS_ERR_ARG;
  return gram_chain_part(N, n, ranks, E, S, tmp, ws, ws_elems, part, static_cast<cudaStream_t>(stream));
}

int64_t trals_cholesky_aux_elems(int m) {
  if (m <= kInvMax) return static_cast<int64_t>(m) * m;                        // V = U^{-T}
  return blocked_aux_elems(m) + 4 * static_cast<int64_t>(m) * m;             // block inverses + split-K
}

int trals_cholesky_f64(const double* S, int m, double* U, double* F, double* aux, int check_degen, int* info,
                       void* stream) {
  if (!S || !U || !F || !aux || !info || m < 1) return TRALS_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (m > kInvMax) {
    double* gws = aux + blocked_aux_elems(m);
    return blocked_cholesky(S, m, U, F, aux, gws, 4 * static_cast<int64_t>(m) * m, check_degen, info, s);
  }
  const size_t npad = (m + 7) & ~7;
  const size_t smem = sizeof(double) * npad * (2 * npad + 4);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  chol_inv_kernel<<<1, 512, smem, s>>>(S, m, U, F, aux, check_degen, info);
  return launch_status();
}

int64_t trals_chol_solve_ws_elems(int64_t rows, int m) {
  const int64_t base = rows * m;
  return base + std::max(gemm_ws(1, rows, m, m), m > kInvMax ? 8 * base : int64_t(0));
}

int trals_chol_solve_f64(const double* U, const double* F, const double* aux, int m, const double* Mr, int64_t rows,
                         double* Z, double* ws, int64_t ws_elems, void* stream) {
  if (!U || !F || !aux || !Mr || !Z || !ws || m < 1) return TRALS_ERR_ARG;
  if (rows <= 0) return TRALS_OK;
  if (ws_elems < trals_chol_solve_ws_elems(rows, m)) return TRALS_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* gws = ws + rows * m;
  const int64_t gws_elems = ws_elems - rows * m;
  if (m > kInvMax) {
    const size_t smem = fused_solve_smem(m);
    if (smem <= 200 * 1024) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(fused_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
      }
      const unsigned blocks = static_cast<unsigned>((rows + kFsRows - 1) / kFsRows);
      fused_solve_kernel<<<blocks, 256, smem, s>>>(U, F, aux, m, Mr, rows, Z);
      return launch_status();
    }
    return blocked_solve(U, F, aux, m, Mr, rows, Z, ws, gws, gws_elems, s);
  }
  // Z = M U^{-1} U^{-T} = (M W) V
  const CMap rm = rowmajor(m);
  int st = gemm(Mr, 0, m, 1, 1, rows, m, m, F, m, ws, rm, 0, gws, gws_elems, s);
  if (st) return st;
  return gemm(ws, 0, m, 1, 1, rows, m, m, aux, m, Z, rm, 0, gws, gws_elems, s);
}

int trals_solve_refine_f64(const double* F, const double* aux, const double* S, int m, const double* Mr,
                           int64_t rows, double* Z, int* info, void* stream) {
  if (!F || !aux || !S || !Mr || !Z || !info || m < 1 || m > kInvMax) return TRALS_ERR_ARG;
  if (rows <= 0) return TRALS_OK;
  refine_kernel<<<static_cast<unsigned>(std::min<int64_t>(rows, 65535)), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      F, aux, S, m, Mr, rows, Z, info);
  return launch_status();
}

int64_t trals_sumsq_ws_elems(void) { return 2 * kSumsqBlocks; }

int trals_sumsq_f64(const double* x, int64_t n, double* out, double* ws, void* stream) {
  if (!x || !out || !ws || n < 0) return TRALS_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  sumsq_partial_kernel<double><<<kSumsqBlocks, 512, 0, s>>>(x, n, ws);
  ++g_launches;
  sum_final_kernel<<<1, 1024, 0, s>>>(ws, kSumsqBlocks, out);
  return launch_status();
}

int trals_sumsq_f32(const float* x, int64_t n, double* out, double* ws, void* stream) {
  if (!x || !out || !ws || n < 0) return TRALS_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  sumsq_partial_kernel<float><<<kSumsqBlocks, 512, 0, s>>>(x, n, ws);
  ++g_launches;
  sum_final_kernel<<<1, 1024, 0, s>>>(ws, kSumsqBlocks, out);
  return launch_status();
}

int64_t trals_error_ws_elems(int64_t rows, int m) {
  return static_cast<int64_t>(m) * m + gemm_ws(1, m, rows, m);
}

int trals_error_terms_f64(const double* Mr, const double* Z, const double* S, int64_t rows, int m,
                          const double* xnorm2, double* out, double* ws, int64_t ws_elems, void* stream) {
  if (!Mr || !Z || !S || !xnorm2 || !out || !ws || m < 1 || rows < 1) return TRALS_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t mm = static_cast<int64_t>(m) * m;
  if (ws_elems < mm) return TRALS_ERR_WORKSPACE;
  double* G = ws;
  // G = Z^T Z : A(m=c, k=i) = Z[i*m + c]
  int st = gemm(Z, 0, 1, m, 1, m, rows, m, Z, m, G, rowmajor(m), 0, ws + mm, ws_elems - mm, s);
  if (st) return st;
  error_terms_kernel<<<1, 1024, 0, s>>>(Mr, Z, rows * m, S, G, mm, xnorm2, out);
  return launch_status();
}

int64_t trals_mttsp_ws_elems(int N, const int64_t* dims, const int32_t* ranks, int n) {
  if (N < 2 || !dims || !ranks || n < 0 || n >= N) return -1;
  return mttsp_total_ws(plan_mttsp(N, dims, ranks, n));
}

int trals_mttsp_f64(const double* X, int N, const int64_t* dims, const int32_t* ranks, int n,
                    const double* const* cc, const double* const* cs, const double* const* czt, double* M,
                    double* ws, int64_t ws_elems, void* stream) {
  if (!X || N < 2 || !dims || !ranks || n < 0 || n >= N || !cc || !cs || !czt || !M || !ws) return TRALS_ERR_ARG;
  return run_mttsp(X, N, dims, ranks, n, cc, cs, czt, M, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

int64_t trals_residual_ws_elems(int64_t pre, int64_t post) { return residual_blocks(pre, post); }

int trals_residual_f64(const double* X, int64_t pre, int64_t post, const double* HL, const double* HRt, int64_t K,
                       const double* xnorm2, double* out, double* ws, int64_t ws_elems, void* stream) {
  if (!X || !HL || !HRt || !out || !ws || pre < 1 || post < 1 || K < 1) return TRALS_ERR_ARG;
  if (ws_elems < residual_blocks(pre, post)) return TRALS_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int st = residual(HL, pre, K, HRt, post, X, ws, s);
  if (st) return st;
  residual_final_kernel<<<1, 1024, 0, s>>>(ws, static_cast<int>(residual_blocks(pre, post)), xnorm2, out);
  return launch_status();
}

int64_t trals_residual_oz64_ws_elems(int64_t pre, int64_t post, int64_t K) {
  return pre < 1 || post < 1 || K < 1 ? 0 : residual_oz64_layout(pre, post, K).total;
}

int trals_residual_oz64(const double* X, int64_t pre, int64_t post, const double* HL, const double* HRt, int64_t K,
                        const double* xnorm2, double* out, double* ws, int64_t ws_elems, void* stream) {
  using SC = trals::OzF64;
  if (!X || !HL || !HRt || !out || !ws || pre < 1 || post < 1 || K < 1 || K > SC::KMAX || pre > INT32_MAX ||
      post > INT32_MAX)
    return TRALS_ERR_ARG;
  const ResOzWs w = residual_oz64_layout(pre, post, K);
  if (ws_elems < w.total) return TRALS_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int8_t* adig = reinterpret_cast<int8_t*>(ws + w.adig);
  int32_t* aexp = reinterpret_cast<int32_t*>(ws + w.aexp);
  int8_t* bdig = reinterpret_cast<int8_t*>(ws + w.bdig);
  int32_t* bexp = reinterpret_cast<int32_t*>(ws + w.bexp);
  // A = HL [pre][K] by rows; B = the columns of HRt [K][post] (transposed slicing)
  if (int st = oz_split<double, SC>(HL, pre, K, 0, adig, aexp, ws + w.amx, pre, s)) return st;
  const int bn = kResBN;
  if (int st = launch_colmax<double>(HRt, K, post, post, ws + w.bmx, s)) return st;
  {
    const trals::OzRowTiles bt = oz_b_tiles(post, bn);
    const int64_t gy = (bt.rows_pad() + 63) / 64;
    if (gy > 65535) return TRALS_ERR_UNSUPPORTED;
    dim3 grid(static_cast<unsigned>((K + 63) / 64), static_cast<unsigned>(gy));
    trals::oz_digits_tiled_t_kernel<double, SC><<<grid, 256, 0, s>>>(HRt, K, post, post, ws + w.bmx, bdig, bt, bexp);
    if (int st = launch_status()) return st;
  }
  trals::OzArgs g{};
  g.M = pre; g.K = K; g.N = post; g.kchunk = K; g.splits = 1;
  g.mtiles = static_cast<int>((pre + trals::kOzBM - 1) / trals::kOzBM);
  g.nt = oz_b_tiles(post, bn);
  g.ntiles = g.nt.ntiles;
  g.rotate = 1;
  g.fixup = 0;
  g.kblocks = (K + SC::BK - 1) / SC::BK;
  g.ad = adig; g.bd = bdig; g.ea = aexp; g.eb = bexp;
  g.cmap = rowmajor(post); g.C = nullptr; g.ws = nullptr;
  g.X = X; g.ldx = post; g.rpart = ws + w.part;
  const int64_t tiles = static_cast<int64_t>(g.mtiles) * g.ntiles;
  if (tiles > INT32_MAX) return TRALS_ERR_UNSUPPORTED;
  const int grid = static_cast<int>(std::min<int64_t>(tiles, kSMs));
  if (int st = launch_oz<kResBN, SC, true>(g, grid, s)) return st;
  residual_final_kernel<<<1, 1024, 0, s>>>(ws + w.part, grid, xnorm2, out);
  return launch_status();
}

int64_t trals_spd_fallback_ws_elems(int64_t rows, int m) {
  const int64_t m2 = (m + 1) & ~1;
  return m2 * m + m2 * m2 + m2 + rows * m2;
}

int trals_spd_fallback_f64(const double* S, int m, const double* Mr, int64_t rows, double* Z, int* info, int mode,
                           double rcond, double* ws, int64_t ws_elems, void* stream) {
  if (!S || !Mr || !Z || !info || !ws || m < 1 || rows < 1 || mode < 0 || mode > 2) return TRALS_ERR_ARG;
  if (ws_elems < trals_spd_fallback_ws_elems(rows, m)) return TRALS_ERR_WORKSPACE;
  pinv_fallback_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(S, m, Mr, rows, Z, info, mode, rcond, ws,
                                                                           m, 0);
  return launch_status();
}

int trals_tri_fallback_f64(const double* R0, int Lr, int m, const double* Mr, int64_t rows, double* Z, int* info,
                           int mode, double rcond, double* ws, int64_t ws_elems, void* stream) {
  if (!R0 || !Mr || !Z || !info || !ws || m < 1 || Lr < 1 || Lr > m || rows < 1 || mode < 1 || mode > 3)
    return TRALS_ERR_ARG;
  if (ws_elems < trals_spd_fallback_ws_elems(rows, m)) return TRALS_ERR_WORKSPACE;
  pinv_fallback_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(R0, m, Mr, rows, Z, info, mode, rcond, ws,
                                                                           Lr, 1);
  return launch_status();
}

int64_t trals_oz_range_ws_elems(int64_t rows, int64_t cols, int transpose) { return transpose ? cols : rows; }

int trals_oz_range_f64(const double* x, int64_t rows, int64_t cols, int transpose, double* out, double* ws,
                       int64_t ws_elems, void* stream) {
  if (!x || !out || !ws || rows < 1 || cols < 1 || (transpose != 0 && transpose != 1)) return TRALS_ERR_ARG;
  const int64_t out_rows = transpose ? cols : rows;
  if (ws_elems < out_rows) return TRALS_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!transpose) {
    const int blocks = static_cast<int>(std::min<int64_t>((rows + 7) / 8, 16 * kSMs));
    oz_range_rows_kernel<<<blocks, 256, 0, s>>>(x, rows, cols, ws);
  } else {
    oz_range_cols_kernel<<<static_cast<unsigned>((cols + 31) / 32), 256, 0, s>>>(x, rows, cols, ws);
  }
  if (int st = launch_status()) return st;
  max_reduce_kernel<<<1, 1024, 0, s>>>(ws, out_rows, out);
  return launch_status();
}

int trals_dd_transfer_f64(const double* Rc, int Ra, int k, int Rb, double* Ehi, double* Elo, void* stream) {
  if (!Rc || !Ehi || !Elo || Ra < 1 || k < 1 || Rb < 1) return TRALS_ERR_ARG;
  const int64_t total = static_cast<int64_t>(Ra) * Ra * Rb * Rb;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * kSMs));
  dd_transfer_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(Rc, Ra, k, Rb, Ehi, Elo);
  return launch_status();
}

int64_t trals_dd_r0_ws_elems(int N, const int32_t* ranks) {
  if (N < 2 || !ranks) return -1;
  return dd_ws(N, ranks).total;
}

int trals_dd_r0_f64(int N, int n, const int32_t* ranks, const double* const* Ehi, const double* const* Elo,
                    double* S, double* R0, double* ws, int64_t ws_elems, void* stream) {
  if (N < 2 || n < 0 || n >= N || !ranks || !Ehi || !Elo || !R0 || !ws) return TRALS_ERR_ARG;
  const DdWs w = dd_ws(N, ranks);
  if (ws_elems < w.total) return TRALS_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int m = ranks[n] * ranks[(n + 1) % N];
  double* Shi = ws + w.s;
  double* Slo = Shi + static_cast<int64_t>(m) * m;
  if (int st = dd_gram_chain(N, n, ranks, Ehi, Elo, Shi, Slo, ws, s)) return st;
  if (S && cudaMemcpyAsync(S, Shi, sizeof(double) * m * m, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return TRALS_ERR_CUDA;
  return dd_cholesky(Shi, Slo, m, R0, ws, w, s);
}

int trals_tri_prepare_f64(double* U, int m, double* F, double* aux, int check_degen, int* info, void* stream) {
  if (!U || !F || !aux || !info || m < 1) return TRALS_ERR_ARG;
  return tri_prepare(U, m, F, aux, check_degen, info, static_cast<cudaStream_t>(stream));
}

int64_t trals_core_qr_ws_elems(int I, int RR) { return hh_supported(I, RR) ? hh_plan(I, RR).ws : -1; }

int trals_core_qr_f64(const double* Gzt, int I, int RR, double* R, double* ws, int64_t ws_elems, void* stream) {
  if (!Gzt || !R || I < 1 || RR < 1) return TRALS_ERR_ARG;
  return hh_qr(Gzt, I, RR, R, ws, ws_elems, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
