// kernels.cuh -- the sm_100a kernels of the multiword modular product.
//
//   (1) pack_a / pack_b : word decomposition (balanced signed digits) written
//       straight into the DMMA-fragment-native tiled layout the GEMM streams
//       with TMA bulk copies (one contiguous chunk per CTA per K-stage).
//   (2) mwgemm          : fused multiword modular GEMM.  All u*v word-pair
//       accumulators live in registers, DMMA.8x8x4 (mma.sync .f64) does the
//       exact FP64 contraction, an in-register reduction runs every lambda_k
//       terms, and
//   (3) the epilogue reconstructs C = sum_ij gamma_ij T_ij mod p (Shoup
//       integer mulmod) so no A_i B_j product ever reaches HBM.
//   Plus the reference-compatible helpers: decompose_ref (bit-identical to
//   multiword.hpp:29-54), recompose (words -> residues) and accumulate (the
//   GemmKernel::accumulate plugin, exact C += A B).
#pragma once

#include <cstdint>

#include "device_common.cuh"

namespace fpmm_b200 {

using i64 = std::int64_t;

// ---------------------------------------------------------------- layouts
// Fragment packing of a (rows x K) operand X (A itself, or B transposed):
// chunk (rb, kb) covers rows [rb*BR, +BR) and k [kb*16, +16) for all W words
// and is contiguous: [kk 0..3][w][mtp 0..BR/16)[lane 0..31][pair 0..1], where
// row = rb*BR + (2*mtp+pair)*8 + lane/4 and k = kb*16 + kk*4 + lane%4.  A
// warp's fragment pair for one (kk, w, mtp) is 512 contiguous bytes: one
// conflict-free LDS.128 delivers the DMMA A (or B) operand of two 8-row tiles.
template <int W, int BR>
struct Packing {
  static constexpr int kChunk = BR * 16 * W;  // doubles per (rb, kb) chunk
  __host__ __device__ static i64 offset(i64 rb, i64 kb, i64 KB, int kk, int w, int mtp, int lane,
                                        int pair) {
    return (rb * KB + kb) * kChunk + (((kk * W + w) * (BR / 16) + mtp) * 32 + lane) * 2 + pair;
  }
};

struct DigitParams {
  long long p;      // modulus
  long long half_p; // floor(p/2)
  long long alpha;  // word base
  long long h;      // floor(alpha/2)
  double inv_alpha; // fl(1/alpha), estimate only
};

// balanced signed digits of x in [0,p): see rules.hpp SignedWords
template <int W>
__device__ __forceinline__ void signed_digits(long long x, const DigitParams& dp, double* d) {
  x = x > dp.half_p ? x - dp.p : x;
#pragma unroll
  for (int i = 0; i + 1 < W; ++i) {
    const long long t = x + dp.h;
    long long q = static_cast<long long>(floor(static_cast<double>(t) * dp.inv_alpha));
    long long r = t - q * dp.alpha;
    if (r < 0) { --q; r += dp.alpha; }
    else if (r >= dp.alpha) { ++q; r -= dp.alpha; }
    d[i] = static_cast<double>(r - dp.h);
    x = q;
  }
  d[W - 1] = static_cast<double>(x);
}

__device__ __forceinline__ bool is_residue(double v, long long p) {
  return v >= 0.0 && v < static_cast<double>(p) && v == floor(v);
}

// FPMM_B200_CHECK_INPUTS for engines whose packers do not validate
__global__ void check_residues_kernel(const double* __restrict__ M, i64 ld, i64 rows, i64 cols,
                                      unsigned long long p, int* err) {
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<i64>(gridDim.x) * blockDim.x)
    if (!is_residue(M[(e / cols) * ld + e % cols], static_cast<long long>(p))) atomicOr(err, 1);
}

// (1) A (m x k, lda) -> packed signed words.  Thread: rows r, r+8 of one
// 16-row group, one column; consecutive threads walk k (coalesced reads).
template <int W, int BR>
__global__ void __launch_bounds__(256) pack_a_kernel(const double* __restrict__ A, i64 lda, i64 m,
                                                     i64 k, i64 KB, i64 mpad, DigitParams dp,
                                                     double* __restrict__ out, int* err) {
  const i64 kp = KB * 16, total = (mpad / 2) * kp;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 rp = idx / kp, c = idx % kp;  // row pair, column
    const i64 r0 = (rp / 8) * 16 + (rp % 8), r1 = r0 + 8;
    double v0 = 0.0, v1 = 0.0;
    if (c < k) {
      if (r0 < m) v0 = A[r0 * lda + c];
      if (r1 < m) v1 = A[r1 * lda + c];
      if (err && ((r0 < m && !is_residue(v0, dp.p)) || (r1 < m && !is_residue(v1, dp.p)))) atomicOr(err, 1);
    }
    double d0[W], d1[W];
    signed_digits<W>(static_cast<long long>(v0), dp, d0);
    signed_digits<W>(static_cast<long long>(v1), dp, d1);
    const i64 rb = r0 / BR;
    const int rr = static_cast<int>(r0 % BR);
    const int mt = rr / 8, lane = (rr % 8) * 4 + static_cast<int>(c % 4);
    const i64 kb = c / 16;
    const int kk = static_cast<int>((c % 16) / 4);
#pragma unroll
    for (int w = 0; w < W; ++w)
      *reinterpret_cast<double2*>(out + Packing<W, BR>::offset(rb, kb, KB, kk, w, mt / 2, lane, 0)) =
          make_double2(d0[w], d1[w]);
  }
}

// (1) B (k x n, ldb) -> packed signed words of B^T.  Thread: columns
// n0, n0+8 of one 16-column group, one k row; consecutive threads walk n.
template <int W, int BR>
__global__ void __launch_bounds__(256) pack_b_kernel(const double* __restrict__ B, i64 ldb, i64 k,
                                                     i64 n, i64 KB, i64 npad, DigitParams dp,
                                                     double* __restrict__ out, int* err) {
  const i64 np2 = npad / 2, total = np2 * KB * 16;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    // a warp covers 8 column pairs x 4 k rows = one fragment's 32 lanes, so
    // its 16-byte stores form one contiguous 512-byte run
    const int c4 = static_cast<int>(idx % 4), nn = static_cast<int>((idx / 4) % 8);
    const i64 rest = idx / 32, g16 = rest % (np2 / 8), kq = rest / (np2 / 8);
    const i64 c = kq * 4 + c4;                   // k row
    const i64 n0 = g16 * 16 + nn, n1 = n0 + 8;   // column pair
    double v0 = 0.0, v1 = 0.0;
    if (c < k) {
      if (n0 < n) v0 = B[c * ldb + n0];
      if (n1 < n) v1 = B[c * ldb + n1];
      if (err && ((n0 < n && !is_residue(v0, dp.p)) || (n1 < n && !is_residue(v1, dp.p)))) atomicOr(err, 1);
    }
    double d0[W], d1[W];
    signed_digits<W>(static_cast<long long>(v0), dp, d0);
    signed_digits<W>(static_cast<long long>(v1), dp, d1);
    const i64 rb = n0 / BR;
    const int rr = static_cast<int>(n0 % BR);
    const int mt = rr / 8, lane = (rr % 8) * 4 + static_cast<int>(c % 4);
    const i64 kb = c / 16;
    const int kk = static_cast<int>((c % 16) / 4);
#pragma unroll
    for (int w = 0; w < W; ++w)
      *reinterpret_cast<double2*>(out + Packing<W, BR>::offset(rb, kb, KB, kk, w, mt / 2, lane, 0)) =
          make_double2(d0[w], d1[w]);
  }
}

// ------------------------------------------------------------ fused GEMM
template <int U, int V, int MT, int NT>
struct GemmCfg {
  static constexpr int kWarpsM = 2, kWarpsN = 4, kWarps = 8, kThreads = 256;
  static constexpr int BM = kWarpsM * MT * 8, BN = kWarpsN * NT * 8, BK = 16;
  static constexpr int kStages = 4;
  static constexpr int kAElems = BM * BK * U, kBElems = BN * BK * V;  // doubles per stage
  static constexpr int kSmem = kStages * (kAElems + kBElems) * 8 + 2 * kStages * 8;
  static_assert(MT % 2 == 0 && NT % 2 == 0, "fragment pairs");
};

constexpr int kMaxPairs = 8;

struct GemmParams {
  const double* apack;
  const double* bpack;
  double* C;
  i64 ldc, m, n;
  int MB, NB, KB;
  int red_every;   // k4-steps between in-register reductions (lambda_k / 4)
  double pf, q;    // p, fl(1/p)
  int* overflow;   // CHECK_EXACTNESS: |accumulator| > 2^53 seen before a reduction -> *overflow |= 2
  unsigned long long p;
  unsigned long long gamma[kMaxPairs], gamma_sh[kMaxPairs];  // alpha^i beta^j mod p, Shoup consts
};

// Instrumented mode (the reference's shadow replay, shadow.hpp:125-162, run by
// `fpmm check --checked`): every accumulator must be an exact integer of
// magnitude <= 2^53 when it is reduced, i.e. no DMMA partial sum left the
// exactly representable range.  One flag word per call; off unless asked.
template <int U, int V, int MT, int NT>
__device__ __forceinline__ void check_exact(const double (&acc)[U][V][MT][NT][2], int* flag) {
  bool bad = false;
#pragma unroll
  for (int i = 0; i < U; ++i)
#pragma unroll
    for (int j = 0; j < V; ++j)
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) bad |= fabs(acc[i][j][a][b][e]) > 9007199254740992.0;
  if (bad) atomicOr(flag, 2);
}

template <int U, int V, int MT, int NT>
__global__ void __launch_bounds__(256, 1) mwgemm_kernel(const __grid_constant__ GemmParams P) {
  using Cfg = GemmCfg<U, V, MT, NT>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, S = Cfg::kStages;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + S * Cfg::kAElems;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * Cfg::kBElems);
  uint64_t* empty = full + S;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / Cfg::kWarpsN, wn = warp % Cfg::kWarpsN;

  // grouped rasterisation: GROUP tile-rows share B panels in L2
  constexpr int GROUP = 8;
  const int pid = blockIdx.x;
  const int in_group = GROUP * P.NB;
  const int first_m = (pid / in_group) * GROUP;
  const int gsz = min(P.MB - first_m, GROUP);
  const int tm = first_m + (pid % in_group) % gsz;
  const int tn = (pid % in_group) / gsz;

  const double* gA = P.apack + static_cast<i64>(tm) * P.KB * Cfg::kAElems;
  const double* gB = P.bpack + static_cast<i64>(tn) * P.KB * Cfg::kBElems;
  constexpr uint32_t kStageBytes = (Cfg::kAElems + Cfg::kBElems) * 8;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], Cfg::kThreads);  // every consumer thread releases its own reads
    }
    dev::fence_barrier_init();
  }
  __syncthreads();
  if (tid == 0) {
    const int pre = min(S, P.KB);
    for (int s = 0; s < pre; ++s) {
      dev::mbar_arrive_expect_tx(&full[s], kStageBytes);
      dev::bulk_g2s(sA + s * Cfg::kAElems, gA + static_cast<i64>(s) * Cfg::kAElems, Cfg::kAElems * 8, &full[s]);
      dev::bulk_g2s(sB + s * Cfg::kBElems, gB + static_cast<i64>(s) * Cfg::kBElems, Cfg::kBElems * 8, &full[s]);
    }
  }

  double acc[U][V][MT][NT][2];
#pragma unroll
  for (int i = 0; i < U; ++i)
#pragma unroll
    for (int j = 0; j < V; ++j)
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) acc[i][j][a][b][0] = acc[i][j][a][b][1] = 0.0;

  const double pf = P.pf, q = P.q;
  int cnt = 0;
  for (int it = 0; it < P.KB; ++it) {
    const int s = it % S;
    dev::mbar_wait(&full[s], (it / S) & 1);
    const double* a_st = sA + s * Cfg::kAElems;
    const double* b_st = sB + s * Cfg::kBElems;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      double fa[U][MT], fb[V][NT];
#pragma unroll
      for (int w = 0; w < U; ++w)
#pragma unroll
        for (int mp = 0; mp < MT / 2; ++mp) {
          const double2 t = dev::lds128(a_st + (((kk * U + w) * (BM / 16) + wm * (MT / 2) + mp) * 32 + lane) * 2);
          fa[w][2 * mp] = t.x;
          fa[w][2 * mp + 1] = t.y;
        }
#pragma unroll
      for (int w = 0; w < V; ++w)
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {
          const double2 t = dev::lds128(b_st + (((kk * V + w) * (BN / 16) + wn * (NT / 2) + np) * 32 + lane) * 2);
          fb[w][2 * np] = t.x;
          fb[w][2 * np + 1] = t.y;
        }
#pragma unroll
      for (int i = 0; i < U; ++i)
#pragma unroll
        for (int j = 0; j < V; ++j)
#pragma unroll
          for (int a = 0; a < MT; ++a)
#pragma unroll
            for (int b = 0; b < NT; ++b) dev::dmma884(acc[i][j][a][b][0], acc[i][j][a][b][1], fa[i][a], fb[j][b]);
      if (++cnt == P.red_every) {
        cnt = 0;
        if (P.overflow) check_exact<U, V, MT, NT>(acc, P.overflow);
#pragma unroll
        for (int i = 0; i < U; ++i)
#pragma unroll
          for (int j = 0; j < V; ++j)
#pragma unroll
            for (int a = 0; a < MT; ++a)
#pragma unroll
              for (int b = 0; b < NT; ++b) {
                acc[i][j][a][b][0] = dev::reduce_signed(acc[i][j][a][b][0], pf, q);
                acc[i][j][a][b][1] = dev::reduce_signed(acc[i][j][a][b][1], pf, q);
              }
      }
    }
    dev::mbar_arrive(&empty[s]);  // release: this thread's LDS reads of stage s are done
    // refill the stage consumed in the previous iteration (its empty barrier
    // is normally complete by now, so the producer rarely waits)
    if (tid == 0 && it >= 1) {
      const int nxt = it - 1 + S;
      if (nxt < P.KB) {
        const int ps = (it - 1) % S;
        dev::mbar_wait(&empty[ps], ((it - 1) / S) & 1);
        dev::mbar_arrive_expect_tx(&full[ps], kStageBytes);
        dev::bulk_g2s(sA + ps * Cfg::kAElems, gA + static_cast<i64>(nxt) * Cfg::kAElems, Cfg::kAElems * 8, &full[ps]);
        dev::bulk_g2s(sB + ps * Cfg::kBElems, gB + static_cast<i64>(nxt) * Cfg::kBElems, Cfg::kBElems * 8, &full[ps]);
      }
    }
  }

  // (3) epilogue: canonical residues of every pair, gamma-weighted sum mod p
  if (P.overflow) check_exact<U, V, MT, NT>(acc, P.overflow);
  const unsigned long long p = P.p;
  const i64 row_base = static_cast<i64>(tm) * BM + wm * MT * 8 + lane / 4;
  const i64 col_base = static_cast<i64>(tn) * BN + wn * NT * 8 + 2 * (lane % 4);
#pragma unroll
  for (int a = 0; a < MT; ++a) {
    const i64 row = row_base + a * 8;
#pragma unroll
    for (int b = 0; b < NT; ++b) {
      const i64 col = col_base + b * 8;
      double outv[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        unsigned long long sum = 0;
#pragma unroll
        for (int i = 0; i < U; ++i)
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const double r = dev::reduce_signed(acc[i][j][a][b][e], pf, q);
            long long t = static_cast<long long>(r);
            t += t < 0 ? static_cast<long long>(p) : 0;
            unsigned long long term = static_cast<unsigned long long>(t);
            if (i + j > 0) term = dev::shoup_mulmod(term, P.gamma[i * V + j], P.gamma_sh[i * V + j], p);
            sum += term;
            sum -= sum >= p ? p : 0;
          }
        outv[e] = static_cast<double>(sum);
      }
      if (row < P.m) {
        double* dst = P.C + row * P.ldc + col;
        if (col + 1 < P.n && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          *reinterpret_cast<double2*>(dst) = make_double2(outv[0], outv[1]);
        } else {
          if (col < P.n) dst[0] = outv[0];
          if (col + 1 < P.n) dst[1] = outv[1];
        }
      }
    }
  }
}

// ------------------------------------------- reference-compatible helpers
// multiword.hpp:29-54: r = floor(T * fl(1/alpha)); w = fma(-alpha, r, T); T = r
__global__ void decompose_ref_kernel(const double* __restrict__ M, i64 ld, i64 rows, i64 cols, int u,
                                     double alpha, double inv_alpha, double* __restrict__ words,
                                     i64 word_stride) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const i64 r = e / cols, c = e % cols;
  double t = M[r * ld + c];
  for (int i = 0; i + 1 < u; ++i) {
    const double q = floor(t * inv_alpha);
    words[i * word_stride + e] = __fma_rn(-alpha, q, t);
    t = q;
  }
  words[static_cast<i64>(u - 1) * word_stride + e] = t;
}

// words -> residues: x = sum_i alpha^i w_i mod p (Horner, Shoup mulmod)
__global__ void recompose_kernel(const double* __restrict__ words, i64 word_stride, i64 ld, i64 rows,
                                 i64 cols, int u, unsigned long long alpha_mod,
                                 unsigned long long alpha_sh, unsigned long long p,
                                 double* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const i64 r = e / cols, c = e % cols;
  unsigned long long x = 0;
  for (int i = u - 1; i >= 0; --i) {
    const unsigned long long w = static_cast<unsigned long long>(words[i * word_stride + r * ld + c]) % p;
    x = dev::shoup_mulmod(x, alpha_mod, alpha_sh, p) + w;
    x -= x >= p ? p : 0;
  }
  out[e] = static_cast<double>(x);
}

// GemmKernel<double>::accumulate: exact C += A B (plugin contract).  64x64
// CTA tile, 4 warps of 32x32, k-tiles of 16 staged through shared memory,
// DMMA.8x8x4.  Panels are strided views; bounds are checked.
__global__ void __launch_bounds__(128) accumulate_kernel(double* __restrict__ C, i64 ldc,
                                                         const double* __restrict__ A, i64 lda,
                                                         const double* __restrict__ B, i64 ldb,
                                                         i64 m, i64 w, i64 n) {
  __shared__ double sa[64][17];
  __shared__ double sb[16][65];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / 2, wn = warp % 2;
  const i64 m0 = static_cast<i64>(blockIdx.y) * 64, n0 = static_cast<i64>(blockIdx.x) * 64;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (i64 k0 = 0; k0 < w; k0 += 16) {
    for (int e = tid; e < 64 * 16; e += 128) {
      const int r = e / 16, c = e % 16;
      sa[r][c] = (m0 + r < m && k0 + c < w) ? A[(m0 + r) * lda + k0 + c] : 0.0;
      const int kr = e / 64, nc = e % 64;
      sb[kr][nc] = (k0 + kr < w && n0 + nc < n) ? B[(k0 + kr) * ldb + n0 + nc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      double fa[4], fb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = sa[wm * 32 + a * 8 + lane / 4][kk * 4 + lane % 4];
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = sb[kk * 4 + lane % 4][wn * 32 + b * 8 + lane / 4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dev::dmma884(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const i64 row = m0 + wm * 32 + a * 8 + lane / 4, col = n0 + wn * 32 + b * 8 + 2 * (lane % 4) + e;
        if (row < m && col < n) C[row * ldc + col] += acc[a][b][e];
      }
}

}  // namespace fpmm_b200

namespace fpmm_b200 {

// block_gemm_mod helpers (block_product.hpp:62-73 on the device).
// M <- M mod p in place: exact (fmod of a non-negative integer below 2^53).
__global__ void reduce_mod_kernel(double* __restrict__ M, i64 ld, i64 rows, i64 cols, double p) {
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    double* x = M + (e / cols) * ld + e % cols;
    *x = fmod(*x, p);
  }
}

// C <- (C + T) mod p for residues C, T < p (< 2^52: the sum is exact)
__global__ void add_mod_kernel(double* __restrict__ Cm, i64 ldc, const double* __restrict__ T, i64 ldt, i64 rows,
                               i64 cols, double p) {
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = e / cols, c = e % cols;
    const double x = Cm[r * ldc + c] + T[r * ldt + c];
    Cm[r * ldc + c] = x >= p ? x - p : x;
  }
}

// the contract's operand scan: max entry (atomicMax) and whether every entry
// is a non-negative integer below 2^53 (err bit 1 otherwise)
__global__ void max_scan_kernel(const double* __restrict__ M, i64 ld, i64 rows, i64 cols,
                                unsigned long long* maxv, int* err) {
  unsigned long long mx = 0;
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double v = M[(e / cols) * ld + e % cols];
    if (!(v >= 0.0 && v < 9007199254740992.0 && v == floor(v))) {
      atomicOr(err, 1);
      continue;
    }
    mx = max(mx, static_cast<unsigned long long>(v));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_down_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxv, mx);
}

// Device-side synthetic residues for large benchmarks: element e of a
// rows x cols slice starting at global row row0 (global index g = (row0+i)*cols + j) is the first draw r = splitmix64(seed ^ (g * 2^8 + t)),
// t = 0, 1, ..., below reject_at (the largest multiple of p), reduced mod p:
// uniform on [0,p), deterministic, independent of launch geometry.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void random_residues_kernel(double* __restrict__ M, i64 ld, i64 rows, i64 cols,
                                       i64 row0, unsigned long long p, unsigned long long reject_at,
                                       unsigned long long seed) {
  const i64 total = rows * cols;
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 i = e / cols, j = e % cols;
    const unsigned long long g = static_cast<unsigned long long>((row0 + i) * cols + j);  // global index
    unsigned long long t = 0, r;
    do r = splitmix64(seed ^ ((g << 8) + t++));
    while (r >= reject_at);
    M[i * ld + j] = static_cast<double>(r % p);
  }
}

// FP64 tensor-pipe peak probe: 8 independent DMMA.8x8x4 chains per warp.
__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* out) {
  double d[8][2];
  const double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
#pragma unroll
  for (int c = 0; c < 8; ++c) d[c][0] = c, d[c][1] = -c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dev::dmma884(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

}  // namespace fpmm_b200
