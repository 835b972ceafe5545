// rnsengine.cuh -- residue-number-system multiword engine on tcgen05 int8.
//
// The multiword idea with the words taken in a residue number system instead
// of a positional base: every centred residue x' = x - p [x > p/2] is
// represented by its residues modulo N pairwise-coprime moduli m_i <= 256
// (one byte each).  The exact integer X = sum_k a'_k b'_k satisfies
// |X| <= K floor(p/2)^2, so with M = prod m_i >= 2.03 K floor(p/2)^2 it is
// recovered from its residues r_i = X mod m_i by the CRT, and reduced mod p
// without ever forming X:
//   Z = sum_i r_i y_i M_i  (M_i = M/m_i, y_i = M_i^{-1} mod m_i),  Z = X + t M,
//   t = round(sum_i r_i y_i / m_i)  (|X|/M <= 1/2.03, fixed point 2^-19),
//   X mod p = (sum_i r_i W_i - t (M mod p)) mod p,  W_i = y_i M_i mod p.
// Each r_i is one exact int8 GEMM: T_i = A_i B_i (u8 x u8 -> s32 in TMEM,
// exact while K_seg 255^2 < 2^32), r_i = T_i mod m_i.  N grows like
// (2 bits(p) + log2 K) / 8 against D^2 = ceil(bits/8)^2 digit products for
// the base-256 engine (15 vs 49 at 52 bits, K = 8192).
//
// Three kernels per product:
//   pack_a_rns / pack_b_rns: the residues of every operand element modulo each
//     m_i, written as canonical K-major UMMA chunks (one plane per modulus);
//   rns_kernel: persistent CTA pairs (clusters of 2) computing 256 x 256 tiles
//     with tcgen05.mma.cta_group::2.kind::i8, one modulus per pass, passes in
//     modulus-major order over the grid; the epilogue reduces T_i mod m_i and
//     parks one byte per element and modulus in HBM;
//   rns_crt_kernel: the CRT above, from the parked bytes into C.
// No int32 product leaves the SM; the parked residues are n bytes per output
// element.
//
// rns_kernel warp roles (18 warps): 0 TMA producer (2-CTA tensor-map loads
// completing on the leader's barrier), 1 TMEM allocator + (leader) the MMA
// issuer, a converged warp whose elect.sync lane issues, or (rank 1) the
// long-K pacing monitor, 2..17 epilogue (TMEM lane quadrant w % 4; two groups
// of eight on alternate passes for one-segment passes, else 64 columns each).
#pragma once

#include <cuda.h>

#include <cstdint>

#include "device_common.cuh"
#include "i8engine.cuh"

namespace fpmm_b200 {
namespace rns {

using i64 = std::int64_t;

constexpr int kMaxMod = 20;
constexpr int kBM = 128;             // rows per CTA (each CTA's half of the pair's M = 256)
constexpr int kNT = 256;             // columns per tile (MMA N)
constexpr int kBH = kNT / 2;         // B columns held by each CTA of the pair
constexpr int kPairM = 2 * kBM;      // rows per pair tile
// k bytes per pipeline stage: 128 (four K=32 MMAs per stage barrier) ran the
// 8192^3 residue GEMMs 9% faster than 64 (two); 256 (three 64 KB stages, eight
// MMAs per barrier) another 2-3% at 8192^3 and 5-6% at 32768^3 / 4096 x 262144
// x 4096, where the one thread that waits, issues and commits per stage is on
// the critical path (profiles/round2/ab_bk256.txt)
#ifndef FPMM_B200_RNS_BK
#define FPMM_B200_RNS_BK 256
#endif
constexpr int kBK = FPMM_B200_RNS_BK;
constexpr int kKSteps = kBK / 32;    // MMA K = 32 for kind::i8
constexpr int kAStage = kBM * kBK;   // this CTA's 128 rows of A (32 KB)
constexpr int kBStage = kBH * kBK;   // this CTA's 128 columns of B (32 KB)
constexpr int kStageBytes = kAStage + kBStage;
constexpr int kStages = 12 * 64 / kBK;  // 192 KB of stages (kBK 64, 128, 192, 256)
#ifndef FPMM_B200_RNS_EPI_WARPS
#define FPMM_B200_RNS_EPI_WARPS 16
#endif
constexpr int kEpiWarps = FPMM_B200_RNS_EPI_WARPS;  // 8 or 16: 4 TMEM lane quadrants x column groups
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiCols = 4 * kNT / kEpiWarps;        // accumulator columns per epilogue warp
static_assert(kEpiWarps == 8 || kEpiWarps == 16, "epilogue warps");
// epilogue: drain all of a warp's accumulator columns, release, then reduce
// (1) or release after the last 32-column load (0)
// MMA issuer: the whole warp 1 of the leader CTA with elect.sync (1) or its
// lane 0 alone (0)
#ifndef FPMM_B200_RNS_MMA_WARP
#define FPMM_B200_RNS_MMA_WARP 1
#endif
#ifndef FPMM_B200_RNS_DRAIN_FIRST
#define FPMM_B200_RNS_DRAIN_FIRST 1
#endif
static_assert(kBK % 64 == 0 && kBK <= 256, "stage k-depth: 64, 128 or 256 bytes");
constexpr int kSmem = kStages * kStageBytes + 1024;
constexpr int kSlotPerMod = kBM * kNT;  // scratch bytes per modulus per CTA tile (32 KB)
constexpr int kGroup = 16;              // pair-tile rows per rasterisation group

// ------------------------------------------------------------------ CRT
// C = X mod p from the parked residue bytes of every tile (summed over the
// split-K slices mod m_i first: residues are additive):
//   X mod p = (sum r_i W_i - t (M mod p)) mod p,  t = round(sum r_i y_i / m_i),
// W_i = y_i M_i mod p (7 bytes), g_i = round(2^19 y_i / m_i) (3 bytes).  Both
// sums are evaluated byte-plane by byte-plane with dp4a over groups of four
// moduli: the residue words of four moduli are transposed (PRMT) so one word
// holds one element's four residues, and plane b accumulates
// sum_i r_i byte_b(W_i) (< 20 * 255^2 < 2^21).  That is 10 dp4a per element
// per four moduli.  The fixed-point error of t is <= n 255 2^-20 <= 0.005,
// inside the plan's range margin (|X| / M <= 1/2.03).
constexpr int kCrtPlanes = 10;                 // 7 byte planes of W, 3 of g
constexpr int kCrtGroups = (kMaxMod + 3) / 4;  // groups of four moduli
struct CrtParams {
  const uint8_t* R;  // residue blocks, as parked by rns_kernel
  double* C;
  i64 ldc, m, n;
  int MB, NB, nmod, splits, group;
  unsigned long long p, mu, two32, two32_sh, Mp, Mp_sh;
  // n <= 16 finalisation (S < 16 * 255 * p): q = umulhi(S >> s_shift, inv32)
  // is floor(S/p) - {0,1,2}; t (M mod p) by a 32-bit Shoup product
  int s_shift;     // max(0, bits(p) - 20): S >> s_shift < 2^32 and 2^s_shift < p
  uint32_t inv32;  // floor(2^(s_shift + 32) / p)
  uint32_t Mp_sh32;  // floor((M mod p) 2^32 / p)
  uint32_t mod[kMaxMod];
  uint32_t wb[kCrtGroups][kCrtPlanes];  // byte b of W_i (b < 7) / g_i (b >= 7) for the group's 4 moduli
  // one-reduction finalisation (rns_crt_spec_kernel, host-checked bounds):
  // R = S + (T0 - t) (M mod p) + C0 == X (mod p), R <= R_max < 2^64, and
  // q = umulhi(R >> s2, inv2) is floor(R/p) or one less, so one conditional
  // subtract finishes R mod p (see crt_plan_final in engine.cu)
  int comb;
  uint32_t T0, s2, inv2;
  unsigned long long C0, negp;  // (p - T0 (M mod p) mod p) mod p, 2^64 - p
  // the same R on the FP64 pipe when R_max < 2^53 (p <= 2^40): S, (T0 - t) Mp and C0
  // are exact doubles, R mod p = R - rint(R fl(1/p)) p (+ p when negative)
  int fp64fin;
  double Mp_d, C0_d, p_d, invp_d;
};

// Per-modulus constants (host: rns_plan in rules.cpp).
struct Params {
  // 2-D byte views (128-byte rows) of the packed operands for the pair TMA
  // loads; a chunk of kAStage bytes is one 128 x (kAStage / 128) box
  CUtensorMap tmA, tmB;
  const uint8_t* apack;  // [128-row block][k-block][modulus] chunks of kAStage bytes
  const uint8_t* bpack;  // [128-column block][k-block][modulus] chunks of kBStage bytes
  double* C;
  uint8_t* scratch;      // residue blocks: [item][CTA rank] x nmod * kSlotPerMod bytes
  i64 ldc, m, n;
  int MB, NB, KB;    // pair tiles (256 x 256) along m and n; 64-byte k-blocks
  int nmod;
  int seg_kb;        // k-blocks per exact int32 segment
  int kb_per_split;  // split-K: k-blocks per slice
  int splits;
  int group;         // pair-tile rows per rasterisation group
  int small_t;       // seg_kb * kBK * 255^2 < 2^24: products reduce without the 16-bit split
  int flat;          // PassIter order (see there)
  int debug;         // timing experiments only (wrong C): 1 no residue stores, 2 no reduction or stores, 4 no MMAs,
                     // 8 MMAs do not wait for the epilogue's drain, 16 no operand loads (stage barriers only);
                     // 22 (= 16 + 4 + 2) does not complete with the converged-warp MMA issuer (not investigated)
  int pingpong;      // 16 epilogue warps as two groups of 8 taking alternate passes (kEpiWarps == 16;
                     // one K segment per pass)
  unsigned epi_sleep_ns;  // epilogue's accumulator wait: sleep between polls (ns), 0 = suspending try_wait
  // pacing (long K): each pair's producer publishes the k-blocks it has issued
  // in progress[pair] and stays at most pace_kb k-blocks ahead of the slowest
  // pair, so the pairs that share a wave's panels stream them in lockstep and
  // the panels are read from DRAM about once (0 = off)
  int* progress;
  int pace_kb;
  // rns_tile_kernel (rnstile.cuh): pipeline stages, byte offsets of the shared
  // residue planes and of the barriers in dynamic shared memory, residue
  // planes held in shared memory (the rest in TMEM), TMEM accumulators
  int stages, res_off, bar_off, smem_mods, naccs;
  int pp_pairs;  // pingpong drain: two 32-column TMEM loads per wait (see the epilogue)
  i64 split_stride;
  unsigned long long p, mu;            // Barrett: mu = floor(2^64 / p)
  unsigned long long two32, two32_sh;  // 2^32 mod p and its Shoup quotient
  unsigned long long Mp, Mp_sh;        // M mod p and its Shoup quotient
  uint32_t mod[kMaxMod];
  uint32_t c16[kMaxMod];    // 2^16 mod m
  uint32_t negm[kMaxMod];   // -m mod 2^32
  uint32_t magic[kMaxMod];  // ceil(2^32 / m): floor(s/m) = umulhi(s, magic) for s < 2^32 / m
  uint32_t g[kMaxMod];      // round(2^24 y_i / m_i)
  uint32_t w_lo[kMaxMod], w_hi[kMaxMod];  // W_i = y_i M_i mod p
  CrtParams crt;  // rns_tile_kernel: the reconstruction constants and C (crt.R unused)
  int wpl;        // byte planes of W_i (ceil(bits(p - 1) / 8))
};

struct PackParams {
  double half_p;  // floor(p/2): x > half_p is centred to x - p
  double pf;      // p
  int nmod;
  // residues of modulus pairs from x' mod (m_a m_b) on the FP64 pipe
  // (residues16_pair; 0 = base-256 digits and dp4a, residues16).  A form with
  // one DFMA quotient and the rest in 32-bit integers (u = lo32(x') - q L + L)
  // measured 0-12% slower at 8192^2 (packs are not ALU-bound there) and 3%
  // faster at 4096 x 262144: profiles/round2/ab_packmode.txt
  int fp64_pairs;
  double L[kMaxMod / 2], invL[kMaxMod / 2], offL[kMaxMod / 2];  // m_2j m_2j+1 (or m_2j alone), fl(1/L), 2^52 + L
  uint32_t mod[kMaxMod];
  uint32_t wlo[kMaxMod];    // bytes (256^j mod m), j = 0..3
  uint32_t whi[kMaxMod];    // bytes (256^j mod m), j = 4..6, and (m - p mod m) mod m in byte 3
  uint32_t negm[kMaxMod];
  uint32_t magic[kMaxMod];
};

// s mod m for s < 2^32 / m with magic = ceil(2^32 / m) and negm = -m (mod
// 2^32): floor(s magic / 2^32) = floor(s/m + s e / (m 2^32)), e < m, and the
// second term is < 1/m <= 1 - frac(s/m), so one IMAD.HI + one IMAD suffice.
__device__ __forceinline__ uint32_t mod_small(uint32_t s, uint32_t negm, uint32_t magic) {
  return __umulhi(s, magic) * negm + s;
}

// four values < 256 -> one little-endian word, by byte permutes (byte 3 of
// r0 / r2 is zero and fills the upper bytes of the halves)
__device__ __forceinline__ uint32_t pack4(uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  return __byte_perm(__byte_perm(r0, r1, 0x3340), __byte_perm(r2, r3, 0x3340), 0x5410);
}

// x < 2^52 as two words of base-256 digits: lo = digits 0..3, hi = digits
// 4..6 plus the centring flag [x > p/2] in byte 3.  The residue of the
// centred value mod m is then dp4a(lo, wlo) + dp4a(hi, whi) (< 2^19) mod m.
__device__ __forceinline__ void digits16(const double (&xs)[16], double half_p, uint32_t (&lo)[16],
                                         uint32_t (&hi)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    // 2^52 + x has the integer x in its significand (x < 2^52)
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(xs[e] + 4503599627370496.0));
    lo[e] = static_cast<uint32_t>(b);
    hi[e] = (static_cast<uint32_t>(b >> 32) & 0xFFFFFu) | (xs[e] > half_p ? 0x1000000u : 0u);
  }
}

// 16 residues (one 16-byte k row of a core matrix) of modulus i
__device__ __forceinline__ uint4 residues16(const uint32_t (&lo)[16], const uint32_t (&hi)[16], const PackParams& P,
                                            int i) {
  const uint32_t nm = P.negm[i], wl = P.wlo[i], wh = P.whi[i], mg = P.magic[i];
  uint32_t r[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t s = __dp4a(lo[e], wl, __dp4a(hi[e], wh, 0u));  // < 2^19
    r[e] = mod_small(s, nm, mg);
  }
  // byte packing with PRMT (ALU pipe): dp4a and the IMADs of mod_small
  // already saturate the FMA-heavy pipe, where shift-by-IMAD would also go
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) w[q] = pack4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// The residues of moduli 2j and 2j+1 from the centred values xc (exact,
// |xc| <= p/2 < 2^51): y = xc - rint(xc fl(1/L)) L with L = m_2j m_2j+1 < 2^16
// is exact and |y| < L/2 + 1 (the quotient estimate is within 2^-16 of xc/L),
// the low word of y + 2^52 + L is u = y + L in [0, 2L), and u mod m_2j, u mod
// m_2j+1 are two mod_small each.  Four FP64-pipe ops per pair and two IMADs
// per residue, against two dp4a and two IMADs per residue on the FMA-heavy
// pipe for the digit form; centred values need no more registers than digits.
__device__ __forceinline__ void residues16_pair(const double (&xc)[16], const PackParams& P, int j, uint4& out0,
                                                uint4& out1) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double L = P.L[j], inv = P.invL[j], off = P.offL[j];
  const int i0 = 2 * j, i1 = min(2 * j + 1, P.nmod - 1);
  const uint32_t n0 = P.negm[i0], g0 = P.magic[i0], n1 = P.negm[i1], g1 = P.magic[i1];
  uint32_t r0[16], r1[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const double q = __fma_rn(xc[e], inv, M) - M;
    const double y = __fma_rn(-q, L, xc[e]);
    const uint32_t u = static_cast<uint32_t>(__double2loint(y + off));
    r0[e] = mod_small(u, n0, g0);
    r1[e] = mod_small(u, n1, g1);
  }
  uint32_t w0[4], w1[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w0[q] = pack4(r0[4 * q], r0[4 * q + 1], r0[4 * q + 2], r0[4 * q + 3]);
    w1[q] = pack4(r1[4 * q], r1[4 * q + 1], r1[4 * q + 2], r1[4 * q + 3]);
  }
  out0 = make_uint4(w0[0], w0[1], w0[2], w0[3]);
  out1 = make_uint4(w1[0], w1[1], w1[2], w1[3]);
}

__device__ __forceinline__ void centre16(const double (&xs)[16], const PackParams& P, double (&xc)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) xc[e] = xs[e] > P.half_p ? xs[e] - P.pf : xs[e];
}

// Every residue plane of one 16-element k row: out + i * plane for modulus i.
// MODE = PackParams::fp64_pairs (compile-time: each form has its own register budget).
template <int MODE>
__device__ __forceinline__ void store_residue_planes(const double (&xs)[16], const PackParams& P, uint8_t* out,
                                                     i64 plane) {
  if constexpr (MODE == 1) {
    double xc[16];
    centre16(xs, P, xc);
#pragma unroll 1
    for (int j = 0; 2 * j < P.nmod; ++j) {
      uint4 a, b;
      residues16_pair(xc, P, j, a, b);
      *reinterpret_cast<uint4*>(out + (2 * j) * plane) = a;
      if (2 * j + 1 < P.nmod) *reinterpret_cast<uint4*>(out + (2 * j + 1) * plane) = b;
    }
  } else {
    uint32_t lo[16], hi[16];
    digits16(xs, P.half_p, lo, hi);
#pragma unroll 1
    for (int i = 0; i < P.nmod; ++i) *reinterpret_cast<uint4*>(out + i * plane) = residues16(lo, hi, P, i);
  }
}

// A: m x k residues -> N residue planes in the canonical K-major core-matrix
// layout.  Chunk (rb, kb, i), kAStage bytes: [k16 c (kBK / 16)][row group g (16)][row (8)][16 B];
// the n moduli of a k-block are adjacent chunks, so a thread's n 16-byte stores
// land within n * kAStage bytes (with the modulus outermost they were KB *
// kAStage apart: 32 MB at k = 262144)
// Thread (row, 16-element k chunk): reads 16 doubles, writes N x 16 bytes.
template <int MODE>
__global__ void __launch_bounds__(256) pack_a_rns(const double* __restrict__ A, i64 lda, i64 m, i64 k, int KB,
                                                  i64 mpad, const __grid_constant__ PackParams P,
                                                  uint8_t* __restrict__ out) {
  const i64 kchunks = static_cast<i64>(KB) * (kBK / 16);
  const i64 total = mpad * kchunks;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 grp = idx / 32;
    const int lane = static_cast<int>(idx % 32);
    const int r8 = lane % 8, c4 = lane / 8;
    const i64 rows8 = mpad / 8;
    const i64 rg = grp % rows8, cq = grp / rows8;
    const i64 row = rg * 8 + r8;
    const i64 kc = cq * 4 + c4;
    if (kc >= kchunks) continue;
    double xs[16];
    if (row < m) {
      const double* src = A + row * lda + kc * 16;
      if (kc * 16 + 16 <= k && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const double2 t = __ldg(reinterpret_cast<const double2*>(src + e));
          xs[e] = t.x;
          xs[e + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) xs[e] = kc * 16 + e < k ? src[e] : 0.0;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) xs[e] = 0.0;
    }
    const i64 rb = row / kBM, kb = kc / (kBK / 16);
    const int c = static_cast<int>(kc % (kBK / 16)), g = static_cast<int>((row % kBM) / 8);
    uint8_t* base = out + ((rb * KB + kb) * P.nmod) * static_cast<i64>(kAStage) + ((c * (kBM / 8) + g) * 8 + r8) * 16;
    store_residue_planes<MODE>(xs, P, base, static_cast<i64>(kAStage));
  }
}

// B: k x n residues -> N residue planes of 128-column blocks, K-major.
// Chunk (cb, kb, i), kBStage bytes: [k16 c (kBK / 16)][column group (16)][column (8)][16 B].
// A 128-thread block transposes a 64 (k) x 32 (column) tile through shared memory.
// k-blocks [kb_begin, kb_begin + kb_count) only (the multi-GPU path packs B's
// k-chunks as their broadcast lands); KB is the layout's k-block count.
template <int MODE>
__global__ void __launch_bounds__(128) pack_b_rns(const double* __restrict__ B, i64 ldb, i64 k, i64 n, int KB,
                                                  int NB128, int kb_begin, int kb_count,
                                                  const __grid_constant__ PackParams P, uint8_t* __restrict__ out) {
  constexpr int SW = 32, SUB = kBH / SW, TK = 64, KSUB = kBK / TK;  // 64 (k) x 32 (column) tiles
  __shared__ double tile[TK][SW + 1];
  const i64 tiles = static_cast<i64>(kb_count) * KSUB * NB128 * SUB;
  for (i64 t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int sb = static_cast<int>(t % SUB);
    const i64 cb = (t / SUB) % NB128, kq = t / (SUB * static_cast<i64>(NB128));
    const i64 kb = kb_begin + kq / KSUB;
    const int ks = static_cast<int>(kq % KSUB);  // 64-row slice of the k-block
    __syncthreads();
    for (int e = threadIdx.x; e < TK * SW; e += blockDim.x) {
      const int kr = e / SW, cc = e % SW;
      const i64 kk = kb * kBK + ks * TK + kr, col = cb * kBH + sb * SW + cc;
      tile[kr][cc] = (kk < k && col < n) ? B[kk * ldb + col] : 0.0;
    }
    __syncthreads();
    const int cc = threadIdx.x % SW;  // column
    {
      const int qt = threadIdx.x / SW;     // k16 chunk within the tile
      const int q = ks * (TK / 16) + qt;   // ... within the k-block
      double xs[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) xs[e] = tile[qt * 16 + e][cc];
      const int nn = sb * SW + cc, g = nn / 8, r8 = nn % 8;
      uint8_t* base =
          out + ((cb * KB + kb) * P.nmod) * static_cast<i64>(kBStage) + ((q * (kBH / 8) + g) * 8 + r8) * 16;
      store_residue_planes<MODE>(xs, P, base, static_cast<i64>(kBStage));
    }
  }
}

// The same packing without the shared-memory transpose: thread (k16 chunk,
// column) reads its 16 k values straight from B, consecutive threads walking
// consecutive columns, so each of the 16 loads of a warp is 256 contiguous
// bytes of one row of B; the stores are pack_a_rns's.
template <int MODE>
__global__ void __launch_bounds__(256) pack_b_rns_direct(const double* __restrict__ B, i64 ldb, i64 k, i64 n, int KB,
                                                         int NB128, int kb_begin, int kb_count,
                                                         const __grid_constant__ PackParams P,
                                                         uint8_t* __restrict__ out) {
  // grid: x over 256-column groups of the padded width, y strided over k16
  // chunks (no 64-bit division per item; a full chunk loads unconditionally)
  const i64 col = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 chunks = static_cast<i64>(kb_count) * (kBK / 16);
  const i64 cb = col / kBH;
  const int nn = static_cast<int>(col % kBH), g = nn / 8, r8 = nn % 8;
  uint8_t* const colbase = out + (cb * KB * P.nmod) * static_cast<i64>(kBStage) + (g * 8 + r8) * 16;
  for (i64 cq = blockIdx.y; cq < chunks; cq += gridDim.y) {
    const i64 kc = static_cast<i64>(kb_begin) * (kBK / 16) + cq;  // global k16 chunk
    const i64 k0 = kc * 16;
    double xs[16];
    if (col < n) {
      const double* src = B + k0 * ldb + col;
      if (k0 + 16 <= k) {
#pragma unroll
        for (int e = 0; e < 16; ++e, src += ldb) xs[e] = __ldg(src);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) xs[e] = k0 + e < k ? __ldg(src + e * ldb) : 0.0;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) xs[e] = 0.0;
    }
    const i64 kb = kc / (kBK / 16);
    const int q = static_cast<int>(kc % (kBK / 16));
    uint8_t* base = colbase + (kb * P.nmod) * static_cast<i64>(kBStage) + (q * (kBH / 8)) * 8 * 16;
    store_residue_planes<MODE>(xs, P, base, static_cast<i64>(kBStage));
  }
}

// ------------------------------------------------------------------ GEMM
// Work item t (0 <= t < MB * NB * splits) -> pair tile (tm, tn), split ks;
// grouped rasterisation keeps a wave's panels of one modulus in L2.
struct Item {
  int tm, tn, ks;
};
__device__ __forceinline__ Item item_of(int t, const Params& P) {
  const int tiles = P.MB * P.NB;
  const int r = t % tiles;
  const int in_group = P.group * P.NB;
  const int first_m = (r / in_group) * P.group;
  const int gsz = min(P.MB - first_m, P.group);
  Item it;
  it.tm = first_m + (r % in_group) % gsz;
  it.tn = (r % in_group) / gsz;
  it.ks = t / tiles;
  return it;
}

// a * b + c with a 32 x 32 -> 64-bit product (one IMAD.WIDE.U32)
__device__ __forceinline__ unsigned long long mad_wide(uint32_t a, uint32_t b, unsigned long long c) {
  unsigned long long d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

__device__ __forceinline__ uint64_t barrett(uint64_t x, uint64_t p, uint64_t mu) {
  const uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * p;
  return r >= p ? r - p : r;
}

// Scratch addressing (per CTA slot): [modulus][half][c16 (8)][row (128)][16 B]
__device__ __forceinline__ uint4* scratch_at(uint8_t* slot, int i, int half, int c16, int row) {
  return reinterpret_cast<uint4*>(slot + ((((static_cast<i64>(i) * 2 + half) * 8 + c16) * kBM + row) * 16));
}

// Reduce 32 TMEM columns (one tcgen05.ld) mod m and park them as 2 x 16 bytes.
// SMALL: every product is below 2^24 (K segments of <= 258 terms, e.g. the
// k = 256 outer-product shape), so mod_small applies to it directly.
template <bool SMALL>
__device__ __forceinline__ void reduce32(const uint32_t (&v)[32], uint32_t negm, uint32_t c16, uint32_t magic,
                                         uint32_t (&w)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t t = v[q * 4 + e];
      const uint32_t s = SMALL ? t : (t >> 16) * c16 + (t & 0xFFFFu);  // < 2^24 <= 2^32 / m, == t mod m
      r[e] = mod_small(s, negm, magic);
    }
    w[q] = pack4(r[0], r[1], r[2], r[3]);
  }
}

template <bool SMALL>
__device__ __forceinline__ void park32(const uint32_t (&v)[32], uint32_t m, uint32_t negm, uint32_t c16, uint32_t magic,
                                       bool acc, uint4* dst0, uint4* dst1) {
  uint32_t w[8];
  reduce32<SMALL>(v, negm, c16, magic, w);
  if (acc) {  // earlier K segments: add the parked residues mod m
    const uint4 o0 = *dst0, o1 = *dst1;
    const uint32_t o[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t s = ((w[q] >> (8 * e)) & 0xFFu) + ((o[q] >> (8 * e)) & 0xFFu);
        s = s >= m ? s - m : s;
        word |= s << (8 * e);
      }
      w[q] = word;
    }
  }
  // streaming stores: read back only by the CRT kernel
  __stcs(dst0, make_uint4(w[0], w[1], w[2], w[3]));
  __stcs(dst1, make_uint4(w[4], w[5], w[6], w[7]));
}

// The n residue words of 4-column step c (SPLIT: the slices' residues summed mod m_i).
template <bool SPLIT>
__device__ __forceinline__ void crt_load(const CrtParams& P, const uint8_t* __restrict__ pthr, i64 slice_stride, int c,
                                         uint32_t (&rw)[kMaxMod]) {
  const uint8_t* pc = pthr + (c >> 2) * (16 * kBM) + (c & 3) * 4;
#pragma unroll
  for (int i = 0; i < kMaxMod; ++i) {
    if (i >= P.nmod) {
      rw[i] = 0;
    } else if (!SPLIT) {
      rw[i] = __ldg(reinterpret_cast<const uint32_t*>(pc + i * kSlotPerMod));
    } else {
      uint32_t r = *reinterpret_cast<const uint32_t*>(pc + i * kSlotPerMod);
      for (int s = 1; s < P.splits; ++s) {  // add the other slices' residues mod m_i
        const uint32_t o = *reinterpret_cast<const uint32_t*>(pc + s * slice_stride + i * kSlotPerMod);
        uint32_t out = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t v = ((r >> (8 * e)) & 0xFFu) + ((o >> (8 * e)) & 0xFFu);
          v = v >= P.mod[i] ? v - P.mod[i] : v;
          out |= v << (8 * e);
        }
        r = out;
      }
      rw[i] = r;
    }
  }
}

// CRT of the 4 columns of step c from their residue words -> C.
template <int WPL>
__device__ __forceinline__ void crt_step(const CrtParams& P, int c, i64 colh, double* __restrict__ dst_row,
                                         const uint32_t (&rw)[kMaxMod]) {
  const i64 col0 = colh + c * 4;
  if (col0 >= P.n) return;
  const unsigned long long p = P.p;
  const int ngroups = (P.nmod + 3) / 4;
  uint32_t acc[4][kCrtPlanes];
#pragma unroll
  for (int e = 0; e < 4; ++e)
#pragma unroll
    for (int b = 0; b < kCrtPlanes; ++b) acc[e][b] = 0;  // planes WPL..6 stay zero
#pragma unroll
  for (int gi = 0; gi < kCrtGroups; ++gi) {
    if (gi >= ngroups) break;
    // transpose: t[e] = the four moduli's residues of column e
    const uint32_t a0 = rw[4 * gi], a1 = rw[4 * gi + 1], a2 = rw[4 * gi + 2], a3 = rw[4 * gi + 3];
    const uint32_t u0 = __byte_perm(a0, a1, 0x5140), u1 = __byte_perm(a0, a1, 0x7362);
    const uint32_t u2 = __byte_perm(a2, a3, 0x5140), u3 = __byte_perm(a2, a3, 0x7362);
    const uint32_t t[4] = {__byte_perm(u0, u2, 0x5410), __byte_perm(u0, u2, 0x7632), __byte_perm(u1, u3, 0x5410),
                           __byte_perm(u1, u3, 0x7632)};
#pragma unroll
    for (int b = 0; b < kCrtPlanes; ++b) {
      if (b >= WPL && b < 7) continue;  // W_i < p < 2^(8 WPL): planes WPL..6 are zero
      const uint32_t wb = P.wb[gi][b];
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e][b] = __dp4a(t[e], wb, acc[e][b]);
    }
  }
  double out[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t* a = acc[e];
    // t = round(F / 2^19), F = a7 + 2^8 a8 + 2^16 a9: with u = a8 + 2^8 a9 + (a7 >> 8),
    // F = 2^8 u + (a7 & 255) and t = (u + 2^10) >> 11 exactly (32-bit)
    const uint32_t tt = (a[8] + (a[9] << 8) + (a[7] >> 8) + 1024u) >> 11;
    // S = sum_i r_i W_i = sum_b 2^(8b) a_b (b < WPL)
    unsigned long long sm;
    if (P.nmod <= 16) {  // S = sum_i r_i W_i <= 16 * 255 * (p - 1) < 2^64
      // planes 0..3 by 32x32 -> 64-bit multiply-adds, planes 4..6 on the high
      // word in 32-bit wrap-around (S < 2^64 makes the sum exact mod 2^64)
      unsigned long long S = a[0];
#pragma unroll
      for (int b = 1; b < (WPL < 4 ? WPL : 4); ++b) S = mad_wide(a[b], 1u << (8 * b), S);
      if (WPL > 4) {
        uint32_t hi = a[4];
#pragma unroll
        for (int b = 5; b < WPL; ++b) hi += a[b] << (8 * (b - 4));
        S += static_cast<unsigned long long>(hi) << 32;
      }
      // q = floor(S/p) - {0,1,2}: (S >> s) < 2^32, inv32 = floor(2^(s+32)/p)
      const uint32_t q = __umulhi(static_cast<uint32_t>(S >> P.s_shift), P.inv32);
      unsigned long long r = S - mad_wide(q, static_cast<uint32_t>(p), 0ull) - (static_cast<unsigned long long>(q * static_cast<uint32_t>(p >> 32)) << 32);
      r = r >= p ? r - p : r;
      sm = r >= p ? r - p : r;
    } else {
      const unsigned long long lo = a[0] + (static_cast<unsigned long long>(a[1]) << 8) +
                                    (static_cast<unsigned long long>(a[2]) << 16) +
                                    (static_cast<unsigned long long>(a[3]) << 24);  // < 2^45
      const unsigned long long hi = a[4] + (static_cast<unsigned long long>(a[5]) << 8) +
                                    (static_cast<unsigned long long>(a[6]) << 16);  // < 2^37
      sm = barrett(dev::shoup_mulmod(hi, P.two32, P.two32_sh, p) + lo, p, P.mu);
    }
    // t M mod p: t < 2^12 (n <= 16), a 32-bit Shoup product leaves [0, 2p)
    unsigned long long tmod;
    if (P.nmod <= 16) {
      const uint32_t qt = __umulhi(tt, P.Mp_sh32);
      const unsigned long long tm = mad_wide(tt, static_cast<uint32_t>(P.Mp), 0ull) +
                                    (static_cast<unsigned long long>(tt * static_cast<uint32_t>(P.Mp >> 32)) << 32) -
                                    mad_wide(qt, static_cast<uint32_t>(p), 0ull) -
                                    (static_cast<unsigned long long>(qt * static_cast<uint32_t>(p >> 32)) << 32);
      tmod = tm >= p ? tm - p : tm;
    } else {
      tmod = dev::shoup_mulmod(tt, P.Mp, P.Mp_sh, p);
    }
    const unsigned long long r = sm >= tmod ? sm - tmod : sm + p - tmod;
    out[e] = __longlong_as_double(static_cast<long long>(r | 0x4330000000000000ull)) - 4503599627370496.0;
  }
  double* dst = dst_row + c * 4;
  if (col0 + 4 <= P.n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    *reinterpret_cast<double2*>(dst) = make_double2(out[0], out[1]);
    *reinterpret_cast<double2*>(dst + 2) = make_double2(out[2], out[3]);
  } else {
    for (int e = 0; e < 4 && col0 + e < P.n; ++e) dst[e] = out[e];
  }
}

// CRT of one thread's 128 columns, four per step; all n residue words of a
// step are loaded before any is used.  (Pipelining the next step's loads
// measured 15-20% slower: the extra registers cost a resident block per SM.)
template <int WPL, bool SPLIT>
__device__ __forceinline__ void crt_row(const CrtParams& P, const uint8_t* __restrict__ pthr, i64 slice_stride,
                                        i64 colh, double* __restrict__ dst_row) {
#pragma unroll 1
  for (int c = 0; c < (kNT / 2) / 4; ++c) {
    if (colh + c * 4 >= P.n) break;
    uint32_t rw[kMaxMod];
    crt_load<SPLIT>(P, pthr, slice_stride, c, rw);
    crt_step<WPL>(P, c, colh, dst_row, rw);
  }
}

// ---- CRT specialised on the plane and group counts (splits == 1) ----
// The generic crt_step above spends ~156 instructions per element at n = 15
// (ncu source page, profiles/round2): runtime modulus / plane checks, the
// accumulators zeroed before the first dp4a, constants fetched with LDC, one
// 4-byte load per modulus and 4 columns.  With WPL (byte planes of W_i) and
// NG (groups of four moduli) compile-time, every dp4a takes its weight word
// straight from the constant bank, the first group initialises the planes,
// and each modulus' 16-byte chunk of a row is loaded once (CW columns per
// load) for CW / 4 steps.

// 4 columns -> 4 outputs mod p from the n residue words of the columns
// (rw[i]: modulus i, bytes = columns).  Same arithmetic as crt_step.
// FIN64: the finalisation on the FP64 pipe where the host allows it (P.fp64fin):
// rns_tile_kernel, whose epilogue is bound by the FMA-heavy pipe (C5 -1.2%); the
// standalone CRT kernel is not, and ran 2-4% slower with it
template <int WPL, int NG, bool FIN64 = false>
__device__ __forceinline__ void crt4_spec(const CrtParams& P, const uint32_t (&rw)[4 * NG], double (&out)[4]) {
  constexpr int NP = WPL + 3;  // planes: W bytes 0..WPL-1, then g bytes 0..2
  uint32_t acc[4][NP];
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    const uint32_t a0 = rw[4 * gi], a1 = rw[4 * gi + 1], a2 = rw[4 * gi + 2], a3 = rw[4 * gi + 3];
    const uint32_t u0 = __byte_perm(a0, a1, 0x5140), u1 = __byte_perm(a0, a1, 0x7362);
    const uint32_t u2 = __byte_perm(a2, a3, 0x5140), u3 = __byte_perm(a2, a3, 0x7362);
    const uint32_t t[4] = {__byte_perm(u0, u2, 0x5410), __byte_perm(u0, u2, 0x7632), __byte_perm(u1, u3, 0x5410),
                           __byte_perm(u1, u3, 0x7632)};
#pragma unroll
    for (int pb = 0; pb < NP; ++pb) {
      const uint32_t wb = P.wb[gi][pb < WPL ? pb : 7 + (pb - WPL)];
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e][pb] = __dp4a(t[e], wb, gi == 0 ? 0u : acc[e][pb]);
    }
  }
  const unsigned long long p = P.p;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t* a = acc[e];
    const uint32_t g0 = a[WPL], g1 = a[WPL + 1], g2 = a[WPL + 2];
    // t = round(F / 2^19), F = g0 + 2^8 g1 + 2^16 g2 (see crt_step)
    const uint32_t tt = (g1 + (g2 << 8) + (g0 >> 8) + 1024u) >> 11;
    if (FIN64 && WPL <= 5 && NG <= 4 && P.fp64fin) {
      // R = S + (T0 - t) Mp + C0 on the FP64 pipe (idle in this kernel; the
      // integer pipes carry the dp4a planes).  Host-checked R_max < 2^53: every
      // partial sum is a non-negative integer below R_max, so exact; q =
      // rint(R fl(1/p)) is within 1/2 + 2^-11 of R/p, so r = R - q p (exact,
      // |r| <= p/2 + 1) needs one conditional + p.
      const double two52 = 4503599627370496.0, M = 6755399441055744.0;
      double S = __hiloint2double(0x43300000, static_cast<int>(a[0])) - two52;
#pragma unroll
      for (int b = 1; b < WPL; ++b)
        S = __fma_rn(__hiloint2double(0x43300000, static_cast<int>(a[b])) - two52, static_cast<double>(1ull << (8 * b)), S);
      const double ud = __hiloint2double(0x43300000, static_cast<int>(P.T0 - tt)) - two52;
      const double R = __fma_rn(ud, P.Mp_d, S) + P.C0_d;
      const double q = __fma_rn(R, P.invp_d, M) - M;
      const double r = __fma_rn(-q, P.p_d, R);
      out[e] = r < 0.0 ? r + P.p_d : r;
      continue;
    }
    if (NG <= 4 && P.comb) {
      // R = C0 + S + (T0 - t) Mp, every term non-negative, R < 2^64
      // planes 0 and 1 in 32 bits (each plane < 16 255^2 < 2^20, so a0 + 2^8 a1 < 2^29):
      // one ALU LEA instead of a 64-bit multiply-add on the FMA-heavy pipe
      unsigned long long R = P.C0 + (WPL > 1 ? a[0] + (a[1] << 8) : a[0]);
#pragma unroll
      for (int b = 2; b < (WPL < 4 ? WPL : 4); ++b) R = mad_wide(a[b], 1u << (8 * b), R);
      uint32_t hi = 0;
#pragma unroll
      for (int b = 4; b < WPL; ++b) hi += a[b] << (8 * (b - 4));
      const uint32_t u = P.T0 - tt;
      R = mad_wide(u, static_cast<uint32_t>(P.Mp), R);
      R += static_cast<unsigned long long>(hi + u * static_cast<uint32_t>(P.Mp >> 32)) << 32;
      const uint32_t q = __umulhi(static_cast<uint32_t>(R >> P.s2), P.inv2);
      unsigned long long r = mad_wide(q, static_cast<uint32_t>(P.negp), R) +
                             (static_cast<unsigned long long>(q * static_cast<uint32_t>(P.negp >> 32)) << 32);
      r = r >= p ? r - p : r;
      out[e] = __longlong_as_double(static_cast<long long>(r | 0x4330000000000000ull)) - 4503599627370496.0;
      continue;
    }
    unsigned long long sm, tmod;
    if (NG <= 4) {  // n <= 16: S = sum_i r_i W_i <= 16 * 255 * (p - 1) < 2^64
      unsigned long long S = a[0];
#pragma unroll
      for (int b = 1; b < (WPL < 4 ? WPL : 4); ++b) S = mad_wide(a[b], 1u << (8 * b), S);
      if (WPL > 4) {
        uint32_t hi = a[4];
#pragma unroll
        for (int b = 5; b < WPL; ++b) hi += a[b] << (8 * (b - 4));
        S += static_cast<unsigned long long>(hi) << 32;
      }
      const uint32_t q = __umulhi(static_cast<uint32_t>(S >> P.s_shift), P.inv32);
      unsigned long long r = S - mad_wide(q, static_cast<uint32_t>(p), 0ull) -
                             (static_cast<unsigned long long>(q * static_cast<uint32_t>(p >> 32)) << 32);
      r = r >= p ? r - p : r;
      sm = r >= p ? r - p : r;
      const uint32_t qt = __umulhi(tt, P.Mp_sh32);
      const unsigned long long tm = mad_wide(tt, static_cast<uint32_t>(P.Mp), 0ull) +
                                    (static_cast<unsigned long long>(tt * static_cast<uint32_t>(P.Mp >> 32)) << 32) -
                                    mad_wide(qt, static_cast<uint32_t>(p), 0ull) -
                                    (static_cast<unsigned long long>(qt * static_cast<uint32_t>(p >> 32)) << 32);
      tmod = tm >= p ? tm - p : tm;
    } else {
      unsigned long long lo = a[0];
#pragma unroll
      for (int b = 1; b < (WPL < 4 ? WPL : 4); ++b) lo += static_cast<unsigned long long>(a[b]) << (8 * b);
      unsigned long long hi = 0;
#pragma unroll
      for (int b = 4; b < WPL; ++b) hi += static_cast<unsigned long long>(a[b]) << (8 * (b - 4));
      sm = barrett(dev::shoup_mulmod(hi, P.two32, P.two32_sh, p) + lo, p, P.mu);
      tmod = dev::shoup_mulmod(tt, P.Mp, P.Mp_sh, p);
    }
    const unsigned long long r = sm >= tmod ? sm - tmod : sm + p - tmod;
    out[e] = __longlong_as_double(static_cast<long long>(r | 0x4330000000000000ull)) - 4503599627370496.0;
  }
}

// columns per residue load (4, 8 or 16 bytes): the whole 16-byte chunk for up
// to 8 moduli (more bytes in flight per thread, coalesced 512-byte warp
// loads), 8 bytes above (register budget)
#ifndef FPMM_B200_CRT_PREFETCH
#define FPMM_B200_CRT_PREFETCH 1
#endif
template <int NG>
constexpr int crt_cw() {
  return NG <= 2 ? 16 : 8;
}

template <int CW>
struct CrtWord;
template <>
struct CrtWord<4> {
  using T = uint32_t;
  static __device__ __forceinline__ void split(T v, uint32_t (&w)[1]) { w[0] = v; }
};
template <>
struct CrtWord<8> {
  using T = uint2;
  static __device__ __forceinline__ void split(T v, uint32_t (&w)[2]) { w[0] = v.x, w[1] = v.y; }
};
template <>
struct CrtWord<16> {
  using T = uint4;
  static __device__ __forceinline__ void split(T v, uint32_t (&w)[4]) { w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w; }
};

// One CTA per (tile, CTA half of the pair), one thread per row half: the
// 128 columns of its row half in 16-column chunks ([i][half][c16][row][16 B]).
template <int WPL, int NG>
__global__ void __launch_bounds__(256) rns_crt_spec_kernel(const __grid_constant__ CrtParams P) {
  constexpr int kCrtCW = crt_cw<NG>();
  using W = CrtWord<kCrtCW>;
  const int tile = blockIdx.x >> 1, rank = blockIdx.x & 1;
  const int row_in_tile = threadIdx.x % kBM, half = threadIdx.x / kBM;
  Params q{};
  q.MB = P.MB, q.NB = P.NB, q.splits = 1, q.group = P.group;
  const Item it = item_of(tile, q);
  const i64 row = (2 * static_cast<i64>(it.tm) + rank) * kBM + row_in_tile;
  if (row >= P.m) return;
  const i64 colh = static_cast<i64>(it.tn) * kNT + half * (kNT / 2);
  const uint8_t* pthr = P.R + (static_cast<i64>(tile) * 2 + rank) * P.nmod * kSlotPerMod +
                        (static_cast<i64>(half) * 8 * kBM + row_in_tile) * 16;
  double* dst_row = P.C + row * P.ldc + colh;
  // the residue words of chunk cl (register double buffer: the next chunk's
  // loads are in flight while this one is reconstructed)
  auto load = [&](int cl, uint32_t (&w)[4 * NG][kCrtCW / 4]) {
    const uint8_t* pc = pthr + (cl / 16) * (16 * kBM) + (cl % 16);
#pragma unroll
    for (int i = 0; i < 4 * NG; ++i) {
      typename W::T v{};
      if (i < 4 * (NG - 1) || i < P.nmod) v = __ldg(reinterpret_cast<const typename W::T*>(pc + i * kSlotPerMod));
      W::split(v, w[i]);
    }
  };
  // prefetch up to 8 moduli (20-25 bits at K = 8192: 0.285 -> 0.241 ms);
  // beyond, the second buffer costs more occupancy than it hides latency
  // (36 bits: flat, 52 bits: 0.32 -> 0.39 ms)
  constexpr bool kPF = FPMM_B200_CRT_PREFETCH && NG <= 2;
  auto emit = [&](int cl, const uint32_t (&cur)[4 * NG][kCrtCW / 4]) {
#pragma unroll
    for (int s = 0; s < kCrtCW / 4; ++s) {
      const i64 col0 = colh + cl + 4 * s;
      if (col0 >= P.n) break;
      uint32_t rw[4 * NG];
#pragma unroll
      for (int i = 0; i < 4 * NG; ++i) rw[i] = cur[i][s];
      double out[4];
      crt4_spec<WPL, NG>(P, rw, out);
      double* dst = dst_row + cl + 4 * s;
      if (col0 + 4 <= P.n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        *reinterpret_cast<double2*>(dst) = make_double2(out[0], out[1]);
        *reinterpret_cast<double2*>(dst + 2) = make_double2(out[2], out[3]);
      } else {
        for (int e = 0; e < 4 && col0 + e < P.n; ++e) dst[e] = out[e];
      }
    }
  };
  if constexpr (kPF) {
    const int cend = static_cast<int>(min(static_cast<i64>(kNT / 2), P.n - colh));
    uint32_t w[4 * NG][kCrtCW / 4];
    if (cend > 0) load(0, w);
#pragma unroll 1
    for (int cl = 0; cl < cend; cl += kCrtCW) {
      uint32_t cur[4 * NG][kCrtCW / 4];
#pragma unroll
      for (int i = 0; i < 4 * NG; ++i)
#pragma unroll
        for (int s = 0; s < kCrtCW / 4; ++s) cur[i][s] = w[i][s];
      if (cl + kCrtCW < cend) load(cl + kCrtCW, w);
      emit(cl, cur);
    }
  } else {
#pragma unroll 1
    for (int cl = 0; cl < kNT / 2; cl += kCrtCW) {
      if (colh + cl >= P.n) break;
      const uint8_t* pc = pthr + (cl / 16) * (16 * kBM) + (cl % 16);
      uint32_t w[4 * NG][kCrtCW / 4];
#pragma unroll
      for (int i = 0; i < 4 * NG; ++i) {
        typename W::T v{};
        if (i < 4 * (NG - 1) || i < P.nmod) v = __ldg(reinterpret_cast<const typename W::T*>(pc + i * kSlotPerMod));
        W::split(v, w[i]);
      }
#pragma unroll
      for (int s = 0; s < kCrtCW / 4; ++s) {
        const i64 col0 = colh + cl + 4 * s;
        if (col0 >= P.n) break;
        uint32_t rw[4 * NG];
#pragma unroll
        for (int i = 0; i < 4 * NG; ++i) rw[i] = w[i][s];
        double out[4];
        crt4_spec<WPL, NG>(P, rw, out);
        double* dst = dst_row + cl + 4 * s;
        if (col0 + 4 <= P.n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          *reinterpret_cast<double2*>(dst) = make_double2(out[0], out[1]);
          *reinterpret_cast<double2*>(dst + 2) = make_double2(out[2], out[3]);
        } else {
          for (int e = 0; e < 4 && col0 + e < P.n; ++e) dst[e] = out[e];
        }
      }
    }
  }
}

// WPL = byte planes of W_i (ceil(bits(p - 1) / 8)): the kernel skips the zero planes.
template <int WPL>
__global__ void __launch_bounds__(256) rns_crt_kernel(const __grid_constant__ CrtParams P) {
  const int tile = blockIdx.x >> 1, rank = blockIdx.x & 1;
  const int row_in_tile = threadIdx.x % kBM, half = threadIdx.x / kBM;
  Params q{};
  q.MB = P.MB, q.NB = P.NB, q.splits = P.splits, q.group = P.group;
  const Item it = item_of(tile, q);  // the tile of items t = tile + s * tiles (s = split)
  const i64 row = (2 * static_cast<i64>(it.tm) + rank) * kBM + row_in_tile;
  if (row >= P.m) return;
  const i64 colh = static_cast<i64>(it.tn) * kNT + half * (kNT / 2);
  const i64 tiles = static_cast<i64>(P.MB) * P.NB;
  // this thread's bytes in the tile's residue block: modulus i, 8-column step c at
  // i * kSlotPerMod + (c / 2) * 16 kBM + (c % 2) * 8 (see scratch_at)
  const uint8_t* pthr = P.R + (static_cast<i64>(tile) * 2 + rank) * P.nmod * kSlotPerMod +
                        (static_cast<i64>(half) * 8 * kBM + row_in_tile) * 16;
  const i64 slice_stride = tiles * 2 * P.nmod * kSlotPerMod;
  double* dst_row = P.C + row * P.ldc + colh;
  if (P.splits == 1) crt_row<WPL, false>(P, pthr, slice_stride, colh, dst_row);
  else crt_row<WPL, true>(P, pthr, slice_stride, colh, dst_row);
}

// ---- CTA-pair plumbing ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(dev::smem_u32(p)), "r"(rank));
  return out;
}
// Arrive on a (possibly remote) barrier of the pair, default .release.cta
// semantics.  Only the epilogue's TMEM drain uses it: its tcgen05.ld values are
// already in registers (tcgen05.wait::ld + fence::before_thread_sync), so the
// MMA may overwrite the accumulator.  A .release.cluster arrive also waited for
// the thread's earlier streaming stores of parked residues to reach L2 (an
// ERRBAR: 24% of the stall samples at k = 256, where passes are short).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra LAB_DONE;\n"
      "bra LAB_WAIT;\n"
      "LAB_DONE:\n"
      "}\n" ::"r"(dev::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z));
}
// Pair TMA load of one stage chunk (row `row` of the 128-byte view) into this
// CTA's shared memory, completing on the LEADER's barrier at the same offset
// (peer bit cleared), so the leader's one barrier tracks both halves.
__device__ __forceinline__ void tma_pair_load(void* dst, const CUtensorMap* map, int row, uint64_t* bar) {
  const uint32_t leader_bar = dev::smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(dev::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(leader_bar)
      : "memory");
}
// arrive on the barrier at this offset in both CTAs of the pair once the MMAs issued so far completed
// The same from a converged warp: every lane executes the asm with identical
// (warp-uniform) operands, so they stay in uniform registers, and the one lane
// elect.sync picks issues the instruction (the single-thread form moved every
// descriptor to uniform registers with R2UR inside a BRA.U.ANY loop per MMA).
__device__ __forceinline__ void mma_i8_pair_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5, %5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z));
}
__device__ __forceinline__ void commit_pair_warp(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
      "}\n" ::"r"(dev::smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          dev::smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}

// Pacing (long K): rank 0's producer of every pair publishes the k-blocks it
// has issued in progress[pair] (relaxed: a hint, never a correctness
// condition).  Warp 1 of rank 1 (idle otherwise) is the pair's monitor: it
// keeps the minimum over all pairs in both CTAs' shared memory, and a producer
// that is pace_kb k-blocks ahead of that minimum sleeps until the slowest pair
// catches up (bounded: after ~2 ms of waiting it stops pacing).
__device__ __forceinline__ void pace_publish(int* slot, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;\n" ::"l"(slot), "r"(v) : "memory");
}
__device__ __forceinline__ int pace_load(const int* slot) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(slot) : "memory");
  return v;
}
__device__ __forceinline__ void st_shared_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}

// The pair's work items (modulus i, item t) in order.  flat: one sequence over i * total + t, so every pair runs the same number of items (+-1) and
// the pairs that share a wave's panels stay in lockstep across moduli;
// otherwise each modulus restarts at t = pair (pairs with one item fewer per
// modulus run ahead into the next modulus).
struct PassIter {
  int i, t;
  __device__ __forceinline__ PassIter(int pair) : i(0), t(pair) {}
  __device__ __forceinline__ void next(const Params& P, int pair, int npairs, int total) {
    if (P.flat) {  // g = i * total + t advances by npairs
      t += npairs;
      while (t >= total) t -= total, ++i;
    } else {
      t += npairs;
      if (t >= total) ++i, t = pair;
    }
  }
  __device__ __forceinline__ bool valid(const Params& P, int total) const { return i < P.nmod && t < total; }
};

// The pair (cluster of 2 CTAs on neighbouring SMs) computes a 256 x 256 tile:
// CTA r holds rows 128 r.. of A and columns 128 r.. of B in its shared
// memory and rows 128 r.. of the accumulator in its TMEM; the leader (r = 0)
// issues M=256 N=256 K=32 cta_group::2 MMAs that read both halves.  Each SM
// so streams 4 KB of A and 4 KB of B per 128-cycle K=32 step (64 B/clk); a
// stage holds kBK / 32 such steps.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) rns_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);  // leader: both halves landed
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;   // [2] leader: both CTAs drained accumulator b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  volatile int* pace_floor = reinterpret_cast<volatile int*>(tmem_slot + 1);  // monitor's min over pairs

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int total = P.MB * P.NB * P.splits;

  if (threadIdx.x == 0) {
    *pace_floor = 0;
    for (int s = 0; s < kStages; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      dev::mbar_init(&tmem_full[b], 1);
      dev::mbar_init(&tmem_empty[b], 2 * (P.pingpong ? kEpiWarps / 2 : kEpiWarps));
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        dev::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  i8::fence_before();
  cluster_sync();
  i8::fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own A rows, own B columns) ----------------
    // The leader's full[s] expects both CTAs' bytes; each CTA's loads
    // complete on it, so the leader's one wait covers the pair.
    if (lane == 0) {
      // (measured and rejected: L2 evict_last/evict_first hints for A/B, -2..10%;
      // cp.async.bulk.prefetch.L2 8..64 k-blocks ahead, -9..19%)
      int g = 0;
      bool pace = P.pace_kb > 0 && P.progress != nullptr;
      for (PassIter pi(pair); pi.valid(P, total); pi.next(P, pair, npairs, total)) {
        {
          const int i = pi.i, t = pi.t;
          const Item it = item_of(t, P);
          const int kb0 = it.ks * P.kb_per_split;
          const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
          const i64 rb = 2 * static_cast<i64>(it.tm) + rank, cb = 2 * static_cast<i64>(it.tn) + rank;
          // chunk (block, kb, i) of the [block][k-block][modulus] layout: k-blocks nmod chunks apart
          const int rowA = static_cast<int>(((rb * P.KB + kb0) * P.nmod + i) * (kAStage / 128));
          const int rowB = static_cast<int>(((cb * P.KB + kb0) * P.nmod + i) * (kBStage / 128));
          const int kstep = P.nmod * (kAStage / 128);
          for (int kb = 0; kb < nkb; ++kb, ++g) {
            const int s = g % kStages;
            if (pace && g - P.pace_kb > *pace_floor) {
              for (int spin = 0; g - P.pace_kb > *pace_floor; ++spin) {
                if (spin == 20000) {  // ~2 ms: a pair that never started; stop pacing
                  pace = false;
                  break;
                }
                __nanosleep(100);
              }
            }
            if (g >= kStages) dev::mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
            if (P.debug & 16) {  // timing experiment: the barrier skeleton without loads
              if (rank == 0) dev::mbar_arrive(&full[s]);
              continue;
            }
            if (rank == 0) dev::mbar_arrive_expect_tx(&full[s], 2 * kStageBytes);
            tma_pair_load(sA + s * kAStage, &P.tmA, rowA + kb * kstep, &full[s]);
            tma_pair_load(sB + s * kBStage, &P.tmB, rowB + kb * kstep, &full[s]);
            if (pace && rank == 0 && (g & 7) == 7) pace_publish(P.progress + pair, g + 1);
          }
        }
      }
      if (pace && rank == 0) pace_publish(P.progress + pair, 0x7fffffff);  // done: never wait for this pair
    }
  } else if (warp == 1) {
    if (rank == 1 && P.pace_kb > 0 && P.progress != nullptr) {
      // ---------------- pacing monitor (rank 1: warp 1 has no MMA role) ----------------
      const uint32_t peer_floor = peer_addr(const_cast<int*>(pace_floor), 0);
      for (int it = 0;; ++it) {
        int v = 0x7fffffff;
        for (int q = lane; q < npairs; q += 32) v = min(v, pace_load(P.progress + q));
        v = __reduce_min_sync(0xffffffffu, v);
        if (lane == 0) {
          *pace_floor = v;
          st_shared_cluster(peer_floor, v);
        }
        if (v == 0x7fffffff || it > 4000000) break;  // every pair's producer is done
        __nanosleep(500);
      }
    }
#if FPMM_B200_RNS_MMA_WARP
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA, warp 1 converged) ----------------
      // Every lane runs the loop, so descriptors and counters are warp-uniform
      // and live in uniform registers; elect.sync picks the lane that issues
      // each MMA and commit (mma_i8_pair_warp).  The descriptors are the stage
      // bases plus byte offsets >> 4 (address field of the descriptor).
      constexpr uint32_t idesc = i8::instr_desc(kPairM, kNT);
      const uint64_t adesc0 = i8::smem_desc(dev::smem_u32(sA), (kBM / 8) * 128, 128);
      const uint64_t bdesc0 = i8::smem_desc(dev::smem_u32(sB), (kBH / 8) * 128, 128);
      const bool issue = !(P.debug & 4);
      int g = 0, pass = 0;
      for (PassIter pi(pair); pi.valid(P, total); pi.next(P, pair, npairs, total)) {
        const int ks = P.splits == 1 ? 0 : pi.t / (P.MB * P.NB);
        const int kb0 = ks * P.kb_per_split;
        const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
        const int nseg = nkb <= P.seg_kb ? 1 : (nkb + P.seg_kb - 1) / P.seg_kb;
        int kb = 0;
        for (int seg = 0; seg < nseg; ++seg, ++pass) {
          const int b = pass & 1;
          if (!(P.debug & 8)) mbar_wait_cluster(&tmem_empty[b], ((pass >> 1) & 1) ^ 1);
          i8::fence_after();
          const uint32_t tacc = tbase + b * kNT;
          const int kend = min(nkb, kb + P.seg_kb);
          const int kstart = kb;
          for (; kb < kend; ++kb, ++g) {
            const int s = g % kStages;
            dev::mbar_wait(&full[s], (g / kStages) & 1);
            i8::fence_after();
            const uint64_t ad = adesc0 + static_cast<uint64_t>((s * kAStage) >> 4);
            const uint64_t bd = bdesc0 + static_cast<uint64_t>((s * kBStage) >> 4);
#pragma unroll
            for (int tk = 0; tk < kKSteps; ++tk) {
              if (issue)
                mma_i8_pair_warp(tacc, ad + static_cast<uint64_t>((tk * 2 * (kBM / 8) * 128) >> 4),
                                 bd + static_cast<uint64_t>((tk * 2 * (kBH / 8) * 128) >> 4), idesc,
                                 (kb > kstart || tk > 0) ? 1u : 0u);
            }
            commit_pair_warp(&empty[s]);  // frees stage s in both CTAs
          }
          commit_pair_warp(&tmem_full[b]);  // accumulator b complete in both CTAs
        }
      }
    }
#else
    if (rank == 0 && lane == 0) {
      // ---------------- MMA issuer (leader CTA, one thread) ----------------
      constexpr uint32_t idesc = i8::instr_desc(kPairM, kNT);
      int g = 0, pass = 0;
      for (PassIter pi(pair); pi.valid(P, total); pi.next(P, pair, npairs, total)) {
        {
          // only the slice matters here (one thread on the critical path of
          // every pass: no tile arithmetic when there is one slice)
          const int ks = P.splits == 1 ? 0 : pi.t / (P.MB * P.NB);
          const int kb0 = ks * P.kb_per_split;
          const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
          const int nseg = nkb <= P.seg_kb ? 1 : (nkb + P.seg_kb - 1) / P.seg_kb;
          int kb = 0;
          for (int seg = 0; seg < nseg; ++seg, ++pass) {
            const int b = pass & 1;
            if (!(P.debug & 8)) mbar_wait_cluster(&tmem_empty[b], ((pass >> 1) & 1) ^ 1);
            i8::fence_after();
            const uint32_t tacc = tbase + b * kNT;
            const int kend = min(nkb, kb + P.seg_kb);
            const int kstart = kb;
            for (; kb < kend; ++kb, ++g) {
              const int s = g % kStages;
              dev::mbar_wait(&full[s], (g / kStages) & 1);
              i8::fence_after();
              const uint32_t a0 = dev::smem_u32(sA + s * kAStage), b0 = dev::smem_u32(sB + s * kBStage);
#pragma unroll
              for (int tk = 0; tk < kKSteps; ++tk) {
                const uint64_t ad = i8::smem_desc(a0 + tk * 2 * (kBM / 8) * 128, (kBM / 8) * 128, 128);
                const uint64_t bd = i8::smem_desc(b0 + tk * 2 * (kBH / 8) * 128, (kBH / 8) * 128, 128);
                if (!(P.debug & 4)) mma_i8_pair(tacc, ad, bd, idesc, (kb > kstart || tk > 0) ? 1u : 0u);
              }
              commit_pair(&empty[s]);  // frees stage s in both CTAs
            }
            commit_pair(&tmem_full[b]);  // accumulator b complete in both CTAs
          }
        }
      }
    }
#endif
  } else {
    // ---------------- epilogue: warps 2..9 of both CTAs ----------------
    // Pass (modulus i, tile t): T_i mod m_i is parked in the tile's residue
    // block in HBM; rns_crt_kernel rebuilds C after the kernel (the on-chip
    // alternative is rns_tile_kernel, rnstile.cuh).
    // pingpong: warps 2..9 take the even passes (accumulator 0), 10..17 the
    // odd ones, each warp 128 columns; a group reduces and stores one pass
    // while the other drains the next, so short-K passes (k = 256: about as
    // long as their epilogue) no longer serialise MMA and epilogue.
    const bool pp = kEpiWarps == 16 && P.pingpong;
    const int ew = warp - 2;
    const int group = pp ? ew / 8 : 0;
    const int wcols = pp ? 128 : kEpiCols;  // accumulator columns of this warp
    const int quad = warp % 4;
    const int col0 = pp ? ((ew % 8) / 4) * 128 : (ew / 4) * kEpiCols;  // this warp's first accumulator column
    const int half = col0 / (kNT / 2);
    const int row_in_tile = quad * 32 + lane;
    const uint32_t tlane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t leader_tmem_empty = peer_addr(tmem_empty, 0);
    int pass = 0;
    for (PassIter pi(pair); pi.valid(P, total); pi.next(P, pair, npairs, total)) {
      const int i = pi.i, t = pi.t;
      const uint32_t m = P.mod[i], nm = P.negm[i], c16 = P.c16[i], mg = P.magic[i];
      {
        const Item it = item_of(t, P);
        const int kb0 = it.ks * P.kb_per_split;
        const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
        const int nseg = max(1, (nkb + P.seg_kb - 1) / P.seg_kb);
        uint8_t* slot = P.scratch + (static_cast<i64>(t) * 2 + rank) * P.nmod * kSlotPerMod;
        for (int seg = 0; seg < nseg; ++seg, ++pass) {
          const int b = pass & 1;
          if (pp && b != group) continue;  // the other group's pass
          if (P.epi_sleep_ns) dev::mbar_wait_sleep(&tmem_full[b], (pass >> 1) & 1, P.epi_sleep_ns);
          else dev::mbar_wait(&tmem_full[b], (pass >> 1) & 1);
          i8::fence_after();
          const uint32_t tcol = tbase + tlane + b * kNT + half * (kNT / 2);
#if FPMM_B200_RNS_DRAIN_FIRST
          if (!pp) {
            // drain every column of this warp into registers first, then hand
            // the accumulator back and reduce: the MMAs of pass + 2 no longer
            // wait for the reduction and stores (short-K passes, e.g. the
            // k = 256 outer product, are as short as the epilogue itself)
            const int cb = col0 % (kNT / 2);
            uint32_t v[kEpiCols / 32][32];
#pragma unroll
            for (int q = 0; q < kEpiCols / 32; ++q) i8::tmem_ld32(tcol + cb + 32 * q, v[q]);
            i8::tmem_wait_ld();
            i8::fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(leader_tmem_empty + b * 8);
#pragma unroll
            for (int q = 0; q < kEpiCols / 32; ++q) {
              const int c0 = cb + 32 * q;
              uint4* d0 = scratch_at(slot, i, half, c0 / 16, row_in_tile);
              uint4* d1 = scratch_at(slot, i, half, c0 / 16 + 1, row_in_tile);
              if (P.small_t) park32<true>(v[q], m, nm, c16, mg, seg > 0, d0, d1);
              else park32<false>(v[q], m, nm, c16, mg, seg > 0, d0, d1);
            }
          } else if (pp && P.pp_pairs && !(P.debug & 3)) {
            // two 32-column loads per wait: half the drain's load round trips
            // before the release (the MMAs of pass + 2 wait for it)
            const int cend = col0 % (kNT / 2) + wcols;
#pragma unroll 1
            for (int c0 = col0 % (kNT / 2); c0 < cend; c0 += 64) {
              uint32_t v[2][32];
              i8::tmem_ld32(tcol + c0, v[0]);
              i8::tmem_ld32(tcol + c0 + 32, v[1]);
              i8::tmem_wait_ld();
              if (c0 + 64 == cend) {
                i8::fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(leader_tmem_empty + b * 8);
              }
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                uint4* d0 = scratch_at(slot, i, half, (c0 + 32 * q) / 16, row_in_tile);
                uint4* d1 = scratch_at(slot, i, half, (c0 + 32 * q) / 16 + 1, row_in_tile);
                if (P.small_t) park32<true>(v[q], m, nm, c16, mg, seg > 0, d0, d1);
                else park32<false>(v[q], m, nm, c16, mg, seg > 0, d0, d1);
              }
            }
          } else
#endif
#pragma unroll 1
          for (int c0 = col0 % (kNT / 2); c0 < col0 % (kNT / 2) + wcols; c0 += 32) {
            uint32_t v[32];
            i8::tmem_ld32(tcol + c0, v);
            i8::tmem_wait_ld();
            if (c0 + 32 == col0 % (kNT / 2) + wcols) {  // all of this warp's columns are in registers: release
              i8::fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(leader_tmem_empty + b * 8);
            }
            if (P.debug & 2) continue;
            uint4* d0 = scratch_at(slot, i, half, c0 / 16, row_in_tile);
            uint4* d1 = scratch_at(slot, i, half, c0 / 16 + 1, row_in_tile);
            if (P.debug & 1) {  // reduction without the stores (the result kept live)
              uint32_t x = 0;
#pragma unroll
              for (int e = 0; e < 32; ++e) x += mod_small(v[e], nm, mg);
              if (x == 0xFFFFFFFFu) *d0 = make_uint4(x, x, x, x);
              continue;
            }
            if (P.small_t) park32<true>(v, m, nm, c16, mg, seg > 0, d0, d1);
            else park32<false>(v, m, nm, c16, mg, seg > 0, d0, d1);
          }
        }
      }
    }
  }
  i8::fence_before();
  cluster_sync();
  if (warp == 1) {
    i8::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

}  // namespace rns
}  // namespace fpmm_b200
