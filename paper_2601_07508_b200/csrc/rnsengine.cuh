// rnsengine.cuh -- residue-number-system multiword engine on tcgen05 int8.
//
// The multiword idea with the words taken in a residue number system instead
// of a positional base: every centred residue x' = x - p [x > p/2] is
// represented by its residues modulo N pairwise-coprime moduli m_i <= 256
// (one byte each).  The exact integer X = sum_k a'_k b'_k satisfies
// |X| <= K floor(p/2)^2, so with M = prod m_i > 2.001 K floor(p/2)^2 it is
// recovered from its residues r_i = X mod m_i by the CRT, and reduced mod p
// without ever forming X:
//   Z = sum_i r_i y_i M_i  (M_i = M/m_i, y_i = M_i^{-1} mod m_i),  Z = X + t M,
//   t = round(sum_i r_i y_i / m_i)  (|X|/M < 1/2 - 2e-4, fixed point 2^-24),
//   X mod p = (sum_i r_i W_i - t (M mod p)) mod p,  W_i = y_i M_i mod p.
// Each r_i is one exact int8 GEMM: T_i = A_i B_i (u8 x u8 -> s32 in TMEM,
// exact while K_seg 255^2 < 2^32), r_i = T_i mod m_i.  N grows like
// (2 bits(p) + log2 K) / 8 against D^2 = ceil(bits/8)^2 digit products for
// the base-256 engine (15 vs 49 at 52 bits, K = 8192).
//
// One CTA computes a 128 x 256 tile of C, one modulus per pass (N passes),
// M=128 N=256 K=32 MMAs into one of two 256-column TMEM accumulators, so the
// epilogue of pass i overlaps the MMAs of pass i+1.  The epilogue reduces
// T_i mod m_i and parks the residue bytes in a per-CTA L2 scratch slot; after
// the last pass of the tile the same threads read their bytes back and run
// the CRT above, storing C.  No product word ever reaches HBM.
//
// Warp roles (10 warps): 0 TMA producer (1-D bulk copies of pre-packed
// chunks), 1 TMEM allocator + single-thread MMA issuer, 2..9 epilogue (TMEM
// lane quadrant w % 4, column half (w - 2) / 4).
#pragma once

#include <cstdint>

#include "device_common.cuh"
#include "i8engine.cuh"

namespace fpmm_b200 {
namespace rns {

using i64 = std::int64_t;

constexpr int kMaxMod = 20;
constexpr int kBM = 128;            // rows per tile (MMA M)
constexpr int kNT = 256;            // columns per tile (MMA N)
constexpr int kBK = 64;             // k bytes per pipeline stage
constexpr int kKSteps = kBK / 32;   // MMA K = 32 for kind::i8
constexpr int kAStage = kBM * kBK;  // 8 KB
constexpr int kBStage = kNT * kBK;  // 16 KB
constexpr int kStageBytes = kAStage + kBStage;
constexpr int kStages = 8;
constexpr int kThreads = 320;       // 10 warps
constexpr int kEpiWarps = 8;
constexpr int kSmem = kStages * kStageBytes + 1024;
constexpr int kSlotPerMod = kBM * kNT;  // scratch bytes per modulus per tile (32 KB)
constexpr int kGroup = 12;              // tile-rows per rasterisation group

// Per-modulus constants (host: rns_plan in rules.cpp).
struct Params {
  const uint8_t* apack;  // [m-block][modulus][k-block] chunks of kAStage bytes
  const uint8_t* bpack;  // [n-block][modulus][k-block] chunks of kBStage bytes
  double* C;
  uint8_t* scratch;      // per CTA: nmod * kSlotPerMod bytes
  i64 ldc, m, n;
  int MB, NB, KB;
  int nmod;
  int seg_kb;        // k-blocks per exact int32 segment
  int kb_per_split;  // split-K: k-blocks per slice
  int splits;
  i64 split_stride;
  unsigned long long p, mu;            // Barrett: mu = floor(2^64 / p)
  unsigned long long two32, two32_sh;  // 2^32 mod p and its Shoup quotient
  unsigned long long Mp, Mp_sh;        // M mod p and its Shoup quotient
  uint32_t mod[kMaxMod];
  uint32_t c16[kMaxMod];    // 2^16 mod m
  uint32_t magic[kMaxMod];  // ceil(2^37 / m): floor(s/m) = umulhi(s, magic) >> 5 for s < 2^29
  uint32_t g[kMaxMod];      // round(2^24 y_i / m_i)
  uint32_t w_lo[kMaxMod], w_hi[kMaxMod];  // W_i = y_i M_i mod p
};

struct PackParams {
  unsigned long long half_p;  // floor(p/2): x > half_p is centred to x - p
  int nmod;
  uint32_t mod[kMaxMod];
  uint32_t c1[kMaxMod];      // 2^18 mod m
  uint32_t c2[kMaxMod];      // 2^36 mod m
  uint32_t negadd[kMaxMod];  // (m - p mod m) mod m: residue offset of x - p
  uint32_t magic[kMaxMod];
};

__device__ __forceinline__ uint32_t mod_small(uint32_t s, uint32_t m, uint32_t magic) {
  return s - (__umulhi(s, magic) >> 5) * m;
}

// 16 residues (one 16-byte k row of a core matrix) of modulus i
__device__ __forceinline__ uint4 residues16(const uint32_t (&x0)[16], const uint32_t (&x1)[16],
                                            const uint32_t (&x2)[16], const uint32_t (&ng)[16],
                                            const PackParams& P, int i) {
  const uint32_t m = P.mod[i], c1 = P.c1[i], c2 = P.c2[i], na = P.negadd[i], mg = P.magic[i];
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t s = x0[e] + x1[e] * c1 + x2[e] * c2 + ng[e] * na;  // < 2^27
    w[e / 4] |= mod_small(s, m, mg) << (8 * (e % 4));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void split16(const double (&xs)[16], unsigned long long half_p, uint32_t (&x0)[16],
                                        uint32_t (&x1)[16], uint32_t (&x2)[16], uint32_t (&ng)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const unsigned long long x = static_cast<unsigned long long>(xs[e]);
    x0[e] = static_cast<uint32_t>(x) & 0x3FFFFu;
    x1[e] = static_cast<uint32_t>(x >> 18) & 0x3FFFFu;
    x2[e] = static_cast<uint32_t>(x >> 36);
    ng[e] = x > half_p ? 1u : 0u;
  }
}

// A: m x k residues -> N residue planes in the canonical K-major core-matrix
// layout.  Chunk (rb, i, kb), kAStage bytes: [k16 c (4)][row group g (16)][row (8)][16 B].
// Thread (row, 16-element k chunk): reads 16 doubles, writes N x 16 bytes.
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
    uint32_t x0[16], x1[16], x2[16], ng[16];
    split16(xs, P.half_p, x0, x1, x2, ng);
    const i64 rb = row / kBM, kb = kc / (kBK / 16);
    const int c = static_cast<int>(kc % (kBK / 16)), g = static_cast<int>((row % kBM) / 8);
    uint8_t* base = out + ((rb * P.nmod) * KB + kb) * static_cast<i64>(kAStage) + ((c * (kBM / 8) + g) * 8 + r8) * 16;
#pragma unroll 1
    for (int i = 0; i < P.nmod; ++i)
      *reinterpret_cast<uint4*>(base + static_cast<i64>(i) * KB * kAStage) = residues16(x0, x1, x2, ng, P, i);
  }
}

// B: k x n residues -> N residue planes of 256-column blocks, K-major.
// Chunk (cb, i, kb), kBStage bytes: [k16 c (4)][column group (32)][column (8)][16 B].
// A 128-thread block transposes a 64 (k) x 32 (column) tile through shared memory.
__global__ void __launch_bounds__(128) pack_b_rns(const double* __restrict__ B, i64 ldb, i64 k, i64 n, int KB,
                                                  int NB, const __grid_constant__ PackParams P,
                                                  uint8_t* __restrict__ out) {
  constexpr int SW = 32, SUB = kNT / SW;
  __shared__ double tile[kBK][SW + 1];
  const i64 tiles = static_cast<i64>(KB) * NB * SUB;
  for (i64 t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int sb = static_cast<int>(t % SUB);
    const i64 cb = (t / SUB) % NB, kb = t / (SUB * static_cast<i64>(NB));
    __syncthreads();
    for (int e = threadIdx.x; e < kBK * SW; e += blockDim.x) {
      const int kr = e / SW, cc = e % SW;
      const i64 kk = kb * kBK + kr, col = cb * kNT + sb * SW + cc;
      tile[kr][cc] = (kk < k && col < n) ? B[kk * ldb + col] : 0.0;
    }
    __syncthreads();
    const int cc = threadIdx.x % SW, q = threadIdx.x / SW;  // column, k16 chunk
    double xs[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) xs[e] = tile[q * 16 + e][cc];
    uint32_t x0[16], x1[16], x2[16], ng[16];
    split16(xs, P.half_p, x0, x1, x2, ng);
    const int nn = sb * SW + cc, g = nn / 8, r8 = nn % 8;
    uint8_t* base = out + ((cb * P.nmod) * KB + kb) * static_cast<i64>(kBStage) + ((q * (kNT / 8) + g) * 8 + r8) * 16;
#pragma unroll 1
    for (int i = 0; i < P.nmod; ++i)
      *reinterpret_cast<uint4*>(base + static_cast<i64>(i) * KB * kBStage) = residues16(x0, x1, x2, ng, P, i);
  }
}

// ------------------------------------------------------------------ GEMM
struct Item {
  int tm, tn, ks;
};
__device__ __forceinline__ Item item_of(int t, const Params& P) {
  const int tiles = P.MB * P.NB;
  const int r = t % tiles;
  const int in_group = kGroup * P.NB;
  const int first_m = (r / in_group) * kGroup;
  const int gsz = min(P.MB - first_m, kGroup);
  Item it;
  it.tm = first_m + (r % in_group) % gsz;
  it.tn = (r % in_group) / gsz;
  it.ks = t / tiles;
  return it;
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
__device__ __forceinline__ void park32(const uint32_t (&v)[32], uint32_t m, uint32_t c16, uint32_t magic, bool acc,
                                       uint4* dst0, uint4* dst1) {
  uint32_t w[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t t = v[q * 4 + e];
      const uint32_t s = (t >> 16) * c16 + (t & 0xFFFFu);  // < 2^25, == t mod m
      word |= mod_small(s, m, magic) << (8 * e);
    }
    w[q] = word;
  }
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
  *dst0 = make_uint4(w[0], w[1], w[2], w[3]);
  *dst1 = make_uint4(w[4], w[5], w[6], w[7]);
}

// CRT of 8 columns (half `sub` of a 16-byte residue row) of one row -> C.
__device__ __forceinline__ void crt8(const Params& P, uint8_t* slot, int half, int c16, int sub, int row_in_tile,
                                     i64 row, i64 col0, double* dst) {
  unsigned long long s_lo[8], s_hi[8], f[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s_lo[e] = s_hi[e] = f[e] = 0;
#pragma unroll 2
  for (int i = 0; i < P.nmod; ++i) {
    const uint4 r4 = *scratch_at(slot, i, half, c16, row_in_tile);
    const uint32_t rw[2] = {sub ? r4.z : r4.x, sub ? r4.w : r4.y};
    const uint32_t wl = P.w_lo[i], wh = P.w_hi[i], g = P.g[i];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t r = (rw[e / 4] >> (8 * (e % 4))) & 0xFFu;
      s_lo[e] += static_cast<unsigned long long>(r) * wl;
      s_hi[e] += static_cast<unsigned long long>(r) * wh;
      f[e] += static_cast<unsigned long long>(r) * g;
    }
  }
  if (row >= P.m) return;
  const unsigned long long p = P.p;
  double out[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const unsigned long long t = (f[e] + (1ull << 23)) >> 24;  // round(Z / M)
    const unsigned long long hi = dev::shoup_mulmod(s_hi[e], P.two32, P.two32_sh, p);
    const unsigned long long s = barrett(hi + s_lo[e], p, P.mu);
    const unsigned long long tm = dev::shoup_mulmod(t, P.Mp, P.Mp_sh, p);
    out[e] = static_cast<double>(s >= tm ? s - tm : s + p - tm);
  }
  if (col0 + 8 <= P.n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int e = 0; e < 8; e += 2) *reinterpret_cast<double2*>(dst + e) = make_double2(out[e], out[e + 1]);
  } else {
    for (int e = 0; e < 8 && col0 + e < P.n; ++e) dst[e] = out[e];
  }
}

__global__ void __launch_bounds__(kThreads, 1) rns_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int total = P.MB * P.NB * P.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      dev::mbar_init(&tmem_full[b], 1);
      dev::mbar_init(&tmem_empty[b], kEpiWarps);
    }
    dev::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        dev::smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  i8::fence_before();
  __syncthreads();
  i8::fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int g = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Item it = item_of(t, P);
        const int kb0 = it.ks * P.kb_per_split;
        const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
        for (int i = 0; i < P.nmod; ++i) {
          const uint8_t* gA = P.apack + ((static_cast<i64>(it.tm) * P.nmod + i) * P.KB + kb0) * kAStage;
          const uint8_t* gB = P.bpack + ((static_cast<i64>(it.tn) * P.nmod + i) * P.KB + kb0) * kBStage;
          for (int kb = 0; kb < nkb; ++kb, ++g) {
            const int s = g % kStages;
            if (g >= kStages) dev::mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
            dev::mbar_arrive_expect_tx(&full[s], kStageBytes);
            dev::bulk_g2s(sA + s * kAStage, gA + static_cast<i64>(kb) * kAStage, kAStage, &full[s]);
            dev::bulk_g2s(sB + s * kBStage, gB + static_cast<i64>(kb) * kBStage, kBStage, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      constexpr uint32_t idesc = i8::instr_desc(kBM, kNT);
      int g = 0, pass = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Item it = item_of(t, P);
        const int kb0 = it.ks * P.kb_per_split;
        const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
        const int nseg = max(1, (nkb + P.seg_kb - 1) / P.seg_kb);
        for (int i = 0; i < P.nmod; ++i) {
          int kb = 0;
          for (int seg = 0; seg < nseg; ++seg, ++pass) {
            const int b = pass & 1;
            dev::mbar_wait(&tmem_empty[b], ((pass >> 1) & 1) ^ 1);
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
                const uint64_t bd = i8::smem_desc(b0 + tk * 2 * (kNT / 8) * 128, (kNT / 8) * 128, 128);
                i8::mma_i8(tacc, ad, bd, idesc, (kb > kstart || tk > 0) ? 1u : 0u);
              }
              i8::mma_commit(&empty[s]);
            }
            i8::mma_commit(&tmem_full[b]);
          }
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..9 ----------------
    const int quad = warp % 4;
    const int half = (warp - 2) / 4;
    const int row_in_tile = quad * 32 + lane;
    const uint32_t tlane = static_cast<uint32_t>(quad * 32) << 16;
    uint8_t* slot = P.scratch + static_cast<i64>(blockIdx.x) * P.nmod * kSlotPerMod;
    int pass = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const Item it = item_of(t, P);
      const int kb0 = it.ks * P.kb_per_split;
      const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
      const int nseg = max(1, (nkb + P.seg_kb - 1) / P.seg_kb);
      for (int i = 0; i < P.nmod; ++i) {
        const uint32_t m = P.mod[i], c16 = P.c16[i], mg = P.magic[i];
        for (int seg = 0; seg < nseg; ++seg, ++pass) {
          const int b = pass & 1;
          dev::mbar_wait(&tmem_full[b], (pass >> 1) & 1);
          i8::fence_after();
          const uint32_t tcol = tbase + tlane + b * kNT + half * (kNT / 2);
#pragma unroll 1
          for (int c0 = 0; c0 < kNT / 2; c0 += 32) {
            uint32_t v[32];
            i8::tmem_ld32(tcol + c0, v);
            i8::tmem_wait_ld();
            if (c0 + 32 == kNT / 2) {  // every column of this buffer is in registers: release it
              i8::fence_before();
              __syncwarp();
              if (lane == 0) dev::mbar_arrive(&tmem_empty[b]);
            }
            park32(v, m, c16, mg, seg > 0, scratch_at(slot, i, half, c0 / 16, row_in_tile),
                   scratch_at(slot, i, half, c0 / 16 + 1, row_in_tile));
          }
        }
      }
      // CRT over the parked residues of this thread's row / column half
      const i64 row = static_cast<i64>(it.tm) * kBM + row_in_tile;
      const i64 colh = static_cast<i64>(it.tn) * kNT + half * (kNT / 2);
      double* dst_row = P.C + static_cast<i64>(it.ks) * P.split_stride + row * P.ldc + colh;
#pragma unroll 1
      for (int c = 0; c < (kNT / 2) / 8; ++c) {
        if (colh + c * 8 >= P.n) break;
        crt8(P, slot, half, c / 2, c % 2, row_in_tile, row, colh + c * 8, dst_row + c * 8);
      }
    }
  }
  i8::fence_before();
  __syncthreads();
  if (warp == 1) {
    i8::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

}  // namespace rns
}  // namespace fpmm_b200
