// i8engine.cuh -- int8 multiword engine on the 5th-gen tensor cores (tcgen05).
//
// The same multiword method with 8-bit words: every residue x < p < 2^(8D) is
// split into D unsigned base-256 digits, x = sum_i 256^i x_i.  Then
//   A B = sum_s 256^s T_s,   T_s = sum_{i+j=s} A_i B_j   (s = 0 .. 2D-2)
// and each T_s is an exact integer sum of digit products (<= 255^2 each)
// computed by tcgen05.mma.kind::i8 into int32 TMEM accumulators.  Read as
// unsigned, a T_s block is exact while pairs(s) * Kseg * 255^2 < 2^32, so K is
// processed in segments of at most Kseg; the epilogue reduces every block mod p
// and forms sum_s (256^s mod p) T_s with independent Shoup products (no Horner
// chain), accumulating the segments.
//
// One CTA computes a 128 x NT tile of C, NT = 256/128/64/64/32/32/32 for
// D = 1..7 (the widest with (2D-1) NT <= 512 TMEM columns and D NT <= 256).
// B's digits are concatenated along N (B_cat = [B_0 | .. | B_{D-1}],
// N_mma = D NT) and the MMA of A digit i is issued at TMEM column offset
// NT i, so digit pair (i, j) lands in column block i + j = s: one MMA per A
// digit per k-step builds every T_s at once.
//
// Warp roles: warp 0 TMA producer (1-D bulk copies of pre-packed chunks),
// warp 1 TMEM allocator + single-thread MMA issuer, warps 2-5 epilogue
// (TMEM -> registers -> mod-p fold -> C).
#pragma once

#include <cstdint>

#include "device_common.cuh"

namespace fpmm_b200 {
namespace i8 {

using i64 = std::int64_t;

constexpr int kBM = 128;      // rows per CTA tile (MMA M)
constexpr int kBK = 64;       // k bytes (int8 elements) per pipeline stage
constexpr int kKSteps = kBK / 32;  // MMA K = 32 for kind::i8
constexpr int kThreads = 192;      // 6 warps

// Output columns per CTA tile (NT): the widest NT (a multiple of 8) with
// (2D-1) NT <= 512 TMEM columns and N_mma = D NT <= 256, N_mma % 16 == 0.  Wider tiles read
// less shared memory per MMA (A is re-read once per MMA) and amortise the
// per-tile epilogue over more work.
// A narrow B (n <= 32, e.g. the unbalanced scenario's 32 columns) uses NT = 32.
template <int D>
constexpr int kWideNT = D == 1 ? 256 : D == 2 ? 128 : D == 3 ? 80 : D == 4 ? 64 : D == 5 ? 48 : D == 6 ? 40 : 32;
template <int D, int NT_ = kWideNT<D>>
struct Cfg {
  static constexpr int kNT = NT_;
  static constexpr int kAStage = D * kBM * kBK;        // bytes: D digit tiles of 128 x 64
  static constexpr int kBStage = D * kNT * kBK;        // bytes: B_cat tile of (NT D) x 64
  static constexpr int kStageBytes = kAStage + kBStage;
  static constexpr int kStages = (220 * 1024) / kStageBytes > 8 ? 8 : (220 * 1024) / kStageBytes;
  static constexpr int kBlocks = 2 * D - 1;            // weight blocks s = 0 .. 2D-2
  static constexpr int kTmemCols = kBlocks * kNT;
  static constexpr int kTmemAlloc = kTmemCols <= 32 ? 32 : kTmemCols <= 64 ? 64 : kTmemCols <= 128 ? 128
                                    : kTmemCols <= 256 ? 256 : 512;
  static constexpr int kSmem = kStages * kStageBytes + 1024;  // + barriers / tmem slot
  static constexpr int kNmma = D * kNT;
  static_assert(kStages >= 2, "pipeline needs two stages");
  static_assert(kTmemCols <= 512 && kNmma <= 256 && kNmma % 16 == 0, "tile does not fit the MMA / TMEM");
};

// ------------------------------------------------------------ descriptors
// UMMA shared-memory descriptor, K-major, no swizzle (canonical
// ((8,n),2):((16B,SBO),LBO)): 8-row x 16-byte core matrices, LBO = byte step
// between the two 16-byte K halves of one MMA, SBO = byte step between
// 8-row groups.  Version 1 (sm_100), layout type 0.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  return d;
}

// Instruction descriptor: kind::i8, D = S32, A = B = unsigned 8-bit, both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z));
}

// From a converged warp: identical operands on every lane, one lane picked by
// elect.sync issues (no per-MMA R2UR / BRA.U.ANY sequence of the one-thread form)
__device__ __forceinline__ void mma_i8_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  const uint32_t z = 0;
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(z));
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(dev::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   dev::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st32_zero(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr),
      "r"(z)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                   taddr),
               "r"(z)
               : "memory");
}
__device__ __forceinline__ void tmem_st8_zero(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr), "r"(z)
               : "memory");
}
template <int W>
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, uint32_t* r) {
  if constexpr (W == 32) tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
  else if constexpr (W == 16) tmem_ld16(taddr, r);
  else tmem_ld8(taddr, r);
}
template <int W>
__device__ __forceinline__ void tmem_zerow(uint32_t taddr) {
  if constexpr (W == 32) tmem_st32_zero(taddr);
  else if constexpr (W == 16) tmem_st16_zero(taddr);
  else tmem_st8_zero(taddr);
}
// zero every TMEM column of the 2D-1 blocks this lane quadrant owns
template <int NBLK, int NT>
__device__ __forceinline__ void tmem_zero_all(uint32_t trow) {
  constexpr int FULL = NT - NT % 32;
#pragma unroll 1
  for (int b = 0; b < NBLK; ++b) {
#pragma unroll
    for (int c0 = 0; c0 < FULL; c0 += 32) tmem_st32_zero(trow + b * NT + c0);
    if constexpr (NT % 32 != 0) tmem_zerow<NT % 32>(trow + b * NT + FULL);
  }
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// x mod p for x < 2^64 with mu = floor(2^64 / p): q = mulhi(x, mu) is floor(x/p)
// or one less, so a single correction lands in [0, p).
__device__ __forceinline__ uint64_t barrett(uint64_t x, uint64_t p, uint64_t mu) {
  const uint64_t q = __umul64hi(x, mu);
  uint64_t r = x - q * p;
  return r >= p ? r - p : r;
}

struct Params {
  const uint8_t* apack;  // [m-block][k-block] chunks of kAStage bytes
  const uint8_t* bpack;  // [n-block][k-block] chunks of kBStage bytes
  double* C;
  i64 ldc, m, n;
  int MB, NB, KB;       // tiles along m, n and 64-byte k-blocks
  int seg_kb;           // k-blocks per exact accumulation segment
  int kb_per_split;     // split-K: k-blocks per slice (== KB when unsplit)
  int splits;           // split-K: number of slices
  i64 split_stride;     // split-K: C offset (elements) between the slices' partial outputs
  unsigned long long p, mu;
  unsigned long long gam[13], gam_sh[13];  // 256^s mod p and Shoup constants, s = 0 .. 2D-2
};

// --------------------------------------------------------------- packing
// A: m x k residues -> D unsigned digit planes in the MMA's canonical
// K-major layout.  Chunk (rb, kb) (contiguous, kAStage bytes):
//   [digit i][k16 c (4)][row group g (16)][row r (8)][16 bytes]
// Thread (row, 16-byte k chunk): reads 16 residues, writes D x 16 bytes.
template <int D>
__global__ void __launch_bounds__(256) pack_a_i8(const double* __restrict__ A, i64 lda, i64 m, i64 k,
                                                 int KB, i64 mpad, uint8_t* __restrict__ out) {
  const i64 kchunks = static_cast<i64>(KB) * (kBK / 16);
  const i64 total = mpad * kchunks;
  for (i64 idx = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<i64>(gridDim.x) * blockDim.x) {
    // warp covers 8 rows x 4 chunks so each 128-byte core matrix line is written whole
    const i64 grp = idx / 32;
    const int lane = static_cast<int>(idx % 32);
    const int r8 = lane % 8, c4 = lane / 8;
    const i64 rows8 = mpad / 8;
    const i64 rg = grp % rows8, cq = grp / rows8;  // row group of 8, chunk quad
    const i64 row = rg * 8 + r8;
    const i64 kc = cq * 4 + c4;  // 16-byte chunk index along k
    if (kc >= kchunks) continue;
    uint32_t w[D][4];
#pragma unroll
    for (int i = 0; i < D; ++i) w[i][0] = w[i][1] = w[i][2] = w[i][3] = 0;
    if (row < m) {
      const double* src = A + row * lda + kc * 16;
      double xs[16];
      if (kc * 16 + 16 <= k && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
#pragma unroll
        for (int e = 0; e < 16; e += 2) {  // 16-byte loads
          const double2 t = __ldg(reinterpret_cast<const double2*>(src + e));
          xs[e] = t.x;
          xs[e + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) xs[e] = kc * 16 + e < k ? src[e] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const unsigned long long x = static_cast<unsigned long long>(xs[e]);
#pragma unroll
        for (int i = 0; i < D; ++i) w[i][e / 4] |= static_cast<uint32_t>((x >> (8 * i)) & 0xFF) << (8 * (e % 4));
      }
    }
    const i64 rb = row / kBM, kb = kc / (kBK / 16);
    const int c = static_cast<int>(kc % (kBK / 16)), g = static_cast<int>((row % kBM) / 8);
    uint8_t* base = out + (rb * KB + kb) * static_cast<i64>(Cfg<D>::kAStage);
#pragma unroll
    for (int i = 0; i < D; ++i)
      *reinterpret_cast<uint4*>(base + i * (kBM * kBK) + ((c * (kBM / 8) + g) * 8 + r8) * 16) =
          make_uint4(w[i][0], w[i][1], w[i][2], w[i][3]);
  }
}

// B: k x n residues -> B_cat digit rows (digit j, column c) -> row NT j + c,
// K-major.  Chunk (cb, kb) (contiguous, kBStage bytes):
//   [k16 c (4)][row group g (NT D / 8)][row r (8)][16 bytes]
// A block transposes 64 (k) x 32 (col) sub-tiles through shared memory.
template <int D, int NT>
__global__ void __launch_bounds__(256) pack_b_i8(const double* __restrict__ B, i64 ldb, i64 k, i64 n,
                                                 int KB, int NB, uint8_t* __restrict__ out) {
  constexpr int SW = NT % 32 == 0 ? 32 : NT % 16 == 0 ? 16 : 8;  // sub-block columns
  constexpr int SUB = NT / SW;
  __shared__ unsigned long long tile[kBK][SW + 1];
  const i64 tiles = static_cast<i64>(KB) * NB * SUB;
  for (i64 t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int sb = static_cast<int>(t % SUB);
    const i64 cb = (t / SUB) % NB, kb = t / (SUB * static_cast<i64>(NB));
    __syncthreads();
    for (int e = threadIdx.x; e < kBK * SW; e += blockDim.x) {
      const int kr = e / SW, cc = e % SW;
      const i64 kk = kb * kBK + kr, col = cb * NT + sb * SW + cc;
      tile[kr][cc] = (kk < k && col < n) ? static_cast<unsigned long long>(B[kk * ldb + col]) : 0ull;
    }
    __syncthreads();
    uint8_t* base = out + (cb * KB + kb) * static_cast<i64>(Cfg<D, NT>::kBStage);
    // units: (digit j, column cc, k16 chunk q): 16 bytes each
    for (int u = threadIdx.x; u < D * SW * (kBK / 16); u += blockDim.x) {
      // lanes walk the 32 columns: 2-way (64-bit) bank access, and 32
      // consecutive 16-byte rows of one core-matrix column -> 512 B stores
      const int cc = u % SW, q = (u / SW) % (kBK / 16), j = u / ((kBK / 16) * SW);
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int e = 0; e < 16; ++e)
        w[e / 4] |= static_cast<uint32_t>((tile[q * 16 + e][cc] >> (8 * j)) & 0xFF) << (8 * (e % 4));
      const int nn = j * NT + sb * SW + cc, g = nn / 8, r8 = nn % 8;
      *reinterpret_cast<uint4*>(base + ((q * (D * NT / 8) + g) * 8 + r8) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ------------------------------------------------------------------ GEMM
// Work item t (0 <= t < MB * NB * splits) -> output tile (tm, tn), split ks.
// Grouped rasterisation: the 148 items in flight cover GROUP tile-rows x ~37
// tile-columns, so their A panels (GROUP x 7 MB at D=7, K=8192) and B_cat
// panels stay resident in the 126 MB L2.
struct Item {
  int tm, tn, ks;
};
__device__ __forceinline__ Item item_of(int t, const Params& P) {
  constexpr int GROUP = 4;
  const int tiles = P.MB * P.NB;
  const int r = t % tiles;
  const int in_group = GROUP * P.NB;
  const int first_m = (r / in_group) * GROUP;
  const int gsz = min(P.MB - first_m, GROUP);
  Item it;
  it.tm = first_m + (r % in_group) % gsz;
  it.tn = (r % in_group) / gsz;
  it.ks = t / tiles;
  return it;
}

// x * g mod p for x < 2^32 (Shoup: gs = floor(g 2^64 / p)); result in [0, p)
__device__ __forceinline__ uint64_t shoup32(uint32_t x, uint64_t g, uint64_t gs, uint64_t p) {
  const uint64_t q = __umul64hi(static_cast<uint64_t>(x), gs);
  const uint64_t r = static_cast<uint64_t>(x) * g - q * p;
  return r >= p ? r - p : r;
}

// One W-column chunk of the epilogue: sum_s (256^s mod p) T_s over the
// weight blocks (re-zeroing each as it is read), optional release of TMEM,
// then the C store (read-modify-write when earlier K segments were parked).
template <int W, int NBLK, int NT>
__device__ __forceinline__ void epi_chunk(const Params& P, uint32_t trow, int c0, bool last, uint64_t* tmem_empty,
                                          int lane, int seg, i64 row, i64 col_base, double* dst_row) {
  const unsigned long long p = P.p;
  unsigned long long acc[W];
#pragma unroll
  for (int c = 0; c < W; ++c) acc[c] = 0;
#pragma unroll 1
  for (int b = 0; b < NBLK; ++b) {
    uint32_t v[W];
    tmem_ldw<W>(trow + b * NT + c0, v);
    tmem_wait_ld();
    tmem_zerow<W>(trow + b * NT + c0);
    const unsigned long long g = P.gam[b], gs = P.gam_sh[b];
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const unsigned long long s2 = acc[c] + shoup32(v[c], g, gs, p);
      acc[c] = s2 >= p ? s2 - p : s2;
    }
  }
  if (last) {  // every block consumed and re-zeroed: release TMEM to the MMA warp
    tmem_wait_st();
    fence_before();
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(tmem_empty);
  }
  if (row < P.m) {
    double* dst = dst_row + c0;
    const i64 col0 = col_base + c0;
    if (seg > 0) {  // earlier segments' residues were parked in C by this thread
      for (int c = 0; c < W && col0 + c < P.n; ++c) {
        const unsigned long long s2 = acc[c] + static_cast<unsigned long long>(dst[c]);
        acc[c] = s2 >= p ? s2 - p : s2;
      }
    }
    if (col0 + W <= P.n && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
      for (int c = 0; c < W; c += 2)
        *reinterpret_cast<double2*>(dst + c) = make_double2(static_cast<double>(acc[c]), static_cast<double>(acc[c + 1]));
    } else {
      for (int c = 0; c < W && col0 + c < P.n; ++c) dst[c] = static_cast<double>(acc[c]);
    }
  }
}

// Persistent: one CTA per SM loops over work items (TMEM allocation, barrier
// set-up and the pipeline fill are paid once per SM, and the TMA producer
// runs ahead into the next item while the epilogue reconstructs the last).
template <int D, int NTC>
__global__ void __launch_bounds__(kThreads, 1) mwi8_kernel(const __grid_constant__ Params P) {
  using CF = Cfg<D, NTC>;
  constexpr int S = CF::kStages, NT = CF::kNT, NB_ = CF::kBlocks;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * CF::kAStage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * CF::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tmem_full = empty + S;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int total = P.MB * P.NB * P.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    dev::mbar_init(tmem_full, 1);
    dev::mbar_init(tmem_empty, 4);  // one arrive per epilogue warp
    dev::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     dev::smem_u32(tmem_slot)),
                 "r"(CF::kTmemAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int g = 0;  // k-blocks issued by this CTA (stage ring position)
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Item it = item_of(t, P);
        const int kb0 = it.ks * P.kb_per_split;
        const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
        const uint8_t* gA = P.apack + (static_cast<i64>(it.tm) * P.KB + kb0) * CF::kAStage;
        const uint8_t* gB = P.bpack + (static_cast<i64>(it.tn) * P.KB + kb0) * CF::kBStage;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % S;
          if (g >= S) dev::mbar_wait(&empty[s], ((g / S) - 1) & 1);
          dev::mbar_arrive_expect_tx(&full[s], CF::kStageBytes);
          dev::bulk_g2s(sA + s * CF::kAStage, gA + static_cast<i64>(kb) * CF::kAStage, CF::kAStage, &full[s]);
          dev::bulk_g2s(sB + s * CF::kBStage, gB + static_cast<i64>(kb) * CF::kBStage, CF::kBStage, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (the converged warp; elect.sync issues) ----------------
    {
      constexpr uint32_t idesc = instr_desc(kBM, CF::kNmma);
      int g = 0, e = 0;  // stage ring position, accumulator generation
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const Item it = item_of(t, P);
        const int kb0 = it.ks * P.kb_per_split;
        const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
        const int nseg = max(1, (nkb + P.seg_kb - 1) / P.seg_kb);
        int kb = 0;
        for (int seg = 0; seg < nseg; ++seg, ++e) {
          dev::mbar_wait(tmem_empty, e & 1);  // epilogue drained and re-zeroed the accumulators
          fence_after();
          const int kend = min(nkb, kb + P.seg_kb);
          for (; kb < kend; ++kb, ++g) {
            const int s = g % S;
            dev::mbar_wait(&full[s], (g / S) & 1);
            fence_after();
            const uint32_t a0 = dev::smem_u32(sA + s * CF::kAStage), b0 = dev::smem_u32(sB + s * CF::kBStage);
#pragma unroll
            for (int tk = 0; tk < kKSteps; ++tk) {
              const uint64_t bd = smem_desc(b0 + tk * 2 * (CF::kNmma / 8) * 128, (CF::kNmma / 8) * 128, 128);
#pragma unroll
              for (int i = 0; i < D; ++i) {
                const uint64_t ad = smem_desc(a0 + i * (kBM * kBK) + tk * 2 * (kBM / 8) * 128, (kBM / 8) * 128, 128);
                mma_i8_warp(tbase + i * NT, ad, bd, idesc, 1u);
              }
            }
            mma_commit_warp(&empty[s]);  // frees the stage once these MMAs have read it
          }
          mma_commit_warp(tmem_full);    // this segment's accumulators are complete
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5 ----------------
    // Reconstruct straight from TMEM: sum_s (256^s mod p) T_s with Shoup
    // products (independent terms, no Horner chain), re-zero each block as it
    // is consumed, release the accumulators, then store C.  (Draining TMEM to
    // an L2 scratch to overlap this with the next item's MMAs was measured
    // slower: the 208 KB/item scratch traffic cost more power than the
    // overlap won on this power-capped part.)
    const int quad = warp % 4;                 // TMEM lane quadrant this warp may access
    const int row_in_tile = quad * 32 + lane;  // TMEM lane == tile row
    const uint32_t trow = tbase + (static_cast<uint32_t>(quad * 32) << 16);
    tmem_zero_all<NB_, NT>(trow);
    tmem_wait_st();
    fence_before();
    __syncwarp();
    if (lane == 0) dev::mbar_arrive(tmem_empty);
    constexpr int FULL = NT - NT % 32;
    int e = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const Item it = item_of(t, P);
      const int kb0 = it.ks * P.kb_per_split;
      const int nkb = max(0, min(P.KB, kb0 + P.kb_per_split) - kb0);
      const int nseg = max(1, (nkb + P.seg_kb - 1) / P.seg_kb);
      const i64 row = static_cast<i64>(it.tm) * kBM + row_in_tile;
      const i64 col_base = static_cast<i64>(it.tn) * NT;
      double* dst_row = P.C + static_cast<i64>(it.ks) * P.split_stride + row * P.ldc + col_base;
      for (int seg = 0; seg < nseg; ++seg, ++e) {
        dev::mbar_wait(tmem_full, e & 1);
        fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < FULL; c0 += 32)
          epi_chunk<32, NB_, NT>(P, trow, c0, NT % 32 == 0 && c0 + 32 >= NT, tmem_empty, lane, seg, row, col_base,
                                 dst_row);
        if constexpr (NT % 32 != 0)
          epi_chunk<NT % 32, NB_, NT>(P, trow, FULL, true, tmem_empty, lane, seg, row, col_base, dst_row);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "r"(CF::kTmemAlloc));
  }
}

// split-K combine: C[i][j] = sum_s W[s][i][j] mod p (W slices are residues)
__global__ void splitk_reduce_kernel(const double* __restrict__ W, i64 slice, int splits, double* __restrict__ C,
                                     i64 ldc, i64 rows, i64 cols, unsigned long long p) {
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    unsigned long long acc = 0;
    for (int s = 0; s < splits; ++s) {
      acc += static_cast<unsigned long long>(W[s * slice + e]);
      acc -= acc >= p ? p : 0;
    }
    C[(e / cols) * ldc + e % cols] = static_cast<double>(acc);
  }
}

// Tensor-pipe int8 peak probe: one thread per CTA issues `iters` back-to-back
// M=128 N=256 K=32 kind::i8 MMAs on zero operands (one CTA per SM).
__global__ void __launch_bounds__(64, 1) i8_peak_kernel(int iters, int* out) {
  __shared__ __align__(1024) uint8_t ops[kBM * 32 + 256 * 32];
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  // random operand bytes: realistic toggling (zero operands draw ~1/3 of the power)
  for (int e = threadIdx.x; e < static_cast<int>(sizeof(ops)) / 4; e += blockDim.x)
    reinterpret_cast<uint32_t*>(ops)[e] = static_cast<uint32_t>(e * 2654435761u + blockIdx.x * 40503u) ^ 0x5bd1e995u;
  if (threadIdx.x == 0) {
    dev::mbar_init(&done, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(dev::smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = dev::smem_u32(ops), b = a + kBM * 32;
    const uint64_t ad = smem_desc(a, (kBM / 8) * 128, 128), bd = smem_desc(b, (256 / 8) * 128, 128);
    constexpr uint32_t idesc = instr_desc(kBM, 256);
    for (int it = 0; it < iters; ++it) mma_i8(tbase, ad, bd, idesc, it > 0 ? 1u : 0u);
    mma_commit(&done);
    dev::mbar_wait(&done, 0);
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    uint32_t v[32];
    tmem_ld32(tbase + (32u << 16), v);  // warp 1 owns TMEM lanes 32..63
    tmem_wait_ld();
    if (v[0] == 12345u) out[0] = 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tbase));
  }
}

// ---- cta_group::2 probe: a CTA pair (cluster of 2) issues M=256 N=256 K=32
// kind::i8 MMAs from the leader; each CTA holds its 128-row A half and half
// of B.  Used to measure the pair's sustained rate against the 1-CTA probe.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
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
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          dev::smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1) i8_peak2_kernel(int iters, int* out) {
  __shared__ __align__(1024) uint8_t ops[kBM * 32 + 128 * 32];  // A half (128x32) + B half (128 rows x 32)
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = cluster_rank();
  for (int e = threadIdx.x; e < static_cast<int>(sizeof(ops)) / 4; e += blockDim.x)
    reinterpret_cast<uint32_t*>(ops)[e] = static_cast<uint32_t>(e * 2654435761u + blockIdx.x * 40503u) ^ 0x5bd1e995u;
  if (threadIdx.x == 0) {
    dev::mbar_init(&done, 1);
    dev::fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(dev::smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  fence_before();
  cluster_sync_all();
  fence_after();
  const uint32_t tbase = slot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t a = dev::smem_u32(ops), b = a + kBM * 32;
    const uint64_t ad = smem_desc(a, (kBM / 8) * 128, 128), bd = smem_desc(b, (128 / 8) * 128, 128);
    constexpr uint32_t idesc = instr_desc(256, 256);
    for (int it = 0; it < iters; ++it) mma_i8_2sm(tbase, ad, bd, idesc, it > 0 ? 1u : 0u);
    mma_commit_2sm(&done, 0x3);
  }
  if (threadIdx.x == 0) dev::mbar_wait(&done, 0);
  fence_before();
  cluster_sync_all();
  if (warp == 1) {
    fence_after();
    uint32_t v[32];
    tmem_ld32(tbase + (32u << 16), v);
    tmem_wait_ld();
    if (v[0] == 12345u) out[0] = 1;
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;\n" ::"r"(tbase));
  }
}

}  // namespace i8
}  // namespace fpmm_b200
