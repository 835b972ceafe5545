// rnstile.cuh -- the RNS engine with the CRT on chip (rns_tile_kernel).
//
// rns_kernel (rnsengine.cuh) parks T_i mod m_i in HBM, n bytes per output
// element, and rns_crt_spec_kernel reads them back: at k = 256 (C5) that round
// trip and the separate CRT launch are more than half of the product.  Here a
// CTA pair owns a 256 x 128 output tile for all n moduli back to back
// (tile-major passes) and keeps the residues of the tile on chip; the CRT
// (crt4_spec, the same arithmetic as the standalone kernel) writes only C.
//
// Per CTA (128 rows x 128 columns of the tile, TMEM lanes = rows):
//   shared memory  `stages` pipeline stages of 48 KB (A 128 rows x kBK bytes,
//                  B 64 columns x kBK bytes), at most 8;
//   shared memory  residue planes of moduli 0..smem_mods-1 (16 KB each),
//                  [i][4-column group (32)][row (128)] words;
//   TMEM           `naccs` (2..4) s32 accumulators of 128 columns, used in
//                  turn by consecutive passes, then the residue planes of
//                  moduli smem_mods..n-1: 32 columns each, column c holding
//                  the residues of tile columns 4c..4c+3 (one byte each).
// Each epilogue thread produces and consumes only its own row's words (TMEM
// lane = its row, shared words indexed by its row), so the residues need no
// synchronisation beyond tcgen05.wait::st.
//
// Measured (profiles/round2/tile_kernel.md): the MMAs of the next tile stall
// while the epilogue runs a tile's CRT (16 warps at ~0.5 IPC per scheduler),
// so the kernel wins only where the parked path's residue round trip costs
// more: k <= 256 up to 40 bits (C5 -9%).  Streaming each tile's CRT through
// the next tile's passes (residue words re-slotted through an involution so
// no pass overwrites an unread word) was correct but 25% slower again: the
// per-word TMEM loads and waits of 16 latency-bound warps cost more than the
// stall they removed.  At long K the 256 x 128 pair tile needs 96 B/clk of
// operands per SM against the ~60 B/clk L2 delivers (8192^3: 48% tensor
// activity against rns_kernel's 94%), and tile-major passes lose the L2
// reuse of the modulus-major order (DRAM reads 2.9 -> 8.2 GB).
//
// The MMA is tcgen05.mma.cta_group::2.kind::i8 M256 N128 K32: CTA r supplies
// rows 128 r.. of A and columns 64 r.. of the tile's B block.  B is packed
// exactly as for rns_kernel (128-column blocks, [k16][column group][8][16 B]);
// a 3-D tensor map (16-byte rows, 16 column groups, k16 slices) loads the
// 8 column groups of this CTA's half.
//
// Needs one exact K segment (k <= 66048, no split-K) and n <= 16.
// Reference being replaced: the gamma-scaled accumulation of the products'
// words, proj/include/fpmm/multiword.hpp:94-105 and :121-129.
#pragma once

#include "rnsengine.cuh"

namespace fpmm_b200 {
namespace rns {

constexpr int kTNT = 128;                  // pair tile columns (MMA N)
constexpr int kTBH = kTNT / 2;             // B columns per CTA
constexpr int kTBStage = kTBH * kBK;       // 16 KB
constexpr int kTStageBytes = kAStage + kTBStage;
constexpr int kTEpiWarps = 16;             // 4 per TMEM lane quadrant, 32 columns each
constexpr int kTThreads = 64 + 32 * kTEpiWarps;
constexpr int kTMaxAccs = 4;
constexpr int kTResBytes = kBM * kTNT;     // one shared residue plane (16 KB)
constexpr int kTMaxMod = 16;
constexpr int kTMaxStages = 8;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&w)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n" : "=r"(a), "=r"(b) : "r"(taddr));
}

// Pair TMA load of this CTA's half of a B stage: 8 column groups (y = 8 rank)
// of kBK / 16 k16 slices starting at slice z, completing on the leader's barrier.
__device__ __forceinline__ void tma_pair_load3(void* dst, const CUtensorMap* map, int y, int z, uint64_t* bar) {
  const uint32_t leader_bar = dev::smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];\n" ::"r"(dev::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(y), "r"(z), "r"(leader_bar)
      : "memory");
}

// The pair's tiles t = pair, pair + npairs, ... (P.NB counts 128-column
// tiles), each for moduli 0..n-1.
template <int WPL, int NG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTThreads, 1)
    rns_tile_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int S = P.stages;
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kAStage;
  uint32_t* sres = reinterpret_cast<uint32_t*>(smem + P.res_off);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P.bar_off);  // leader: both halves landed
  uint64_t* empty = full + kTMaxStages;
  uint64_t* tmem_full = empty + kTMaxStages;       // [naccs]
  uint64_t* tmem_empty = tmem_full + kTMaxAccs;    // [naccs] leader: both CTAs drained accumulator a
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + kTMaxAccs);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int tiles = P.MB * P.NB;
  const int nmod = P.nmod, KB = P.KB, NA = P.naccs;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NA; ++a) {
      dev::mbar_init(&tmem_full[a], 1);
      dev::mbar_init(&tmem_empty[a], 2 * kTEpiWarps);
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
    // ---------------- TMA producer (both CTAs: own A rows, own half of B) ----------------
    if (lane == 0) {
      int s = 0, round = 0;
      for (int t = pair; t < tiles; t += npairs) {
        const Item it = item_of(t, P);
        const i64 rb = 2 * static_cast<i64>(it.tm) + rank, cb = it.tn;
        for (int i = 0; i < nmod; ++i) {
          const int rowA = static_cast<int>(((rb * KB) * nmod + i) * (kAStage / 128));
          const int zB = static_cast<int>(((cb * KB) * nmod + i) * (kBK / 16));
          for (int kb = 0; kb < KB; ++kb) {
            if (round > 0) dev::mbar_wait(&empty[s], (round - 1) & 1);
            if (rank == 0) dev::mbar_arrive_expect_tx(&full[s], 2 * kTStageBytes);
            // [block][k-block][modulus] chunks: consecutive k-blocks are nmod chunks apart
            tma_pair_load(sA + s * kAStage, &P.tmA, rowA + kb * nmod * (kAStage / 128), &full[s]);
            tma_pair_load3(sB + s * kTBStage, &P.tmB, 8 * static_cast<int>(rank), zB + kb * nmod * (kBK / 16),
                           &full[s]);
            if (++s == S) s = 0, ++round;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------- MMA issuer (leader CTA, converged warp; elect.sync issues) ----------------
      constexpr uint32_t idesc = i8::instr_desc(kPairM, kTNT);
      const uint64_t adesc0 = i8::smem_desc(dev::smem_u32(sA), (kBM / 8) * 128, 128);
      const uint64_t bdesc0 = i8::smem_desc(dev::smem_u32(sB), (kTBH / 8) * 128, 128);
      int s = 0, round = 0, a = 0, around = 0;
      for (int t = pair; t < tiles; t += npairs) {
        for (int i = 0; i < nmod; ++i) {
          mbar_wait_cluster(&tmem_empty[a], (around & 1) ^ 1);
          i8::fence_after();
          const uint32_t tacc = tbase + a * kTNT;
          for (int kb = 0; kb < KB; ++kb) {
            dev::mbar_wait(&full[s], round & 1);
            i8::fence_after();
            const uint64_t ad = adesc0 + static_cast<uint64_t>((s * kAStage) >> 4);
            const uint64_t bd = bdesc0 + static_cast<uint64_t>((s * kTBStage) >> 4);
#pragma unroll
            for (int tk = 0; tk < kKSteps; ++tk)
              mma_i8_pair_warp(tacc, ad + static_cast<uint64_t>((tk * 2 * (kBM / 8) * 128) >> 4),
                               bd + static_cast<uint64_t>((tk * 2 * (kTBH / 8) * 128) >> 4), idesc,
                               (kb > 0 || tk > 0) ? 1u : 0u);
            commit_pair_warp(&empty[s]);  // frees stage s in both CTAs
            if (++s == S) s = 0, ++round;
          }
          commit_pair_warp(&tmem_full[a]);  // accumulator a complete in both CTAs
          if (++a == NA) a = 0, ++around;
        }
      }
    }
  } else {
    // ---------------- epilogue: warps 2..17 of both CTAs ----------------
    // warp -> (TMEM lane quadrant warp % 4, 32-column group wq = (warp - 2) / 4)
    const int quad = warp % 4, wq = (warp - 2) / 4;
    const int row_in_tile = quad * 32 + lane;
    const uint32_t tlane = tbase + (static_cast<uint32_t>(quad * 32) << 16);
    const uint32_t leader_tmem_empty = peer_addr(tmem_empty, 0);
    const bool small = P.small_t != 0;
    const int SM = P.smem_mods;
    const uint32_t tres = tlane + NA * kTNT - SM * (kTNT / 4);  // TMEM plane of modulus i >= SM: tres + 32 i
    int a = 0, around = 0;
    for (int t = pair; t < tiles; t += npairs) {
      for (int i = 0; i < nmod; ++i) {
        dev::mbar_wait(&tmem_full[a], around & 1);
        i8::fence_after();
        uint32_t v[32];
        i8::tmem_ld32(tlane + a * kTNT + wq * 32, v);
        i8::tmem_wait_ld();
        i8::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tmem_empty + a * 8);
        if (++a == NA) a = 0, ++around;
        uint32_t w[8];
        if (small) reduce32<true>(v, P.negm[i], P.c16[i], P.magic[i], w);
        else reduce32<false>(v, P.negm[i], P.c16[i], P.magic[i], w);
        if (i >= SM) {
          tmem_st8(tres + i * (kTNT / 4) + wq * 8, w);
        } else {
          uint32_t* dst = sres + (i * (kTNT / 4) + wq * 8) * kBM + row_in_tile;
#pragma unroll
          for (int q = 0; q < 8; ++q) dst[q * kBM] = w[q];
        }
      }
      // every residue of this thread's 32 columns is on chip: C = X mod p
      i8::tmem_wait_st();
      const Item it = item_of(t, P);
      const i64 row = (2 * static_cast<i64>(it.tm) + rank) * kBM + row_in_tile;
      const i64 col0 = static_cast<i64>(it.tn) * kTNT + wq * 32;
      double* dst_row = P.crt.C + (row < P.crt.m ? row : 0) * P.crt.ldc;
#pragma unroll 1
      for (int c8 = 0; c8 < 4; ++c8) {  // 8 columns (two residue words per modulus) per step
        if (col0 + 8 * c8 >= P.crt.n) break;  // warp-uniform
        uint32_t r2[4 * NG][2];
#pragma unroll
        for (int i = 0; i < 4 * NG; ++i) {
          if (i >= nmod) {
            r2[i][0] = r2[i][1] = 0;
          } else if (i >= SM) {
            tmem_ld2(tres + i * (kTNT / 4) + wq * 8 + 2 * c8, r2[i][0], r2[i][1]);
          } else {
            const uint32_t* src = sres + (i * (kTNT / 4) + wq * 8 + 2 * c8) * kBM + row_in_tile;
            r2[i][0] = src[0];
            r2[i][1] = src[kBM];
          }
        }
        i8::tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t rw[4 * NG];
#pragma unroll
          for (int i = 0; i < 4 * NG; ++i) rw[i] = r2[i][h];
          double out[4];
          crt4_spec<WPL, NG, true>(P.crt, rw, out);
          const i64 c = col0 + 8 * c8 + 4 * h;
          if (row < P.crt.m && c < P.crt.n) {
            double* d = dst_row + c;
            if (c + 4 <= P.crt.n && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
              *reinterpret_cast<double2*>(d) = make_double2(out[0], out[1]);
              *reinterpret_cast<double2*>(d + 2) = make_double2(out[2], out[3]);
            } else {
              for (int e = 0; e < 4 && c + e < P.crt.n; ++e) d[e] = out[e];
            }
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
