/*
 * fpmm_b200.h -- C-ABI of the B200-native multiword modular matrix product.
 *
 * C = A B mod p for primes (or, via the workspace variant, composites)
 * 5 <= p < 2^52, following arXiv 2601.07508.  Plain pointers and sizes only:
 * no torch or C++ types cross this boundary.  Matrices are dense row-major
 * binary64 arrays holding exact integers, element (i,j) at data[i*ld + j],
 * exactly the layout of the reference's Mat<T>/MatView<T>
 * (/root/reference/proj/include/fpmm/mat.hpp:13-26,42).
 *
 * Every entry point returns an fpmm_b200_status; on failure the message is
 * available from fpmm_b200_last_error() (thread-local).  Status codes mirror
 * the reference's exception taxonomy (/root/reference/proj/include/fpmm/
 * errors.hpp:9-33) so the C++ shim (include/fpmm_b200/fpmm.hpp) rethrows the
 * matching fpmm:: exception.  There is NO CPU fallback: a CUDA failure is
 * returned as FPMM_B200_ECUDA.
 *
 * Reference interfaces each entry point replaces are cited per declaration.
 */
#ifndef FPMM_B200_H
#define FPMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPMM_B200_VERSION 1

typedef enum {
  FPMM_B200_OK = 0,
  FPMM_B200_EERROR = 1,      /* fpmm::Error           (errors.hpp:9-12)  */
  FPMM_B200_EINFEASIBLE = 2, /* fpmm::InfeasibleError (errors.hpp:22-25) */
  FPMM_B200_ENOINVERSE = 3,  /* fpmm::NoInverseError  (errors.hpp:29-31) */
  FPMM_B200_ECONTRACT = 4,   /* fpmm::ContractError   (errors.hpp:17-19) */
  FPMM_B200_ECUDA = 10,      /* CUDA runtime / launch failure             */
  FPMM_B200_ENCCL = 11,      /* NCCL failure                              */
  FPMM_B200_ENOMEM = 12      /* device allocation failure                 */
} fpmm_b200_status;

/* flags for the product entry points */
#define FPMM_B200_ALLOW_COMPOSITE 0x1u /* FpContext::make(p, allow_composite=true) (fp_context.hpp:36) */
#define FPMM_B200_CHECK_INPUTS 0x2u    /* FPMM_CONTRACTS analogue: verify A, B hold residues in [0,p) */
#define FPMM_B200_INPLACE_INVERSES 0x4u /* mw_product semantics: require alpha, beta invertible mod p
                                           (multiword.hpp:76-86); NoInverseError otherwise */
#define FPMM_B200_BCAST_RAW_B 0x8u     /* multi-GPU: broadcast raw B and pack locally (default: B words) */
/* engine selection (same results, different tensor-core path):
 *   DMMA: the paper's FP64 multiword product on the FP64 tensor pipe (mma.sync .f64)
 *   I8  : base-256 multiword words on tcgen05.mma.kind::i8 (int32 TMEM accumulators)
 *   RNS : byte residues modulo pairwise-coprime m_i <= 256, one kind::i8 GEMM per
 *         modulus (epilogue parks T_i mod m_i, one byte per element), then one
 *         CRT reconstruction kernel mod p; for k <= 256 with <= 12 moduli the
 *         residues stay on chip and the CRT runs in the GEMM's epilogue
 * no flag = the library default: I8 or RNS, whichever a B200 time model
 * predicts faster for (m, k, n, p) (I8 for prepared A, where n is unknown) */
#define FPMM_B200_ENGINE_DMMA 0x10u
#define FPMM_B200_ENGINE_I8 0x20u
#define FPMM_B200_ENGINE_RNS 0x40u
/* FP64 engine: use exactly the caller's (u,v) words.  By default the engine may
 * use other word counts where the caller's collapse the exact K-block
 * (lambda_k = 4 at the rule's limits, e.g. (2,2) at 52 bits); C is the same. */
#define FPMM_B200_DMMA_EXACT_WORDS 0x80u
/* Instrumented mode, the analogue of the reference's shadow replay
 * (shadow.hpp:125-162, `fpmm check --checked`): the FP64 engine verifies at
 * every in-register reduction (and before its epilogue) that each accumulator
 * is at most 2^53 in magnitude, i.e. still exact; a violation fails the call
 * with FPMM_B200_ECONTRACT.  The int8 engines are exact by construction. */
#define FPMM_B200_CHECK_EXACTNESS 0x200u

/* product variants (multiword.hpp:113-254); all map to the same fused kernel */
typedef enum {
  FPMM_B200_PLAIN = 0,     /* mw_product / mw_product_words        */
  FPMM_B200_WORKSPACE = 1, /* mw_product_workspace(_words)          */
  FPMM_B200_CONCAT = 2     /* mw_product_concat(_words)             */
} fpmm_b200_variant;

/* planner.hpp:57-65 ProductPlan */
typedef struct {
  int u, v;
  uint64_t lambda;
  int concat; /* 0 none, 1 a, 2 b (ConcatChoice) */
  uint64_t predicted_products;
  uint64_t predicted_reductions;
  uint64_t storage_entries;
} fpmm_b200_plan;

/* optional per-call timing (CUDA events on the call's stream, milliseconds) */
typedef struct {
  double h2d_ms;       /* host -> device copies (host-buffer entry points)   */
  double pack_ms;      /* decomposition kernels (A and B words)              */
  double gemm_ms;      /* product kernel(s): GEMM and its fused epilogue      */
  double comm_ms;      /* NCCL broadcast / gather                            */
  double d2h_ms;       /* device -> host copy of C                           */
  double total_ms;     /* whole call                                         */
  int64_t lambda_k;    /* K-block between in-register reductions (terms)     */
  int32_t launches;    /* kernels launched by this call (all devices)        */
  int32_t ngpus;       /* devices used                                       */
  int32_t engine;      /* engine that ran: 0x10 DMMA, 0x20 I8, 0x40 RNS (FPMM_B200_ENGINE_*) */
  int32_t words;       /* words per residue: u*v (DMMA), base-256 digits D (I8), moduli (RNS) */
  double recon_ms;     /* reconstruction kernels after the product kernel (RNS CRT, int8 split-K
                          combine); gemm_ms is the product kernel alone where this is set */
} fpmm_b200_timing;

/* ------------------------------------------------------------ diagnostics */
const char* fpmm_b200_last_error(void);
int fpmm_b200_version(void);
int fpmm_b200_device_count(int* out);

/* --------------------------------------------------- host-side rule layer */
/* primality.hpp:8-11 */
int fpmm_b200_is_prime(uint64_t n);
uint64_t fpmm_b200_prev_prime(uint64_t limit);
/* FpContext<double>::make validation (fp_context.hpp:36-48): 5 <= p < 2^52, prime unless allowed */
int fpmm_b200_context_check(uint64_t p, int allow_composite);
/* multiword.cpp:7-19 word_base; multiword.hpp:16 word_bound */
int fpmm_b200_word_base(uint64_t p, int u, uint64_t* out);
/* block_product.hpp:13-22 max_block_size; *out = 0 encodes std::nullopt */
int fpmm_b200_max_block_size(uint64_t max_a, uint64_t max_b, uint64_t p, int t, uint64_t* out);
/* planner.hpp:29-31 mw_block_size; *out = 0 encodes std::nullopt */
int fpmm_b200_mw_block_size(int u, int v, uint64_t p, int t, uint64_t* out);
/* planner.cpp:20-28 variant_bit_limit (scan from b=2) */
int fpmm_b200_variant_bit_limit(int u, int v, int t, int* out);
/* planner.cpp:93-101 select_variant / plan_for_modulus */
int fpmm_b200_select_variant(int bits, int64_t m, int64_t k, int64_t n, int t, uint64_t min_lambda,
                             int64_t concat_threshold, fpmm_b200_plan* out);
int fpmm_b200_plan_for_modulus(uint64_t p, int64_t m, int64_t k, int64_t n, int t,
                               uint64_t min_lambda, int64_t concat_threshold, fpmm_b200_plan* out);
/* planner.cpp:30-42 finish_plan */
int fpmm_b200_finish_plan(fpmm_b200_plan* plan, int64_t m, int64_t k, int64_t n);
/* the fused kernel's internal K-block (terms between in-register reductions)
 * for balanced signed words; >= 4 for every (u,v,p) the reference admits */
int fpmm_b200_kernel_block(uint64_t p, int u, int v, int64_t* lambda_k);
/* RNS engine words: the smallest count n of the fixed pairwise-coprime byte
 * moduli (256, 255, 253, 251, ...) whose product M covers the centred exact
 * sum, 1000 M >= 2030 K floor(p/2)^2, and the CRT constants:
 * y_i = (M/m_i)^-1 mod m_i, g_i = round(2^24 y_i / m_i),
 * W_i = y_i (M/m_i) mod p, Mp = M mod p.  Arrays hold FPMM_B200_RNS_MAX_MODULI. */
#define FPMM_B200_RNS_MAX_MODULI 20
/* The engine the library default (no ENGINE_* flag) runs for an m x k by k x n
 * product mod p: FPMM_B200_ENGINE_I8 or FPMM_B200_ENGINE_RNS (B200 time model). */
int fpmm_b200_select_engine(int64_t m, int64_t k, int64_t n, uint64_t p, unsigned* engine_flag);
int fpmm_b200_rns_plan(uint64_t p, int64_t k, int* nmod, uint32_t* moduli, uint32_t* y, uint32_t* g,
                       uint64_t* W, uint64_t* Mp);

/* mat.hpp:92-120 random_mat + driver.cpp:14-20 matrix_seed (synthetic inputs) */
uint64_t fpmm_b200_mix_seed(uint64_t a, uint64_t b);
uint64_t fpmm_b200_matrix_seed(uint64_t seed, int bits, int64_t m, int64_t k, int64_t n,
                               uint64_t which);
int fpmm_b200_random_mat(int64_t rows, int64_t cols, uint64_t p, uint64_t seed, double* out);

/* ------------------------------------------------ products, host buffers */
/* multiword.hpp:133-139 mw_product (+ _workspace :248-254, _concat :211-218).
 * A: m x k (lda), B: k x n (ldb), C: m x n (ldc), all caller-owned host memory
 * (pinned memory gives full PCIe bandwidth).  lambda is validated exactly as
 * check_mw_inputs (multiword.hpp:58-70).  ngpus >= 1 row-shards C across
 * devices 0..ngpus-1 of this process (B words broadcast over NCCL). */
int fpmm_b200_mw_product(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t m, int64_t k, int64_t n, uint64_t p, int u, int v,
                         uint64_t lambda, int variant, int ngpus, unsigned flags,
                         fpmm_b200_timing* timing);

/* multiword.hpp:113-131 mw_product_words: host word planes (words[i] at
 * Awords + i*a_word_stride, each m x k with lda), bases alpha/beta as in
 * WordDecomposition (multiword.hpp:19-24). */
int fpmm_b200_mw_product_words(const double* Awords, int64_t a_word_stride, int64_t lda,
                               uint64_t alpha, int u, const double* Bwords,
                               int64_t b_word_stride, int64_t ldb, uint64_t beta, int v,
                               double* C, int64_t ldc, int64_t m, int64_t k, int64_t n,
                               uint64_t p, uint64_t lambda, int variant, unsigned flags,
                               fpmm_b200_timing* timing);

/* multiword.hpp:29-54 decompose, bit-identical words (reference loop
 * r = floor(T*fl(1/alpha)), w = fma(-alpha, r, T)); words[i] written at
 * words + i*word_stride with leading dimension cols. */
int fpmm_b200_decompose(const double* M, int64_t ld, int64_t rows, int64_t cols, uint64_t p,
                        int u, double* words, int64_t word_stride, uint64_t* base);

/* block_product.hpp:62-73 block_gemm_mod: C <- C + A B mod p, C reduced */
int fpmm_b200_block_gemm_mod(double* C, int64_t ldc, const double* A, int64_t lda,
                             const double* B, int64_t ldb, int64_t m, int64_t k, int64_t n,
                             uint64_t lambda, uint64_t p, unsigned flags);

/* GemmKernel<double>::accumulate (gemm_kernel.hpp:13-19): exact C += A B on
 * panels whose every partial dot product stays <= 2^53 (the plugin contract,
 * gemm_kernel.hpp:9-12).  Host buffers. */
int fpmm_b200_accumulate(double* C, int64_t ldc, const double* A, int64_t lda, const double* B,
                         int64_t ldb, int64_t m, int64_t w, int64_t n);

/* ---------------------------------------------- products, device buffers */
/* Same as fpmm_b200_mw_product on device-resident A, B, C of `device`,
 * enqueued on `stream` (cudaStream_t, NULL = the library's stream for that
 * device).  Workspace is owned by the library (per device, grown on demand).
 * The call is synchronous unless FPMM_B200_ASYNC is passed in flags. */
#define FPMM_B200_ASYNC 0x100u
int fpmm_b200_mw_product_device(const double* dA, int64_t lda, const double* dB, int64_t ldb,
                                double* dC, int64_t ldc, int64_t m, int64_t k, int64_t n,
                                uint64_t p, int u, int v, uint64_t lambda, int variant,
                                int device, void* stream, unsigned flags,
                                fpmm_b200_timing* timing);
int fpmm_b200_decompose_device(const double* dM, int64_t ld, int64_t rows, int64_t cols,
                               uint64_t p, int u, double* dwords, int64_t word_stride,
                               uint64_t* base, int device, void* stream);
int fpmm_b200_accumulate_device(double* dC, int64_t ldc, const double* dA, int64_t lda,
                                const double* dB, int64_t ldb, int64_t m, int64_t w, int64_t n,
                                int device, void* stream);

/* ------------------------------------------ prepared (resident) A words */
/* The unbalanced scenario (driver.cpp:215-218) reuses A's
 * word decomposition across iterated products: decompose / pack A once,
 * keep the words resident in HBM, multiply by many B.  The engine flag of
 * prepare_a fixes the engine of every product made from the handle. */
typedef struct fpmm_b200_prepared fpmm_b200_prepared;
int fpmm_b200_prepare_a_device(const double* dA, int64_t lda, int64_t m, int64_t k, uint64_t p, int u, int v,
                               unsigned flags, int device, void* stream, fpmm_b200_prepared** out);
/* C (m x n) = A B mod p from the prepared A (mw_product_words with fixed da) */
int fpmm_b200_mw_product_prepared_device(const fpmm_b200_prepared* a, const double* dB, int64_t ldb, double* dC,
                                         int64_t ldc, int64_t n, uint64_t lambda, void* stream, unsigned flags,
                                         fpmm_b200_timing* timing);
int fpmm_b200_prepared_free(fpmm_b200_prepared* a);

/* ------------------------------------- multi-process partitioner (NCCL) */
/* One process per GPU.  Rank 0 creates the id, the host bootstrap (e.g. a
 * torch.distributed / MPI broadcast) ships the 128 bytes to every rank. */
int fpmm_b200_nccl_id_size(void);
int fpmm_b200_nccl_get_unique_id(void* id);
int fpmm_b200_dist_init(const void* id, int nranks, int rank, int device);
int fpmm_b200_dist_finalize(void);
/* Row partition used by the partitioner: rows [*row0, *row0 + *rows) of m. */
int fpmm_b200_dist_rows(int64_t m, int nranks, int rank, int u, int v, int64_t* row0,
                        int64_t* rows);
/* Row chunks [starts[i], starts[i] + lens[i]) of a rank block of `rows` rows
 * in which the row-sharded product computes and, with a gather, ships C to
 * root (chunk i's transfer overlaps chunk i+1's compute).  At most
 * FPMM_B200_DIST_MAX_CHUNKS chunks; the same function on every rank, so root
 * knows each rank's chunks. */
#define FPMM_B200_DIST_MAX_CHUNKS 4
int fpmm_b200_dist_chunks(int64_t m, int64_t k, int64_t n, uint64_t p, int u, int v, unsigned flags,
                          int64_t rows, int* count, int64_t* starts, int64_t* lens);
/* Row-sharded product.  Every rank passes its own A row block (dA_rows:
 * rows x k, this rank's slice from fpmm_b200_dist_rows) and receives its C
 * row block in dC_rows.  dB (k x n) is read on `root` only and its words are
 * broadcast.  If dC_full != NULL on root, the row blocks are gathered there. */
int fpmm_b200_dist_mw_product_device(const double* dA_rows, int64_t lda, const double* dB,
                                     int64_t ldb, double* dC_rows, int64_t ldc, double* dC_full,
                                     int64_t ldc_full, int64_t m, int64_t k, int64_t n, uint64_t p,
                                     int u, int v, uint64_t lambda, int root, void* stream,
                                     unsigned flags, fpmm_b200_timing* timing);

/* ------------------------------------------------------ benchmark support */
/* Uniform residues in [0,p) generated on the device (counter-based
 * splitmix64 with rejection; for inputs too large for the host mt19937_64
 * generator of mat.hpp:112-120).  Rows [row0, row0+rows) of the global
 * matrix, so row-sharded ranks generate consistent slices.  Synchronous
 * when stream is NULL. */
int fpmm_b200_random_residues_device(double* dM, int64_t ld, int64_t rows, int64_t cols, int64_t row0,
                                     uint64_t p, uint64_t seed, int device, void* stream);
/* Exact on-device check of a device-resident product C = A B mod p, for sizes
 * a CPU recomputation cannot reach (the analogue of the reference's
 * oracle-equivalence check, driver.cpp:37-140 / first_mismatch at
 * oracle.hpp:71-81).  All arithmetic is exact (128-bit dot products):
 *   counts[0] = entries of C that are not integers in [0, p)
 *   counts[1] = rows with A (B s) != C s (mod p), summed over `trials`
 *               Freivalds trials with uniform s in [0, p)^n (a wrong C passes
 *               one trial with probability <= 1/p)
 *   counts[2] = wrong entries among `samples` sampled (i, j) (corners first)
 *   counts[3], counts[4] = (i, j) of the first wrong sample, or -1
 * Synchronous on `stream` (NULL = the library's stream for `device`). */
int fpmm_b200_verify_device(const double* dA, int64_t lda, const double* dB, int64_t ldb, const double* dC,
                            int64_t ldc, int64_t m, int64_t k, int64_t n, uint64_t p, uint64_t seed, int trials,
                            int samples, int device, void* stream, int64_t* counts);
/* Measured FP64 tensor-pipe peak (TFLOP/s): a DMMA.8x8x4-only loop. */
int fpmm_b200_fp64_peak(int device, int iters, double* tflops);
/* Measured int8 tensor-core peak (TOP/s): back-to-back tcgen05.mma.kind::i8
 * M=128 N=256 K=32 on every SM. */
int fpmm_b200_i8_peak(int device, int iters, double* tops);
/* Diagnostic tensor-pipe probe: mode 0 = one CTA per SM (M128 N256), mode 1 =
 * CTA pairs issuing cta_group::2 M256 N256 MMAs.  Long `iters` measure the
 * sustained (power-capped) rate. */
int fpmm_b200_i8_probe(int device, int iters, int mode, double* tops);

/* release every device workspace, stream and communicator */
int fpmm_b200_finalize(void);

#ifdef __cplusplus
}
#endif
#endif /* FPMM_B200_H */
