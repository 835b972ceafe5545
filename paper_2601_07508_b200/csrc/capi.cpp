// capi.cpp -- extern "C" boundary (include/fpmm_b200.h).  Every entry point
// converts library failures into an fpmm_b200_status plus a thread-local
// message; nothing throws across the ABI.
#include <cstring>
#include <exception>
#include <string>

#include "engine.hpp"
#include "fpmm_b200.h"
#include "rules.hpp"

using namespace fpmm_b200;

namespace {
thread_local std::string g_last;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last.clear();
    return FPMM_B200_OK;
  } catch (const Failure& e) {
    g_last = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last = "host allocation failed";
    return FPMM_B200_ENOMEM;
  } catch (const std::exception& e) {
    g_last = e.what();
    return FPMM_B200_EERROR;
  }
}

void to_c(const Plan& pl, fpmm_b200_plan* out) {
  out->u = pl.u;
  out->v = pl.v;
  out->lambda = pl.lambda;
  out->concat = pl.concat;
  out->predicted_products = pl.products;
  out->predicted_reductions = pl.reductions;
  out->storage_entries = pl.storage;
}

void check_variant(int variant) {
  if (variant < FPMM_B200_PLAIN || variant > FPMM_B200_CONCAT)
    throw Failure(FPMM_B200_EERROR, "unknown product variant " + std::to_string(variant));
}

// the plain (in-place) variant needs alpha^-1 / beta^-1 (multiword.hpp:76-86)
unsigned variant_flags(int variant, unsigned flags) {
  return variant == FPMM_B200_PLAIN ? (flags | FPMM_B200_INPLACE_INVERSES) : flags;
}
}  // namespace

extern "C" {

const char* fpmm_b200_last_error(void) { return g_last.c_str(); }
int fpmm_b200_version(void) { return FPMM_B200_VERSION; }
int fpmm_b200_device_count(int* out) {
  return guarded([&] { *out = device_count(); });
}

int fpmm_b200_is_prime(uint64_t n) { return is_prime(n) ? 1 : 0; }
uint64_t fpmm_b200_prev_prime(uint64_t limit) { return prev_prime(limit); }

int fpmm_b200_context_check(uint64_t p, int allow_composite) {
  return guarded([&] { context_check(p, allow_composite != 0); });
}

int fpmm_b200_word_base(uint64_t p, int u, uint64_t* out) {
  return guarded([&] { *out = word_base(p, u); });
}

int fpmm_b200_max_block_size(uint64_t max_a, uint64_t max_b, uint64_t p, int t, uint64_t* out) {
  return guarded([&] {
    if (t < 3 || t > 62) throw Failure(FPMM_B200_EERROR, "t out of range");
    *out = max_block_size(max_a, max_b, p, t);
  });
}

int fpmm_b200_mw_block_size(int u, int v, uint64_t p, int t, uint64_t* out) {
  return guarded([&] {
    if (t < 3 || t > 62) throw Failure(FPMM_B200_EERROR, "t out of range");
    *out = mw_block_size(u, v, p, t);
  });
}

int fpmm_b200_variant_bit_limit(int u, int v, int t, int* out) {
  return guarded([&] { *out = variant_bit_limit(u, v, t); });
}

int fpmm_b200_select_variant(int bits, int64_t m, int64_t k, int64_t n, int t, uint64_t min_lambda,
                             int64_t concat_threshold, fpmm_b200_plan* out) {
  return guarded([&] { to_c(select_variant(bits, m, k, n, t, min_lambda, concat_threshold), out); });
}

int fpmm_b200_plan_for_modulus(uint64_t p, int64_t m, int64_t k, int64_t n, int t,
                               uint64_t min_lambda, int64_t concat_threshold, fpmm_b200_plan* out) {
  return guarded([&] { to_c(plan_for_modulus(p, m, k, n, t, min_lambda, concat_threshold), out); });
}

int fpmm_b200_finish_plan(fpmm_b200_plan* plan, int64_t m, int64_t k, int64_t n) {
  return guarded([&] {
    Plan pl;
    pl.u = plan->u;
    pl.v = plan->v;
    pl.lambda = plan->lambda;
    pl.concat = plan->concat;
    finish_plan(pl, m, k, n);
    to_c(pl, plan);
  });
}

int fpmm_b200_kernel_block(uint64_t p, int u, int v, int64_t* lambda_k) {
  return guarded([&] {
    if (u < 1 || v < 1) throw Failure(FPMM_B200_EERROR, "word counts must be positive");
    *lambda_k = kernel_block(p, u, v, 4);
  });
}

int fpmm_b200_rns_plan(uint64_t p, int64_t k, int* nmod, uint32_t* moduli, uint32_t* y, uint32_t* g,
                       uint64_t* W, uint64_t* Mp) {
  return guarded([&] {
    if (k < 0) throw Failure(FPMM_B200_EERROR, "k must be nonnegative");
    const RnsPlan pl = rns_plan(p, k);
    *nmod = pl.n;
    for (int i = 0; i < pl.n; ++i) {
      if (moduli) moduli[i] = pl.mod[i];
      if (y) y[i] = pl.y[i];
      if (g) g[i] = pl.g[i];
      if (W) W[i] = pl.W[i];
    }
    if (Mp) *Mp = pl.Mp;
  });
}

int fpmm_b200_select_engine(int64_t m, int64_t k, int64_t n, uint64_t p, unsigned* engine_flag) {
  return guarded([&] { *engine_flag = select_engine(m, k, n, p); });
}

// mat.hpp:104-110 (splitmix64 step)
uint64_t fpmm_b200_mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ull * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// driver.cpp:14-20
uint64_t fpmm_b200_matrix_seed(uint64_t seed, int bits, int64_t m, int64_t k, int64_t n,
                               uint64_t which) {
  uint64_t h = fpmm_b200_mix_seed(seed, static_cast<uint64_t>(bits));
  h = fpmm_b200_mix_seed(h, static_cast<uint64_t>(m));
  h = fpmm_b200_mix_seed(h, static_cast<uint64_t>(k));
  h = fpmm_b200_mix_seed(h, static_cast<uint64_t>(n));
  return fpmm_b200_mix_seed(h, which);
}

int fpmm_b200_random_mat(int64_t rows, int64_t cols, uint64_t p, uint64_t seed, double* out);

int fpmm_b200_mw_product(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t m, int64_t k, int64_t n, uint64_t p, int u, int v,
                         uint64_t lambda, int variant, int ngpus, unsigned flags,
                         fpmm_b200_timing* timing) {
  return guarded([&] {
    check_variant(variant);
    ProductArgs a{A, lda, B, ldb, C, ldc, m, k, n, p, u, v, lambda, variant_flags(variant, flags)};
    product_host(a, ngpus, timing);
  });
}

int fpmm_b200_mw_product_words(const double* Awords, int64_t a_word_stride, int64_t lda,
                               uint64_t alpha, int u, const double* Bwords,
                               int64_t b_word_stride, int64_t ldb, uint64_t beta, int v,
                               double* C, int64_t ldc, int64_t m, int64_t k, int64_t n,
                               uint64_t p, uint64_t lambda, int variant, unsigned flags,
                               fpmm_b200_timing* timing) {
  return guarded([&] {
    check_variant(variant);
    product_words_host(Awords, a_word_stride, lda, alpha, u, Bwords, b_word_stride, ldb, beta, v, C, ldc,
                       m, k, n, p, lambda, variant_flags(variant, flags), timing);
  });
}

int fpmm_b200_decompose(const double* M, int64_t ld, int64_t rows, int64_t cols, uint64_t p,
                        int u, double* words, int64_t word_stride, uint64_t* base) {
  return guarded([&] { decompose_host(M, ld, rows, cols, p, u, words, word_stride, base); });
}

int fpmm_b200_block_gemm_mod(double* C, int64_t ldc, const double* A, int64_t lda,
                             const double* B, int64_t ldb, int64_t m, int64_t k, int64_t n,
                             uint64_t lambda, uint64_t p, unsigned flags) {
  return guarded([&] { block_gemm_mod_host(C, ldc, A, lda, B, ldb, m, k, n, lambda, p, flags); });
}

int fpmm_b200_accumulate(double* C, int64_t ldc, const double* A, int64_t lda, const double* B,
                         int64_t ldb, int64_t m, int64_t w, int64_t n) {
  return guarded([&] { accumulate_host(C, ldc, A, lda, B, ldb, m, w, n); });
}

int fpmm_b200_mw_product_device(const double* dA, int64_t lda, const double* dB, int64_t ldb,
                                double* dC, int64_t ldc, int64_t m, int64_t k, int64_t n,
                                uint64_t p, int u, int v, uint64_t lambda, int variant,
                                int device, void* stream, unsigned flags,
                                fpmm_b200_timing* timing) {
  return guarded([&] {
    check_variant(variant);
    ProductArgs a{dA, lda, dB, ldb, dC, ldc, m, k, n, p, u, v, lambda, variant_flags(variant, flags)};
    product_device(a, device, stream, timing);
  });
}

int fpmm_b200_decompose_device(const double* dM, int64_t ld, int64_t rows, int64_t cols,
                               uint64_t p, int u, double* dwords, int64_t word_stride,
                               uint64_t* base, int device, void* stream) {
  return guarded([&] { decompose_device(dM, ld, rows, cols, p, u, dwords, word_stride, base, device, stream); });
}

int fpmm_b200_accumulate_device(double* dC, int64_t ldc, const double* dA, int64_t lda,
                                const double* dB, int64_t ldb, int64_t m, int64_t w, int64_t n,
                                int device, void* stream) {
  return guarded([&] { accumulate_device(dC, ldc, dA, lda, dB, ldb, m, w, n, device, stream); });
}

int fpmm_b200_prepare_a_device(const double* dA, int64_t lda, int64_t m, int64_t k, uint64_t p, int u, int v,
                               unsigned flags, int device, void* stream, fpmm_b200_prepared** out) {
  return guarded([&] {
    *out = reinterpret_cast<fpmm_b200_prepared*>(prepare_a_device(dA, lda, m, k, p, u, v, flags, device, stream));
  });
}

int fpmm_b200_mw_product_prepared_device(const fpmm_b200_prepared* a, const double* dB, int64_t ldb, double* dC,
                                         int64_t ldc, int64_t n, uint64_t lambda, void* stream, unsigned flags,
                                         fpmm_b200_timing* timing) {
  return guarded([&] {
    product_prepared_device(reinterpret_cast<const Prepared*>(a), dB, ldb, dC, ldc, n, lambda, stream, flags, timing);
  });
}

int fpmm_b200_prepared_free(fpmm_b200_prepared* a) {
  return guarded([&] { prepared_free(reinterpret_cast<Prepared*>(a)); });
}

int fpmm_b200_nccl_id_size(void) { return nccl_id_size(); }
int fpmm_b200_nccl_get_unique_id(void* id) {
  return guarded([&] { nccl_unique_id(id); });
}
int fpmm_b200_dist_init(const void* id, int nranks, int rank, int device) {
  return guarded([&] { dist_init(id, nranks, rank, device); });
}
int fpmm_b200_dist_finalize(void) {
  return guarded([&] { dist_finalize(); });
}
int fpmm_b200_dist_rows(int64_t m, int nranks, int rank, int u, int v, int64_t* row0,
                        int64_t* rows) {
  return guarded([&] {
    i64 a = 0, b = 0;
    dist_rows(m, nranks, rank, u, v, &a, &b);
    *row0 = a;
    *rows = b;
  });
}
int fpmm_b200_dist_chunks(int64_t m, int64_t k, int64_t n, uint64_t p, int u, int v, unsigned flags,
                          int64_t rows, int* count, int64_t* starts, int64_t* lens) {
  return guarded([&] {
    if (rows < 0) throw Failure(FPMM_B200_EERROR, "rows must be nonnegative");
    dist_chunks(m, k, n, p, u, v, flags, rows, count, starts, lens);
  });
}
int fpmm_b200_dist_mw_product_device(const double* dA_rows, int64_t lda, const double* dB,
                                     int64_t ldb, double* dC_rows, int64_t ldc, double* dC_full,
                                     int64_t ldc_full, int64_t m, int64_t k, int64_t n, uint64_t p,
                                     int u, int v, uint64_t lambda, int root, void* stream,
                                     unsigned flags, fpmm_b200_timing* timing) {
  return guarded([&] {
    dist_product_device(dA_rows, lda, dB, ldb, dC_rows, ldc, dC_full, ldc_full, m, k, n, p, u, v, lambda, root,
                        stream, flags, timing);
  });
}

int fpmm_b200_random_residues_device(double* dM, int64_t ld, int64_t rows, int64_t cols, int64_t row0,
                                     uint64_t p, uint64_t seed, int device, void* stream) {
  return guarded([&] { random_residues_device(dM, ld, rows, cols, row0, p, seed, device, stream); });
}

int fpmm_b200_verify_device(const double* dA, int64_t lda, const double* dB, int64_t ldb, const double* dC,
                            int64_t ldc, int64_t m, int64_t k, int64_t n, uint64_t p, uint64_t seed, int trials,
                            int samples, int device, void* stream, int64_t* counts) {
  return guarded([&] {
    if (!counts) throw Failure(FPMM_B200_EERROR, "verify: counts must not be NULL");
    verify_device(dA, lda, dB, ldb, dC, ldc, m, k, n, p, seed, trials, samples, device, stream, counts);
  });
}

int fpmm_b200_fp64_peak(int device, int iters, double* tflops) {
  return guarded([&] { *tflops = fp64_peak_tflops(device, iters); });
}

int fpmm_b200_i8_peak(int device, int iters, double* tops) {
  return guarded([&] { *tops = i8_peak_tops(device, iters); });
}

int fpmm_b200_i8_probe(int device, int iters, int mode, double* tops) {
  return guarded([&] { *tops = i8_probe_tops(device, iters, mode); });
}

int fpmm_b200_finalize(void) {
  return guarded([&] { finalize_all(); });
}

}  // extern "C"
