// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" veneer over the UNMODIFIED reference library, compiled
// from its sources where they lie (/root/reference/proj/src/*.cpp, see
// oracle/Makefile) into oracle/_ref/libfpmm_ref.so.  It lets the Python tests
// and bench.py's reference arm drive the reference's own mw_product /
// decompose / planner code paths.  Nothing here re-implements reference
// arithmetic; only driver.cpp's 5-line matrix_seed (driver.cpp:14-20, which
// cannot be compiled because driver.cpp includes the boost oracle) is
// restated.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>

#include "fpmm/block_product.hpp"
#include "fpmm/fp_context.hpp"
#include "fpmm/gemm_kernel.hpp"
#include "fpmm/mat.hpp"
#include "fpmm/multiword.hpp"
#include "fpmm/planner.hpp"
#include "fpmm/primality.hpp"

using namespace fpmm;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

Mat<double> from_ptr(const double* p, int64_t r, int64_t c) {
  Mat<double> m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

const GemmKernel<double>& pick(int accelerated) {
  if (accelerated && blas_kernel_available()) return blas_kernel<double>();
  return naive_kernel<double>();
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const InfeasibleError& e) {
    return fail(e, 2);
  } catch (const NoInverseError& e) {
    return fail(e, 3);
  } catch (const ContractError& e) {
    return fail(e, 4);
  } catch (const Error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 5);
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_blas_available() { return blas_kernel_available() ? 1 : 0; }
void ref_set_threads(int n) { set_blas_threads(n); }

uint64_t ref_prev_prime(uint64_t limit) { return prev_prime(limit); }
int ref_is_prime(uint64_t n) { return is_prime_u64(n) ? 1 : 0; }

int ref_word_base(uint64_t p, int u, uint64_t* out) {
  return guard([&] { *out = word_base(p, u); });
}

// 0 = nullopt
int ref_mw_block_size(int u, int v, uint64_t p, int t, uint64_t* out) {
  return guard([&] {
    auto l = mw_block_size(u, v, p, t);
    *out = l ? *l : 0;
  });
}

// the shipped rule (planner.cpp:20-28); throws for u*v > 1
int ref_variant_bit_limit(int u, int v, int t, int* out) {
  return guard([&] { *out = variant_bit_limit(u, v, t); });
}

int ref_plan_for_modulus(uint64_t p, int64_t m, int64_t k, int64_t n, int t, int* u, int* v,
                         uint64_t* lambda) {
  return guard([&] {
    ProductPlan pl = plan_for_modulus(p, m, k, n, t);
    *u = pl.u;
    *v = pl.v;
    *lambda = pl.lambda;
  });
}

// driver.cpp:14-20
uint64_t ref_matrix_seed(uint64_t seed, int bits, int64_t m, int64_t k, int64_t n,
                         uint64_t which) {
  uint64_t h = mix_seed(seed, static_cast<uint64_t>(bits));
  h = mix_seed(h, static_cast<uint64_t>(m));
  h = mix_seed(h, static_cast<uint64_t>(k));
  h = mix_seed(h, static_cast<uint64_t>(n));
  return mix_seed(h, which);
}

void ref_random_mat(int64_t rows, int64_t cols, uint64_t p, uint64_t seed, double* out) {
  Mat<double> m = random_mat<double>(rows, cols, p, seed);
  std::memcpy(out, m.data(), sizeof(double) * m.size());
}

int ref_decompose(const double* M, int64_t rows, int64_t cols, uint64_t p, int u, double* words,
                  uint64_t* base) {
  return guard([&] {
    auto F = FpContext<double>::make(p, true);
    auto d = decompose(from_ptr(M, rows, cols), u, F);
    *base = d.base;
    for (int i = 0; i < u; ++i)
      std::memcpy(words + static_cast<size_t>(i) * rows * cols, d.words[i].data(),
                  sizeof(double) * static_cast<size_t>(rows * cols));
  });
}

// variant: 0 plain (Alg 3.2), 1 workspace, 2 concat auto, 3 concat a, 4 concat b
int ref_mw_product(const double* A, const double* B, int64_t m, int64_t k, int64_t n, uint64_t p,
                   int u, int v, uint64_t lambda, int variant, int accelerated,
                   int allow_composite, double* C) {
  return guard([&] {
    auto F = FpContext<double>::make(p, allow_composite != 0);
    Mat<double> a = from_ptr(A, m, k), b = from_ptr(B, k, n);
    a.set_max_hint(p - 1);
    b.set_max_hint(p - 1);
    const auto& K = pick(accelerated);
    Mat<double> c;
    switch (variant) {
      case 0: c = mw_product(a, b, u, v, lambda, F, K); break;
      case 1: c = mw_product_workspace(a, b, u, v, lambda, F, K); break;
      case 2: c = mw_product_concat(a, b, u, v, lambda, F, K, ConcatSide::auto_pick); break;
      case 3: c = mw_product_concat(a, b, u, v, lambda, F, K, ConcatSide::a); break;
      default: c = mw_product_concat(a, b, u, v, lambda, F, K, ConcatSide::b); break;
    }
    std::memcpy(C, c.data(), sizeof(double) * c.size());
  });
}

// run_bench's square-scenario timed region (driver.cpp:222-243): lambda from
// the rule, decompose(B), decompose(A), mw_product_words, `runs` times.
// Returns the mean seconds per run in *t_avg.
int ref_bench_square(const double* A, const double* B, int64_t m, int64_t k, int64_t n,
                     uint64_t p, int u, int v, int accelerated, int runs, double* C,
                     double* t_avg) {
  return guard([&] {
    constexpr int t = FpContext<double>::t;
    auto F = FpContext<double>::make(p);
    Mat<double> a = from_ptr(A, m, k), b = from_ptr(B, k, n);
    a.set_max_hint(p - 1);
    b.set_max_hint(p - 1);
    const auto& K = pick(accelerated);
    double total = 0.0;
    Mat<double> c;
    for (int r = 0; r < runs; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const auto lam0 = mw_block_size(u, v, p, t);
      if (!lam0) throw InfeasibleError("no block size");
      const u64 lambda = std::min<u64>(*lam0, static_cast<u64>(k));
      WordDecomposition<double> db = decompose(b, v, F);
      WordDecomposition<double> da = decompose(a, u, F);
      c = mw_product_words(da, db, m, k, n, lambda, F, K);
      const auto t1 = std::chrono::steady_clock::now();
      total += std::chrono::duration<double>(t1 - t0).count();
    }
    *t_avg = total / runs;
    std::memcpy(C, c.data(), sizeof(double) * c.size());
  });
}

}  // extern "C"
