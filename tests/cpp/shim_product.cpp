// A reference-style program against the C++ drop-in header, on the GPU:
// fpmm::mw_product with the planned (u,v,lambda) for every kernel name, the
// workspace and concat variants, all bit-identical and checked entry by entry
// against an exact __int128 dot product.
#include <cstdio>

#include "fpmm_b200/fpmm.hpp"

#define REQUIRE(c)                                              \
  do {                                                          \
    if (!(c)) {                                                 \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);   \
      return 1;                                                 \
    }                                                           \
  } while (0)

int main() {
  using namespace fpmm;
  for (int bits : {20, 33, 47, 52}) {
    const u64 p = prev_prime(u64{1} << bits);
    const index_t m = 130, k = 517, n = 70;
    const auto A = random_mat<double>(m, k, p, 1000 + bits);
    const auto B = random_mat<double>(k, n, p, 2000 + bits);
    const auto F = FpContext<double>::make(p);
    const ProductPlan pl = plan_for_modulus(p, m, k, n, 53);
    const Mat<double> C = mw_product(A, B, pl.u, pl.v, pl.lambda, F, *kernel_by_name<double>("b200"));
    for (const char* nm : {"b200-rns", "b200-i8", "b200-dmma"})
      REQUIRE(mw_product(A, B, pl.u, pl.v, pl.lambda, F, *kernel_by_name<double>(nm)) == C);
    REQUIRE(mw_product_workspace(A, B, pl.u, pl.v, pl.lambda, F, b200_kernel<double>()) == C);
    REQUIRE(mw_product_concat(A, B, pl.u, pl.v, pl.lambda, F, b200_kernel<double>()) == C);
    for (index_t i = 0; i < m; i += 13)
      for (index_t j = 0; j < n; j += 7) {
        unsigned __int128 acc = 0;
        for (index_t t = 0; t < k; ++t)
          acc += static_cast<unsigned __int128>(static_cast<u64>(A(i, t))) * static_cast<u64>(B(t, j));
        REQUIRE(static_cast<u64>(C(i, j)) == static_cast<u64>(acc % p));
      }
  }
  std::printf("OK\n");
  return 0;
}
