// Host-rule checks through the C++ drop-in header (no GPU needed).
#include <cstdio>
#include <cstdlib>

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
  REQUIRE(prev_prime(u64{1} << 52) == (u64{1} << 52) - 47);
  REQUIRE(is_prime_u64(97) && !is_prime_u64(91));
  REQUIRE(word_base(97, 2) == 10 && word_base(101, 3) == 5);
  REQUIRE(variant_bit_limit(1, 1, 53) == 26 && variant_bit_limit(1, 2, 53) == 35);
  REQUIRE(variant_bit_limit(1, 3, 53) == 39 && variant_bit_limit(1, 4, 53) == 42);
  REQUIRE(variant_bit_limit(2, 2, 53) == 52 && variant_bit_limit(2, 3, 53) == 52);
  auto F = FpContext<double>::make((u64{1} << 50) - 27);
  auto lam = mw_block_size(2, 2, F);
  REQUIRE(lam && *lam == 7);
  ProductPlan pl = plan_for_modulus(F.p(), 1024, 1024, 1024, 53);
  REQUIRE(pl.u == 2 && pl.v == 2 && pl.lambda == 7);
  REQUIRE(select_variant(37, 1024, 1024, 1024, 53).variant() == (Variant{1, 3}));
  bool threw = false;
  try {
    FpContext<double>::make(91);
  } catch (const Error&) {
    threw = true;
  }
  REQUIRE(threw);
  threw = false;
  try {
    Mat<double> A(2, 2), B(2, 2);
    mw_product(A, B, 2, 2, 2, FpContext<double>::make((u64{1} << 52) - 47));
  } catch (const InfeasibleError&) {
    threw = true;
  }
  REQUIRE(threw);
  // kernel names pin an engine (plugin conformance: name() round-trips)
  REQUIRE(kernel_by_name<double>("b200") == &b200_kernel<double>());
  REQUIRE(kernel_by_name<double>("accelerated") == &b200_kernel<double>());
  for (const char* nm : {"b200-rns", "b200-i8", "b200-dmma"}) {
    const GemmKernel<double>* k = kernel_by_name<double>(nm);
    REQUIRE(k && k->name() == nm);
  }
  REQUIRE(detail::engine_of(*kernel_by_name<double>("b200-rns")) == FPMM_B200_ENGINE_RNS);
  REQUIRE(detail::engine_of(b200_kernel<double>()) == 0u);
  REQUIRE(kernel_by_name<double>("naive") == nullptr);
  auto M = random_mat<double>(3, 4, 31, 1);
  REQUIRE(M.max_bound() <= 30);
  std::printf("OK\n");
  return 0;
}
