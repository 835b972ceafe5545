// rules.hpp -- host-side exact integer rules of the multiword product.
//
// Re-implements (from the paper and the reference's documented behaviour) the
// prime rule, FpContext validation, word bases, block-size bounds and the
// (u,v) planner, plus the B200 kernel's own exactness budget for balanced
// signed words.  All arithmetic is exact (unsigned __int128).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace fpmm_b200 {

using u64 = std::uint64_t;
using i64 = std::int64_t;
using u128 = unsigned __int128;

// Status-carrying exception used inside the library; the C-ABI maps it to
// fpmm_b200_status and a thread-local message.
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

constexpr int kT = 53;  // binary64 significand bits (FpContext<double>::t)

int bitsize(u64 n);
u64 mulmod(u64 a, u64 b, u64 m);
u64 powmod(u64 b, u64 e, u64 m);
bool is_prime(u64 n);
u64 prev_prime(u64 limit);

// FpContext<double>::make (fp_context.hpp:36-48); throws Failure
void context_check(u64 p, bool allow_composite);

u64 word_base(u64 p, int u);   // multiword.cpp:7-19
u64 word_bound(u64 p, int u);  // multiword.hpp:16
u64 max_block_size(u64 max_a, u64 max_b, u64 p, int t);  // 0 == nullopt
u64 mw_block_size(int u, int v, u64 p, int t);           // 0 == nullopt
int variant_bit_limit(int u, int v, int t);

struct Plan {
  int u = 1, v = 1;
  u64 lambda = 1;
  int concat = 0;
  u64 products = 1, reductions = 0, storage = 0;
};
void finish_plan(Plan& pl, i64 m, i64 k, i64 n);
Plan select_variant(int bits, i64 m, i64 k, i64 n, int t, u64 min_lambda, i64 concat_threshold);
Plan plan_for_modulus(u64 p, i64 m, i64 k, i64 n, int t, u64 min_lambda, i64 concat_threshold);

// check_mw_inputs (multiword.hpp:58-70)
void check_mw_inputs(i64 k, i64 bk, int u, int v, u64 lambda, u64 p);

// ---------------------------------------------------------------------------
// Balanced signed words used by the B200 kernel.
//
// x in [0,p) is first centred, x' = x - p [x > p/2], then split in base
// alpha = word_base(p,u) into digits d_i = (x'_i + h) mod alpha - h, h =
// floor(alpha/2), x'_{i+1} = floor((x'_i + h)/alpha); the last digit is
// what remains.  So x' = sum alpha^i d_i exactly, |d_i| <= h for i < u-1 and
// the top digit is bounded by simulating the (monotone) recursion on the two
// extreme centred values.
struct SignedWords {
  int u = 1;
  u64 alpha = 0;      // base (== p when u == 1)
  u64 half = 0;       // floor(alpha/2)
  u64 max_digit = 0;  // max |d_i| over all digits and all x in [0,p)
};
SignedWords signed_words(u64 p, int u);

// Largest K-block L (a multiple of `step`) with L*Pmax + Rmax <= 2^53, where
// Pmax = max|a_i| max|b_j| and Rmax bounds the carried residue after the
// kernel's reduction r = x - rint(x fl(1/p)) p.  0 if not even `step` fits.
i64 kernel_block(u64 p, int u, int v, int step = 4);

// floor(w * 2^64 / p): Shoup constant for a fixed multiplier w < p
u64 shoup(u64 w, u64 p);

}  // namespace fpmm_b200

namespace fpmm_b200 {

// ---------------------------------------------------------------------------
// Residue-number-system words for the RNS engine (rnsengine.cuh).
//
// Centred residues x' = x - p [x > p/2] are represented modulo n pairwise
// coprime moduli m_i <= 256 (one byte each).  n is the smallest count with
// 1000 M >= 2030 K floor(p/2)^2 (M = prod m_i), so the exact integer
// X = sum_k a'_k b'_k (|X| <= K floor(p/2)^2, |X| / M <= 1/2.03) is recovered
// by the CRT with the rounding of t = round(sum r_i y_i / m_i) (fixed point
// 2^-19, error <= n 255 2^-20 <= 0.005) kept clear of the +-1/2 boundary.
constexpr int kRnsMaxMod = 20;
struct RnsPlan {
  int n = 0;
  std::uint32_t mod[kRnsMaxMod] = {};
  std::uint32_t y[kRnsMaxMod] = {};       // (M/m_i)^{-1} mod m_i
  std::uint32_t g[kRnsMaxMod] = {};       // round(2^24 y_i / m_i) (the C-ABI's exported scale)
  u64 W[kRnsMaxMod] = {};                 // y_i (M/m_i) mod p
  u64 Mp = 0;                             // M mod p
  double log2M = 0, log2X = 0;            // log2 M and log2(2 K floor(p/2)^2)
};
// The fixed modulus list (descending, pairwise coprime).
const std::uint32_t* rns_moduli_list();
// Plan for residues < p and a contraction length k (the CRT range bound);
// throws Failure(EINFEASIBLE) when kRnsMaxMod moduli do not suffice.
RnsPlan rns_plan(u64 p, i64 k);

}  // namespace fpmm_b200
