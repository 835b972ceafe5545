// rules.cpp -- exact host-side rules (see rules.hpp).
#include "rules.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "fpmm_b200.h"

namespace fpmm_b200 {

int bitsize(u64 n) { return n ? 64 - __builtin_clzll(n) : 0; }

u64 mulmod(u64 a, u64 b, u64 m) { return static_cast<u64>((static_cast<u128>(a) * b) % m); }

u64 powmod(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  for (b %= m; e; e >>= 1, b = mulmod(b, b, m))
    if (e & 1) r = mulmod(r, b, m);
  return r;
}

// Deterministic Miller-Rabin: the first twelve primes as bases decide every
// n < 3.3e24 (primality.cpp:21-38 uses the same witness set).
bool is_prime(u64 n) {
  static constexpr u64 kBases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 b : kBases) {
    if (n == b) return true;
    if (n % b == 0) return false;
  }
  const int s = __builtin_ctzll(n - 1);
  const u64 d = (n - 1) >> s;
  for (u64 a : kBases) {
    u64 x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool witness = true;
    for (int i = 1; i < s && witness; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) witness = false;
    }
    if (witness) return false;
  }
  return true;
}

// Largest prime strictly below limit (primality.cpp:40-49); 0 if none.
u64 prev_prime(u64 limit) {
  if (limit <= 2) return 0;
  if (limit == 3) return 2;
  u64 n = (limit - 1) | 1;
  if (n >= limit) n -= 2;
  for (; n >= 3; n -= 2)
    if (is_prime(n)) return n;
  return 2;
}

void context_check(u64 p, bool allow_composite) {
  if (p < 5) throw Failure(FPMM_B200_EERROR, "modulus must be at least 5, got " + std::to_string(p));
  if (p >= (u64{1} << (kT - 1)))
    throw Failure(FPMM_B200_EERROR, "modulus must be below 2^" + std::to_string(kT - 1));
  if (!allow_composite && !is_prime(p))
    throw Failure(FPMM_B200_EERROR, "modulus " + std::to_string(p) +
                                        " is composite; pass allow_composite to use the workspace product");
}

namespace {
// a^e saturated at cap
u128 pow_sat(u128 a, int e, u128 cap) {
  u128 r = 1;
  for (int i = 0; i < e; ++i) {
    if (a && r > cap / a) return cap;
    r *= a;
    if (r > cap) return cap;
  }
  return r;
}
}  // namespace

// Smallest integer alpha with alpha^u >= p: a floating root as the first
// guess, then exact integer correction.
u64 word_base(u64 p, int u) {
  if (p < 2) throw Failure(FPMM_B200_EERROR, "word_base: p must exceed 1");
  if (u < 1) throw Failure(FPMM_B200_EERROR, "word_base: word count must be positive");
  if (u == 1) return p;
  const u128 cap = u128{1} << 100;
  u64 a = static_cast<u64>(std::llround(std::pow(static_cast<double>(p), 1.0 / u)));
  a = std::max<u64>(a, 1);
  while (pow_sat(a, u, cap) < p) ++a;
  while (a > 1 && pow_sat(a - 1, u, cap) >= p) --a;
  return a;
}

u64 word_bound(u64 p, int u) { return u == 1 ? p - 1 : word_base(p, u); }

u64 max_block_size(u64 max_a, u64 max_b, u64 p, int t) {
  const u128 budget = (u128{1} << t) - (p - 1);
  const u128 ab = static_cast<u128>(max_a) * max_b;
  if (ab == 0) return std::numeric_limits<u64>::max();
  if (ab > budget) return 0;
  const u128 l = budget / ab;
  return l > std::numeric_limits<u64>::max() ? std::numeric_limits<u64>::max() : static_cast<u64>(l);
}

u64 mw_block_size(int u, int v, u64 p, int t) {
  return max_block_size(word_bound(p, u), word_bound(p, v), p, t);
}

namespace {
bool feasible(int u, int v, u64 p, int t, u64 min_lambda) {
  const u64 l = mw_block_size(u, v, p, t);
  return l != 0 && l >= min_lambda;
}
constexpr int kVariants[6][2] = {{1, 1}, {1, 2}, {1, 3}, {1, 4}, {2, 2}, {2, 3}};
}  // namespace

// Largest bitsize b whose worst-case modulus 2^b - 1 admits lambda >= 1.  The
// scan starts at b = 2: the reference starts at b = 1 (planner.cpp:24) whose
// surrogate modulus 1 makes word_base throw for every multiword variant
// (SURVEY.md F1); b = 2 reproduces Table 3.1 (26/35/39/42/52/52).
int variant_bit_limit(int u, int v, int t) {
  if (u < 1 || v < 1) throw Failure(FPMM_B200_EERROR, "variant_bit_limit: word counts must be positive");
  if (t < 3 || t > 62) throw Failure(FPMM_B200_EERROR, "variant_bit_limit: t out of range");
  int best = 0;
  for (int b = 2; b <= t - 1; ++b)
    if (feasible(u, v, (u64{1} << b) - 1, t, 1)) best = b;
  return best;
}

void finish_plan(Plan& pl, i64 m, i64 k, i64 n) {
  const u64 um = static_cast<u64>(m), uk = static_cast<u64>(k), un = static_cast<u64>(n);
  pl.products = static_cast<u64>(pl.u) * pl.v;
  const u64 panels = pl.lambda ? (uk + pl.lambda - 1) / pl.lambda : 0;
  pl.reductions = pl.products * um * un * (panels + 2);
  pl.storage = uk * (static_cast<u64>(pl.u) * um + static_cast<u64>(pl.v) * un) + um * un;
  if (pl.concat) pl.storage += static_cast<u64>(pl.concat == 2 ? pl.v : pl.u) * um * un;
}

namespace {
// planner.cpp:46-89: minimal uv; ties -> (concat ? larger : smaller) u+v, then smaller u
Plan plan_common(int bits, u64 p_lambda, i64 m, i64 k, i64 n, int t, u64 min_lambda,
                 i64 concat_threshold) {
  if (bits < 1) throw Failure(FPMM_B200_EERROR, "select_variant: bitsize must be positive");
  if (bits > t - 1)
    throw Failure(FPMM_B200_EINFEASIBLE, "modulus unrepresentable: bitsize " + std::to_string(bits) +
                                             " needs p < 2^" + std::to_string(t - 1));
  int concat = 0;
  if (std::min(m, n) < concat_threshold && m != n) concat = n < m ? 2 : 1;
  int best = -1;
  for (int i = 0; i < 6; ++i) {
    const int u = kVariants[i][0], v = kVariants[i][1];
    if (bits > variant_bit_limit(u, v, t) || !feasible(u, v, p_lambda, t, min_lambda)) continue;
    if (best < 0) {
      best = i;
      continue;
    }
    const int bu = kVariants[best][0], bv = kVariants[best][1];
    const int su = u + v, sb = bu + bv;
    if (u * v < bu * bv) best = i;
    else if (u * v == bu * bv && ((concat && su > sb) || (!concat && su < sb) || (su == sb && u < bu)))
      best = i;
  }
  if (best < 0)
    throw Failure(FPMM_B200_EINFEASIBLE, "no (u,v) variant admits bitsize " + std::to_string(bits) +
                                             " with block size >= " + std::to_string(min_lambda));
  Plan pl;
  pl.u = kVariants[best][0];
  pl.v = kVariants[best][1];
  pl.lambda = std::min<u64>(mw_block_size(pl.u, pl.v, p_lambda, t), static_cast<u64>(std::max<i64>(k, 1)));
  pl.concat = concat;
  finish_plan(pl, m, k, n);
  return pl;
}
}  // namespace

Plan select_variant(int bits, i64 m, i64 k, i64 n, int t, u64 min_lambda, i64 concat_threshold) {
  if (bits > 62) throw Failure(FPMM_B200_EINFEASIBLE, "modulus unrepresentable");
  return plan_common(bits, bits >= 1 ? (u64{1} << bits) - 1 : 0, m, k, n, t, min_lambda,
                     concat_threshold);
}

Plan plan_for_modulus(u64 p, i64 m, i64 k, i64 n, int t, u64 min_lambda, i64 concat_threshold) {
  return plan_common(bitsize(p), p, m, k, n, t, min_lambda, concat_threshold);
}

void check_mw_inputs(i64 k, i64 bk, int u, int v, u64 lambda, u64 p) {
  if (u < 1 || v < 1) throw Failure(FPMM_B200_EERROR, "multiword product: word counts must be positive");
  if (k != bk) throw Failure(FPMM_B200_EERROR, "multiword product: dimension mismatch");
  if (lambda < 1) throw Failure(FPMM_B200_EINFEASIBLE, "block size infeasible");
  const u128 peak = static_cast<u128>(lambda) * word_bound(p, u) * word_bound(p, v) + (p - 1);
  if (peak > (u128{1} << kT))
    throw Failure(FPMM_B200_EINFEASIBLE, "multiword product: lambda alpha beta + p - 1 exceeds 2^t");
}

namespace {
// floor((x + h) / a) for signed x, a > 0
i64 floor_div(i64 x, i64 a) {
  i64 q = x / a;
  if ((x % a != 0) && (x < 0)) --q;
  return q;
}
// top digit of the balanced expansion of the centred value x
i64 top_digit(i64 x, int u, i64 a, i64 h) {
  for (int i = 0; i + 1 < u; ++i) x = floor_div(x + h, a);
  return x;
}
}  // namespace

SignedWords signed_words(u64 p, int u) {
  SignedWords s;
  s.u = u;
  s.alpha = word_base(p, u);
  const i64 hi = static_cast<i64>(p / 2);             // largest centred value
  const i64 lo = static_cast<i64>(p / 2) - static_cast<i64>(p) + 1;  // smallest (<= 0)
  if (u == 1) {
    s.half = 0;
    s.max_digit = static_cast<u64>(std::max(hi, -lo));
    return s;
  }
  const i64 a = static_cast<i64>(s.alpha), h = a / 2;
  s.half = static_cast<u64>(h);
  const i64 t_hi = top_digit(hi, u, a, h), t_lo = top_digit(lo, u, a, h);
  s.max_digit = static_cast<u64>(std::max<i64>({h, t_hi, -t_lo}));
  return s;
}

// Rmax: |x - rint(x q) p| <= p/2 + |x| 2^-52 (1 + 2^-50) for |x| <= 2^53 gives
// at most floor(p/2) + 2; one more unit of slack is kept.
i64 kernel_block(u64 p, int u, int v, int step) {
  const SignedWords a = signed_words(p, u), b = signed_words(p, v);
  const u128 pmax = static_cast<u128>(a.max_digit) * b.max_digit;
  const u128 rmax = p / 2 + 3;
  const u128 lim = u128{1} << kT;
  if (pmax == 0) return i64{1} << 40;
  if (rmax + pmax * step > lim) return 0;
  u128 L = (lim - rmax) / pmax;
  if (L > (u128{1} << 40)) L = u128{1} << 40;
  return static_cast<i64>(L) / step * step;
}

u64 shoup(u64 w, u64 p) { return static_cast<u64>((static_cast<u128>(w) << 64) / p); }

}  // namespace fpmm_b200

namespace fpmm_b200 {

namespace {
constexpr std::uint32_t kRnsModuli[kRnsMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227,
                                                  223, 217, 211, 199, 197, 193, 191, 181, 179, 173};

// little-endian base-2^32 magnitudes
using Big = std::vector<std::uint32_t>;
void big_mul(Big& a, u64 f) {
  u128 carry = 0;
  for (auto& x : a) {
    const u128 t = static_cast<u128>(x) * f + carry;
    x = static_cast<std::uint32_t>(t);
    carry = t >> 32;
  }
  for (; carry; carry >>= 32) a.push_back(static_cast<std::uint32_t>(carry));
}
bool big_ge(const Big& a, const Big& b) {
  size_t na = a.size(), nb = b.size();
  while (na > 1 && a[na - 1] == 0) --na;
  while (nb > 1 && b[nb - 1] == 0) --nb;
  if (na != nb) return na > nb;
  for (size_t i = na; i-- > 0;)
    if (a[i] != b[i]) return a[i] > b[i];
  return true;
}
}  // namespace

const std::uint32_t* rns_moduli_list() { return kRnsModuli; }

RnsPlan rns_plan(u64 p, i64 k) {
  if (p < 2) throw Failure(FPMM_B200_EERROR, "rns_plan: p must exceed 1");
  const u64 h = p / 2, kk = static_cast<u64>(std::max<i64>(k, 1));
  Big need{1};  // 2030 K h^2
  big_mul(need, 2030);
  big_mul(need, kk);
  big_mul(need, h);
  big_mul(need, h);
  Big M{1000};
  RnsPlan pl;
  for (int n = 1; n <= kRnsMaxMod; ++n) {
    big_mul(M, kRnsModuli[n - 1]);
    if (big_ge(M, need)) {
      pl.n = n;
      break;
    }
  }
  if (pl.n == 0)
    throw Failure(FPMM_B200_EINFEASIBLE, "rns_plan: " + std::to_string(kRnsMaxMod) +
                                             " byte moduli cannot cover K = " + std::to_string(k) + " at p = " +
                                             std::to_string(p));
  const int n = pl.n;
  pl.Mp = 1 % p;
  pl.log2M = 0;
  for (int i = 0; i < n; ++i) {
    pl.mod[i] = kRnsModuli[i];
    pl.Mp = mulmod(pl.Mp, kRnsModuli[i] % p, p);
    pl.log2M += std::log2(static_cast<double>(kRnsModuli[i]));
  }
  pl.log2X = 1.0 + std::log2(static_cast<double>(kk)) + 2.0 * std::log2(static_cast<double>(std::max<u64>(h, 1)));
  for (int i = 0; i < n; ++i) {
    const std::uint32_t mi = pl.mod[i];
    u64 Mi_mod_mi = 1, Mi_mod_p = 1 % p;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      Mi_mod_mi = Mi_mod_mi * (pl.mod[j] % mi) % mi;
      Mi_mod_p = mulmod(Mi_mod_p, pl.mod[j] % p, p);
    }
    std::uint32_t y = 0;
    for (std::uint32_t c = 1; c < mi; ++c)
      if (Mi_mod_mi * c % mi == 1) {
        y = c;
        break;
      }
    if (y == 0 && mi > 1) throw Failure(FPMM_B200_EERROR, "rns_plan: moduli are not pairwise coprime");
    pl.y[i] = y;
    pl.g[i] = static_cast<std::uint32_t>(((static_cast<u64>(y) << 24) + mi / 2) / mi);
    pl.W[i] = mulmod(y % p, Mi_mod_p, p);
  }
  return pl;
}

}  // namespace fpmm_b200
