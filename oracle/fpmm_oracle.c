/*
 * fpmm_oracle.c -- TEST INFRASTRUCTURE ONLY (see fpmm_oracle.h).
 *
 * Plain-C restatement of the reference algorithms, one function per reference
 * routine, each citing the file:line it follows under /root/reference/proj.
 * Exact ground truth uses unsigned __int128 and never touches floating point.
 */
#include "fpmm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef __int128 i128;

#define T53 53

/* ---------------------------------------------------------------- integers */

/* int_utils.hpp:15 bitsize = bit_width */
int fo_bitsize(uint64_t n) { return n ? 64 - __builtin_clzll(n) : 0; }

/* int_utils.hpp:17-19 */
uint64_t fo_mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)(((u128)a * b) % m); }

/* int_utils.hpp:21-30 */
uint64_t fo_powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = fo_mulmod(r, b, m);
    b = fo_mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}

/* int_utils.hpp:33-41 */
static u128 pow_saturating(u128 a, int e, u128 cap) {
  u128 r = 1;
  for (int i = 0; i < e; ++i) {
    if (a != 0 && r > cap / a) return cap;
    r *= a;
    if (r > cap) return cap;
  }
  return r;
}

/* primality.cpp:11-19 */
static int mr_composite(uint64_t n, uint64_t a, uint64_t d, int r) {
  uint64_t x = fo_powmod(a, d, n);
  if (x == 1 || x == n - 1) return 0;
  for (int i = 1; i < r; ++i) {
    x = fo_mulmod(x, x, n);
    if (x == n - 1) return 0;
  }
  return 1;
}

/* primality.cpp:21-38: deterministic Miller-Rabin with the first 12 primes */
int fo_is_prime(uint64_t n) {
  static const uint64_t w[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) {
    if (n == w[i]) return 1;
    if (n % w[i] == 0) return 0;
  }
  int r = 0;
  uint64_t d = n - 1;
  while ((d & 1) == 0) d >>= 1, ++r;
  for (int i = 0; i < 12; ++i)
    if (mr_composite(n, w[i], d, r)) return 0;
  return 1;
}

/* primality.cpp:40-49: largest prime strictly below limit, 0 if none */
uint64_t fo_prev_prime(uint64_t limit) {
  if (limit <= 2) return 0;
  uint64_t n = limit - 1;
  if (n == 2) return 2;
  if ((n & 1) == 0) --n;
  for (; n >= 3; n -= 2)
    if (fo_is_prime(n)) return n;
  return 2;
}

/* ------------------------------------------------------------ seeded inputs */

/* std::mt19937_64 (the engine random_mat uses, mat.hpp:112-114) */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (s->idx >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    for (; i < 311; ++i) {
      uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    }
    uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1) ? A : 0);
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* mat.hpp:94-102 bounded_u64: rejection above the largest multiple of bound */
static uint64_t bounded_u64(mt64* s, uint64_t bound) {
  const uint64_t reject_above = UINT64_MAX - UINT64_MAX % bound;
  uint64_t r;
  do r = mt64_next(s);
  while (r >= reject_above);
  return r % bound;
}

/* mat.hpp:104-110 mix_seed (splitmix64 step) */
uint64_t fo_mix_seed(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* driver.cpp:14-20 matrix_seed */
uint64_t fo_matrix_seed(uint64_t seed, int bits, int64_t m, int64_t k, int64_t n, uint64_t which) {
  uint64_t h = fo_mix_seed(seed, (uint64_t)bits);
  h = fo_mix_seed(h, (uint64_t)m);
  h = fo_mix_seed(h, (uint64_t)k);
  h = fo_mix_seed(h, (uint64_t)n);
  return fo_mix_seed(h, which);
}

/* mat.hpp:112-120 random_mat: row-major uniform residues in [0, p) */
void fo_random_mat(int64_t rows, int64_t cols, uint64_t p, uint64_t seed, double* out) {
  mt64 s;
  mt64_seed(&s, seed);
  for (int64_t e = 0; e < rows * cols; ++e) out[e] = (double)bounded_u64(&s, p);
}

uint64_t fo_fnv1a64_f64(const double* x, int64_t count) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < count; ++i) {
    uint64_t v = (uint64_t)x[i];
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xff;
      h *= 0x100000001b3ULL;
    }
  }
  return h;
}

/* ------------------------------------------------------- scalar algorithms */

/* scalar_ops.hpp:19-30, Alg 2.1 */
double fo_fp_reduce(double x, double p, double q) {
  double b = x * q;
  double c = floor(b);
  double d = fma(-c, p, x);
  if (d >= p) d -= p;
  if (d < 0.0) d += p;
  return d;
}

/* scalar_ops.hpp:36-51, Alg 2.2 */
double fo_fp_mul_reduce(double x, double y, double p, double q) {
  double h = x * y;
  double l = fma(x, y, -h);
  double b = h * q;
  double c = floor(b);
  double d = fma(-c, p, h);
  double e = d + l;
  if (e >= p) e -= p;
  if (e < 0.0) e += p;
  return e;
}

/* fp_context.hpp:56-69 residue_fp_safe = 3(p-1)^2 <= 2^(t-1) p */
static int residue_fp_safe(uint64_t p) {
  return (u128)3 * (p - 1) * (p - 1) <= ((u128)1 << (T53 - 1)) * p;
}

/* scalar_ops.hpp:56-60 */
double fo_residue_mul_mod(double x, double y, uint64_t p) {
  if (residue_fp_safe(p)) return fo_fp_mul_reduce(x, y, (double)p, 1.0 / (double)p);
  return (double)fo_mulmod((uint64_t)x, (uint64_t)y, p);
}

/* scalar_ops.hpp:64-76 */
double fo_mod_pow(double base, uint64_t e, uint64_t p) {
  double r = 1.0, b = base;
  while (e) {
    if (e & 1) r = fo_residue_mul_mod(r, b, p);
    b = fo_residue_mul_mod(b, b, p);
    e >>= 1;
  }
  return r;
}

/* scalar_ops.hpp:80-104 extended Euclid */
int fo_mod_inv(uint64_t a, uint64_t p, uint64_t* out) {
  if (a % p == 0) return FO_ENOINVERSE;
  int64_t t0 = 0, t1 = 1, r0 = (int64_t)p, r1 = (int64_t)(a % p);
  while (r1 != 0) {
    int64_t q = r0 / r1, tmp = t0 - q * t1;
    t0 = t1;
    t1 = tmp;
    tmp = r0 - q * r1;
    r0 = r1;
    r1 = tmp;
  }
  if (r0 != 1) return FO_ENOINVERSE;
  *out = (uint64_t)(t0 < 0 ? t0 + (int64_t)p : t0);
  return FO_OK;
}

/* --------------------------------------------------------------------- rule */

/* multiword.cpp:7-19 word_base: smallest a with a^u >= p */
int fo_word_base(uint64_t p, int u, uint64_t* out) {
  if (p < 2 || u < 1) return FO_EERROR;
  if (u == 1) {
    *out = p;
    return FO_OK;
  }
  const u128 cap = (u128)1 << 100;
  uint64_t c = (uint64_t)llround(pow((double)p, 1.0 / u));
  if (c < 1) c = 1;
  while (pow_saturating(c, u, cap) < p) ++c;
  while (c > 1 && pow_saturating(c - 1, u, cap) >= p) --c;
  *out = c;
  return FO_OK;
}

/* multiword.hpp:16 */
uint64_t fo_word_bound(uint64_t p, int u) {
  uint64_t b = 0;
  if (u == 1) return p - 1;
  fo_word_base(p, u, &b);
  return b;
}

/* block_product.hpp:13-22 (returns 0 for nullopt; UINT64_MAX for unbounded) */
uint64_t fo_max_block_size(uint64_t max_a, uint64_t max_b, uint64_t p, int t) {
  const u128 budget = ((u128)1 << t) - (p - 1);
  const u128 ab = (u128)max_a * max_b;
  if (ab == 0) return UINT64_MAX;
  if (ab > budget) return 0;
  const u128 l = budget / ab;
  return l > UINT64_MAX ? UINT64_MAX : (uint64_t)l;
}

/* planner.hpp:29-31 */
uint64_t fo_mw_block_size(int u, int v, uint64_t p, int t) {
  if (p < 2) return 0; /* word_base throws for p < 2 (multiword.cpp:8) */
  return fo_max_block_size(fo_word_bound(p, u), fo_word_bound(p, v), p, t);
}

/* planner.cpp:11-14 */
static int feasible_at(int u, int v, uint64_t p, int t, uint64_t min_lambda) {
  uint64_t l = fo_mw_block_size(u, v, p, t);
  return l != 0 && l >= min_lambda;
}

/* planner.cpp:20-28 with the scan starting at b=2 (the shipped
 * scan starts at b=1 whose surrogate modulus 2^1-1 = 1 makes word_base throw) */
int fo_variant_bit_limit(int u, int v, int t) {
  if (u < 1 || v < 1 || t < 3 || t > 62) return -1;
  int best = 0;
  for (int b = 2; b <= t - 1; ++b)
    if (feasible_at(u, v, (1ULL << b) - 1, t, 1)) best = b;
  return best;
}

static const int kVariants[6][2] = {{1, 1}, {1, 2}, {1, 3}, {1, 4}, {2, 2}, {2, 3}};

/* planner.cpp:30-42 */
static void finish_plan(fo_plan* pl, int64_t m, int64_t k, int64_t n) {
  const uint64_t um = (uint64_t)m, uk = (uint64_t)k, un = (uint64_t)n;
  const uint64_t uv = (uint64_t)pl->u * pl->v;
  pl->products = uv;
  const uint64_t panels = pl->lambda == 0 ? 0 : (uk + pl->lambda - 1) / pl->lambda;
  pl->reductions = uv * um * un * (panels + 2);
  pl->storage = uk * ((uint64_t)pl->u * um + (uint64_t)pl->v * un) + um * un;
  if (pl->concat != 0)
    pl->storage += (pl->concat == 2 ? (uint64_t)pl->v : (uint64_t)pl->u) * um * un;
}

/* planner.cpp:46-89 plan_common */
static int plan_common(int bits, uint64_t p_for_lambda, int64_t m, int64_t k, int64_t n, int t,
                       uint64_t min_lambda, int64_t concat_threshold, fo_plan* out) {
  if (bits < 1) return FO_EERROR;
  if (bits > t - 1) return FO_EINFEASIBLE;
  int concat = 0;
  if ((m < n ? m : n) < concat_threshold && m != n) concat = (n < m) ? 2 : 1;
  int best = -1;
  for (int i = 0; i < 6; ++i) {
    const int u = kVariants[i][0], v = kVariants[i][1];
    if (bits > fo_variant_bit_limit(u, v, t)) continue;
    if (!feasible_at(u, v, p_for_lambda, t, min_lambda)) continue;
    if (best < 0) {
      best = i;
      continue;
    }
    const int bu = kVariants[best][0], bv = kVariants[best][1];
    if (u * v < bu * bv) {
      best = i;
    } else if (u * v == bu * bv) {
      const int wide = concat != 0, su = u + v, sb = bu + bv;
      if ((wide && su > sb) || (!wide && su < sb) || (su == sb && u < bu)) best = i;
    }
  }
  if (best < 0) return FO_EINFEASIBLE;
  out->u = kVariants[best][0];
  out->v = kVariants[best][1];
  uint64_t lam = fo_mw_block_size(out->u, out->v, p_for_lambda, t);
  uint64_t kk = (uint64_t)(k > 1 ? k : 1);
  out->lambda = lam < kk ? lam : kk;
  out->concat = concat;
  finish_plan(out, m, k, n);
  return FO_OK;
}

/* planner.cpp:93-96 */
int fo_select_variant(int bits, int64_t m, int64_t k, int64_t n, int t, uint64_t min_lambda,
                      int64_t concat_threshold, fo_plan* out) {
  if (bits < 1 || bits > 62) return bits < 1 ? FO_EERROR : FO_EINFEASIBLE;
  return plan_common(bits, (1ULL << bits) - 1, m, k, n, t, min_lambda, concat_threshold, out);
}

/* planner.cpp:98-101 */
int fo_plan_for_modulus(uint64_t p, int64_t m, int64_t k, int64_t n, int t, uint64_t min_lambda,
                        int64_t concat_threshold, fo_plan* out) {
  return plan_common(fo_bitsize(p), p, m, k, n, t, min_lambda, concat_threshold, out);
}

/* ------------------------------------------------- matrix algorithms (fp64) */

/* multiword.hpp:29-54 decompose: r = floor(T * fl(1/alpha)); w = fma(-alpha, r, T) */
int fo_decompose(const double* M, int64_t rows, int64_t cols, uint64_t p, int u, double* words,
                 uint64_t* base) {
  if (u < 1) return FO_EERROR;
  uint64_t b;
  if (fo_word_base(p, u, &b)) return FO_EERROR;
  *base = b;
  const int64_t sz = rows * cols;
  const double alpha = (double)b, inv = 1.0 / alpha;
  double* t = words + (int64_t)(u - 1) * sz; /* last word holds T */
  memcpy(t, M, sizeof(double) * (size_t)sz);
  for (int i = 0; i + 1 < u; ++i) {
    double* w = words + (int64_t)i * sz;
    for (int64_t e = 0; e < sz; ++e) {
      double r = floor(t[e] * inv);
      w[e] = fma(-alpha, r, t[e]);
      t[e] = r;
    }
  }
  return FO_OK;
}

/* gemm_kernel.hpp:24-34 NaiveKernel::accumulate on strided panels */
static void naive_accumulate(double* C, int64_t ldc, const double* A, int64_t lda, const double* B,
                             int64_t ldb, int64_t m, int64_t w, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    double* crow = C + i * ldc;
    for (int64_t l = 0; l < w; ++l) {
      const double a = A[i * lda + l];
      if (a == 0.0) continue;
      const double* brow = B + l * ldb;
      for (int64_t j = 0; j < n; ++j) crow[j] += a * brow[j];
    }
  }
}

/* block_product.hpp:30-36 */
static void elementwise_reduce(double* C, int64_t count, double p, double q) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e) C[e] = fo_fp_reduce(C[e], p, q);
}

/* block_product.hpp:62-73 Alg 2.3 */
int fo_block_gemm_mod(double* C, const double* A, int64_t lda, const double* B, int64_t ldb,
                      int64_t m, int64_t k, int64_t n, uint64_t lambda, uint64_t p) {
  if (lambda < 1) return FO_EINFEASIBLE;
  const int64_t lam = (int64_t)(lambda < (uint64_t)k ? lambda : (uint64_t)k);
  const double pf = (double)p, q = 1.0 / pf;
  for (int64_t j0 = 0; j0 < k; j0 += lam) {
    const int64_t w = lam < k - j0 ? lam : k - j0;
    naive_accumulate(C, n, A + j0, lda, B + j0 * ldb, ldb, m, w, n);
    elementwise_reduce(C, m * n, pf, q);
  }
  return FO_OK;
}

/* multiword.hpp:58-70 check_mw_inputs */
static int check_mw(int u, int v, uint64_t lambda, uint64_t p) {
  if (u < 1 || v < 1) return FO_EERROR;
  if (lambda < 1) return FO_EINFEASIBLE;
  const u128 peak = (u128)lambda * fo_word_bound(p, u) * fo_word_bound(p, v) + (p - 1);
  if (peak > ((u128)1 << T53)) return FO_EINFEASIBLE;
  return FO_OK;
}

/* multiword.hpp:88-92 gamma_factor */
static double gamma_factor(uint64_t alpha, uint64_t beta, int i, int j, uint64_t p) {
  return fo_residue_mul_mod(fo_mod_pow((double)(alpha % p), (uint64_t)i, p),
                            fo_mod_pow((double)(beta % p), (uint64_t)j, p), p);
}

/* multiword.hpp:94-99 scale_mod */
static void scale_mod(double* M, int64_t count, double f, uint64_t p) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e) M[e] = fo_residue_mul_mod(M[e], f, p);
}

int fo_mw_product(const double* A, const double* B, int64_t m, int64_t k, int64_t n, uint64_t p,
                  int u, int v, uint64_t lambda, int variant, double* C) {
  int st = check_mw(u, v, lambda, p);
  if (st) return st;
  const double pf = (double)p, q = 1.0 / pf;
  double* da = (double*)malloc(sizeof(double) * (size_t)(u * m * k + 1));
  double* db = (double*)malloc(sizeof(double) * (size_t)(v * k * n + 1));
  uint64_t alpha = 0, beta = 0;
  fo_decompose(A, m, k, p, u, da, &alpha);
  fo_decompose(B, k, n, p, v, db, &beta);
  memset(C, 0, sizeof(double) * (size_t)(m * n));
  if (variant == 0) {
    /* multiword.hpp:113-131: in-place delta / gamma scaling, needs inverses */
    for (int i = 0; i < u && !st; ++i)
      for (int j = 0; j < v && !st; ++j) {
        const uint64_t a = alpha % p, b = beta % p;
        const double gamma = gamma_factor(alpha, beta, i, j, p);
        double dA = 1.0, dB = 1.0;
        uint64_t inv;
        if (i > 0) {
          if ((st = fo_mod_inv(a, p, &inv))) break;
          dA = fo_mod_pow((double)inv, (uint64_t)i, p);
        }
        if (j > 0) {
          if ((st = fo_mod_inv(b, p, &inv))) break;
          dB = fo_mod_pow((double)inv, (uint64_t)j, p);
        }
        const double delta = fo_residue_mul_mod(dA, dB, p);
        scale_mod(C, m * n, delta, p);
        fo_block_gemm_mod(C, da + i * m * k, k, db + j * k * n, n, m, k, n, lambda, p);
        scale_mod(C, m * n, gamma, p);
      }
  } else if (variant == 1) {
    /* multiword.hpp:222-246 workspace (inverse-free) */
    double* work = (double*)malloc(sizeof(double) * (size_t)(m * n + 1));
    for (int i = 0; i < u; ++i)
      for (int j = 0; j < v; ++j) {
        memset(work, 0, sizeof(double) * (size_t)(m * n));
        fo_block_gemm_mod(work, da + i * m * k, k, db + j * k * n, n, m, k, n, lambda, p);
        scale_mod(work, m * n, gamma_factor(alpha, beta, i, j, p), p);
        for (int64_t e = 0; e < m * n; ++e) C[e] = fo_fp_reduce(C[e] + work[e], pf, q);
      }
    free(work);
  } else {
    /* multiword.hpp:155-209 concatenated: side b stacks B words horizontally,
     * side a stacks A words vertically; auto picks a when n > m */
    int side_a = variant == 3 || (variant == 2 && n > m);
    if (!side_a) {
      double* bcat = (double*)malloc(sizeof(double) * (size_t)(k * n * v + 1));
      double* work = (double*)malloc(sizeof(double) * (size_t)(m * n * v + 1));
      for (int j = 0; j < v; ++j)
        for (int64_t r = 0; r < k; ++r)
          memcpy(bcat + r * n * v + j * n, db + j * k * n + r * n, sizeof(double) * (size_t)n);
      for (int i = 0; i < u; ++i) {
        memset(work, 0, sizeof(double) * (size_t)(m * n * v));
        /* block_gemm_mod over the m x nv workspace */
        const int64_t lam = (int64_t)(lambda < (uint64_t)k ? lambda : (uint64_t)k);
        for (int64_t j0 = 0; j0 < k; j0 += lam) {
          const int64_t w = lam < k - j0 ? lam : k - j0;
          naive_accumulate(work, n * v, da + i * m * k + j0, k, bcat + j0 * n * v, n * v, m, w,
                           n * v);
          elementwise_reduce(work, m * n * v, pf, q);
        }
        for (int j = 0; j < v; ++j) {
          const double g = gamma_factor(alpha, beta, i, j, p);
          for (int64_t r = 0; r < m; ++r)
            for (int64_t c = 0; c < n; ++c) {
              double* t = work + r * n * v + j * n + c;
              *t = fo_residue_mul_mod(*t, g, p);
              C[r * n + c] = fo_fp_reduce(C[r * n + c] + *t, pf, q);
            }
        }
      }
      free(bcat);
      free(work);
    } else {
      /* A words stacked: acat (um x k) */
      double* work = (double*)malloc(sizeof(double) * (size_t)(m * u * n + 1));
      for (int j = 0; j < v; ++j) {
        memset(work, 0, sizeof(double) * (size_t)(m * u * n));
        fo_block_gemm_mod(work, da, k, db + j * k * n, n, m * u, k, n, lambda, p);
        for (int i = 0; i < u; ++i) {
          const double g = gamma_factor(alpha, beta, i, j, p);
          for (int64_t r = 0; r < m; ++r)
            for (int64_t c = 0; c < n; ++c) {
              double* t = work + (i * m + r) * n + c;
              *t = fo_residue_mul_mod(*t, g, p);
              C[r * n + c] = fo_fp_reduce(C[r * n + c] + *t, pf, q);
            }
        }
      }
      free(work);
    }
  }
  free(da);
  free(db);
  return st;
}

/* ---------------------------------------------------- exact ground truth */

#define RED_EVERY (1 << 20) /* 2^20 products < 2^104 each stay below 2^124 */

/* oracle.cpp:5-16 (row order), restated with u128 instead of cpp_int */
void fo_exact_mod_gemm(const double* A, const double* B, int64_t m, int64_t k, int64_t n,
                       uint64_t p, double* C, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel
  {
    u128* acc = (u128*)malloc(sizeof(u128) * (size_t)(n + 1));
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; ++i) {
      memset(acc, 0, sizeof(u128) * (size_t)n);
      for (int64_t l = 0; l < k; ++l) {
        const uint64_t a = (uint64_t)A[i * k + l];
        if (!a) continue;
        const double* brow = B + l * n;
        for (int64_t j = 0; j < n; ++j) acc[j] += (u128)a * (uint64_t)brow[j];
        if ((l + 1) % RED_EVERY == 0)
          for (int64_t j = 0; j < n; ++j) acc[j] %= p;
      }
      for (int64_t j = 0; j < n; ++j) C[i * n + j] = (double)(uint64_t)(acc[j] % p);
    }
    free(acc);
  }
}

/* oracle.cpp:18-30 column order (independent second route) */
void fo_exact_mod_gemm_colmajor(const double* A, const double* B, int64_t m, int64_t k,
                                int64_t n, uint64_t p, double* C) {
  u128* col = (u128*)malloc(sizeof(u128) * (size_t)(m + 1));
  for (int64_t j = 0; j < n; ++j) {
    memset(col, 0, sizeof(u128) * (size_t)m);
    for (int64_t l = 0; l < k; ++l) {
      const uint64_t b = (uint64_t)B[l * n + j];
      if (!b) continue;
      for (int64_t i = 0; i < m; ++i) col[i] += (u128)(uint64_t)A[i * k + l] * b;
      if ((l + 1) % RED_EVERY == 0)
        for (int64_t i = 0; i < m; ++i) col[i] %= p;
    }
    for (int64_t i = 0; i < m; ++i) C[i * n + j] = (double)(uint64_t)(col[i] % p);
  }
  free(col);
}

void fo_exact_mod_entries(const double* A, const double* B, int64_t m, int64_t k, int64_t n,
                          uint64_t p, const int64_t* rows, const int64_t* cols, int64_t count,
                          uint64_t* out, int threads) {
  (void)m;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t e = 0; e < count; ++e) {
    u128 acc = 0;
    const int64_t i = rows[e], j = cols[e];
    for (int64_t l = 0; l < k; ++l) {
      acc += (u128)(uint64_t)A[i * k + l] * (uint64_t)B[l * n + j];
      if ((l + 1) % RED_EVERY == 0) acc %= p;
    }
    out[e] = (uint64_t)(acc % p);
  }
}

/* y[i] = sum_l M[i][l] x[l] mod p */
static void matvec_mod(const double* M, const uint64_t* x, int64_t rows, int64_t cols, uint64_t p,
                       uint64_t* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    u128 acc = 0;
    const double* r = M + i * cols;
    for (int64_t l = 0; l < cols; ++l) {
      acc += (u128)(uint64_t)r[l] * x[l];
      if ((l + 1) % RED_EVERY == 0) acc %= p;
    }
    y[i] = (uint64_t)(acc % p);
  }
}

int fo_freivalds(const double* A, const double* B, const double* C, int64_t m, int64_t k,
                 int64_t n, uint64_t p, uint64_t seed, int trials, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  /* C must hold canonical residues */
  int64_t bad_range = 0;
#pragma omp parallel for reduction(+ : bad_range)
  for (int64_t e = 0; e < m * n; ++e) {
    const double c = C[e];
    if (!(c >= 0.0 && c < (double)p && c == floor(c))) ++bad_range;
  }
  if (bad_range) return trials + 1;
  uint64_t* s = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
  uint64_t* bs = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(k + 1));
  uint64_t* abs_ = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m + 1));
  uint64_t* cs = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m + 1));
  mt64 g;
  mt64_seed(&g, seed);
  int fails = 0;
  for (int t = 0; t < trials; ++t) {
    for (int64_t j = 0; j < n; ++j) s[j] = bounded_u64(&g, p);
    matvec_mod(B, s, k, n, p, bs);
    matvec_mod(A, bs, m, k, p, abs_);
    matvec_mod(C, s, m, n, p, cs);
    for (int64_t i = 0; i < m; ++i)
      if (abs_[i] != cs[i]) {
        ++fails;
        break;
      }
  }
  free(s);
  free(bs);
  free(abs_);
  free(cs);
  return fails;
}
