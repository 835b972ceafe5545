// verify.cuh -- on-device exact check of a product C = A B mod p at any size.
//
// The analogue of the reference's oracle-equivalence check (driver.cpp:37-140,
// first_mismatch at oracle.hpp:71-81) for products too large for a CPU
// recomputation (C3: 32768^3 takes hours on the host).  Three independent
// tests, each exact in integer arithmetic:
//   range    every C entry is an integer in [0, p);
//   Freivalds  A (B s) == C s (mod p) for uniform random s in [0, p)^n: a
//            wrong C passes one trial with probability <= 1/p (p > 2^19 in
//            the sweep), trials are independent;
//   samples  C[i][j] == sum_l A[i][l] B[l][j] mod p at random (i, j).
// Every dot product is accumulated exactly as a 128-bit integer (entries
// < 2^53, vector entries < p < 2^52, up to 2^18 terms: < 2^123) and reduced
// mod p once.  This is a checker of outputs, run outside any timed region.
#pragma once

#include <cstdint>

namespace fpmm_b200 {
namespace verify {

using i64 = std::int64_t;
using u64 = std::uint64_t;

__device__ __forceinline__ u64 mix64(u64 z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// (hi 2^64 + lo) mod p for p < 2^52: hi mod p, then eight byte steps (r < p,
// so r 2^8 + byte < 2^60 never overflows)
__device__ __forceinline__ u64 mod128(u64 hi, u64 lo, u64 p) {
  u64 r = hi % p;
#pragma unroll
  for (int b = 7; b >= 0; --b) r = ((r << 8) | ((lo >> (8 * b)) & 0xFFull)) % p;
  return r;
}

// 128-bit accumulate of a * b
__device__ __forceinline__ void mac128(u64 a, u64 b, u64& lo, u64& hi) {
  const u64 pl = a * b, ph = __umul64hi(a, b);
  lo += pl;
  hi += ph + (lo < pl ? 1ull : 0ull);
}

__device__ __forceinline__ void warp_sum128(u64& lo, u64& hi) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const u64 olo = __shfl_down_sync(0xffffffffu, lo, off), ohi = __shfl_down_sync(0xffffffffu, hi, off);
    lo += olo;
    hi += ohi + (lo < olo ? 1ull : 0ull);
  }
}

// x[i] uniform in [0, p): splitmix64 draws with rejection above reject_at
__global__ void rand_vec_kernel(u64* __restrict__ x, i64 n, u64 p, u64 reject_at, u64 seed) {
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    u64 t = 0, r;
    do r = mix64(seed ^ ((static_cast<u64>(i) << 8) + t++));
    while (r >= reject_at);
    x[i] = r % p;
  }
}

// out[r] = (sum_c M[r][c] x[c]) mod p, one warp per row (coalesced row reads)
__global__ void __launch_bounds__(256) matvec_mod_kernel(const double* __restrict__ M, i64 ld, i64 rows, i64 cols,
                                                         const u64* __restrict__ x, u64 p, u64* __restrict__ out) {
  const int lane = threadIdx.x % 32;
  const i64 warps = static_cast<i64>(gridDim.x) * (blockDim.x / 32);
  for (i64 r = static_cast<i64>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
    const double* row = M + r * ld;
    u64 lo = 0, hi = 0;
    for (i64 c = lane; c < cols; c += 32) mac128(static_cast<u64>(row[c]), x[c], lo, hi);
    warp_sum128(lo, hi);
    if (lane == 0) out[r] = mod128(hi, lo, p);
  }
}

// counts[1] += #{r : z[r] != w[r]}
__global__ void compare_kernel(const u64* __restrict__ z, const u64* __restrict__ w, i64 n,
                               unsigned long long* counts) {
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    if (z[i] != w[i]) atomicAdd(&counts[1], 1ull);
}

// counts[0] += #{entries of C that are not integers in [0, p)}
__global__ void range_kernel(const double* __restrict__ Cm, i64 ld, i64 rows, i64 cols, u64 p,
                             unsigned long long* counts) {
  const double pf = static_cast<double>(p);
  for (i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * cols;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double v = Cm[(e / cols) * ld + e % cols];
    const bool bad = !(v >= 0.0 && v < pf && v == floor(v));
    const unsigned mask = __ballot_sync(__activemask(), bad);
    if (bad && (threadIdx.x % 32) == static_cast<unsigned>(__ffs(mask) - 1)) atomicAdd(&counts[0], __popc(mask));
  }
}

// counts[2] += wrong sampled entries; sample s is (i, j) from mix64(seed, s),
// one warp per sample.  The first bad sample's (i, j) goes to first[0..1].
__global__ void __launch_bounds__(256) sample_kernel(const double* __restrict__ A, i64 lda, const double* __restrict__ B,
                                                     i64 ldb, const double* __restrict__ Cm, i64 ldc, i64 m, i64 k,
                                                     i64 n, u64 p, u64 seed, int samples, unsigned long long* counts,
                                                     long long* first) {
  const int lane = threadIdx.x % 32;
  const int warps = gridDim.x * (blockDim.x / 32);
  for (int s = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; s < samples; s += warps) {
    const u64 h = mix64(seed ^ (0x5A5A000000000000ull + static_cast<u64>(s)));
    // the four corners first (ragged tile edges), then uniform positions
    i64 i, j;
    if (s < 4) {
      i = (s & 1) ? m - 1 : 0;
      j = (s & 2) ? n - 1 : 0;
    } else {
      i = static_cast<i64>((h >> 32) % static_cast<u64>(m));
      j = static_cast<i64>((h & 0xFFFFFFFFull) % static_cast<u64>(n));
    }
    u64 lo = 0, hi = 0;
    for (i64 l = lane; l < k; l += 32) mac128(static_cast<u64>(A[i * lda + l]), static_cast<u64>(B[l * ldb + j]), lo, hi);
    warp_sum128(lo, hi);
    if (lane == 0) {
      const u64 want = mod128(hi, lo, p);
      const double got = Cm[i * ldc + j];
      if (!(got >= 0.0 && got == floor(got) && static_cast<u64>(got) == want)) {
        if (atomicAdd(&counts[2], 1ull) == 0ull) first[0] = i, first[1] = j;
      }
    }
  }
}

}  // namespace verify
}  // namespace fpmm_b200
