// FP64 pipe microbenchmarks for sm_100a (B200).
//
// Questions this answers before the fused multiword kernel is designed:
//   1. DMMA (mma.sync .f64) throughput for m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16.
//   2. DFMA, DMUL, DADD, FRND (rint / floor) throughput.
//   3. Whether DMMA and the DFMA-class ops share one pipe (mixed kernels).
//   4. Throughput of the two candidate in-register reductions:
//        rint form : c = rint(x*q); r = fma(-c, p, x)
//        magic form: t = fma(x, q, M); c = t - M; r = fma(-c, p, x)
//   5. DMMA exactness at the 2^53 edge with integer operands.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo fp64_pipes.cu -o fp64_pipes
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1684(double* d, double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void dmma1688(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void dmma16816(double* d, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

constexpr int CH = 8;  // independent chains per thread

__global__ void k_dmma884(int iters, double* out, double seed) {
  double d[CH][2];
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma884(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_dmma1684(int iters, double* out, double seed) {
  double d[CH][4];
  double a0 = seed + threadIdx.x * 1e-3, a1 = seed * 0.5, b = seed - threadIdx.x * 1e-3;
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; d[c][2] = 0; d[c][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma1684(d[c], a0, a1, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_dmma1688(int iters, double* out, double seed) {
  double d[CH][4];
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed + i + threadIdx.x * 1e-3;
  b[0] = seed; b[1] = seed * 0.25;
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; d[c][2] = 0; d[c][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma1688(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_dmma16816(int iters, double* out, double seed) {
  double d[CH / 2][4];
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i + threadIdx.x * 1e-3;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed * (i + 1);
#pragma unroll
  for (int c = 0; c < CH / 2; ++c) { d[c][0] = c; d[c][1] = -c; d[c][2] = 0; d[c][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH / 2; ++c) dmma16816(d[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH / 2; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_dfma(int iters, double* out, double seed) {
  double x[CH];
  double a = seed + threadIdx.x * 1e-9, b = 0.999999;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], b, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_dmul(int iters, double* out, double seed) {
  double x[CH];
  double b = 0.9999999 + threadIdx.x * 1e-12;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = seed + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * b;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// FRND: x = rint(x) + h keeps a dependency through FRND and one DADD
__global__ void k_frnd(int iters, double* out, double seed) {
  double x[CH];
  double h = 0.75 + threadIdx.x * 1e-12;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = seed + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = rint(x[c]) - h;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_dadd(int iters, double* out, double seed) {
  double x[CH];
  double h = 0.75 + threadIdx.x * 1e-12;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = seed + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] - h;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// reduction: r = x - rint(x q) p ; then x = r + big (keeps values integer, large)
__global__ void k_red_rint(int iters, double* out, double p, double q, double big) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = big + c + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double cq = rint(x[c] * q);
      x[c] = fma(-cq, p, x[c]) + big;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

__global__ void k_red_magic(int iters, double* out, double p, double q, double big) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = big + c + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      double t = fma(x[c], q, M);
      double cq = t - M;
      x[c] = fma(-cq, p, x[c]) + big;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// mixed: per iteration, CH DMMA884 + R DFMA (independent chains)
template <int R>
__global__ void k_mix_dmma_dfma(int iters, double* out, double seed) {
  double d[CH][2];
  double x[R];
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
#pragma unroll
  for (int c = 0; c < R; ++c) x[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma884(d[c][0], d[c][1], a, b);
#pragma unroll
    for (int c = 0; c < R; ++c) x[c] = fma(x[c], 0.999999, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
#pragma unroll
  for (int c = 0; c < R; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// mixed: CH DMMA884 + reductions (rint form) on R independent values
template <int R>
__global__ void k_mix_dmma_red(int iters, double* out, double p, double q, double big) {
  double d[CH][2];
  double x[R];
  double a = 3.0 + threadIdx.x, b = 5.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) { d[c][0] = c; d[c][1] = -c; }
#pragma unroll
  for (int c = 0; c < R; ++c) x[c] = big + c + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma884(d[c][0], d[c][1], a, b);
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double cq = rint(x[c] * q);
      x[c] = fma(-cq, p, x[c]) + big;
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
#pragma unroll
  for (int c = 0; c < R; ++c) s += x[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

// exactness of DMMA on integers: A (8x4 row), B (4x8 col), C (8x8) integer
// valued with every partial sum <= 2^53; compare with u128 host result.
__global__ void k_dmma_exact(const double* A, const double* B, const double* C, double* D) {
  int t = threadIdx.x;
  double a = A[(t / 4) * 4 + (t % 4)];
  double b = B[(t % 4) * 8 + (t / 4)];  // B[k][n]
  double d0 = C[(t / 4) * 8 + 2 * (t % 4)], d1 = C[(t / 4) * 8 + 2 * (t % 4) + 1];
  dmma884(d0, d1, a, b);
  D[(t / 4) * 8 + 2 * (t % 4)] = d0;
  D[(t / 4) * 8 + 2 * (t % 4) + 1] = d1;
}

template <typename K, typename... Args>
float timeit(K kern, int blocks, int threads, Args... args) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  kern<<<blocks, threads>>>(args...);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(args...);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  printf("device %s sms=%d\n", prop.name, sms);
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int iters = argc > 1 ? atoi(argv[1]) : 4096;
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb;
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      double warps = double(blocks) * wpb;
      float ms;
      ms = timeit(k_dmma884, blocks, threads, iters, out, 1.0);
      double fl884 = warps * iters * CH * 256.0 * 2;
      printf("wpb=%2d bps=%d dmma m8n8k4   : %8.2f TFLOP/s (%.3f ms)\n", wpb, bps, fl884 / ms / 1e9, ms);
      ms = timeit(k_dmma1684, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d dmma m16n8k4  : %8.2f TFLOP/s\n", wpb, bps, warps * iters * CH * 512.0 * 2 / ms / 1e9);
      ms = timeit(k_dmma1688, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d dmma m16n8k8  : %8.2f TFLOP/s\n", wpb, bps, warps * iters * CH * 1024.0 * 2 / ms / 1e9);
      ms = timeit(k_dmma16816, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d dmma m16n8k16 : %8.2f TFLOP/s\n", wpb, bps, warps * iters * (CH / 2) * 2048.0 * 2 / ms / 1e9);
      double thr = double(blocks) * threads;
      ms = timeit(k_dfma, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d dfma          : %8.2f TFLOP/s  (%.1f Gop/s)\n", wpb, bps, thr * iters * CH * 2 / ms / 1e9,
             thr * iters * CH / ms / 1e6);
      ms = timeit(k_dmul, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d dmul          : %8.1f Gop/s\n", wpb, bps, thr * iters * CH / ms / 1e6);
      ms = timeit(k_dadd, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d dadd          : %8.1f Gop/s\n", wpb, bps, thr * iters * CH / ms / 1e6);
      ms = timeit(k_frnd, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d frnd+dadd     : %8.1f Gpair/s\n", wpb, bps, thr * iters * CH / ms / 1e6);
      const double p = 4503599627370449.0;  // 2^52 - 47
      const double q = 1.0 / p;
      ms = timeit(k_red_rint, blocks, threads, iters, out, p, q, 4.0 * p);
      printf("wpb=%2d bps=%d red rint(+add): %8.1f Gred/s\n", wpb, bps, thr * iters * CH / ms / 1e6);
      ms = timeit(k_red_magic, blocks, threads, iters, out, p, q, 4.0 * p);
      printf("wpb=%2d bps=%d red magic(+add):%8.1f Gred/s\n", wpb, bps, thr * iters * CH / ms / 1e6);
      ms = timeit(k_mix_dmma_dfma<4>, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d mix 8dmma+4dfma : %8.3f ms (dmma-only %.3f)\n", wpb, bps, ms,
             timeit(k_dmma884, blocks, threads, iters, out, 1.0));
      ms = timeit(k_mix_dmma_dfma<16>, blocks, threads, iters, out, 1.0);
      printf("wpb=%2d bps=%d mix 8dmma+16dfma: %8.3f ms (dfma-only x16 est %.3f)\n", wpb, bps, ms,
             2 * timeit(k_dfma, blocks, threads, iters, out, 1.0));
      ms = timeit(k_mix_dmma_red<4>, blocks, threads, iters, out, p, q, 4.0 * p);
      printf("wpb=%2d bps=%d mix 8dmma+4red  : %8.3f ms\n", wpb, bps, ms);
      ms = timeit(k_mix_dmma_red<8>, blocks, threads, iters, out, p, q, 4.0 * p);
      printf("wpb=%2d bps=%d mix 8dmma+8red  : %8.3f ms\n", wpb, bps, ms);
    }
  }
  // exactness
  {
    double hA[32], hB[32], hC[64], hD[64];
    double *dA, *dB, *dC, *dD;
    CK(cudaMalloc(&dA, 256));
    CK(cudaMalloc(&dB, 256));
    CK(cudaMalloc(&dC, 512));
    CK(cudaMalloc(&dD, 512));
    int bad = 0, cases = 0;
    uint64_t s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; };
    for (int trial = 0; trial < 20000; ++trial) {
      // products up to 2^50 (signed), C up to 2^51, total <= 2^53
      for (int i = 0; i < 32; ++i) hA[i] = double((int64_t)(rnd() % (1ull << 26)) - (1ll << 25));
      for (int i = 0; i < 32; ++i) hB[i] = double((int64_t)(rnd() % (1ull << 26)) - (1ll << 25));
      if (trial % 3 == 0) {  // extreme: all max magnitude
        for (int i = 0; i < 32; ++i) hA[i] = (1ll << 25), hB[i] = (i & 1) ? (1ll << 25) : (1ll << 25);
      }
      for (int i = 0; i < 64; ++i) hC[i] = double((int64_t)(rnd() % (1ull << 52)) - (1ll << 51));
      if (trial % 3 == 0) for (int i = 0; i < 64; ++i) hC[i] = double((1ll << 51) - 1 - (rnd() & 1023));
      CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dC, hC, 512, cudaMemcpyHostToDevice));
      k_dmma_exact<<<1, 32>>>(dA, dB, dC, dD);
      CK(cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost));
      for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) {
          __int128 acc = (__int128)(int64_t)hC[r * 8 + c];
          for (int k = 0; k < 4; ++k) acc += (__int128)(int64_t)hA[r * 4 + k] * (int64_t)hB[k * 8 + c];
          ++cases;
          if ((double)(int64_t)acc != hD[r * 8 + c] || (int64_t)hD[r * 8 + c] != (int64_t)acc) ++bad;
        }
    }
    printf("dmma exactness: %d bad of %d\n", bad, cases);
  }
  return 0;
}
