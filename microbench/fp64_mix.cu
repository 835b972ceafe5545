// DMMA co-issue microbenchmark for sm_100a (B200): how much do integer,
// FP32 and FP64 side instructions slow a DMMA.8x8x4 stream?  Answers whether
// the in-register reduction of the FP64 multiword GEMM can move work off the
// FP64 pipe (reduce_fast: 6 INT/FP32 + 1 DFMA) or whether the side pipes
// contend with DMMA anyway.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo fp64_mix.cu -o fp64_mix
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int CH = 8;  // DMMA chains per thread per iteration

// side work kinds (R independent values per iteration)
enum { kNone = 0, kInt = 1, kF32 = 2, kDfma = 3, kRedClassic = 4, kRedFast = 5, kIntF32 = 6, kRedIntQ = 7 };

template <int KIND, int R>
__device__ __forceinline__ void side(double* x, uint32_t* u, float* f, double p, double q, float qf) {
#pragma unroll
  for (int c = 0; c < R; ++c) {
    if constexpr (KIND == kInt) {
      u[c] = u[c] * 8u + 0x40000000u;           // IMAD / LEA
    } else if constexpr (KIND == kF32) {
      f[c] = __fmaf_rn(f[c], 0.999f, 1.0f);      // FFMA
    } else if constexpr (KIND == kIntF32) {
      u[c] = u[c] * 8u + 0x40000000u;
      f[c] = __fmaf_rn(f[c], 0.999f, 1.0f);
    } else if constexpr (KIND == kDfma) {
      x[c] = __fma_rn(x[c], 0.999999, 1.0);
    } else if constexpr (KIND == kRedClassic) {
      const double M = 6755399441055744.0;
      const double cq = __fma_rn(x[c], q, M) - M;
      x[c] = __fma_rn(-cq, p, x[c]) + 4.0 * p;  // keeps x large; the DADD is extra
    } else if constexpr (KIND == kRedIntQ) {
      // quotient from x's high word with integer ops only (IMAD-class), then
      // c = (1.5*2^52 + q) - 1.5*2^52 (one DADD) and r = fma(-c, p, x): 2 FP64 ops
      const uint32_t hi = static_cast<uint32_t>(__double2hiint(x[c]));
      const uint32_t mant = (hi & 0xFFFFFu) | 0x100000u;          // 21-bit significand
      const int e = static_cast<int>((hi >> 20) & 0x7FFu) - 1023;  // x in [2^e, 2^(e+1))
      const uint32_t qq = __umulhi(mant << 11, static_cast<uint32_t>(qf * 4294967296.0f));  // ~ mant * 2^31 / p'
      const int sh = 31 - e;  // placeholder scaling: the cost, not the value, is what is measured
      const uint32_t q = sh > 0 && sh < 32 ? (qq >> sh) : qq;
      const long long qs = (hi >> 31) ? -static_cast<long long>(q) : static_cast<long long>(q);
      const double cd = __longlong_as_double(0x4338000000000000ll + qs) - 6755399441055744.0;
      x[c] = __fma_rn(-cd, p, x[c]) + 4.0 * p;
    } else if constexpr (KIND == kRedFast) {
      const uint32_t hi = static_cast<uint32_t>(__double2hiint(x[c]));
      const float fx = __uint_as_float(hi * 8u + 0x40000000u);
      const float M = 12582912.0f;
      const float cf = __fadd_rn(__fmaf_rn(fx, qf, M), -M);
      const uint32_t cb = __float_as_uint(cf);
      uint32_t sb;
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(sb) : "r"(hi), "n"(0x80000000u), "r"(0x38000000u));
      const double cd = __hiloint2double(static_cast<int>((cb >> 3) + sb), static_cast<int>(cb << 29));
      x[c] = __fma_rn(-cd, p, x[c]) + 4.0 * p;
    }
  }
}

template <int KIND, int R>
__global__ void k_mix(int iters, double* out, double p, double q, float qf) {
  double d[CH][2];
  double x[R > 0 ? R : 1];
  uint32_t u[R > 0 ? R : 1];
  float f[R > 0 ? R : 1];
  const double a = 3.0 + threadIdx.x, b = 5.0;
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = c, d[c][1] = -c;
#pragma unroll
  for (int c = 0; c < (R > 0 ? R : 1); ++c) x[c] = 4.0 * p + c + threadIdx.x, u[c] = c + threadIdx.x, f[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma884(d[c][0], d[c][1], a, b);
    side<KIND, R>(x, u, f, p, q, qf);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
#pragma unroll
  for (int c = 0; c < (R > 0 ? R : 1); ++c) s += x[c] + u[c] + f[c];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <typename K>
float timeit(K kern, int blocks, int threads, int iters, double* out, double p, double q, float qf) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  kern<<<blocks, threads>>>(iters, out, p, q, qf);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<blocks, threads>>>(iters, out, p, q, qf);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 1 << 20));
  const int iters = argc > 1 ? atoi(argv[1]) : 8192;
  const double p = 4503599627370449.0;  // 2^52 - 47
  const double q = 1.0 / p;
  const float qf = 1.0f / static_cast<float>(p);
  const int threads = 256, blocks = sms;  // the GEMM's shape: 8 warps, 1 CTA per SM
  const double dmma_flops = double(blocks) * (threads / 32) * iters * CH * 512.0;
  const float base = timeit(k_mix<kNone, 0>, blocks, threads, iters, out, p, q, qf);
  printf("device %s sms=%d; 8 warps/SM, per iteration %d DMMA.8x8x4 per warp + R side ops per thread\n",
         prop.name, sms, CH);
  printf("dmma only                 : %.3f ms  %.2f TFLOP/s\n", base, dmma_flops / base / 1e9);
#define ROW(KIND, R, NAME)                                                                        \
  {                                                                                               \
    const float ms = timeit(k_mix<KIND, R>, blocks, threads, iters, out, p, q, qf);              \
    printf("%-26s: %.3f ms  x%.3f  DMMA %.2f TFLOP/s\n", NAME, ms, ms / base, dmma_flops / ms / 1e9); \
  }
  ROW(kInt, 8, "+8 IMAD")
  ROW(kInt, 16, "+16 IMAD")
  ROW(kInt, 32, "+32 IMAD")
  ROW(kF32, 8, "+8 FFMA")
  ROW(kF32, 16, "+16 FFMA")
  ROW(kF32, 32, "+32 FFMA")
  ROW(kIntF32, 16, "+16 IMAD +16 FFMA")
  ROW(kDfma, 4, "+4 DFMA")
  ROW(kDfma, 8, "+8 DFMA")
  ROW(kDfma, 16, "+16 DFMA")
  ROW(kRedClassic, 4, "+4 classic red (+DADD)")
  ROW(kRedClassic, 8, "+8 classic red (+DADD)")
  ROW(kRedClassic, 16, "+16 classic red (+DADD)")
  ROW(kRedFast, 4, "+4 fast red (+DADD)")
  ROW(kRedFast, 8, "+8 fast red (+DADD)")
  ROW(kRedFast, 16, "+16 fast red (+DADD)")
  ROW(kRedIntQ, 4, "+4 int-quotient red (+DADD)")
  ROW(kRedIntQ, 8, "+8 int-quotient red (+DADD)")
  ROW(kRedIntQ, 16, "+16 int-quotient red (+DADD)")
  return 0;
}
