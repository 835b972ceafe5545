// Host-side probe: how fast can the host cores narrow fp64 residues (< 2^bits)
// to w-byte integers and widen them back, against plain memcpy?  Decides
// whether a compressed PCIe transfer can beat the raw fp64 copy (e2e path).
//   g++ -O3 -mavx2 -mfma -pthread host_pack.cpp -o host_pack && ./host_pack
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static void narrow(const double* x, uint8_t* out, size_t n, int w) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t v = static_cast<uint64_t>(x[i]);
    std::memcpy(out + i * w, &v, 8 > w ? w : 8);
  }
}
static void narrow4(const double* x, uint32_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(x[i]);
}
static void widen(const uint8_t* in, double* y, size_t n, int w) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t v = 0;
    std::memcpy(&v, in + i * w, w);
    y[i] = static_cast<double>(v);
  }
}

template <class F>
static double par(int T, size_t n, F f) {
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) {
    size_t a = n * t / T, b = n * (t + 1) / T;
    th.emplace_back([=] { f(a, b); });
  }
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  const size_t n = size_t(1) << 26;  // 64 M elements = 512 MB of fp64
  std::vector<double> x(n), y(n);
  std::vector<uint8_t> buf(n * 8);
  for (size_t i = 0; i < n; ++i) x[i] = double((i * 2654435761u) & 0xFFFFFFFFFFull);
  unsigned hw = std::thread::hardware_concurrency();
  std::printf("hardware_concurrency %u\n", hw);
  for (int T : {1, 4, 8, 16, 32}) {
    if (T > int(hw)) break;
    for (int rep = 0; rep < 2; ++rep) {
      double tm = par(T, n, [&](size_t a, size_t b) { std::memcpy(y.data() + a, x.data() + a, (b - a) * 8); });
      double t4 = par(T, n, [&](size_t a, size_t b) { narrow4(x.data() + a, (uint32_t*)buf.data() + a, b - a); });
      double t5 = par(T, n, [&](size_t a, size_t b) { narrow(x.data() + a, buf.data() + a * 5, b - a, 5); });
      double w5 = par(T, n, [&](size_t a, size_t b) { widen(buf.data() + a * 5, y.data() + a, b - a, 5); });
      std::printf("T=%2d memcpy %.1f GB/s | narrow fp64->u32 %.1f GB/s in | fp64->5B %.1f GB/s in | 5B->fp64 %.1f GB/s out\n",
                  T, n * 8 / tm / 1e9, n * 8 / t4 / 1e9, n * 8 / t5 / 1e9, n * 8 / w5 / 1e9);
    }
  }
  return 0;
}
