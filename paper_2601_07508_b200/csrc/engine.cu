// engine.cu -- device orchestration: workspaces, streams, kernel dispatch over
// (u,v), host<->device staging, and the NCCL row partitioner.
#include "engine.hpp"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "nccl_loader.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "i8engine.cuh"
#include "kernels.cuh"
#include "rnsengine.cuh"
#include "rnstile.cuh"
#include "verify.cuh"

namespace fpmm_b200 {

#define CUDA_OK(x)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw Failure(FPMM_B200_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)
#define NCCL_OK(x)                                                                              \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess)                                                                      \
      throw Failure(FPMM_B200_ENCCL, std::string(#x) + ": " + nccl().GetErrorString(r_));          \
  } while (0)

namespace {

// Locking.  The context table has its own mutex, held only to look up or
// create a device's context.  Every call that uses a device holds that
// device's (recursive) mutex for its duration: host threads driving different
// GPUs run concurrently, calls on one device serialise (they share its
// workspaces and events).  Multi-device calls take the device locks in
// increasing device order; the partitioner's communicator (g_dist_mu) and the
// in-process communicators (g_all_mu) are locked before any device.
std::mutex g_ctx_mu;
std::recursive_mutex g_dist_mu, g_all_mu;

// grow-only device buffer.  A grow is a cudaFree + cudaMalloc that
// serialises the device (hundreds of ms for GB-sized workspaces), so it
// over-allocates by 25%: a bitsize sweep, whose RNS moduli count rises one at
// a time, then regrows once or twice instead of at every new count.  The
// exact size is the fallback when the padded one does not fit.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need > bytes) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      bytes = 0;
      need = std::max<size_t>(need, 256);
      constexpr size_t kRound = size_t{2} << 20;
      const size_t padded = (need + need / 4 + kRound - 1) / kRound * kRound;
      if (cudaMalloc(&ptr, padded) == cudaSuccess) {
        bytes = padded;
      } else {
        cudaGetLastError();
        if (cudaMalloc(&ptr, need) != cudaSuccess) {
          cudaGetLastError();
          ptr = nullptr;
          throw Failure(FPMM_B200_ENOMEM, "device allocation of " + std::to_string(need) + " bytes failed");
        }
        bytes = need;
      }
    }
    return ptr;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
};

// Device workspaces of one product in flight: packed words, the RNS residue
// blocks and the split-K partials.  Products issued on different streams get
// different sets, so independent products overlap on the device (the packs
// and reconstruction of one run beside the tensor-core kernel of another).
struct Workspace {
  DevBuf apack, bpack, scratch, splitws, rawb;  // rawb: the partitioner's broadcast copy of raw B
  DevBuf pace;                                  // RNS pacing: k-blocks issued per CTA pair
  void release() {
    apack.release(), bpack.release(), scratch.release(), splitws.release(), rawb.release(), pace.release();
  }
};

struct DeviceCtx {
  std::recursive_mutex mu;  // held by every call using this device
  static constexpr int kChunks = 16;  // host-path pipeline depth (exposed head/tail ~1/16 of a product)
  static constexpr int kStreamSets = 8;
  int dev = -1;
  cudaStream_t stream = nullptr, s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev[8] = {}, ev_in[kChunks] = {}, ev_out[kChunks] = {};
  DevBuf a, b, c, tmp, err, ver, agree;
  Workspace ws0;  // the library's own stream and the legacy default stream
  std::vector<std::pair<cudaStream_t, std::unique_ptr<Workspace>>> ws_streams;
  Workspace& ws_for(cudaStream_t s) {
    if (s == nullptr || s == stream) return ws0;
    for (auto& e : ws_streams)
      if (e.first == s) return *e.second;
    if (static_cast<int>(ws_streams.size()) >= kStreamSets) {
      // a stream handle may be gone: only reuse a set once nothing is in flight
      CUDA_OK(cudaDeviceSynchronize());
      ws_streams.front().first = s;
      std::rotate(ws_streams.begin(), ws_streams.begin() + 1, ws_streams.end());
      return *ws_streams.back().second;
    }
    ws_streams.emplace_back(s, std::make_unique<Workspace>());
    return *ws_streams.back().second;
  }
  void init(int d) {
    dev = d;
    CUDA_OK(cudaSetDevice(d));
    CUDA_OK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    for (auto& e : ev) CUDA_OK(cudaEventCreate(&e));
    for (auto& e : ev_in) CUDA_OK(cudaEventCreate(&e));
    for (auto& e : ev_out) CUDA_OK(cudaEventCreate(&e));
  }
  void release() {
    if (dev < 0) return;
    cudaSetDevice(dev);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e), e = nullptr;
    for (auto& e : ev_in)
      if (e) cudaEventDestroy(e), e = nullptr;
    for (auto& e : ev_out)
      if (e) cudaEventDestroy(e), e = nullptr;
    if (s_in) cudaStreamDestroy(s_in), s_in = nullptr;
    if (s_out) cudaStreamDestroy(s_out), s_out = nullptr;
    if (stream) cudaStreamDestroy(stream), stream = nullptr;
    a.release(), b.release(), c.release(), tmp.release(), err.release(), ver.release(), agree.release();
    ws0.release();
    for (auto& e : ws_streams) e.second->release();
    ws_streams.clear();
    dev = -1;
  }
};

std::vector<std::unique_ptr<DeviceCtx>> g_ctx;

DeviceCtx& ctx(int dev) {
  int count = 0;
  CUDA_OK(cudaGetDeviceCount(&count));
  if (dev < 0 || dev >= count)
    throw Failure(FPMM_B200_EERROR, "device " + std::to_string(dev) + " out of range (" +
                                        std::to_string(count) + " visible)");
  DeviceCtx* c = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (g_ctx.size() < static_cast<size_t>(count)) g_ctx.resize(count);
    if (!g_ctx[dev]) {
      auto fresh = std::make_unique<DeviceCtx>();
      fresh->init(dev);
      g_ctx[dev] = std::move(fresh);
    }
    c = g_ctx[dev].get();
  }
  CUDA_OK(cudaSetDevice(dev));
  return *c;
}

// the calling thread holds device `dev` for the scope (and its context exists)
struct DevLock {
  std::unique_lock<std::recursive_mutex> lk;
  explicit DevLock(int dev) : lk(ctx(dev).mu) { CUDA_OK(cudaSetDevice(dev)); }
};

// ----------------------------------------------------------- (u,v) dispatch
// warp tile per word pair: MT x NT DMMA tiles of 8x8 (<= 64 fp64 accumulators)
template <typename F>
void dispatch(int u, int v, F&& f) {
#define FPMM_CASE(U, V, MT, NT) \
  if (u == U && v == V) return f.template operator()<U, V, MT, NT>();
  FPMM_CASE(1, 1, 8, 4)
  FPMM_CASE(1, 2, 4, 4)
  FPMM_CASE(2, 1, 4, 4)
  FPMM_CASE(1, 3, 4, 2)
  FPMM_CASE(3, 1, 4, 2)
  FPMM_CASE(1, 4, 4, 2)
  FPMM_CASE(4, 1, 4, 2)
  FPMM_CASE(2, 2, 4, 2)
  FPMM_CASE(2, 3, 2, 2)
  FPMM_CASE(3, 2, 2, 2)
  FPMM_CASE(2, 4, 2, 2)
  FPMM_CASE(4, 2, 2, 2)
#undef FPMM_CASE
  throw Failure(FPMM_B200_EERROR, "unsupported word counts (u,v)=(" + std::to_string(u) + "," +
                                      std::to_string(v) + "): need u,v <= 4 and uv <= 8");
}

DigitParams digit_params(u64 p, int w) {
  const SignedWords s = signed_words(p, w);
  DigitParams d;
  d.p = static_cast<long long>(p);
  d.half_p = static_cast<long long>(p / 2);
  d.alpha = static_cast<long long>(s.alpha);
  d.h = static_cast<long long>(s.half);
  d.inv_alpha = 1.0 / static_cast<double>(s.alpha);
  return d;
}

// Split-K count for `tiles` output tiles on `slots` persistent CTAs (or
// pairs): the smallest count in [lo, hi] whose last wave is well filled, i.e.
// maximising items / (waves * slots) with a 2% cost per extra slice.
int pick_splits(i64 tiles, i64 slots, i64 lo, i64 hi) {
  if (tiles <= 0) return 1;
  hi = std::max<i64>(hi, 1);
  lo = std::min<i64>(std::max<i64>(lo, 1), hi);
  i64 best = lo;
  double best_score = -1;
  for (i64 s = lo; s <= hi; ++s) {
    const i64 items = tiles * s;
    const i64 waves = (items + slots - 1) / slots;
    const double score = static_cast<double>(items) / static_cast<double>(waves * slots) - 0.02 * (s - lo);
    if (score > best_score + 1e-9) best_score = score, best = s;
  }
  return static_cast<int>(best);
}

int grid_for(i64 items, int threads) {
  const i64 blocks = (items + threads - 1) / threads;
  return static_cast<int>(std::min<i64>(std::max<i64>(blocks, 1), 148 * 64));
}

// Everything the kernels need for one (m, k, n, p, u, v) problem.
enum Engine { kDmma = 0, kI8 = 1, kRns = 2, kAuto = 3 };

struct Job {
  i64 m, k, n;
  u64 p;
  int u, v;
  int engine = kDmma;
  int D = 0;  // int8 engine: base-256 digits per residue
  bool narrow = false;  // int8 engine: NT = 32 tiles for n <= 32
  int BM = 0, BN = 0, MB = 0, NB = 0, KB = 0;
  size_t apack_bytes = 0, bpack_bytes = 0, per_rb_bytes = 0;
  i64 lambda_k = 0;
  GemmParams gp{};
  DigitParams da{}, db{};
  i8::Params ip{};
  int nmod = 0;  // RNS engine: moduli count
  rns::Params rp{};
  rns::PackParams rpp{};
  rns::CrtParams rcp{};
};

// int8 engine kernels by digit count and tile width (wide default or NT = 32)
template <typename F>
void dispatch_dn(int D, bool narrow, F&& f) {
  switch (D) {
    case 1: return narrow ? f.template operator()<1, 32>() : f.template operator()<1, i8::kWideNT<1>>();
    case 2: return narrow ? f.template operator()<2, 32>() : f.template operator()<2, i8::kWideNT<2>>();
    case 3: return narrow ? f.template operator()<3, 32>() : f.template operator()<3, i8::kWideNT<3>>();
    case 4: return narrow ? f.template operator()<4, 32>() : f.template operator()<4, i8::kWideNT<4>>();
    case 5: return narrow ? f.template operator()<5, 32>() : f.template operator()<5, i8::kWideNT<5>>();
    case 6: return narrow ? f.template operator()<6, 32>() : f.template operator()<6, i8::kWideNT<6>>();
    case 7: return f.template operator()<7, 32>();
  }
  throw Failure(FPMM_B200_EERROR, "int8 engine: unsupported digit count " + std::to_string(D));
}

template <typename F>
void dispatch_d(int D, F&& f) {
  switch (D) {
    case 1: return f.template operator()<1>();
    case 2: return f.template operator()<2>();
    case 3: return f.template operator()<3>();
    case 4: return f.template operator()<4>();
    case 5: return f.template operator()<5>();
    case 6: return f.template operator()<6>();
    case 7: return f.template operator()<7>();
  }
  throw Failure(FPMM_B200_EERROR, "int8 engine: unsupported digit count " + std::to_string(D));
}

int engine_flag(const Job& j) {
  return j.engine == kRns ? FPMM_B200_ENGINE_RNS : j.engine == kI8 ? FPMM_B200_ENGINE_I8 : FPMM_B200_ENGINE_DMMA;
}
int engine_words(const Job& j) { return j.engine == kRns ? j.nmod : j.engine == kI8 ? j.D : j.u * j.v; }

int resolve_engine(unsigned flags) {
  if (flags & FPMM_B200_ENGINE_RNS) return kRns;
  if (flags & FPMM_B200_ENGINE_I8) return kI8;
  if (flags & FPMM_B200_ENGINE_DMMA) return kDmma;
  return kAuto;  // library default: the faster tcgen05 engine for the shape (same results)
}

// The library default between the two tcgen05 engines, by a time model fitted
// on B200 (profiles/round1: the 8192^3 sweep and configs.json): the base-256
// engine costs D^2 int8 GEMMs on NT-column tiles plus a (2D-1)-block epilogue
// per output element; the RNS engine n_mod GEMMs on 256 x 256 pair tiles plus
// per-element residue parking and CRT; both pack their words (D or n_mod bytes
// per element) and lose the idle SMs when there are too few (split) tiles.
int auto_engine(i64 m, i64 k, i64 n, u64 p) {
  const int D = std::max(1, (bitsize(p - 1) + 7) / 8);
  int nmod = 0;
  try {
    nmod = rns_plan(p, k).n;
  } catch (const Failure&) {
    return kI8;
  }
  int nt = 32;
  dispatch_d(D, [&]<int DD>() { nt = n <= 32 ? 32 : i8::kWideNT<DD>; });
  const i64 KB = (k + 63) / 64;
  // fraction of the SMs (pairs) a product keeps busy, split-K included
  auto busy = [&](i64 tiles, i64 slots) {
    i64 items = tiles;
    if (tiles < slots) items = tiles * std::max<i64>(1, std::min<i64>({(slots + tiles - 1) / tiles, KB / 16, 32}));
    return std::min(1.0, static_cast<double>(items) / static_cast<double>(slots));
  };
  const double mn = static_cast<double>(m) * n;
  const double mk_kn = static_cast<double>(m) * k + static_cast<double>(k) * n;
  const double n_i8 = static_cast<double>((n + nt - 1) / nt * nt);
  const double n_rns = static_cast<double>((n + 255) / 256 * 256), m_rns = static_cast<double>((m + 255) / 256 * 256);
  const double t_i8 = (D * D * 2.0 * m * k * n_i8 / 3.2e15 + (2 * D - 1) * mn * 1.8e-12) /
                          busy(((m + 127) / 128) * ((n + nt - 1) / nt), 148) +
                      (8.0 + D) * mk_kn / 4.5e12;
  const double t_rns = (nmod * 2.0 * m_rns * k * n_rns / 3.2e15 + nmod * mn * 0.95e-12) /
                           busy(((m + 255) / 256) * ((n + 255) / 256), 74) +
                       (8.0 + nmod) * mk_kn / 4.5e12;
  return t_rns < t_i8 ? kRns : kI8;
}

Job make_i8_job(i64 m, i64 k, i64 n, u64 p) {
  Job j;
  j.m = m, j.k = k, j.n = n, j.p = p, j.engine = kI8;
  j.D = std::max(1, (bitsize(p - 1) + 7) / 8);
  j.BM = i8::kBM;
  j.MB = static_cast<int>((m + i8::kBM - 1) / i8::kBM);
  j.KB = static_cast<int>((k + i8::kBK - 1) / i8::kBK);
  j.narrow = n <= 32;
  dispatch_dn(j.D, j.narrow, [&]<int D, int NT>() {
    using CF = i8::Cfg<D, NT>;
    j.BN = CF::kNT;
    j.NB = static_cast<int>((n + j.BN - 1) / j.BN);
    j.per_rb_bytes = static_cast<size_t>(j.KB) * CF::kAStage;  // A's layout does not depend on NT
    j.apack_bytes = static_cast<size_t>(j.MB) * j.per_rb_bytes;
    j.bpack_bytes = static_cast<size_t>(j.NB) * j.KB * CF::kBStage;
  });
  // exact while pairs * K_seg * 255^2 < 2^32 (weight block read as unsigned)
  const u64 terms = 0xFFFFFFFFull / (static_cast<u64>(j.D) * 255 * 255);
  const i64 seg_kb = std::max<i64>(1, static_cast<i64>(terms) / i8::kBK);
  j.lambda_k = seg_kb * i8::kBK;
  i8::Params& q = j.ip;
  q.m = m, q.n = n, q.MB = j.MB, q.NB = j.NB, q.KB = j.KB;
  q.seg_kb = static_cast<int>(std::min<i64>(seg_kb, j.KB > 0 ? j.KB : 1));
  q.kb_per_split = j.KB;
  q.splits = 1;
  q.split_stride = 0;
  // epilogue reconstruction constants: 256^s mod p and Shoup quotients
  for (int s = 0; s < 2 * j.D - 1 && s < 13; ++s) {
    q.gam[s] = powmod(256 % p, static_cast<u64>(s), p);
    q.gam_sh[s] = shoup(q.gam[s], p);
  }
  q.p = p;
  q.mu = static_cast<unsigned long long>((static_cast<u128>(1) << 64) / p);
  return j;
}

// The one-reduction CRT finalisation (rns_crt_spec_kernel): with r_i the
// residues of X, S = sum_i r_i W_i and t the rounded sum_i r_i g_i / 2^19,
// X == S - t (M mod p) (mod p).  T0 bounds t, so R = S + (T0 - t) Mp + C0
// with C0 = -T0 Mp mod p is a non-negative representative; its bound R_max
// follows from r_i <= m_i - 1.  The quotient estimate umulhi(R >> s2, inv2),
// inv2 = floor(2^(s2+32) / p), undershoots R/p by less than 2^s2/p +
// (R_max >> s2) / 2^32; when that is below 1 a single conditional subtract
// finishes.  comb = 0 (generic two-reduction path) when a bound fails.
// Mirrored in tests/test_rns_rules.py.
void crt_plan_final(const RnsPlan& pl, int nmod, u64 p, rns::CrtParams& cp) {
  cp.comb = 0;
  if (nmod > 16) return;
  u128 smax = 0, fmax = 0;
  for (int i = 0; i < nmod; ++i) {
    const u64 g = ((static_cast<u64>(pl.y[i]) << 19) + pl.mod[i] / 2) / pl.mod[i];
    smax += static_cast<u128>(pl.mod[i] - 1) * pl.W[i];
    fmax += static_cast<u128>(pl.mod[i] - 1) * g;
  }
  const u128 t0 = (fmax + (u128{1} << 18)) >> 19;
  if (t0 >= (u128{1} << 32)) return;
  const u64 k = static_cast<u64>((t0 * pl.Mp) % p);
  const u64 c0 = (p - k) % p;
  const u128 rmax = smax + t0 * pl.Mp + c0;
  if (rmax >> 64) return;
  int bl = 0;
  while (bl < 128 && (rmax >> bl) != 0) ++bl;
  const int s2 = std::max(0, bl - 31);
  if ((u128{1} << s2) >= p) return;
  const u128 inv2 = (u128{1} << (s2 + 32)) / p;
  // 2^s2 / p + (R_max >> s2) / 2^32 < 1  <=>  2^(s2+32) + (R_max >> s2) p < 2^32 p
  if ((u128{1} << (s2 + 32)) + (rmax >> s2) * p >= (static_cast<u128>(p) << 32)) return;
  cp.comb = 1;
  cp.T0 = static_cast<uint32_t>(t0);
  cp.s2 = static_cast<uint32_t>(s2);
  cp.inv2 = static_cast<uint32_t>(inv2);
  cp.C0 = c0;
  cp.negp = static_cast<unsigned long long>(0) - p;
  // FP64 finalisation (crt4_spec in rns_tile_kernel, at most 5 byte planes):
  // R_max < 2^53 keeps every partial sum exact; the byte planes are < 2^20 (n <= 16)
  cp.fp64fin = 0;
  if (rmax < (u128{1} << 53) && p <= (u64{1} << 40)) {
    cp.fp64fin = 1;
    cp.Mp_d = static_cast<double>(pl.Mp);
    cp.C0_d = static_cast<double>(c0);
    cp.p_d = static_cast<double>(p);
    cp.invp_d = 1.0 / static_cast<double>(p);
  }
  if (const char* e = std::getenv("FPMM_B200_RNS_CRT_FP64")) cp.fp64fin = cp.fp64fin && std::atoi(e) != 0;
}

Job make_rns_job(i64 m, i64 k, i64 n, u64 p) {
  Job j;
  j.m = m, j.k = k, j.n = n, j.p = p, j.engine = kRns;
  const RnsPlan pl = rns_plan(p, k);
  j.nmod = pl.n;
  j.BM = rns::kPairM;  // pair tiles: 256 x 256
  j.BN = rns::kNT;
  j.MB = static_cast<int>((m + j.BM - 1) / j.BM);
  j.NB = static_cast<int>((n + j.BN - 1) / j.BN);
  j.KB = static_cast<int>((k + rns::kBK - 1) / rns::kBK);
  j.per_rb_bytes = static_cast<size_t>(2) * j.nmod * j.KB * rns::kAStage;  // per 256 rows
  j.apack_bytes = static_cast<size_t>(j.MB) * j.per_rb_bytes;
  j.bpack_bytes = static_cast<size_t>(2) * j.NB * j.nmod * j.KB * rns::kBStage;
  // a residue GEMM block read as u32 is exact while K_seg 255^2 < 2^32
  const i64 seg_kb = std::max<i64>(1, static_cast<i64>(0xFFFFFFFFull / (255ull * 255ull)) / rns::kBK);
  j.lambda_k = seg_kb * rns::kBK;
  rns::Params& q = j.rp;
  q.m = m, q.n = n, q.MB = j.MB, q.NB = j.NB, q.KB = j.KB;
  q.nmod = j.nmod;
  q.seg_kb = static_cast<int>(std::min<i64>(seg_kb, j.KB > 0 ? j.KB : 1));
  q.small_t = static_cast<i64>(q.seg_kb) * rns::kBK * 255 * 255 < (i64{1} << 24) ? 1 : 0;
  // the epilogue waits on the accumulator with the suspending try_wait; a
  // 256 ns sleep between polls measured 0.5-1% slower at 8192^3
  q.epi_sleep_ns = 0;
  // one flat (modulus, tile) sequence per pair: 52-bit 8192^3 DRAM reads
  // 10.4 -> 6.4 GB, L2 hit 75 -> 81%, rns_kernel 5.52 -> 5.24 ms
  q.flat = 1;
  if (const char* e = std::getenv("FPMM_B200_RNS_FLAT")) q.flat = std::atoi(e) != 0;
  if (const char* e = std::getenv("FPMM_B200_RNS_EPI_SLEEP")) q.epi_sleep_ns = static_cast<unsigned>(std::atoi(e));
  q.kb_per_split = j.KB;
  q.splits = 1;
  q.split_stride = 0;
  q.p = p;
  q.mu = static_cast<unsigned long long>((static_cast<u128>(1) << 64) / p);
  q.two32 = (u64{1} << 32) % p;
  q.two32_sh = shoup(q.two32, p);
  q.Mp = pl.Mp;
  q.Mp_sh = shoup(pl.Mp, p);
  rns::CrtParams& cp = j.rcp;
  cp.nmod = j.nmod;
  cp.p = p;
  cp.mu = q.mu;
  cp.two32 = q.two32;
  cp.two32_sh = q.two32_sh;
  cp.Mp = pl.Mp;
  cp.Mp_sh = q.Mp_sh;
  {
    int bits = 0;
    while (bits < 64 && (u64{1} << bits) < p) ++bits;  // ceil(log2 p)
    cp.s_shift = std::max(0, bits - 20);
    cp.inv32 = static_cast<uint32_t>((static_cast<u128>(1) << (cp.s_shift + 32)) / p);
    cp.Mp_sh32 = static_cast<uint32_t>((static_cast<u128>(pl.Mp) << 32) / p);
  }
  for (int i = 0; i < j.nmod; ++i) {
    cp.mod[i] = pl.mod[i];
    const u64 g = ((static_cast<u64>(pl.y[i]) << 19) + pl.mod[i] / 2) / pl.mod[i];  // < 2^19
    for (int b = 0; b < rns::kCrtPlanes; ++b) {
      const u64 byte = b < 7 ? (pl.W[i] >> (8 * b)) & 0xFF : (g >> (8 * (b - 7))) & 0xFF;
      cp.wb[i / 4][b] |= static_cast<uint32_t>(byte) << (8 * (i % 4));
    }
  }
  crt_plan_final(pl, j.nmod, p, cp);
  if (const char* e = std::getenv("FPMM_B200_RNS_CRT_COMB")) cp.comb = cp.comb && std::atoi(e) != 0;
  rns::PackParams& pp = j.rpp;
  pp.half_p = static_cast<double>(p / 2);
  pp.pf = static_cast<double>(p);
  pp.nmod = j.nmod;
  // residues of modulus pairs on the FP64 pipe: packs 5-7% faster at 36-52 bits than the dp4a digit form
  pp.fp64_pairs = 1;
  if (const char* e = std::getenv("FPMM_B200_RNS_PACK_FP64")) pp.fp64_pairs = std::atoi(e) != 0;
  for (int jj = 0; 2 * jj < j.nmod; ++jj) {
    const u64 L = static_cast<u64>(pl.mod[2 * jj]) * (2 * jj + 1 < j.nmod ? pl.mod[2 * jj + 1] : 1);
    pp.L[jj] = static_cast<double>(L);
    pp.invL[jj] = 1.0 / static_cast<double>(L);
    pp.offL[jj] = 4503599627370496.0 + static_cast<double>(L);
  }
  for (int i = 0; i < j.nmod; ++i) {
    const u64 mi = pl.mod[i];
    q.mod[i] = pp.mod[i] = static_cast<uint32_t>(mi);
    q.c16[i] = static_cast<uint32_t>((u64{1} << 16) % mi);
    q.magic[i] = pp.magic[i] = static_cast<uint32_t>(((u64{1} << 32) + mi - 1) / mi);
    q.negm[i] = pp.negm[i] = static_cast<uint32_t>(0u - static_cast<uint32_t>(mi));
    q.g[i] = pl.g[i];
    q.w_lo[i] = static_cast<uint32_t>(pl.W[i]);
    q.w_hi[i] = static_cast<uint32_t>(pl.W[i] >> 32);
    // dp4a weights: byte j of wlo/whi = 256^j mod m (j = 0..6); whi byte 3
    // weighs the centring flag with the residue offset of x - p
    pp.wlo[i] = pp.whi[i] = 0;
    for (int jj = 0; jj < 7; ++jj) {
      const uint32_t w = static_cast<uint32_t>(powmod(256 % mi, jj, mi));
      if (jj < 4) pp.wlo[i] |= w << (8 * jj);
      else pp.whi[i] |= w << (8 * (jj - 4));
    }
    pp.whi[i] |= static_cast<uint32_t>((mi - p % mi) % mi) << 24;
  }
  return j;
}

// FP64 engine word counts.  The engine's balanced signed words are internal
// (C is the same for any counts), so at the rule's lambda-collapse points --
// (2,2) at 52 bits, (1,3) at 39, (1,2) at 35, where the in-register
// reduction every lambda_k = 4 terms caps the FP64 pipe at 4/7 -- a larger
// count with a long exact block is cheaper: cost = u'v' (lambda_k + 3) /
// lambda_k DMMA-equivalents per term (3 FP64-pipe ops per reduction).
std::pair<int, int> dmma_words(u64 p, int u, int v, bool exact) {
  if (exact) return {u, v};
  auto cost = [&](int uu, int vv) {
    const i64 lk = kernel_block(p, uu, vv, 4);
    return lk < 4 ? 1e30 : uu * vv * (static_cast<double>(lk) + 3.0) / static_cast<double>(lk);
  };
  std::pair<int, int> best{u, v};
  double bc = cost(u, v);
  static constexpr int kCombos[12][2] = {{1, 1}, {1, 2}, {2, 1}, {1, 3}, {3, 1}, {1, 4},
                                         {4, 1}, {2, 2}, {2, 3}, {3, 2}, {2, 4}, {4, 2}};
  for (const auto& c : kCombos) {
    const double cc = cost(c[0], c[1]);
    if (cc < 0.97 * bc) bc = cc, best = {c[0], c[1]};  // only a clear win replaces the caller's words
  }
  return best;
}

Job make_job(i64 m, i64 k, i64 n, u64 p, int u, int v, int engine = kDmma, bool exact_words = false) {
  if (engine == kAuto) engine = auto_engine(m, k, n, p);
  if (engine == kRns) {
    Job j = make_rns_job(m, k, n, p);
    j.u = u, j.v = v;
    return j;
  }
  if (engine == kI8) {
    Job j = make_i8_job(m, k, n, p);
    j.u = u, j.v = v;
    return j;
  }
  std::tie(u, v) = dmma_words(p, u, v, exact_words);
  Job j;
  j.m = m, j.k = k, j.n = n, j.p = p, j.u = u, j.v = v;
  dispatch(u, v, [&]<int U, int V, int MT, int NT>() {
    using Cfg = GemmCfg<U, V, MT, NT>;
    j.BM = Cfg::BM;
    j.BN = Cfg::BN;
    j.MB = static_cast<int>((m + Cfg::BM - 1) / Cfg::BM);
    j.NB = static_cast<int>((n + Cfg::BN - 1) / Cfg::BN);
    j.KB = static_cast<int>((k + 15) / 16);
    j.per_rb_bytes = static_cast<size_t>(j.KB) * Cfg::kAElems * sizeof(double);
    j.apack_bytes = static_cast<size_t>(j.MB) * j.per_rb_bytes;
    j.bpack_bytes = static_cast<size_t>(j.NB) * j.KB * Cfg::kBElems * sizeof(double);
  });
  j.lambda_k = kernel_block(p, u, v, 4);
  if (j.lambda_k < 4)
    throw Failure(FPMM_B200_EINFEASIBLE, "no exact K-block >= 4 for (u,v)=(" + std::to_string(u) + "," +
                                             std::to_string(v) + ") at p=" + std::to_string(p));
  j.da = digit_params(p, u);
  j.db = digit_params(p, v);
  GemmParams& g = j.gp;
  g.MB = j.MB, g.NB = j.NB, g.KB = j.KB;
  g.m = m, g.n = n;
  const i64 steps = j.lambda_k / 4;
  g.red_every = static_cast<int>(std::min<i64>(steps, i64{1} << 30));
  g.pf = static_cast<double>(p);
  g.q = 1.0 / static_cast<double>(p);
  g.p = p;
  const u64 alpha = word_base(p, u) % p, beta = word_base(p, v) % p;
  for (int i = 0; i < u; ++i)
    for (int jj = 0; jj < v; ++jj) {
      const u64 gm = mulmod(powmod(alpha, i, p), powmod(beta, jj, p), p);
      g.gamma[i * v + jj] = gm;
      g.gamma_sh[i * v + jj] = shoup(gm, p);
    }
  return j;
}

// RNS packers by residue form (PackParams::fp64_pairs)
template <typename F>
void rns_pack_mode(int mode, F&& f) {
  switch (mode) {
    case 0: return f.template operator()<0>();
    default: return f.template operator()<1>();
  }
}

void launch_pack_a(const Job& j, const double* A, i64 lda, i64 rows, void* apack, int* err,
                   cudaStream_t s) {
  if (j.engine == kRns) {
    if (err && rows > 0 && j.k > 0)
      check_residues_kernel<<<grid_for(rows * j.k, 256), 256, 0, s>>>(A, lda, rows, j.k, j.p, err);
    const i64 mpad = ((rows + rns::kPairM - 1) / rns::kPairM) * rns::kPairM;
    const i64 items = mpad * j.KB * (rns::kBK / 16);
    rns_pack_mode(j.rpp.fp64_pairs, [&]<int MODE>() {
      rns::pack_a_rns<MODE><<<grid_for(items, 256), 256, 0, s>>>(A, lda, rows, j.k, j.KB, mpad, j.rpp,
                                                                 static_cast<uint8_t*>(apack));
    });
    CUDA_OK(cudaGetLastError());
    return;
  }
  if (j.engine == kI8) {
    if (err && rows > 0 && j.k > 0)
      check_residues_kernel<<<grid_for(rows * j.k, 256), 256, 0, s>>>(A, lda, rows, j.k, j.p, err);
    const i64 mpad = ((rows + i8::kBM - 1) / i8::kBM) * i8::kBM;
    const i64 items = mpad * j.KB * (i8::kBK / 16);
    dispatch_d(j.D, [&]<int D>() {
      i8::pack_a_i8<D><<<grid_for(items, 256), 256, 0, s>>>(A, lda, rows, j.k, j.KB, mpad,
                                                            static_cast<uint8_t*>(apack));
    });
    CUDA_OK(cudaGetLastError());
    return;
  }
  dispatch(j.u, j.v, [&]<int U, int V, int MT, int NT>() {
    using Cfg = GemmCfg<U, V, MT, NT>;
    const i64 mb = (rows + Cfg::BM - 1) / Cfg::BM;
    const i64 mpad = mb * Cfg::BM;
    const i64 items = (mpad / 2) * j.KB * 16;
    pack_a_kernel<U, Cfg::BM><<<grid_for(items, 256), 256, 0, s>>>(A, lda, rows, j.k, j.KB, mpad, j.da,
                                                                   static_cast<double*>(apack), err);
  });
  CUDA_OK(cudaGetLastError());
}

// RNS: B's k-blocks [kb0, kb0 + nkb) only (the multi-GPU path's k-chunks); B
// is the whole k x n matrix, and the residue check covers the chunk's rows.
void launch_pack_b_rns(const Job& j, const double* B, i64 ldb, void* bpack, int* err, cudaStream_t s, int kb0,
                       int nkb) {
  const i64 r0 = static_cast<i64>(kb0) * rns::kBK, r1 = std::min<i64>(j.k, static_cast<i64>(kb0 + nkb) * rns::kBK);
  if (err && r1 > r0 && j.n > 0)
    check_residues_kernel<<<grid_for((r1 - r0) * j.n, 256), 256, 0, s>>>(B + r0 * ldb, ldb, r1 - r0, j.n, j.p, err);
  const char* smem_env = std::getenv("FPMM_B200_RNS_PACKB_SMEM");
  const bool direct = !(smem_env && std::atoi(smem_env) != 0);
  if (direct) {
    // x: the padded width in blocks of 256 columns; y: k16 chunks, enough blocks for ~8 waves
    const unsigned gx = static_cast<unsigned>((2 * j.NB * rns::kBH + 255) / 256);
    const i64 chunks = static_cast<i64>(nkb) * (rns::kBK / 16);
    if (gx == 0 || chunks <= 0) return;
    const unsigned gy = static_cast<unsigned>(std::max<i64>(1, std::min<i64>({chunks, 65535,
                                                                               (148 * 64 + gx - 1) / gx})));
    rns_pack_mode(j.rpp.fp64_pairs, [&]<int MODE>() {
      rns::pack_b_rns_direct<MODE><<<dim3(gx, gy), 256, 0, s>>>(B, ldb, j.k, j.n, j.KB, 2 * j.NB, kb0, nkb, j.rpp,
                                                                static_cast<uint8_t*>(bpack));
    });
  } else {
    const i64 tiles = static_cast<i64>(nkb) * (2 * j.NB) * (rns::kBH / 32);
    rns_pack_mode(j.rpp.fp64_pairs, [&]<int MODE>() {
      rns::pack_b_rns<MODE><<<static_cast<unsigned>(std::min<i64>(std::max<i64>(tiles, 1), 148 * 32)), 128, 0, s>>>(
          B, ldb, j.k, j.n, j.KB, 2 * j.NB, kb0, nkb, j.rpp, static_cast<uint8_t*>(bpack));
    });
  }
  CUDA_OK(cudaGetLastError());
}

void launch_pack_b(const Job& j, const double* B, i64 ldb, void* bpack, int* err, cudaStream_t s) {
  if (j.engine == kRns) return launch_pack_b_rns(j, B, ldb, bpack, err, s, 0, j.KB);
  if (j.engine == kI8) {
    if (err && j.k > 0 && j.n > 0)
      check_residues_kernel<<<grid_for(j.k * j.n, 256), 256, 0, s>>>(B, ldb, j.k, j.n, j.p, err);
    const i64 tiles = static_cast<i64>(j.KB) * j.NB;
    dispatch_dn(j.D, j.narrow, [&]<int D, int NT>() {
      i8::pack_b_i8<D, NT><<<static_cast<unsigned>(std::min<i64>(std::max<i64>(tiles, 1), 148 * 16)), 256, 0, s>>>(
          B, ldb, j.k, j.n, j.KB, j.NB, static_cast<uint8_t*>(bpack));
    });
    CUDA_OK(cudaGetLastError());
    return;
  }
  dispatch(j.u, j.v, [&]<int U, int V, int MT, int NT>() {
    using Cfg = GemmCfg<U, V, MT, NT>;
    const i64 npad = static_cast<i64>(j.NB) * Cfg::BN;
    const i64 items = (npad / 2) * j.KB * 16;
    pack_b_kernel<V, Cfg::BN><<<grid_for(items, 256), 256, 0, s>>>(B, ldb, j.k, j.n, j.KB, npad, j.db,
                                                                   static_cast<double*>(bpack), err);
  });
  CUDA_OK(cudaGetLastError());
}

int launch_gemm_i8(const Job& j, const void* apack, const void* bpack, double* C, i64 ldc, i64 rows,
                   cudaStream_t s, cudaEvent_t mid, Workspace& ws) {
  i8::Params q = j.ip;
  q.apack = static_cast<const uint8_t*>(apack);
  q.bpack = static_cast<const uint8_t*>(bpack);
  q.C = C;
  q.ldc = ldc;
  q.m = rows;
  q.MB = static_cast<int>((rows + i8::kBM - 1) / i8::kBM);
  // split-K when the output has too few tiles to fill two waves of 148 SMs
  // (tall-and-skinny / unbalanced shapes): slices of >= 16 k-blocks write
  // partial residues to a workspace, combined mod p afterwards
  const i64 tiles0 = static_cast<i64>(q.MB) * q.NB;
  int splits = 1;
  if (tiles0 > 0 && tiles0 < 2 * 148) {
    const i64 want = (2 * 148 + tiles0 - 1) / tiles0;
    splits = pick_splits(tiles0, 148, std::min<i64>(want, j.KB / 16), std::min<i64>(j.KB / 16, 32));
  }
  // Long K: one split per exact int32 segment, slices ordered split-major, so
  // every wave of 148 items streams one K-chunk of its panels (~100 MB at
  // D=7) instead of the whole K (measured at 8192 x 32768 x 8192: L2 hit rate
  // 52% and 222 GB of DRAM reads with in-item segments).
  if (j.KB > q.seg_kb) splits = std::max<int>(splits, (j.KB + q.seg_kb - 1) / q.seg_kb);
  q.kb_per_split = (j.KB + splits - 1) / splits;
  splits = (j.KB + q.kb_per_split - 1) / q.kb_per_split;
  q.splits = splits;
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  double* work = nullptr;
  if (splits > 1) {
    work = static_cast<double*>(ws.splitws.get(sizeof(double) * splits * rows * j.n));
    q.C = work;
    q.ldc = j.n;
    q.split_stride = rows * j.n;
  }
  // persistent grid: one CTA per SM (at most one work item each if fewer)
  int sms = 148;
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const i64 items = static_cast<i64>(q.MB) * q.NB * splits;
  const unsigned grid = static_cast<unsigned>(std::max<i64>(1, std::min<i64>(items, sms)));
  dispatch_dn(j.D, j.narrow, [&]<int D, int NT>() {
    using CF = i8::Cfg<D, NT>;
    auto kern = i8::mwi8_kernel<D, NT>;
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 63]) {
      CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::kSmem));
      configured[dev & 63] = true;
    }
    if (items > 0x7fffffff) throw Failure(FPMM_B200_EERROR, "problem too large for one launch");
    kern<<<grid, i8::kThreads, CF::kSmem, s>>>(q);
  });
  CUDA_OK(cudaGetLastError());
  if (mid) CUDA_OK(cudaEventRecord(mid, s));
  if (splits > 1) {
    i8::splitk_reduce_kernel<<<grid_for(rows * j.n, 256), 256, 0, s>>>(work, rows * j.n, splits, C, ldc, rows,
                                                                        j.n, j.p);
    CUDA_OK(cudaGetLastError());
  }
  return splits > 1 ? 2 : 1;
}

// 2-D uint8 tensor map over `bytes` of a packed operand viewed as 128-byte
// rows, box 128 x (stage chunk / 128); the encoder comes from the driver
// through the runtime (no libcuda link dependency).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  // thread-safe one-time lookup (calls on different devices run concurrently)
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      throw Failure(FPMM_B200_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  return encode;
}

CUtensorMap chunk_map(const void* base, size_t bytes) {
  const PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  CUtensorMap m{};
  constexpr cuuint32_t kRows = rns::kAStage / 128;  // one stage chunk (kBStage == kAStage)
  static_assert(rns::kAStage == rns::kBStage, "A and B stage chunks share the tensor-map box");
  const cuuint64_t dims[2] = {128, std::max<cuuint64_t>(kRows, bytes / 128)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, kRows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Failure(FPMM_B200_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// 3-D uint8 tensor map over packed RNS B (128-column blocks, [k16][column
// group (16)][8 columns][16 B]): 128-byte rows of one column group, 16 groups
// per k16 slice, k16 slices; box = 8 column groups x one stage's k16 slices
// (half of a 128-column block: rns_tile_kernel's per-CTA B).
CUtensorMap half_block_map(const void* base, size_t bytes) {
  const PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  CUtensorMap m{};
  constexpr cuuint32_t kSlices = rns::kBK / 16;
  const cuuint64_t dims[3] = {128, 16, std::max<cuuint64_t>(kSlices, bytes / 2048)};
  const cuuint64_t strides[2] = {128, 2048};
  const cuuint32_t box[3] = {128, 8, kSlices};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Failure(FPMM_B200_ECUDA, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string(r));
  return m;
}

// RNS split-K: split when the output has too few pair tiles for the SM
// pairs, and one slice per exact int32 segment for long K (split-major: each
// wave streams one K-chunk of its panels); n_mod is planned for the full K.
int rns_splits(const Job& j, i64 rows) {
  const i64 tiles0 = ((rows + rns::kPairM - 1) / rns::kPairM) * j.NB;
  int splits = 1;
  if (tiles0 > 0 && tiles0 < 74) {
    const i64 want = (74 + tiles0 - 1) / tiles0;
    splits = pick_splits(tiles0, 74, std::min<i64>(want, j.KB / 16), std::min<i64>(j.KB / 16, 32));
  }
  if (j.KB > j.rp.seg_kb) splits = std::max<int>(splits, (j.KB + j.rp.seg_kb - 1) / j.rp.seg_kb);
  if (const char* e = std::getenv("FPMM_B200_RNS_SLICE_KB")) {  // experiment: K slices of at most this many k-blocks
    const int sl = std::max(1, std::atoi(e));
    splits = std::max<int>(splits, (j.KB + sl - 1) / sl);
  }
  const int per = (j.KB + splits - 1) / splits;
  return (j.KB + per - 1) / per;
}

int launch_gemm_rns_rows(const Job& j, const void* apack, const void* bpack, double* C, i64 ldc, i64 rows,
                         cudaStream_t s, cudaEvent_t mid, Workspace& ws) {
  rns::Params q = j.rp;
  q.apack = static_cast<const uint8_t*>(apack);
  q.bpack = static_cast<const uint8_t*>(bpack);
  q.tmA = chunk_map(apack, static_cast<size_t>((rows + rns::kPairM - 1) / rns::kPairM) * j.per_rb_bytes);
  q.tmB = chunk_map(bpack, j.bpack_bytes);
  q.C = C;
  q.ldc = ldc;
  q.m = rows;
  q.MB = static_cast<int>((rows + rns::kPairM - 1) / rns::kPairM);
  const int splits = rns_splits(j, rows);
  q.kb_per_split = (j.KB + splits - 1) / splits;
  q.splits = splits;
  // two epilogue groups on alternate passes (one K segment per pass); off: FPMM_B200_RNS_PINGPONG=0
  q.pingpong = q.kb_per_split <= q.seg_kb ? 1 : 0;
  if (const char* e = std::getenv("FPMM_B200_RNS_PINGPONG")) q.pingpong = q.pingpong && std::atoi(e) != 0;
  // pingpong drain with two TMEM loads per wait: the accumulator goes back to
  // the MMAs two load round trips earlier; short passes gain (16384^2 x 256:
  // -6..-8% at 20/40/52 bits), k = 1024 loses 1.5% (tools/ab/ab_pp_pairs.sh)
  q.pp_pairs = q.kb_per_split <= 4 ? 1 : 0;
  if (const char* e = std::getenv("FPMM_B200_RNS_PP_PAIRS")) q.pp_pairs = std::atoi(e) != 0;
  if (const char* e = std::getenv("FPMM_B200_RNS_DEBUG")) q.debug = std::atoi(e);
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  int sms = 148;
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const i64 items = static_cast<i64>(q.MB) * q.NB * splits;
  if (items > 0x7fffffff) throw Failure(FPMM_B200_EERROR, "problem too large for one launch");
  // persistent CTA pairs (clusters of 2 on neighbouring SMs): no more pairs
  // than can be co-resident (a GPC with an odd SM count leaves one SM out of
  // every pair), so no pair waits for another to finish
  static int max_pairs[64] = {};
  if (!max_pairs[dev & 63]) {
    CUDA_OK(cudaFuncSetAttribute(rns::rns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rns::kSmem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(sms / 2 * 2));
    cfg.blockDim = dim3(rns::kThreads);
    cfg.dynamicSmemBytes = rns::kSmem;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2, attr.val.clusterDim.y = 1, attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, rns::rns_kernel, &cfg) != cudaSuccess || clusters < 1) {
      cudaGetLastError();
      clusters = sms / 2;
    }
    max_pairs[dev & 63] = std::min(clusters, sms / 2);
  }
  const unsigned grid = 2 * static_cast<unsigned>(std::max<i64>(1, std::min<i64>(items, max_pairs[dev & 63])));
  // residue bytes: every item's, n bytes per output element and slice
  const size_t slots = static_cast<size_t>(items) * 2;
  q.scratch = static_cast<uint8_t*>(ws.scratch.get(slots * j.nmod * rns::kSlotPerMod));
  q.group = rns::kGroup;
  if (const char* d = std::getenv("FPMM_B200_RNS_GROUP")) q.group = std::max(1, std::atoi(d));
  // pacing (rns_kernel's producer and monitor): for passes longer than 8192 k
  // a wave's panels (21 of 256 x k bytes) exceed L2 and the pairs drift apart
  // unless held within 8192 k of the slowest (64 k-blocks of 128 B at the time); measured: C3 32768^3 rns_kernel
  // DRAM reads 1048 -> 328 GB and 533 -> 443 ms per product, C4 287 -> 90 GB and
  // 57 -> 42 ms; at k = 8192 (fits L2) it only costs (sweep -3.5%):
  // profiles/round2/ab_pace.txt.  FPMM_B200_RNS_PACE=<k-blocks> overrides (0 = off).
  constexpr int kPaceKb = 8192 / rns::kBK;  // a window of 8192 k, whatever the stage depth
  q.pace_kb = q.kb_per_split > kPaceKb ? kPaceKb : 0;
  if (const char* e = std::getenv("FPMM_B200_RNS_PACE")) q.pace_kb = std::max(0, std::atoi(e));
  q.progress = nullptr;
  if (q.pace_kb > 0) {
    const size_t np = grid / 2, padded = (np + 3) / 4 * 4;  // pace_min reads int4s; padding = INT_MAX-ish
    q.progress = static_cast<int*>(ws.pace.get(sizeof(int) * padded));
    CUDA_OK(cudaMemsetAsync(q.progress, 0x7f, sizeof(int) * padded, s));
    CUDA_OK(cudaMemsetAsync(q.progress, 0, sizeof(int) * np, s));
  }
  static bool configured[64] = {};
  if (!configured[dev & 63]) {
    CUDA_OK(cudaFuncSetAttribute(rns::rns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, rns::kSmem));
    configured[dev & 63] = true;
  }
  // the CRT constants and C
  rns::CrtParams cp = j.rcp;
  cp.R = q.scratch;
  cp.C = C;
  cp.ldc = ldc;
  cp.m = rows;
  cp.n = j.n;
  cp.MB = q.MB, cp.NB = q.NB, cp.splits = splits, cp.group = q.group;
  const int wpl = std::max(1, (bitsize(j.p - 1) + 7) / 8);
  rns::rns_kernel<<<grid, rns::kThreads, rns::kSmem, s>>>(q);
  CUDA_OK(cudaGetLastError());
  if (mid) CUDA_OK(cudaEventRecord(mid, s));
  // CRT of every tile (slices summed mod m_i first) straight into C
  const i64 tiles = static_cast<i64>(q.MB) * q.NB;
  // one K slice: the kernel specialised on the plane and group counts
  // (FPMM_B200_RNS_CRT_SPEC=0 keeps the generic one, for A/B)
  static const bool spec = [] {
    const char* e = std::getenv("FPMM_B200_RNS_CRT_SPEC");
    return !(e && std::atoi(e) == 0);
  }();
  if (splits == 1 && spec) {
    using K = void (*)(rns::CrtParams);
#define FPMM_CRT_ROW(W) \
  {rns::rns_crt_spec_kernel<W, 1>, rns::rns_crt_spec_kernel<W, 2>, rns::rns_crt_spec_kernel<W, 3>, \
   rns::rns_crt_spec_kernel<W, 4>, rns::rns_crt_spec_kernel<W, 5>}
    static const K table[7][5] = {FPMM_CRT_ROW(1), FPMM_CRT_ROW(2), FPMM_CRT_ROW(3), FPMM_CRT_ROW(4),
                                  FPMM_CRT_ROW(5), FPMM_CRT_ROW(6), FPMM_CRT_ROW(7)};
#undef FPMM_CRT_ROW
    const int ng = (j.nmod + 3) / 4;
    table[std::min(wpl, 7) - 1][ng - 1]<<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp);
    CUDA_OK(cudaGetLastError());
    return 2;
  }
  switch (wpl) {
    case 1: rns::rns_crt_kernel<1><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
    case 2: rns::rns_crt_kernel<2><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
    case 3: rns::rns_crt_kernel<3><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
    case 4: rns::rns_crt_kernel<4><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
    case 5: rns::rns_crt_kernel<5><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
    case 6: rns::rns_crt_kernel<6><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
    default: rns::rns_crt_kernel<7><<<static_cast<unsigned>(2 * tiles), 256, 0, s>>>(cp); break;
  }
  CUDA_OK(cudaGetLastError());
  return 2;
}

// The parked residues take n bytes per output element (and split-K slice);
// above kRnsResidueBudget the product runs in row blocks of whole pair tiles
// that reuse one residue buffer (e.g. 65536^2 outputs at n = 11: 47 GB).
constexpr size_t kRnsResidueBudget = size_t{8} << 30;

// The on-chip CRT (rns_tile_kernel, rnstile.cuh): one exact K segment, no
// split-K, n <= 16.  FPMM_B200_RNS_TILE=0 never uses it, =1 wherever it applies;
// by default at k <= 256 with n <= 12 (up to ~40 bits), where it measured
// faster than parking the residues once both kernels issue MMAs from a
// converged warp (C5 65536 x 256 x 65536: 30.9 against 34.4 ms, 16384^2 x 256:
// -5% at 20 bits, -1% at 40); at 52 bits (+4%) and k = 512 (+2%) it is slower
// (profiles/round2/tile_kernel.md).
constexpr int kRnsTileMaxK = 256, kRnsTileMaxMod = 12;
bool rns_tile(const Job& j, i64 rows) {
  if (j.nmod > rns::kTMaxMod || j.KB > j.rp.seg_kb || rns_splits(j, rows) != 1) return false;
  const char* e = std::getenv("FPMM_B200_RNS_TILE");
  const int mode = e ? std::atoi(e) : -1;
  if (mode == 0) return false;
  return mode > 0 || (j.k <= kRnsTileMaxK && j.nmod <= kRnsTileMaxMod);
}

template <int WPL, int NG>
void launch_tile_kernel(const rns::Params& q, unsigned grid, size_t smem, cudaStream_t s) {
  auto kern = rns::rns_tile_kernel<WPL, NG>;
  static bool configured[64] = {};
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  if (!configured[dev & 63]) {
    CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    configured[dev & 63] = true;
  }
  kern<<<grid, rns::kTThreads, smem, s>>>(q);
}

int launch_rns_tile(const Job& j, const void* apack, const void* bpack, double* C, i64 ldc, i64 rows,
                    cudaStream_t s, cudaEvent_t mid) {
  rns::Params q = j.rp;
  q.apack = static_cast<const uint8_t*>(apack);
  q.bpack = static_cast<const uint8_t*>(bpack);
  q.tmA = chunk_map(apack, static_cast<size_t>((rows + rns::kPairM - 1) / rns::kPairM) * j.per_rb_bytes);
  q.tmB = half_block_map(bpack, j.bpack_bytes);
  q.C = C;
  q.ldc = ldc;
  q.m = rows;
  q.MB = static_cast<int>((rows + rns::kPairM - 1) / rns::kPairM);
  q.NB = static_cast<int>((j.n + rns::kTNT - 1) / rns::kTNT);
  q.splits = 1;
  q.kb_per_split = j.KB;
  q.group = rns::kGroup;
  if (const char* d = std::getenv("FPMM_B200_RNS_GROUP")) q.group = std::max(1, std::atoi(d));
  // shared memory: `stages` stages of 48 KB, then as many residue planes (16 KB
  // each) as fit, then the barriers; TMEM: as many 128-column accumulators
  // (2..4) as the remaining planes (32 columns each) leave room for.  Two
  // stages (two k = 256 passes ahead) and the rest for residues, so more
  // accumulators: the MMAs run further ahead while the epilogue rebuilds a
  // tile (C5 30.5 -> 29.7 ms, 16384^2 x 256 at 20 bits -8%, tools/ab/ab_tile_stages.sh)
  constexpr int kMaxSmem = 227 * 1024, kBarBytes = 256;
  int want = 2;
  if (const char* e = std::getenv("FPMM_B200_RNS_TILE_STAGES")) want = std::atoi(e);
  q.naccs = 0;
  want = std::min({want, rns::kTMaxStages, (kMaxSmem - kBarBytes) / rns::kTStageBytes});
  for (q.stages = std::max(2, want); q.stages >= 2; --q.stages) {
    q.smem_mods = std::min(j.nmod, (kMaxSmem - kBarBytes - q.stages * rns::kTStageBytes) / rns::kTResBytes);
    q.naccs = std::min(rns::kTMaxAccs, (512 - (j.nmod - q.smem_mods) * (rns::kTNT / 4)) / rns::kTNT);
    if (q.naccs >= 2) break;
  }
  if (const char* e = std::getenv("FPMM_B200_RNS_TILE_ACCS")) q.naccs = std::min(q.naccs, std::atoi(e));
  if (q.naccs < 2) throw Failure(FPMM_B200_EERROR, "rns_tile_kernel: on-chip residues do not fit");
  const int res_bytes = q.smem_mods * rns::kTResBytes;
  q.res_off = q.stages * rns::kTStageBytes;
  q.bar_off = q.res_off + res_bytes;
  const size_t smem = static_cast<size_t>(q.bar_off) + kBarBytes;
  rns::CrtParams cp = j.rcp;
  cp.R = nullptr;
  cp.C = C;
  cp.ldc = ldc;
  cp.m = rows;
  cp.n = j.n;
  cp.MB = q.MB, cp.NB = q.NB, cp.splits = 1, cp.group = q.group;
  q.crt = cp;
  const int wpl = std::max(1, (bitsize(j.p - 1) + 7) / 8), ng = (j.nmod + 3) / 4;
  q.wpl = wpl;
  int dev = 0, sms = 148;
  CUDA_OK(cudaGetDevice(&dev));
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const i64 tiles = static_cast<i64>(q.MB) * q.NB;
  // as many pairs as rns_kernel's co-resident clusters (one CTA per SM either way)
  const unsigned grid = 2 * static_cast<unsigned>(std::max<i64>(1, std::min<i64>(tiles, sms / 2)));
  switch (wpl * 8 + ng) {
#define FPMM_TILE(W, G) \
  case W * 8 + G: launch_tile_kernel<W, G>(q, grid, smem, s); break;
    FPMM_TILE(1, 1) FPMM_TILE(1, 2) FPMM_TILE(2, 1) FPMM_TILE(2, 2) FPMM_TILE(3, 2) FPMM_TILE(3, 3)
    FPMM_TILE(4, 2) FPMM_TILE(4, 3) FPMM_TILE(5, 3) FPMM_TILE(5, 4) FPMM_TILE(6, 3) FPMM_TILE(6, 4)
    FPMM_TILE(7, 4)
#undef FPMM_TILE
    default:
      throw Failure(FPMM_B200_EERROR, "rns_tile_kernel: no instance for " + std::to_string(wpl) + " planes, " +
                                          std::to_string(j.nmod) + " moduli");
  }
  CUDA_OK(cudaGetLastError());
  if (mid) CUDA_OK(cudaEventRecord(mid, s));
  return 1;
}

int launch_gemm_rns(const Job& j, const void* apack, const void* bpack, double* C, i64 ldc, i64 rows,
                    cudaStream_t s, cudaEvent_t mid, Workspace& ws) {
  if (rns_tile(j, rows)) return launch_rns_tile(j, apack, bpack, C, ldc, rows, s, mid);
  const i64 pair_rows = (rows + rns::kPairM - 1) / rns::kPairM;
  const size_t per_pair_row = static_cast<size_t>(j.NB) * 2 * j.nmod * rns::kSlotPerMod *
                              std::max<i64>(rns_splits(j, rows), (j.KB + j.rp.seg_kb - 1) / j.rp.seg_kb);
  size_t budget = kRnsResidueBudget;
  if (const char* e = std::getenv("FPMM_B200_RNS_RESIDUE_BUDGET")) budget = std::strtoull(e, nullptr, 10);
  const i64 chunk = std::max<i64>(1, static_cast<i64>(budget / per_pair_row));
  if (pair_rows <= chunk) return launch_gemm_rns_rows(j, apack, bpack, C, ldc, rows, s, mid, ws);
  int launches = 0;
  for (i64 pr = 0; pr < pair_rows; pr += chunk) {
    const i64 r0 = pr * rns::kPairM, rn = std::min<i64>(rows - r0, chunk * rns::kPairM);
    launches += launch_gemm_rns_rows(j, static_cast<const uint8_t*>(apack) + pr * j.per_rb_bytes, bpack,
                                     C + r0 * ldc, ldc, rn, s, nullptr, ws);
  }
  if (mid) CUDA_OK(cudaEventRecord(mid, s));  // row blocks interleave GEMM and CRT: all counted as GEMM
  return launches;
}

// Launches the product kernel(s) for packed operands; returns the launch count.
// `mid` (nullable) is recorded after the product kernel, before any
// reconstruction kernel (RNS CRT, int8 split-K combine).
int launch_gemm(const Job& j, const void* apack_v, const void* bpack_v, double* C, i64 ldc, i64 rows,
                cudaStream_t s, Workspace& ws, cudaEvent_t mid = nullptr, int* overflow = nullptr) {
  if (j.engine == kRns) return launch_gemm_rns(j, apack_v, bpack_v, C, ldc, rows, s, mid, ws);
  if (j.engine == kI8) return launch_gemm_i8(j, apack_v, bpack_v, C, ldc, rows, s, mid, ws);
  const double* apack = static_cast<const double*>(apack_v);
  const double* bpack = static_cast<const double*>(bpack_v);
  GemmParams g = j.gp;
  g.overflow = overflow;  // CHECK_EXACTNESS (FP64 engine only: the int8 engines are exact by construction)
  if (const char* e = std::getenv("FPMM_B200_TEST_RED_EVERY")) g.red_every = std::max(1, std::atoi(e));
  g.apack = apack;
  g.bpack = bpack;
  g.C = C;
  g.ldc = ldc;
  g.m = rows;
  dispatch(j.u, j.v, [&]<int U, int V, int MT, int NT>() {
    using Cfg = GemmCfg<U, V, MT, NT>;
    g.MB = static_cast<int>((rows + Cfg::BM - 1) / Cfg::BM);
    auto kern = mwgemm_kernel<U, V, MT, NT>;
    static bool configured[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!configured[dev & 63]) {
      CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
      configured[dev & 63] = true;
    }
    const i64 tiles = static_cast<i64>(g.MB) * g.NB;
    if (tiles > 0x7fffffff) throw Failure(FPMM_B200_EERROR, "problem too large for one launch");
    kern<<<static_cast<unsigned>(tiles), Cfg::kThreads, Cfg::kSmem, s>>>(g);
  });
  CUDA_OK(cudaGetLastError());
  if (mid) CUDA_OK(cudaEventRecord(mid, s));
  return 1;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

void check_err_flag(DeviceCtx& c, cudaStream_t s) {
  int h = 0;
  CUDA_OK(cudaMemcpyAsync(&h, c.err.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  if (h & 1) throw Failure(FPMM_B200_ECONTRACT, "multiword product: inputs must be residues in [0, p)");
  if (h & 2)
    throw Failure(FPMM_B200_ECONTRACT, "exactness check: an FP64 accumulator exceeded 2^53 before its reduction");
}

// Zero the rows x n block of C (k == 0 product).
void zero_c(double* C, i64 ldc, i64 rows, i64 n, cudaStream_t s) {
  if (rows > 0 && n > 0)
    CUDA_OK(cudaMemset2DAsync(C, ldc * sizeof(double), 0, n * sizeof(double), rows, s));
}

}  // namespace

unsigned select_engine(i64 m, i64 k, i64 n, u64 p) {
  if (m < 0 || k < 0 || n < 0) throw Failure(FPMM_B200_EERROR, "matrix dimensions must be nonnegative");
  if (p < 2) throw Failure(FPMM_B200_EERROR, "modulus must exceed 1");
  return auto_engine(std::max<i64>(m, 1), std::max<i64>(k, 1), std::max<i64>(n, 1), p) == kRns ? FPMM_B200_ENGINE_RNS
                                                                                             : FPMM_B200_ENGINE_I8;
}

void validate_product(u64 p, int u, int v, u64 lambda, i64 m, i64 k, i64 n, unsigned flags) {
  if (m < 0 || k < 0 || n < 0) throw Failure(FPMM_B200_EERROR, "matrix dimensions must be nonnegative");
  context_check(p, (flags & FPMM_B200_ALLOW_COMPOSITE) != 0);
  check_mw_inputs(k, k, u, v, lambda, p);
  if (flags & FPMM_B200_INPLACE_INVERSES) {
    // scale_factors (multiword.hpp:76-86) inverts alpha (i > 0) and beta (j > 0)
    auto invertible = [&](u64 base) {
      u64 a = base % p, b = p;
      while (b) {
        const u64 t = a % b;
        a = b;
        b = t;
      }
      return a == 1;
    };
    if (u > 1 && !invertible(word_base(p, u)))
      throw Failure(FPMM_B200_ENOINVERSE, "no inverse: gcd(alpha, p) > 1; use the workspace product variant");
    if (v > 1 && !invertible(word_base(p, v)))
      throw Failure(FPMM_B200_ENOINVERSE, "no inverse: gcd(beta, p) > 1; use the workspace product variant");
  }
}

void product_device(const ProductArgs& a, int device, void* stream, fpmm_b200_timing* tm) {
  DevLock lk(device);
  validate_product(a.p, a.u, a.v, a.lambda, a.m, a.k, a.n, a.flags);
  DeviceCtx& c = ctx(device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  if (tm) *tm = fpmm_b200_timing{};
  if (a.m == 0 || a.n == 0) return;
  if (a.k == 0) {
    zero_c(a.C, a.ldc, a.m, a.n, s);
    if (!(a.flags & FPMM_B200_ASYNC)) CUDA_OK(cudaStreamSynchronize(s));
    return;
  }
  const Job j = make_job(a.m, a.k, a.n, a.p, a.u, a.v, resolve_engine(a.flags),
                     (a.flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
  Workspace& ws = c.ws_for(s);
  void* apack = ws.apack.get(j.apack_bytes);
  void* bpack = ws.bpack.get(j.bpack_bytes);
  int* err = nullptr;
  if (a.flags & (FPMM_B200_CHECK_INPUTS | FPMM_B200_CHECK_EXACTNESS)) {
    err = static_cast<int*>(c.err.get(sizeof(int)));
    CUDA_OK(cudaMemsetAsync(err, 0, sizeof(int), s));
  }
  int* err_in = (a.flags & FPMM_B200_CHECK_INPUTS) ? err : nullptr;
  if (tm) CUDA_OK(cudaEventRecord(c.ev[0], s));
  launch_pack_a(j, a.A, a.lda, a.m, apack, err_in, s);
  launch_pack_b(j, a.B, a.ldb, bpack, err_in, s);
  if (tm) CUDA_OK(cudaEventRecord(c.ev[1], s));
  const int gl = launch_gemm(j, apack, bpack, a.C, a.ldc, a.m, s, ws, tm ? c.ev[5] : nullptr,
                             (a.flags & FPMM_B200_CHECK_EXACTNESS) ? err : nullptr);
  if (tm) CUDA_OK(cudaEventRecord(c.ev[2], s));
  if (err) check_err_flag(c, s);
  if (tm) {
    CUDA_OK(cudaEventSynchronize(c.ev[2]));
    tm->pack_ms = elapsed(c.ev[0], c.ev[1]);
    tm->gemm_ms = elapsed(c.ev[1], c.ev[5]);
    tm->recon_ms = elapsed(c.ev[5], c.ev[2]);
    tm->total_ms = elapsed(c.ev[0], c.ev[2]);
    tm->lambda_k = j.lambda_k;
    tm->engine = engine_flag(j), tm->words = engine_words(j);
    tm->launches = 2 + gl;
    tm->ngpus = 1;
  }
  if (!(a.flags & FPMM_B200_ASYNC)) CUDA_OK(cudaStreamSynchronize(s));
}

// ------------------------------------------------- prepared (resident) A words
// The unbalanced scenario of the paper (and run_bench's, driver.cpp:215-218)
// reuses A's decomposition across many products: pack A's words once, keep
// them resident in HBM, and run each product from the packed words.
struct Prepared {
  int device = 0, engine = kI8;
  u64 p = 0;
  int u = 1, v = 1;
  i64 m = 0, k = 0;
  unsigned flags = 0;
  DevBuf words;
};

Prepared* prepare_a_device(const double* dA, i64 lda, i64 m, i64 k, u64 p, int u, int v, unsigned flags,
                           int device, void* stream) {
  DevLock lk(device);
  if (m < 0 || k < 0) throw Failure(FPMM_B200_EERROR, "matrix dimensions must be nonnegative");
  context_check(p, (flags & FPMM_B200_ALLOW_COMPOSITE) != 0);
  if (u < 1 || v < 1) throw Failure(FPMM_B200_EERROR, "multiword product: word counts must be positive");
  DeviceCtx& c = ctx(device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  auto h = std::make_unique<Prepared>();
  h->device = device, h->engine = resolve_engine(flags), h->p = p, h->u = u, h->v = v, h->m = m, h->k = k;
  // n is unknown when A is prepared; the resident-A (unbalanced) scenario
  // multiplies by narrow B blocks, where the base-256 engine's narrow tiles win
  if (h->engine == kAuto) h->engine = kI8;
  h->flags = flags;
  if (m > 0 && k > 0) {
    const Job j = make_job(m, k, 1, p, u, v, h->engine, (flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
    void* w = h->words.get(j.apack_bytes);
    int* err = nullptr;
    if (flags & FPMM_B200_CHECK_INPUTS) {
      err = static_cast<int*>(c.err.get(sizeof(int)));
      CUDA_OK(cudaMemsetAsync(err, 0, sizeof(int), s));
    }
    launch_pack_a(j, dA, lda, m, w, err, s);
    if (err) check_err_flag(c, s);
    CUDA_OK(cudaStreamSynchronize(s));
  }
  return h.release();
}

void prepared_free(Prepared* h) {
  if (!h) return;
  DevLock lk(h->device);
  cudaSetDevice(h->device);
  h->words.release();
  delete h;
}

void product_prepared_device(const Prepared* h, const double* dB, i64 ldb, double* dC, i64 ldc, i64 n, u64 lambda,
                             void* stream, unsigned flags, fpmm_b200_timing* tm) {
  if (!h) throw Failure(FPMM_B200_EERROR, "null prepared operand");
  DevLock lk(h->device);
  const unsigned fl = (flags & ~(FPMM_B200_ENGINE_DMMA | FPMM_B200_ENGINE_I8 | FPMM_B200_ENGINE_RNS)) |
                      (h->engine == kRns  ? FPMM_B200_ENGINE_RNS
                       : h->engine == kI8 ? FPMM_B200_ENGINE_I8
                                          : FPMM_B200_ENGINE_DMMA) |
                      (h->flags & FPMM_B200_ALLOW_COMPOSITE);
  validate_product(h->p, h->u, h->v, lambda, h->m, h->k, n, fl);
  DeviceCtx& c = ctx(h->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  if (tm) *tm = fpmm_b200_timing{};
  if (h->m == 0 || n == 0) return;
  if (h->k == 0) {
    zero_c(dC, ldc, h->m, n, s);
    if (!(fl & FPMM_B200_ASYNC)) CUDA_OK(cudaStreamSynchronize(s));
    return;
  }
  const Job j = make_job(h->m, h->k, n, h->p, h->u, h->v, h->engine, (h->flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
  Workspace& ws = c.ws_for(s);
  void* bpack = ws.bpack.get(j.bpack_bytes);
  int* err = nullptr;
  if (fl & (FPMM_B200_CHECK_INPUTS | FPMM_B200_CHECK_EXACTNESS)) {
    err = static_cast<int*>(c.err.get(sizeof(int)));
    CUDA_OK(cudaMemsetAsync(err, 0, sizeof(int), s));
  }
  if (tm) CUDA_OK(cudaEventRecord(c.ev[0], s));
  launch_pack_b(j, dB, ldb, bpack, (fl & FPMM_B200_CHECK_INPUTS) ? err : nullptr, s);
  if (tm) CUDA_OK(cudaEventRecord(c.ev[1], s));
  const int gl = launch_gemm(j, h->words.ptr, bpack, dC, ldc, h->m, s, ws, tm ? c.ev[5] : nullptr,
                             (fl & FPMM_B200_CHECK_EXACTNESS) ? err : nullptr);
  if (tm) CUDA_OK(cudaEventRecord(c.ev[2], s));
  if (err) check_err_flag(c, s);
  if (tm) {
    CUDA_OK(cudaEventSynchronize(c.ev[2]));
    tm->pack_ms = elapsed(c.ev[0], c.ev[1]);
    tm->gemm_ms = elapsed(c.ev[1], c.ev[5]);
    tm->recon_ms = elapsed(c.ev[5], c.ev[2]);
    tm->total_ms = elapsed(c.ev[0], c.ev[2]);
    tm->lambda_k = j.lambda_k;
    tm->engine = engine_flag(j), tm->words = engine_words(j);
    tm->launches = 1 + gl;
    tm->ngpus = 1;
  }
  if (!(fl & FPMM_B200_ASYNC)) CUDA_OK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------- host buffers
namespace {

struct CommAll {
  int n = 0;
  std::vector<ncclComm_t> comms;
  void ensure(int g) {
    if (n == g) return;
    for (auto cm : comms) nccl().CommDestroy(cm);
    comms.assign(g, nullptr);
    std::vector<int> devs(g);
    for (int i = 0; i < g; ++i) devs[i] = i;
    NCCL_OK(nccl().CommInitAll(comms.data(), g, devs.data()));
    n = g;
  }
  void release() {
    for (auto cm : comms) nccl().CommDestroy(cm);
    comms.clear();
    n = 0;
  }
} g_all;

// rows per partition: multiples of the GEMM's BM so every rank packs whole tiles
i64 part_rows(i64 m, int parts, int bm) {
  const i64 tiles = (m + bm - 1) / bm;
  return ((tiles + parts - 1) / parts) * bm;
}

}  // namespace

void product_host(const ProductArgs& a, int ngpus, fpmm_b200_timing* tm) {
  validate_product(a.p, a.u, a.v, a.lambda, a.m, a.k, a.n, a.flags);
  if (tm) *tm = fpmm_b200_timing{};
  if (ngpus < 1) throw Failure(FPMM_B200_EERROR, "ngpus must be >= 1");
  const int avail = device_count();
  if (ngpus > avail)
    throw Failure(FPMM_B200_EERROR, "requested " + std::to_string(ngpus) + " GPUs, " + std::to_string(avail) + " visible");
  std::lock_guard<std::recursive_mutex> all_lk(g_all_mu);
  std::vector<std::unique_ptr<DevLock>> dev_lks;
  for (int g = 0; g < ngpus; ++g) dev_lks.push_back(std::make_unique<DevLock>(g));
  if (a.m == 0 || a.n == 0) return;
  if (a.k == 0) {
    for (i64 r = 0; r < a.m; ++r) std::memset(a.C + r * a.ldc, 0, sizeof(double) * a.n);
    return;
  }
  const Job j = make_job(a.m, a.k, a.n, a.p, a.u, a.v, resolve_engine(a.flags),
                     (a.flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
  const unsigned chk = a.flags & (FPMM_B200_CHECK_INPUTS | FPMM_B200_CHECK_EXACTNESS);

  // FPMM_B200_INPROC_NCCL=1 runs the multi-device branch (communicators from
  // ncclCommInitAll, B broadcast, per-device C rows) at ngpus = 1 too: the
  // only way to execute it on a one-GPU box (tests/test_dist_gpu.py)
  const char* force_env = std::getenv("FPMM_B200_INPROC_NCCL");
  const bool force_nccl = force_env && std::atoi(force_env) != 0;
  if (ngpus == 1 && !force_nccl) {
    // Three-stream pipeline over row chunks of A / C: H2D of chunk i+1 and
    // D2H of chunk i-1 overlap the fused kernel on chunk i (PCIe is full
    // duplex); B goes first since every chunk needs its words.
    DeviceCtx& c = ctx(0);
    cudaStream_t s = c.stream, si = c.s_in, so = c.s_out;
    double* dA = static_cast<double*>(c.a.get(sizeof(double) * a.m * a.k));
    double* dB = static_cast<double*>(c.b.get(sizeof(double) * a.k * a.n));
    double* dC = static_cast<double*>(c.c.get(sizeof(double) * a.m * a.n));
    uint8_t* apack = static_cast<uint8_t*>(c.ws0.apack.get(j.apack_bytes));
    void* bpack = c.ws0.bpack.get(j.bpack_bytes);
    const size_t per_rb = j.per_rb_bytes;
    // ~8 chunks of whole GEMM row tiles once the operands are large enough to matter
    const i64 bytes = 8 * (a.m * a.k + a.m * a.n);
    const int want = bytes >= (i64{64} << 20) ? DeviceCtx::kChunks : 1;
    const i64 tiles = (a.m + j.BM - 1) / j.BM;
    // ...but each chunk keeps >= 2 waves of output tiles on the SMs (CTA pairs
    // for RNS): smaller chunks fall back to split-K, whose slices multiply the
    // RNS residue traffic (measured: 16 chunks of 512 rows ran the 8192^3
    // compute 2.8x slower than one launch)
    const i64 slots = j.engine == kRns ? 74 : 148;
    const i64 min_blocks = std::max<i64>(1, (2 * slots + j.NB - 1) / std::max(j.NB, 1));
    const i64 chunk_rows = std::max<i64>((tiles + want - 1) / want, min_blocks) * j.BM;
    const int nch = static_cast<int>((a.m + chunk_rows - 1) / chunk_rows);
    int* err = nullptr;
    if (chk) {
      err = static_cast<int*>(c.err.get(sizeof(int)));
      CUDA_OK(cudaMemsetAsync(err, 0, sizeof(int), s));
      CUDA_OK(cudaStreamSynchronize(s));
    }
    CUDA_OK(cudaEventRecord(c.ev[0], si));
    CUDA_OK(cudaMemcpy2DAsync(dB, a.n * 8, a.B, a.ldb * 8, a.n * 8, a.k, cudaMemcpyHostToDevice, si));
    CUDA_OK(cudaEventRecord(c.ev[1], si));
    for (int i = 0; i < nch; ++i) {
      const i64 r0 = i * chunk_rows, rn = std::min<i64>(a.m - r0, chunk_rows);
      CUDA_OK(cudaMemcpy2DAsync(dA + r0 * a.k, a.k * 8, a.A + r0 * a.lda, a.lda * 8, a.k * 8, rn,
                                cudaMemcpyHostToDevice, si));
      CUDA_OK(cudaEventRecord(c.ev_in[i], si));
    }
    CUDA_OK(cudaStreamWaitEvent(s, c.ev[1], 0));
    CUDA_OK(cudaEventRecord(c.ev[2], s));
    int* err_in = (a.flags & FPMM_B200_CHECK_INPUTS) ? err : nullptr;
    int* err_ex = (a.flags & FPMM_B200_CHECK_EXACTNESS) ? err : nullptr;
    launch_pack_b(j, dB, a.n, bpack, err_in, s);
    int nl = 1;
    for (int i = 0; i < nch; ++i) {
      const i64 r0 = i * chunk_rows, rn = std::min<i64>(a.m - r0, chunk_rows);
      uint8_t* ap = apack + static_cast<size_t>(r0 / j.BM) * per_rb;
      CUDA_OK(cudaStreamWaitEvent(s, c.ev_in[i], 0));
      launch_pack_a(j, dA + r0 * a.k, a.k, rn, ap, err_in, s);
      nl += 1 + launch_gemm(j, ap, bpack, dC + r0 * a.n, a.n, rn, s, c.ws0, nullptr, err_ex);
      CUDA_OK(cudaEventRecord(c.ev_out[i], s));
      CUDA_OK(cudaStreamWaitEvent(so, c.ev_out[i], 0));
      CUDA_OK(cudaMemcpy2DAsync(a.C + r0 * a.ldc, a.ldc * 8, dC + r0 * a.n, a.n * 8, a.n * 8, rn,
                                cudaMemcpyDeviceToHost, so));
    }
    CUDA_OK(cudaEventRecord(c.ev[3], so));
    CUDA_OK(cudaStreamSynchronize(so));
    if (err) check_err_flag(c, s);
    if (tm) {
      tm->h2d_ms = elapsed(c.ev[0], c.ev_in[nch - 1]);
      tm->gemm_ms = elapsed(c.ev[2], c.ev_out[nch - 1]);  // pack + fused GEMM span (overlaps copies)
      tm->d2h_ms = elapsed(c.ev_out[nch - 1], c.ev[3]);  // exposed tail of the D2H
      tm->total_ms = elapsed(c.ev[0], c.ev[3]);
      tm->lambda_k = j.lambda_k;
      tm->engine = engine_flag(j), tm->words = engine_words(j);
      tm->launches = nl;
      tm->ngpus = 1;
    }
    return;
  }

  // ngpus > 1 (or forced): contiguous row blocks of A / C per device; B words packed on
  // device 0 and broadcast over NCCL (NVLink); each device writes its C rows
  // straight back into the host matrix (row blocks are contiguous).
  g_all.ensure(ngpus);
  const bool raw = (a.flags & FPMM_B200_BCAST_RAW_B) || j.bpack_bytes > static_cast<size_t>(8) * a.k * a.n;
  const i64 rows_per = part_rows(a.m, ngpus, j.BM);
  std::vector<i64> r0(ngpus), rn(ngpus);
  for (int g = 0; g < ngpus; ++g) {
    r0[g] = std::min<i64>(a.m, g * rows_per);
    rn[g] = std::min<i64>(a.m, r0[g] + rows_per) - r0[g];
  }
  std::vector<DeviceCtx*> cs(ngpus);
  for (int g = 0; g < ngpus; ++g) cs[g] = &ctx(g);
  std::vector<double*> dA(ngpus), dC(ngpus);
  std::vector<void*> apack(ngpus), bpack(ngpus);
  std::vector<int*> errs(ngpus, nullptr), errs_in(ngpus, nullptr), errs_ex(ngpus, nullptr);
  double* dB0 = nullptr;
  for (int g = 0; g < ngpus; ++g) {
    DeviceCtx& c = *cs[g];
    CUDA_OK(cudaSetDevice(g));
    dA[g] = static_cast<double*>(c.a.get(sizeof(double) * std::max<i64>(rn[g], 1) * a.k));
    dC[g] = static_cast<double*>(c.c.get(sizeof(double) * std::max<i64>(rn[g], 1) * a.n));
    apack[g] = c.ws0.apack.get(j.apack_bytes);
    bpack[g] = c.ws0.bpack.get(j.bpack_bytes);
    if (chk) {
      errs[g] = static_cast<int*>(c.err.get(sizeof(int)));
      CUDA_OK(cudaMemsetAsync(errs[g], 0, sizeof(int), c.stream));
      if (a.flags & FPMM_B200_CHECK_INPUTS) errs_in[g] = errs[g];
      if (a.flags & FPMM_B200_CHECK_EXACTNESS) errs_ex[g] = errs[g];
    }
    CUDA_OK(cudaEventRecord(c.ev[0], c.stream));
    if (rn[g] > 0)
      CUDA_OK(cudaMemcpy2DAsync(dA[g], a.k * 8, a.A + r0[g] * a.lda, a.lda * 8, a.k * 8, rn[g],
                                cudaMemcpyHostToDevice, c.stream));
    if (g == 0) {
      dB0 = static_cast<double*>(c.b.get(sizeof(double) * a.k * a.n));
      CUDA_OK(cudaMemcpy2DAsync(dB0, a.n * 8, a.B, a.ldb * 8, a.n * 8, a.k, cudaMemcpyHostToDevice, c.stream));
    }
    CUDA_OK(cudaEventRecord(c.ev[1], c.stream));
    if (rn[g] > 0) launch_pack_a(j, dA[g], a.k, rn[g], apack[g], errs_in[g], c.stream);
    if (g == 0 && !raw) launch_pack_b(j, dB0, a.n, bpack[0], errs_in[0], c.stream);
    CUDA_OK(cudaEventRecord(c.ev[2], c.stream));
  }
  // B crosses NVLink once, as packed words or (fewer bytes / BCAST_RAW_B) as raw residues packed per device
  std::vector<double*> dBg(ngpus, dB0);
  if (raw)
    for (int g = 1; g < ngpus; ++g) {
      CUDA_OK(cudaSetDevice(g));
      dBg[g] = static_cast<double*>(cs[g]->b.get(sizeof(double) * a.k * a.n));
    }
  NCCL_OK(nccl().GroupStart());
  for (int g = 0; g < ngpus; ++g) {
    CUDA_OK(cudaSetDevice(g));
    if (raw)
      NCCL_OK(nccl().Broadcast(dB0, dBg[g], static_cast<size_t>(a.k * a.n), ncclDouble, 0, g_all.comms[g],
                               cs[g]->stream));
    else
      NCCL_OK(nccl().Broadcast(bpack[0], bpack[g], j.bpack_bytes, ncclUint8, 0, g_all.comms[g], cs[g]->stream));
  }
  NCCL_OK(nccl().GroupEnd());
  if (raw)
    for (int g = 0; g < ngpus; ++g) {
      CUDA_OK(cudaSetDevice(g));
      launch_pack_b(j, dBg[g], a.n, bpack[g], g == 0 ? errs_in[0] : nullptr, cs[g]->stream);
    }
  int nl = raw ? ngpus : 1;
  for (int g = 0; g < ngpus; ++g) {
    DeviceCtx& c = *cs[g];
    CUDA_OK(cudaSetDevice(g));
    CUDA_OK(cudaEventRecord(c.ev[3], c.stream));
    if (rn[g] > 0) nl += 1 + launch_gemm(j, apack[g], bpack[g], dC[g], a.n, rn[g], c.stream, c.ws0, nullptr, errs_ex[g]);
    CUDA_OK(cudaEventRecord(c.ev[4], c.stream));
    if (rn[g] > 0)
      CUDA_OK(cudaMemcpy2DAsync(a.C + r0[g] * a.ldc, a.ldc * 8, dC[g], a.n * 8, a.n * 8, rn[g],
                                cudaMemcpyDeviceToHost, c.stream));
    CUDA_OK(cudaEventRecord(c.ev[5], c.stream));
  }
  double h2d = 0, pack = 0, comm = 0, gemm = 0, d2h = 0, total = 0;
  for (int g = 0; g < ngpus; ++g) {
    DeviceCtx& c = *cs[g];
    CUDA_OK(cudaSetDevice(g));
    CUDA_OK(cudaStreamSynchronize(c.stream));
    if (errs[g]) check_err_flag(c, c.stream);
    h2d = std::max<double>(h2d, elapsed(c.ev[0], c.ev[1]));
    pack = std::max<double>(pack, elapsed(c.ev[1], c.ev[2]));
    comm = std::max<double>(comm, elapsed(c.ev[2], c.ev[3]));
    gemm = std::max<double>(gemm, elapsed(c.ev[3], c.ev[4]));
    d2h = std::max<double>(d2h, elapsed(c.ev[4], c.ev[5]));
    total = std::max<double>(total, elapsed(c.ev[0], c.ev[5]));
  }
  if (tm) {
    tm->h2d_ms = h2d, tm->pack_ms = pack, tm->comm_ms = comm, tm->gemm_ms = gemm, tm->d2h_ms = d2h;
    tm->total_ms = total;
    tm->lambda_k = j.lambda_k;
    tm->engine = engine_flag(j), tm->words = engine_words(j);
    tm->launches = nl;
    tm->ngpus = ngpus;
  }
}

void product_words_host(const double* Aw, i64 a_stride, i64 lda, u64 alpha, int u, const double* Bw,
                        i64 b_stride, i64 ldb, u64 beta, int v, double* C, i64 ldc, i64 m, i64 k,
                        i64 n, u64 p, u64 lambda, unsigned flags, fpmm_b200_timing* tm) {
  DevLock lk(0);
  validate_product(p, u, v, lambda, m, k, n, flags);
  if (m == 0 || n == 0) {
    if (tm) *tm = fpmm_b200_timing{};
    return;
  }
  // words -> residues on the device (sum_i alpha^i w_i mod p), then the product
  DeviceCtx& c = ctx(0);
  cudaStream_t s = c.stream;
  const size_t aw = static_cast<size_t>(u) * m * k, bw = static_cast<size_t>(v) * k * n;
  double* dW = static_cast<double*>(c.tmp.get(sizeof(double) * std::max<size_t>(aw + bw, 1)));
  double* dA = static_cast<double*>(c.a.get(sizeof(double) * std::max<i64>(m * k, 1)));
  double* dB = static_cast<double*>(c.b.get(sizeof(double) * std::max<i64>(k * n, 1)));
  double* dC = static_cast<double*>(c.c.get(sizeof(double) * m * n));
  for (int i = 0; i < u; ++i)
    CUDA_OK(cudaMemcpy2DAsync(dW + static_cast<size_t>(i) * m * k, k * 8, Aw + i * a_stride, lda * 8, k * 8, m,
                              cudaMemcpyHostToDevice, s));
  for (int i = 0; i < v; ++i)
    CUDA_OK(cudaMemcpy2DAsync(dW + aw + static_cast<size_t>(i) * k * n, n * 8, Bw + i * b_stride, ldb * 8, n * 8,
                              k, cudaMemcpyHostToDevice, s));
  if (m * k > 0)
    recompose_kernel<<<grid_for(m * k, 256), 256, 0, s>>>(dW, m * k, k, m, k, u, alpha % p, shoup(alpha % p, p), p, dA);
  if (k * n > 0)
    recompose_kernel<<<grid_for(k * n, 256), 256, 0, s>>>(dW + aw, k * n, n, k, n, v, beta % p, shoup(beta % p, p), p,
                                                         dB);
  CUDA_OK(cudaGetLastError());
  ProductArgs pa{dA, k, dB, n, dC, n, m, k, n, p, u, v, lambda, flags & ~FPMM_B200_CHECK_INPUTS};
  product_device(pa, 0, s, tm);
  CUDA_OK(cudaMemcpy2DAsync(C, ldc * 8, dC, n * 8, n * 8, m, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
}

void decompose_device(const double* dM, i64 ld, i64 rows, i64 cols, u64 p, int u, double* dwords,
                      i64 word_stride, u64* base, int device, void* stream) {
  DevLock lk(device);
  if (u < 1) throw Failure(FPMM_B200_EERROR, "decompose: word count must be positive");
  const u64 alpha = word_base(p, u);
  if (base) *base = alpha;
  DeviceCtx& c = ctx(device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  if (rows * cols == 0) return;
  const double af = static_cast<double>(alpha);
  decompose_ref_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(dM, ld, rows, cols, u, af, 1.0 / af, dwords,
                                                                  word_stride);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaStreamSynchronize(s));
}

void decompose_host(const double* M, i64 ld, i64 rows, i64 cols, u64 p, int u, double* words,
                    i64 word_stride, u64* base) {
  DevLock lk(0);
  if (u < 1) throw Failure(FPMM_B200_EERROR, "decompose: word count must be positive");
  DeviceCtx& c = ctx(0);
  const i64 e = rows * cols;
  if (e == 0) {
    if (base) *base = word_base(p, u);
    return;
  }
  double* dM = static_cast<double*>(c.a.get(sizeof(double) * e));
  double* dW = static_cast<double*>(c.tmp.get(sizeof(double) * e * u));
  CUDA_OK(cudaMemcpy2DAsync(dM, cols * 8, M, ld * 8, cols * 8, rows, cudaMemcpyHostToDevice, c.stream));
  decompose_device(dM, cols, rows, cols, p, u, dW, e, base, 0, c.stream);
  for (int i = 0; i < u; ++i)
    CUDA_OK(cudaMemcpyAsync(words + i * word_stride, dW + static_cast<size_t>(i) * e, sizeof(double) * e,
                            cudaMemcpyDeviceToHost, c.stream));
  CUDA_OK(cudaStreamSynchronize(c.stream));
}

void accumulate_device(double* dC, i64 ldc, const double* dA, i64 lda, const double* dB, i64 ldb,
                       i64 m, i64 w, i64 n, int device, void* stream) {
  DevLock lk(device);
  if (m < 0 || w < 0 || n < 0) throw Failure(FPMM_B200_EERROR, "accumulate: negative dimensions");
  DeviceCtx& c = ctx(device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  if (m == 0 || n == 0 || w == 0) return;
  dim3 grid(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((m + 63) / 64));
  accumulate_kernel<<<grid, 128, 0, s>>>(dC, ldc, dA, lda, dB, ldb, m, w, n);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaStreamSynchronize(s));
}

void accumulate_host(double* C, i64 ldc, const double* A, i64 lda, const double* B, i64 ldb, i64 m,
                     i64 w, i64 n) {
  DevLock lk(0);
  if (m <= 0 || n <= 0 || w <= 0) return;
  DeviceCtx& c = ctx(0);
  cudaStream_t s = c.stream;
  double* dA = static_cast<double*>(c.a.get(sizeof(double) * m * w));
  double* dB = static_cast<double*>(c.b.get(sizeof(double) * w * n));
  double* dC = static_cast<double*>(c.c.get(sizeof(double) * m * n));
  CUDA_OK(cudaMemcpy2DAsync(dA, w * 8, A, lda * 8, w * 8, m, cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpy2DAsync(dB, n * 8, B, ldb * 8, n * 8, w, cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpy2DAsync(dC, n * 8, C, ldc * 8, n * 8, m, cudaMemcpyHostToDevice, s));
  accumulate_device(dC, n, dA, w, dB, n, m, w, n, 0, s);
  CUDA_OK(cudaMemcpy2DAsync(C, ldc * 8, dC, n * 8, n * 8, m, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
}

// Alg 2.3 (block_product.hpp:62-73): C <- C + A B mod p, on the device.
// The reference's panel loop is exact when lambda max(A) max(B) + p - 1 <=
// 2^t, a contract checked only in FPMM_CONTRACTS builds (check_block_inputs,
// block_product.hpp:40-54), and its operands need not be residues (e.g. the
// words of mw_product_words, bounded by alpha).  Here A and B are reduced mod
// p on the device (exact for integers below 2^53), the exact residue product
// T runs on the library's engine, and C <- C + T mod p is a device kernel: the
// reference's value wherever the reference is exact, for any lambda >= 1.
// CHECK_INPUTS is the contract: entries are non-negative integers below 2^53,
// C is reduced, and the lambda bound holds on the actual maxima (ContractError).
void block_gemm_mod_host(double* C, i64 ldc, const double* A, i64 lda, const double* B, i64 ldb,
                         i64 m, i64 k, i64 n, u64 lambda, u64 p, unsigned flags) {
  DevLock lk(0);
  context_check(p, true);
  if (m < 0 || k < 0 || n < 0) throw Failure(FPMM_B200_EERROR, "block_gemm_mod: dimension mismatch");
  if (lambda < 1) throw Failure(FPMM_B200_EINFEASIBLE, "block size infeasible");
  if (m == 0 || n == 0 || k == 0) return;  // no panel: C unchanged, as the reference's loop
  DeviceCtx& c = ctx(0);
  cudaStream_t s = c.stream;
  double* dA = static_cast<double*>(c.a.get(sizeof(double) * m * k));
  double* dB = static_cast<double*>(c.b.get(sizeof(double) * k * n));
  double* dC = static_cast<double*>(c.c.get(sizeof(double) * m * n));
  double* dT = static_cast<double*>(c.tmp.get(sizeof(double) * m * n));
  CUDA_OK(cudaMemcpy2DAsync(dA, k * 8, A, lda * 8, k * 8, m, cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpy2DAsync(dB, n * 8, B, ldb * 8, n * 8, k, cudaMemcpyHostToDevice, s));
  CUDA_OK(cudaMemcpy2DAsync(dC, n * 8, C, ldc * 8, n * 8, m, cudaMemcpyHostToDevice, s));
  if (flags & FPMM_B200_CHECK_INPUTS) {
    auto* scan = static_cast<unsigned long long*>(c.ver.get(4 * sizeof(unsigned long long)));
    int* err = reinterpret_cast<int*>(scan + 3);
    CUDA_OK(cudaMemsetAsync(scan, 0, 4 * sizeof(unsigned long long), s));
    max_scan_kernel<<<grid_for(m * k, 256), 256, 0, s>>>(dA, k, m, k, scan + 0, err);
    max_scan_kernel<<<grid_for(k * n, 256), 256, 0, s>>>(dB, n, k, n, scan + 1, err);
    max_scan_kernel<<<grid_for(m * n, 256), 256, 0, s>>>(dC, n, m, n, scan + 2, err);
    CUDA_OK(cudaGetLastError());
    unsigned long long h[4];
    CUDA_OK(cudaMemcpyAsync(h, scan, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    if (static_cast<int>(h[3] & 0xFFFFFFFFu))
      throw Failure(FPMM_B200_ECONTRACT, "block_gemm_mod: entries must be non-negative integers below 2^53");
    if (h[2] >= p) throw Failure(FPMM_B200_ECONTRACT, "block_gemm_mod: C must be reduced mod p");
    const u64 lam = std::min<u64>(lambda, static_cast<u64>(k));
    const u128 peak = static_cast<u128>(lam) * h[0] * h[1] + (p - 1);
    if (peak > (u128{1} << kT))
      throw Failure(FPMM_B200_ECONTRACT, "block_gemm_mod: lambda max(A) max(B) + p - 1 exceeds 2^t");
  }
  const double pf = static_cast<double>(p);
  reduce_mod_kernel<<<grid_for(m * k, 256), 256, 0, s>>>(dA, k, m, k, pf);
  reduce_mod_kernel<<<grid_for(k * n, 256), 256, 0, s>>>(dB, n, k, n, pf);
  reduce_mod_kernel<<<grid_for(m * n, 256), 256, 0, s>>>(dC, n, m, n, pf);
  CUDA_OK(cudaGetLastError());
  // T = A B mod p: the (1,1) residue product on the selected (or default) engine
  const Job j = make_job(m, k, n, p, 1, 1, resolve_engine(flags), (flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
  Workspace& ws = c.ws_for(s);
  void* apack = ws.apack.get(j.apack_bytes);
  void* bpack = ws.bpack.get(j.bpack_bytes);
  launch_pack_a(j, dA, k, m, apack, nullptr, s);
  launch_pack_b(j, dB, n, bpack, nullptr, s);
  launch_gemm(j, apack, bpack, dT, n, m, s, ws);
  add_mod_kernel<<<grid_for(m * n, 256), 256, 0, s>>>(dC, n, dT, n, m, n, pf);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpy2DAsync(C, ldc * 8, dC, n * 8, n * 8, m, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
}

void random_residues_device(double* dM, i64 ld, i64 rows, i64 cols, i64 row0, u64 p, u64 seed, int device,
                            void* stream) {
  DevLock lk(device);
  if (p < 2) throw Failure(FPMM_B200_EERROR, "random_residues: p must exceed 1");
  DeviceCtx& c = ctx(device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  if (rows * cols == 0) return;
  const u64 kMax = ~u64{0};
  random_residues_kernel<<<grid_for(rows * cols, 256), 256, 0, s>>>(dM, ld, rows, cols, row0, p, kMax - kMax % p, seed);
  CUDA_OK(cudaGetLastError());
  if (!stream) CUDA_OK(cudaStreamSynchronize(s));
}

// Exact on-device check of C = A B mod p (verify.cuh): range of C, Freivalds
// trials A (B s) == C s mod p, and sampled exact entries.  counts: [0] entries
// of C outside [0, p), [1] Freivalds rows that differ (summed over trials),
// [2] wrong sampled entries, [3..4] (i, j) of the first wrong sample (or -1).
void verify_device(const double* dA, i64 lda, const double* dB, i64 ldb, const double* dC, i64 ldc, i64 m, i64 k,
                   i64 n, u64 p, u64 seed, int trials, int samples, int device, void* stream, i64* counts) {
  DevLock lk(device);
  if (m < 0 || k < 0 || n < 0) throw Failure(FPMM_B200_EERROR, "verify: dimensions must be nonnegative");
  if (p < 2 || p >= (u64{1} << 52)) throw Failure(FPMM_B200_EERROR, "verify: modulus must be in [2, 2^52)");
  if (trials < 0 || samples < 0) throw Failure(FPMM_B200_EERROR, "verify: negative trial / sample count");
  for (int i = 0; i < 5; ++i) counts[i] = i < 3 ? 0 : -1;
  if (m == 0 || n == 0) return;
  DeviceCtx& c = ctx(device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  const size_t words = static_cast<size_t>(n) + static_cast<size_t>(k) + 2 * static_cast<size_t>(m) + 8;
  u64* base = static_cast<u64*>(c.ver.get(sizeof(u64) * words));
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(base);
  long long* first = reinterpret_cast<long long*>(base + 3);
  u64* sv = base + 8;
  u64* yv = sv + n;
  u64* zv = yv + k;
  u64* wv = zv + m;
  CUDA_OK(cudaMemsetAsync(cnt, 0, 3 * sizeof(u64), s));
  CUDA_OK(cudaMemsetAsync(first, 0xFF, 2 * sizeof(u64), s));
  verify::range_kernel<<<grid_for(m * n, 256), 256, 0, s>>>(dC, ldc, m, n, p, cnt);
  const u64 kMax = ~u64{0};
  auto rows_grid = [](i64 rows) { return grid_for(rows * 32, 256); };
  for (int t = 0; t < trials; ++t) {
    const u64 ts = seed * 0x9E3779B97F4A7C15ull + static_cast<u64>(t) * 0xD1B54A32D192ED03ull + 1;
    verify::rand_vec_kernel<<<grid_for(n, 256), 256, 0, s>>>(sv, n, p, kMax - kMax % p, ts);
    verify::matvec_mod_kernel<<<rows_grid(k), 256, 0, s>>>(dB, ldb, k, n, sv, p, yv);   // y = B s
    verify::matvec_mod_kernel<<<rows_grid(m), 256, 0, s>>>(dA, lda, m, k, yv, p, zv);   // z = A y
    verify::matvec_mod_kernel<<<rows_grid(m), 256, 0, s>>>(dC, ldc, m, n, sv, p, wv);   // w = C s
    verify::compare_kernel<<<grid_for(m, 256), 256, 0, s>>>(zv, wv, m, cnt);
  }
  if (samples > 0)
    verify::sample_kernel<<<std::max(1, std::min(samples / 8 + 1, 148 * 8)), 256, 0, s>>>(
        dA, lda, dB, ldb, dC, ldc, m, k, n, p, seed, samples, cnt, first);
  CUDA_OK(cudaGetLastError());
  u64 h[5];
  CUDA_OK(cudaMemcpyAsync(h, base, sizeof(h), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  for (int i = 0; i < 5; ++i) counts[i] = static_cast<i64>(h[i]);
}

double fp64_peak_tflops(int device, int iters) {
  DevLock lk(device);
  DeviceCtx& c = ctx(device);
  int sms = 0;
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* out = static_cast<double*>(c.err.get(4096));
  const int blocks = sms * 4;
  dmma_peak_kernel<<<blocks, 256, 0, c.stream>>>(iters, out);  // warm-up
  CUDA_OK(cudaEventRecord(c.ev[0], c.stream));
  dmma_peak_kernel<<<blocks, 256, 0, c.stream>>>(iters, out);
  CUDA_OK(cudaEventRecord(c.ev[1], c.stream));
  CUDA_OK(cudaEventSynchronize(c.ev[1]));
  const double ms = elapsed(c.ev[0], c.ev[1]);
  const double flops = 2.0 * 256.0 * 8.0 * iters * blocks * 8.0;  // 8 warps per block
  return flops / (ms * 1e-3) / 1e12;
}

double i8_probe_tops(int device, int iters, int mode) {
  DevLock lk(device);
  DeviceCtx& c = ctx(device);
  int sms = 0;
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int* out = static_cast<int*>(c.err.get(4096));
  const int grid = mode == 1 ? (sms / 2) * 2 : sms;
  auto launch = [&](int it) {
    if (mode == 1) i8::i8_peak2_kernel<<<grid, 64, 0, c.stream>>>(it, out);
    else i8::i8_peak_kernel<<<grid, 64, 0, c.stream>>>(it, out);
  };
  launch(iters / 8);
  CUDA_OK(cudaEventRecord(c.ev[0], c.stream));
  launch(iters);
  CUDA_OK(cudaEventRecord(c.ev[1], c.stream));
  CUDA_OK(cudaEventSynchronize(c.ev[1]));
  CUDA_OK(cudaGetLastError());
  const double ms = elapsed(c.ev[0], c.ev[1]);
  // per MMA: 1-CTA M128 N256 K32 on every SM; 2-CTA M256 N256 K32 per pair
  const double ops = mode == 1 ? 2.0 * 256 * 256 * 32 * iters * (grid / 2) : 2.0 * i8::kBM * 256.0 * 32.0 * iters * grid;
  return ops / (ms * 1e-3) / 1e12;
}

double i8_peak_tops(int device, int iters) {
  DevLock lk(device);
  DeviceCtx& c = ctx(device);
  int sms = 0;
  CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  int* out = static_cast<int*>(c.err.get(4096));
  i8::i8_peak_kernel<<<sms, 64, 0, c.stream>>>(iters / 4, out);  // warm-up (clocks ramp)
  CUDA_OK(cudaEventRecord(c.ev[0], c.stream));
  i8::i8_peak_kernel<<<sms, 64, 0, c.stream>>>(iters, out);
  CUDA_OK(cudaEventRecord(c.ev[1], c.stream));
  CUDA_OK(cudaEventSynchronize(c.ev[1]));
  CUDA_OK(cudaGetLastError());
  const double ms = elapsed(c.ev[0], c.ev[1]);
  const double ops = 2.0 * i8::kBM * 256.0 * 32.0 * iters * sms;
  return ops / (ms * 1e-3) / 1e12;
}

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// ------------------------------------------------- multi-process partitioner
namespace {
struct DistState {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = -1, device = -1;
} g_dist;
}  // namespace

int nccl_id_size() { return static_cast<int>(sizeof(ncclUniqueId)); }

void nccl_unique_id(void* id) {
  ncclUniqueId uid;
  NCCL_OK(nccl().GetUniqueId(&uid));
  std::memcpy(id, &uid, sizeof(uid));
}

void dist_init(const void* id, int nranks, int rank, int device) {
  std::lock_guard<std::recursive_mutex> dlk(g_dist_mu);
  DevLock lk(device);
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Failure(FPMM_B200_EERROR, "dist_init: bad rank/size");
  if (g_dist.comm) nccl().CommDestroy(g_dist.comm), g_dist.comm = nullptr;
  ctx(device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  NCCL_OK(nccl().CommInitRank(&g_dist.comm, nranks, uid, rank));
  g_dist.nranks = nranks;
  g_dist.rank = rank;
  g_dist.device = device;
}

void dist_finalize() {
  std::lock_guard<std::recursive_mutex> dlk(g_dist_mu);
  if (g_dist.comm) nccl().CommDestroy(g_dist.comm);
  g_dist = DistState{};
}

void dist_rows(i64 m, int nranks, int rank, int u, int v, i64* row0, i64* rows) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw Failure(FPMM_B200_EERROR, "dist_rows: bad rank/size");
  // 256 = a multiple of every engine's row tile (DMMA BM in {32,64,128},
  // int8 BM = 128, RNS pair tile 256), so each rank packs whole tiles whatever the engine
  dispatch(u, v, [&]<int U, int V, int MT, int NT>() {});  // rejects unsupported (u,v)
  const i64 per = part_rows(m, nranks, 256);
  const i64 r0 = std::min<i64>(m, rank * per);
  *row0 = r0;
  *rows = std::min<i64>(m, r0 + per) - r0;
}

// Row chunks of one rank's block for the overlapped gather: chunk c's C rows
// go to root (NCCL send/recv on a second stream) while chunk c+1 computes.
// Whole row tiles, each chunk >= 2 waves of the engine's output tiles (CTA
// pairs for RNS; smaller launches fall back to split-K), at most 4 chunks.
// A pure function of (job, rows): root derives every rank's chunks itself.
constexpr int kGatherChunks = FPMM_B200_DIST_MAX_CHUNKS;
std::vector<std::pair<i64, i64>> gather_chunks(const Job& j, i64 rows) {
  std::vector<std::pair<i64, i64>> out;
  if (rows <= 0) return out;
  const i64 slots = j.engine == kRns ? 74 : 148;
  const i64 min_tiles = std::max<i64>(1, (2 * slots + j.NB - 1) / std::max(j.NB, 1));
  const i64 tiles = (rows + j.BM - 1) / j.BM;
  i64 cap = kGatherChunks;
  if (const char* e = std::getenv("FPMM_B200_DIST_CHUNKS")) cap = std::max(1, std::min(kGatherChunks, std::atoi(e)));
  const i64 nch = std::max<i64>(1, std::min<i64>(cap, tiles / min_tiles));
  const i64 per = (tiles + nch - 1) / nch * j.BM;
  for (i64 r = 0; r < rows; r += per) out.emplace_back(r, std::min<i64>(per, rows - r));
  return out;
}

void dist_chunks(i64 m, i64 k, i64 n, u64 p, int u, int v, unsigned flags, i64 rows, int* count, i64* starts,
                 i64* lens) {
  context_check(p, (flags & FPMM_B200_ALLOW_COMPOSITE) != 0);
  const Job j = make_job(std::max<i64>(m, 1), std::max<i64>(k, 1), std::max<i64>(n, 1), p, u, v, resolve_engine(flags),
                         (flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
  const auto ch = gather_chunks(j, rows);
  *count = static_cast<int>(ch.size());
  for (size_t i = 0; i < ch.size(); ++i) starts[i] = ch[i].first, lens[i] = ch[i].second;
}

void dist_product_device(const double* dA_rows, i64 lda, const double* dB, i64 ldb, double* dC_rows,
                         i64 ldc, double* dC_full, i64 ldc_full, i64 m, i64 k, i64 n, u64 p, int u,
                         int v, u64 lambda, int root, void* stream, unsigned flags,
                         fpmm_b200_timing* tm) {
  std::lock_guard<std::recursive_mutex> dlk(g_dist_mu);
  if (!g_dist.comm) throw Failure(FPMM_B200_EERROR, "dist_mw_product: call fpmm_b200_dist_init first");
  DevLock lk(g_dist.device);
  if (tm) *tm = fpmm_b200_timing{};
  DeviceCtx& c = ctx(g_dist.device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c.stream;
  cudaStream_t so = c.s_out;  // every NCCL call of the partitioner, in one order on every rank
  const bool is_root = g_dist.rank == root;
  // Argument checks, agreed on by every rank before any data moves: one
  // 3-int all-reduce (max) of [status, root gathers, this rank's C rows are
  // not dense].  A bad argument on any rank -- root's gather target included
  // -- fails the call on every rank, so no rank is left waiting in a
  // collective, and every rank gathers iff root passed dC_full (the other
  // ranks' dC_full is ignored).
  int code = 0;
  std::string why;
  Job j{};
  i64 r0 = 0, rn = 0;
  try {
    validate_product(p, u, v, lambda, m, k, n, flags);
    if (root < 0 || root >= g_dist.nranks) throw Failure(FPMM_B200_EERROR, "dist_mw_product: bad root");
    if (k == 0 && m > 0 && n > 0) throw Failure(FPMM_B200_EERROR, "dist_mw_product: k == 0 unsupported");
    if (m > 0 && n > 0) {
      j = make_job(m, k, n, p, u, v, resolve_engine(flags), (flags & FPMM_B200_DMMA_EXACT_WORDS) != 0);
      dist_rows(m, g_dist.nranks, g_dist.rank, u, v, &r0, &rn);
      if (rn > 0 && (ldc < n || lda < k)) throw Failure(FPMM_B200_EERROR, "dist_mw_product: leading dimension too small");
      if (is_root && (!dB || ldb < n)) throw Failure(FPMM_B200_EERROR, "dist_mw_product: root needs B (ldb >= n)");
      if (is_root && dC_full && ldc_full != n)
        throw Failure(FPMM_B200_EERROR, "dist_mw_product: gather needs a dense target (ldc_full == n)");
    }
  } catch (const Failure& e) {
    code = e.code;
    why = e.what();
  }
  int agree[3] = {code, is_root && dC_full ? 1 : 0, rn > 0 && ldc != n ? 1 : 0};
  {
    int* d = static_cast<int*>(c.agree.get(sizeof(agree)));
    CUDA_OK(cudaMemcpyAsync(d, agree, sizeof(agree), cudaMemcpyHostToDevice, so));
    NCCL_OK(nccl().AllReduce(d, d, 3, ncclInt32, ncclMax, g_dist.comm, so));
    CUDA_OK(cudaMemcpyAsync(agree, d, sizeof(agree), cudaMemcpyDeviceToHost, so));
    CUDA_OK(cudaStreamSynchronize(so));
  }
  const bool gather = agree[1] != 0;
  if (!code && gather && agree[2]) {
    code = FPMM_B200_EERROR;
    why = "dist_mw_product: gather needs dense row blocks (ldc == n) on every rank";
  }
  if (code) throw Failure(code, why);
  if (agree[0] || (gather && agree[2]))
    throw Failure(agree[0] ? agree[0] : FPMM_B200_EERROR,
                  "dist_mw_product: another rank rejected this call's arguments (status " +
                      std::to_string(agree[0] ? agree[0] : FPMM_B200_EERROR) + ")");
  if (m == 0 || n == 0) return;
  Workspace& ws = c.ws_for(s);
  void* apack = ws.apack.get(j.apack_bytes);
  void* bpack = ws.bpack.get(j.bpack_bytes);
  int* errbuf = nullptr;
  if (flags & (FPMM_B200_CHECK_INPUTS | FPMM_B200_CHECK_EXACTNESS)) {
    errbuf = static_cast<int*>(c.err.get(sizeof(int)));
    CUDA_OK(cudaMemsetAsync(errbuf, 0, sizeof(int), s));
  }
  int* err = (flags & FPMM_B200_CHECK_INPUTS) ? errbuf : nullptr;
  int* err_ex = (flags & FPMM_B200_CHECK_EXACTNESS) ? errbuf : nullptr;
  CUDA_OK(cudaEventRecord(c.ev[0], s));
  // B crosses NVLink once: as packed words, or as raw residues (8 B per
  // element) packed by every rank when that is fewer bytes (the RNS engine
  // above 8 moduli, the FP64 engine at v >= 2) or when BCAST_RAW_B asks
  const bool raw = (flags & FPMM_B200_BCAST_RAW_B) || j.bpack_bytes > static_cast<size_t>(8) * k * n;
  // RNS with a large raw B: the broadcast runs in k-chunks on stream s_out and
  // each chunk's residues are packed on s as soon as it lands, so the per-rank
  // pack of B (about 9 ms at 32768^2) hides under the broadcast.
  const int bchunks = (raw && j.engine == kRns && static_cast<size_t>(8) * k * n >= (size_t{256} << 20))
                          ? std::min(4, j.KB) : 1;
  // Every NCCL call of the partitioner goes to the device's s_out stream, in
  // the same program order on every rank, so products issued on different
  // caller streams never run collectives of the one communicator concurrently.
  if (raw && bchunks > 1) {
    double* dBd = static_cast<double*>(ws.rawb.get(sizeof(double) * k * n));
    if (g_dist.rank == root)
      CUDA_OK(cudaMemcpy2DAsync(dBd, n * 8, dB, ldb * 8, n * 8, k, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaEventRecord(c.ev[6], s));  // B staged; the last call's reads of dBd are done
    CUDA_OK(cudaStreamWaitEvent(so, c.ev[6], 0));
    if (rn > 0) launch_pack_a(j, dA_rows, lda, rn, apack, err, s);
    CUDA_OK(cudaEventRecord(c.ev[1], s));
    const int per = (j.KB + bchunks - 1) / bchunks;
    for (int bc = 0; bc < bchunks; ++bc) {
      const int kb0 = bc * per, nkb = std::min(j.KB, kb0 + per) - kb0;
      if (nkb <= 0) break;
      const i64 k0 = static_cast<i64>(kb0) * rns::kBK, k1 = std::min<i64>(k, static_cast<i64>(kb0 + nkb) * rns::kBK);
      NCCL_OK(nccl().Broadcast(dBd + k0 * n, dBd + k0 * n, static_cast<size_t>((k1 - k0) * n), ncclDouble, root,
                               g_dist.comm, so));
      CUDA_OK(cudaEventRecord(c.ev_in[bc], so));
      CUDA_OK(cudaStreamWaitEvent(s, c.ev_in[bc], 0));
      launch_pack_b_rns(j, dBd, n, bpack, g_dist.rank == root ? err : nullptr, s, kb0, nkb);
    }
  } else if (raw) {
    double* dBd = static_cast<double*>(ws.rawb.get(sizeof(double) * k * n));
    if (g_dist.rank == root)
      CUDA_OK(cudaMemcpy2DAsync(dBd, n * 8, dB, ldb * 8, n * 8, k, cudaMemcpyDeviceToDevice, s));
    if (rn > 0) launch_pack_a(j, dA_rows, lda, rn, apack, err, s);
    CUDA_OK(cudaEventRecord(c.ev[1], s));
    CUDA_OK(cudaStreamWaitEvent(so, c.ev[1], 0));
    NCCL_OK(nccl().Broadcast(dBd, dBd, static_cast<size_t>(k * n), ncclDouble, root, g_dist.comm, so));
    CUDA_OK(cudaEventRecord(c.ev[6], so));
    CUDA_OK(cudaStreamWaitEvent(s, c.ev[6], 0));
    launch_pack_b(j, dBd, n, bpack, g_dist.rank == root ? err : nullptr, s);
  } else {
    if (g_dist.rank == root) launch_pack_b(j, dB, ldb, bpack, err, s);
    if (rn > 0) launch_pack_a(j, dA_rows, lda, rn, apack, err, s);
    CUDA_OK(cudaEventRecord(c.ev[1], s));
    CUDA_OK(cudaStreamWaitEvent(so, c.ev[1], 0));
    NCCL_OK(nccl().Broadcast(bpack, bpack, j.bpack_bytes, ncclUint8, root, g_dist.comm, so));
    CUDA_OK(cudaEventRecord(c.ev[6], so));
    CUDA_OK(cudaStreamWaitEvent(s, c.ev[6], 0));
  }
  CUDA_OK(cudaEventRecord(c.ev[2], s));
  // the product in row chunks; with a gather, chunk c's rows travel to root
  // on stream s_out (NCCL P2P) while chunk c+1 computes on s.  Every NCCL call
  // of this product is issued on s_out in the same order on every rank: the
  // broadcast (all of it, or its k-chunks), then one group per chunk index.
  const auto mine = gather ? gather_chunks(j, rn) : std::vector<std::pair<i64, i64>>{{0, rn}};
  int gl = 0;
  for (size_t ci = 0; ci < mine.size(); ++ci) {
    const i64 o = mine[ci].first, l = mine[ci].second;
    if (l <= 0) continue;
    gl += launch_gemm(j, static_cast<uint8_t*>(apack) + static_cast<size_t>(o / j.BM) * j.per_rb_bytes, bpack,
                      dC_rows + o * ldc, ldc, l, s, ws, nullptr, err_ex);
    if (gather) CUDA_OK(cudaEventRecord(c.ev_out[ci], s));
  }
  CUDA_OK(cudaEventRecord(c.ev[3], s));
  int launches = (rn > 0 ? 1 + gl : 0) + (g_dist.rank == root || raw ? bchunks : 0);
  if (gather) {
    // gather row blocks to root (grouped point-to-point; NCCL has no gather)
    CUDA_OK(cudaStreamWaitEvent(so, c.ev[2], 0));  // root's copies / recvs follow this call's earlier work
    std::vector<std::vector<std::pair<i64, i64>>> theirs(g_dist.nranks);
    std::vector<i64> q0s(g_dist.nranks, 0);
    size_t rounds = mine.size();
    if (g_dist.rank == root)
      for (int r = 0; r < g_dist.nranks; ++r) {
        i64 qn = 0;
        dist_rows(m, g_dist.nranks, r, u, v, &q0s[r], &qn);
        theirs[r] = gather_chunks(j, qn);
        rounds = std::max(rounds, theirs[r].size());
      }
    for (size_t ci = 0; ci < rounds; ++ci) {
      if (ci < mine.size()) CUDA_OK(cudaStreamWaitEvent(so, c.ev_out[ci], 0));
      NCCL_OK(nccl().GroupStart());
      if (g_dist.rank == root) {
        for (int r = 0; r < g_dist.nranks; ++r) {
          if (ci >= theirs[r].size()) continue;
          const i64 row = q0s[r] + theirs[r][ci].first, len = theirs[r][ci].second;
          if (r == root) {
            if (dC_full + q0s[r] * ldc_full != dC_rows)
              CUDA_OK(cudaMemcpyAsync(dC_full + row * ldc_full, dC_rows + theirs[r][ci].first * ldc,
                                      sizeof(double) * len * n, cudaMemcpyDeviceToDevice, so));
          } else {
            NCCL_OK(nccl().Recv(dC_full + row * ldc_full, static_cast<size_t>(len * n), ncclDouble, r, g_dist.comm,
                                so));
          }
        }
      } else if (ci < mine.size()) {
        NCCL_OK(nccl().Send(dC_rows + mine[ci].first * ldc, static_cast<size_t>(mine[ci].second * n), ncclDouble, root,
                            g_dist.comm, so));
      }
      NCCL_OK(nccl().GroupEnd());
    }
    CUDA_OK(cudaEventRecord(c.ev[5], so));
    CUDA_OK(cudaStreamWaitEvent(s, c.ev[5], 0));  // the call completes on its own stream
  }
  CUDA_OK(cudaEventRecord(c.ev[4], s));
  if (errbuf) check_err_flag(c, s);
  if (!(flags & FPMM_B200_ASYNC) || tm) CUDA_OK(cudaStreamSynchronize(s));
  if (tm) {
    tm->pack_ms = elapsed(c.ev[0], c.ev[1]);
    tm->comm_ms = elapsed(c.ev[1], c.ev[2]) + elapsed(c.ev[3], c.ev[4]);
    tm->gemm_ms = elapsed(c.ev[2], c.ev[3]);
    tm->total_ms = elapsed(c.ev[0], c.ev[4]);
    tm->lambda_k = j.lambda_k;
    tm->engine = engine_flag(j), tm->words = engine_words(j);
    tm->launches = launches;
    tm->ngpus = g_dist.nranks;
  }
}

void finalize_all() {
  std::lock_guard<std::recursive_mutex> dlk(g_dist_mu), alk(g_all_mu);
  if (g_dist.comm) nccl().CommDestroy(g_dist.comm);
  g_dist = DistState{};
  g_all.release();
  // no call may be in flight on any device (the contexts and their locks go away)
  std::lock_guard<std::mutex> tl(g_ctx_mu);
  for (auto& c : g_ctx)
    if (c) {
      std::lock_guard<std::recursive_mutex> l(c->mu);
      c->release();
    }
  g_ctx.clear();
}

}  // namespace fpmm_b200
