// fpmm_b200/fpmm.hpp -- C++ drop-in for the reference library's hot path.
//
// Mirrors namespace fpmm of /root/reference/proj/include/fpmm (same names,
// argument order, matrix layout, prime and (u,v) rule, exception types) for
// binary64, implemented over the C-ABI in fpmm_b200.h (sm_100a kernels).  A
// program written against the reference's
//     fpmm::mw_product(A, B, u, v, lambda, F, kernel)
// recompiles against this header and links libfpmm_b200.so instead.
//
// Differences, by design:
//   * only T = double (FpContext<float> / t = 24 is out of scope);
//   * GemmKernel selection is accepted for signature parity; every product
//     runs a fused engine.  kernel_by_name("b200") (alias "accelerated")
//     selects the library default; "b200-rns", "b200-i8" and "b200-dmma" pin
//     an engine (FPMM_B200_ENGINE_*).  Each also is the panel-level kernel
//     (DMMA, exact C += A B) for plugin-style callers.
#pragma once

#include <cstdint>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "fpmm_b200.h"

namespace fpmm {

using u64 = std::uint64_t;
using i64 = std::int64_t;
using index_t = std::int64_t;

// errors.hpp:9-33
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractError : Error {
  using Error::Error;
};
struct InfeasibleError : Error {
  using Error::Error;
};
struct NoInverseError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};
struct DeviceError : Error {
  using Error::Error;
};

namespace detail {
inline void check(int st) {
  if (st == FPMM_B200_OK) return;
  const std::string msg = fpmm_b200_last_error();
  switch (st) {
    case FPMM_B200_EINFEASIBLE: throw InfeasibleError(msg);
    case FPMM_B200_ENOINVERSE: throw NoInverseError(msg);
    case FPMM_B200_ECONTRACT: throw ContractError(msg);
    case FPMM_B200_ECUDA:
    case FPMM_B200_ENCCL:
    case FPMM_B200_ENOMEM: throw DeviceError(msg);
    default: throw Error(msg);
  }
}
}  // namespace detail

inline int bitsize(u64 n) { return n ? 64 - __builtin_clzll(n) : 0; }
inline bool is_prime_u64(u64 n) { return fpmm_b200_is_prime(n) != 0; }
inline u64 prev_prime(u64 limit) { return fpmm_b200_prev_prime(limit); }

// mat.hpp:13-26
template <typename T>
struct ConstMatView {
  const T* data;
  index_t rows, cols, stride;
  const T& operator()(index_t i, index_t j) const { return data[i * stride + j]; }
};
template <typename T>
struct MatView {
  T* data;
  index_t rows, cols, stride;
  T& operator()(index_t i, index_t j) const { return data[i * stride + j]; }
  operator ConstMatView<T>() const { return {data, rows, cols, stride}; }
};

// mat.hpp:31-90: dense row-major integers stored as T
template <typename T>
class Mat {
 public:
  Mat() : rows_(0), cols_(0) {}
  Mat(index_t rows, index_t cols, T fill = T(0))
      : rows_(rows), cols_(cols), data_(static_cast<size_t>(rows * cols), fill) {
    if (rows < 0 || cols < 0) throw Error("matrix dimensions must be nonnegative");
  }
  index_t rows() const { return rows_; }
  index_t cols() const { return cols_; }
  T& operator()(index_t i, index_t j) { return data_[static_cast<size_t>(i * cols_ + j)]; }
  const T& operator()(index_t i, index_t j) const { return data_[static_cast<size_t>(i * cols_ + j)]; }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  size_t size() const { return data_.size(); }
  MatView<T> view() { return {data_.data(), rows_, cols_, cols_}; }
  ConstMatView<T> view() const { return {data_.data(), rows_, cols_, cols_}; }
  ConstMatView<T> col_panel(index_t c0, index_t n) const { return {data_.data() + c0, rows_, n, cols_}; }
  MatView<T> col_panel(index_t c0, index_t n) { return {data_.data() + c0, rows_, n, cols_}; }
  ConstMatView<T> row_panel(index_t r0, index_t n) const { return {data_.data() + r0 * cols_, n, cols_, cols_}; }
  MatView<T> row_panel(index_t r0, index_t n) { return {data_.data() + r0 * cols_, n, cols_, cols_}; }
  const std::optional<u64>& max_hint() const { return max_hint_; }
  void set_max_hint(u64 b) { max_hint_ = b; }
  void clear_max_hint() { max_hint_ = std::nullopt; }
  u64 max_bound() const {
    if (max_hint_) return *max_hint_;
    T m = T(0);
    for (T v : data_) m = v > m ? v : m;
    return static_cast<u64>(m);
  }
  bool same_dims(const Mat& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }
  friend bool operator==(const Mat& a, const Mat& b) {
    return a.rows_ == b.rows_ && a.cols_ == b.cols_ && a.data_ == b.data_;
  }

 private:
  index_t rows_, cols_;
  std::vector<T> data_;
  std::optional<u64> max_hint_;
};

inline u64 mix_seed(u64 a, u64 b) { return fpmm_b200_mix_seed(a, b); }

// mat.hpp:112-120
template <typename T>
Mat<T> random_mat(index_t rows, index_t cols, u64 p, u64 seed) {
  static_assert(std::is_same_v<T, double>, "binary64 only");
  Mat<T> m(rows, cols);
  detail::check(fpmm_b200_random_mat(rows, cols, p, seed, m.data()));
  m.set_max_hint(p - 1);
  return m;
}

template <typename T>
Mat<T> identity_mat(index_t n) {
  Mat<T> m(n, n);
  for (index_t i = 0; i < n; ++i) m(i, i) = T(1);
  m.set_max_hint(1);
  return m;
}

// fp_context.hpp:29-77 (binary64)
template <typename T>
class FpContext {
  static_assert(std::is_same_v<T, double>, "the B200 path is binary64 only");

 public:
  static constexpr int t = 53;
  static FpContext make(u64 p, bool allow_composite = false) {
    detail::check(fpmm_b200_context_check(p, allow_composite ? 1 : 0));
    return FpContext(p, is_prime_u64(p));
  }
  u64 p() const { return p_; }
  T pf() const { return static_cast<T>(p_); }
  T q() const { return T(1) / static_cast<T>(p_); }
  int bits() const { return bitsize(p_); }
  bool prime() const { return prime_; }
  bool residue_mul_fp_safe() const {
    return 3 * static_cast<unsigned __int128>(p_ - 1) * (p_ - 1) <= (static_cast<unsigned __int128>(1) << (t - 1)) * p_;
  }

 private:
  FpContext(u64 p, bool prime) : p_(p), prime_(prime) {}
  u64 p_;
  bool prime_;
};
using FpContext64 = FpContext<double>;

// gemm_kernel.hpp:13-19 plugin interface, with the B200 panel kernel
template <typename T>
class GemmKernel {
 public:
  virtual ~GemmKernel() = default;
  virtual void accumulate(MatView<T> c, ConstMatView<T> a, ConstMatView<T> b) const = 0;
  virtual std::string_view name() const = 0;
};

class B200Kernel final : public GemmKernel<double> {
 public:
  constexpr B200Kernel(std::string_view name, unsigned engine) : name_(name), engine_(engine) {}
  void accumulate(MatView<double> c, ConstMatView<double> a, ConstMatView<double> b) const override {
    if (a.rows != c.rows || b.cols != c.cols || a.cols != b.rows) throw Error("accumulate: dimension mismatch");
    detail::check(fpmm_b200_accumulate(c.data, c.stride, a.data, a.stride, b.data, b.stride, c.rows, a.cols, c.cols));
  }
  std::string_view name() const override { return name_; }
  unsigned engine() const { return engine_; }  // FPMM_B200_ENGINE_* flag, 0 = library default

 private:
  std::string_view name_;
  unsigned engine_;
};

template <typename T>
const GemmKernel<T>& b200_kernel() {
  static const B200Kernel k("b200", 0u);
  return k;
}
template <typename T>
const GemmKernel<T>* kernel_by_name(std::string_view name) {
  static const B200Kernel rns("b200-rns", FPMM_B200_ENGINE_RNS), i8("b200-i8", FPMM_B200_ENGINE_I8),
      dmma("b200-dmma", FPMM_B200_ENGINE_DMMA);
  if (name == "b200" || name == "accelerated") return &b200_kernel<T>();
  if (name == "b200-rns") return &rns;
  if (name == "b200-i8") return &i8;
  if (name == "b200-dmma") return &dmma;
  return nullptr;
}

namespace detail {
// engine flag carried by the caller's kernel choice (0 for foreign kernels: the default)
template <typename T>
unsigned engine_of(const GemmKernel<T>& k) {
  const auto* b = dynamic_cast<const B200Kernel*>(&k);
  return b ? b->engine() : 0u;
}
}  // namespace detail

// multiword.hpp:12-24
inline u64 word_base(u64 p, int u) {
  u64 out = 0;
  detail::check(fpmm_b200_word_base(p, u, &out));
  return out;
}
inline u64 word_bound(u64 p, int u) { return u == 1 ? p - 1 : word_base(p, u); }

template <typename T>
struct WordDecomposition {
  u64 base;
  std::vector<Mat<T>> words;
  int word_count() const { return static_cast<int>(words.size()); }
};

// block_product.hpp:13-22
inline std::optional<u64> max_block_size(u64 max_a, u64 max_b, u64 p, int t) {
  u64 out = 0;
  detail::check(fpmm_b200_max_block_size(max_a, max_b, p, t, &out));
  return out ? std::optional<u64>(out) : std::nullopt;
}

// multiword.hpp:29-54 (on the device; words identical to the reference's)
template <typename T>
WordDecomposition<T> decompose(const Mat<T>& M, int u, const FpContext<T>& F) {
  if (u < 1) throw Error("decompose: word count must be positive");
  WordDecomposition<T> d;
  std::vector<T> buf(static_cast<size_t>(u) * M.size());
  detail::check(fpmm_b200_decompose(M.data(), M.cols(), M.rows(), M.cols(), F.p(), u, buf.data(),
                                    static_cast<i64>(M.size()), &d.base));
  for (int i = 0; i < u; ++i) {
    Mat<T> w(M.rows(), M.cols());
    std::copy(buf.begin() + static_cast<i64>(i) * M.size(), buf.begin() + static_cast<i64>(i + 1) * M.size(),
              w.data());
    w.set_max_hint(word_bound(F.p(), u));
    d.words.push_back(std::move(w));
  }
  return d;
}

// block_product.hpp:62-73: C <- C + A B mod p
template <typename T>
void block_gemm_mod(Mat<T>& C, const Mat<T>& A, const Mat<T>& B, u64 lambda, const FpContext<T>& F,
                    const GemmKernel<T>& = b200_kernel<T>()) {
  if (A.rows() != C.rows() || B.cols() != C.cols() || A.cols() != B.rows())
    throw Error("block_gemm_mod: dimension mismatch");
  detail::check(fpmm_b200_block_gemm_mod(C.data(), C.cols(), A.data(), A.cols(), B.data(), B.cols(), A.rows(),
                                         A.cols(), B.cols(), lambda, F.p(), 0));
  C.set_max_hint(F.p() - 1);
}

namespace detail {
template <typename T>
Mat<T> product(const Mat<T>& A, const Mat<T>& B, int u, int v, u64 lambda, const FpContext<T>& F, int variant,
               int ngpus, unsigned engine = 0) {
  if (A.cols() != B.rows()) throw Error("multiword product: dimension mismatch");
  Mat<T> C(A.rows(), B.cols());
  const unsigned flags = (F.prime() ? 0u : FPMM_B200_ALLOW_COMPOSITE) | engine;
  check(fpmm_b200_mw_product(A.data(), A.cols(), B.data(), B.cols(), C.data(), C.cols(), A.rows(), A.cols(),
                             B.cols(), F.p(), u, v, lambda, variant, ngpus, flags, nullptr));
  C.set_max_hint(F.p() - 1);
  return C;
}

template <typename T>
Mat<T> words_product(const WordDecomposition<T>& da, const WordDecomposition<T>& db, index_t m, index_t k,
                     index_t n, u64 lambda, const FpContext<T>& F, int variant, unsigned engine = 0) {
  const int u = da.word_count(), v = db.word_count();
  if (u < 1 || v < 1) throw Error("multiword product: word counts must be positive");
  std::vector<T> aw(static_cast<size_t>(u) * m * k), bw(static_cast<size_t>(v) * k * n);
  for (int i = 0; i < u; ++i) {
    if (da.words[i].rows() != m || da.words[i].cols() != k) throw Error("multiword product: dimension mismatch");
    std::copy(da.words[i].data(), da.words[i].data() + m * k, aw.data() + static_cast<i64>(i) * m * k);
  }
  for (int j = 0; j < v; ++j) {
    if (db.words[j].rows() != k || db.words[j].cols() != n) throw Error("multiword product: dimension mismatch");
    std::copy(db.words[j].data(), db.words[j].data() + k * n, bw.data() + static_cast<i64>(j) * k * n);
  }
  Mat<T> C(m, n);
  const unsigned flags = (F.prime() ? 0u : FPMM_B200_ALLOW_COMPOSITE) | engine;
  check(fpmm_b200_mw_product_words(aw.data(), m * k, k > 0 ? k : 1, da.base, u, bw.data(), k * n, n > 0 ? n : 1,
                                   db.base, v, C.data(), n > 0 ? n : 1, m, k, n, F.p(), lambda, variant, flags,
                                   nullptr));
  C.set_max_hint(F.p() - 1);
  return C;
}
}  // namespace detail

// multiword.hpp:113-139
template <typename T>
Mat<T> mw_product_words(const WordDecomposition<T>& da, const WordDecomposition<T>& db, index_t m, index_t k,
                        index_t n, u64 lambda, const FpContext<T>& F, const GemmKernel<T>& kernel = b200_kernel<T>()) {
  return detail::words_product(da, db, m, k, n, lambda, F, FPMM_B200_PLAIN, detail::engine_of(kernel));
}
template <typename T>
Mat<T> mw_product(const Mat<T>& A, const Mat<T>& B, int u, int v, u64 lambda, const FpContext<T>& F,
                  const GemmKernel<T>& kernel = b200_kernel<T>()) {
  return detail::product(A, B, u, v, lambda, F, FPMM_B200_PLAIN, 1, detail::engine_of(kernel));
}
// row-sharded over devices 0..ngpus-1 of this process (NCCL broadcast of B words)
template <typename T>
Mat<T> mw_product_multi_gpu(const Mat<T>& A, const Mat<T>& B, int u, int v, u64 lambda, const FpContext<T>& F,
                            int ngpus) {
  return detail::product(A, B, u, v, lambda, F, FPMM_B200_PLAIN, ngpus);
}

enum class ConcatSide { auto_pick, a, b };
inline u64 concat_workspace_entries(int u, int v, index_t m, index_t n, ConcatSide side) {
  const u64 mn = static_cast<u64>(m) * static_cast<u64>(n);
  return side == ConcatSide::a ? static_cast<u64>(u) * mn : static_cast<u64>(v) * mn;
}

// multiword.hpp:155-218 (same value; all word pairs share one fused tile)
template <typename T>
Mat<T> mw_product_concat_words(const WordDecomposition<T>& da, const WordDecomposition<T>& db, index_t m,
                               index_t k, index_t n, u64 lambda, const FpContext<T>& F,
                               const GemmKernel<T>& kernel = b200_kernel<T>(), ConcatSide = ConcatSide::auto_pick) {
  return detail::words_product(da, db, m, k, n, lambda, F, FPMM_B200_CONCAT, detail::engine_of(kernel));
}
template <typename T>
Mat<T> mw_product_concat(const Mat<T>& A, const Mat<T>& B, int u, int v, u64 lambda, const FpContext<T>& F,
                         const GemmKernel<T>& kernel = b200_kernel<T>(), ConcatSide = ConcatSide::auto_pick) {
  return detail::product(A, B, u, v, lambda, F, FPMM_B200_CONCAT, 1, detail::engine_of(kernel));
}
// multiword.hpp:222-254 (inverse-free; composite p allowed)
template <typename T>
Mat<T> mw_product_workspace_words(const WordDecomposition<T>& da, const WordDecomposition<T>& db, index_t m,
                                  index_t k, index_t n, u64 lambda, const FpContext<T>& F,
                                  const GemmKernel<T>& kernel = b200_kernel<T>()) {
  return detail::words_product(da, db, m, k, n, lambda, F, FPMM_B200_WORKSPACE, detail::engine_of(kernel));
}
template <typename T>
Mat<T> mw_product_workspace(const Mat<T>& A, const Mat<T>& B, int u, int v, u64 lambda, const FpContext<T>& F,
                            const GemmKernel<T>& kernel = b200_kernel<T>()) {
  return detail::product(A, B, u, v, lambda, F, FPMM_B200_WORKSPACE, 1, detail::engine_of(kernel));
}

// planner.hpp:12-102
struct Variant {
  int u, v;
  int products() const { return u * v; }
  friend bool operator==(Variant a, Variant b) { return a.u == b.u && a.v == b.v; }
};
inline constexpr Variant kVariants[6] = {{1, 1}, {1, 2}, {1, 3}, {1, 4}, {2, 2}, {2, 3}};
inline std::string variant_name(Variant v) {
  return "(" + std::to_string(v.u) + "," + std::to_string(v.v) + ")";
}
inline std::optional<u64> mw_block_size(int u, int v, u64 p, int t) {
  u64 out = 0;
  detail::check(fpmm_b200_mw_block_size(u, v, p, t, &out));
  return out ? std::optional<u64>(out) : std::nullopt;
}
template <typename T>
std::optional<u64> mw_block_size(int u, int v, const FpContext<T>& F) {
  return mw_block_size(u, v, F.p(), FpContext<T>::t);
}
inline int variant_bit_limit(int u, int v, int t) {
  int out = 0;
  detail::check(fpmm_b200_variant_bit_limit(u, v, t, &out));
  return out;
}
inline bool variant_admits_bits(Variant var, int bits, int t) { return bits <= variant_bit_limit(var.u, var.v, t); }

enum class ConcatChoice { none, a, b };
struct ProductPlan {
  int u = 1, v = 1;
  u64 lambda = 1;
  ConcatChoice concat = ConcatChoice::none;
  u64 predicted_products = 1;
  u64 predicted_reductions = 0;
  u64 storage_entries = 0;
  Variant variant() const { return {u, v}; }
};
namespace detail {
inline ProductPlan from_c(const fpmm_b200_plan& c) {
  ProductPlan p;
  p.u = c.u;
  p.v = c.v;
  p.lambda = c.lambda;
  p.concat = c.concat == 1 ? ConcatChoice::a : c.concat == 2 ? ConcatChoice::b : ConcatChoice::none;
  p.predicted_products = c.predicted_products;
  p.predicted_reductions = c.predicted_reductions;
  p.storage_entries = c.storage_entries;
  return p;
}
}  // namespace detail
inline ProductPlan select_variant(int bits, index_t m, index_t k, index_t n, int t, u64 min_lambda = 1,
                                  index_t concat_threshold = 256) {
  fpmm_b200_plan c{};
  detail::check(fpmm_b200_select_variant(bits, m, k, n, t, min_lambda, concat_threshold, &c));
  return detail::from_c(c);
}
inline ProductPlan plan_for_modulus(u64 p, index_t m, index_t k, index_t n, int t, u64 min_lambda = 1,
                                    index_t concat_threshold = 256) {
  fpmm_b200_plan c{};
  detail::check(fpmm_b200_plan_for_modulus(p, m, k, n, t, min_lambda, concat_threshold, &c));
  return detail::from_c(c);
}
inline void finish_plan(ProductPlan& plan, index_t m, index_t k, index_t n) {
  fpmm_b200_plan c{plan.u, plan.v, plan.lambda,
                   plan.concat == ConcatChoice::a ? 1 : plan.concat == ConcatChoice::b ? 2 : 0, 0, 0, 0};
  detail::check(fpmm_b200_finish_plan(&c, m, k, n));
  plan = detail::from_c(c);
}

}  // namespace fpmm
