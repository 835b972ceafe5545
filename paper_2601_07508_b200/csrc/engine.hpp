// engine.hpp -- device orchestration of the multiword product (internal).
#pragma once

#include <cstdint>

#include "fpmm_b200.h"
#include "rules.hpp"

namespace fpmm_b200 {

struct ProductArgs {
  const double* A;
  i64 lda;
  const double* B;
  i64 ldb;
  double* C;
  i64 ldc;
  i64 m, k, n;
  u64 p;
  int u, v;
  u64 lambda;
  unsigned flags;
};

// validation shared by every product entry point (FpContext::make +
// check_mw_inputs + the in-place variant's inverse requirement)
void validate_product(u64 p, int u, int v, u64 lambda, i64 m, i64 k, i64 n, unsigned flags);

// device-resident product on one device / stream (stream may be null)
void product_device(const ProductArgs& a, int device, void* stream, fpmm_b200_timing* tm);
// host-buffer product on devices [0, ngpus)
void product_host(const ProductArgs& a, int ngpus, fpmm_b200_timing* tm);
// host-buffer words product (recompose then product)
void product_words_host(const double* Aw, i64 a_stride, i64 lda, u64 alpha, int u, const double* Bw,
                        i64 b_stride, i64 ldb, u64 beta, int v, double* C, i64 ldc, i64 m, i64 k,
                        i64 n, u64 p, u64 lambda, unsigned flags, fpmm_b200_timing* tm);

struct Prepared;
Prepared* prepare_a_device(const double* dA, i64 lda, i64 m, i64 k, u64 p, int u, int v, unsigned flags,
                           int device, void* stream);
void prepared_free(Prepared* h);
void product_prepared_device(const Prepared* h, const double* dB, i64 ldb, double* dC, i64 ldc, i64 n, u64 lambda,
                             void* stream, unsigned flags, fpmm_b200_timing* tm);

void decompose_device(const double* dM, i64 ld, i64 rows, i64 cols, u64 p, int u, double* dwords,
                      i64 word_stride, u64* base, int device, void* stream);
void decompose_host(const double* M, i64 ld, i64 rows, i64 cols, u64 p, int u, double* words,
                    i64 word_stride, u64* base);
void accumulate_device(double* dC, i64 ldc, const double* dA, i64 lda, const double* dB, i64 ldb,
                       i64 m, i64 w, i64 n, int device, void* stream);
void accumulate_host(double* C, i64 ldc, const double* A, i64 lda, const double* B, i64 ldb, i64 m,
                     i64 w, i64 n);
void block_gemm_mod_host(double* C, i64 ldc, const double* A, i64 lda, const double* B, i64 ldb,
                         i64 m, i64 k, i64 n, u64 lambda, u64 p, unsigned flags);

// library-default engine for a product shape: FPMM_B200_ENGINE_I8 or _RNS
unsigned select_engine(i64 m, i64 k, i64 n, u64 p);

int device_count();
void verify_device(const double* dA, i64 lda, const double* dB, i64 ldb, const double* dC, i64 ldc, i64 m, i64 k,
                   i64 n, u64 p, u64 seed, int trials, int samples, int device, void* stream, i64* counts);
void random_residues_device(double* dM, i64 ld, i64 rows, i64 cols, i64 row0, u64 p, u64 seed, int device,
                            void* stream);
double fp64_peak_tflops(int device, int iters);
double i8_peak_tops(int device, int iters);
double i8_probe_tops(int device, int iters, int mode);
void finalize_all();

// multi-process partitioner
int nccl_id_size();
void nccl_unique_id(void* id);
void dist_init(const void* id, int nranks, int rank, int device);
void dist_finalize();
void dist_rows(i64 m, int nranks, int rank, int u, int v, i64* row0, i64* rows);
void dist_chunks(i64 m, i64 k, i64 n, u64 p, int u, int v, unsigned flags, i64 rows, int* count, i64* starts,
                 i64* lens);
void dist_product_device(const double* dA_rows, i64 lda, const double* dB, i64 ldb, double* dC_rows,
                         i64 ldc, double* dC_full, i64 ldc_full, i64 m, i64 k, i64 n, u64 p, int u,
                         int v, u64 lambda, int root, void* stream, unsigned flags,
                         fpmm_b200_timing* tm);

}  // namespace fpmm_b200
