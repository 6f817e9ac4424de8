// Launch interface of assemble.cu
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace afsai {
__global__ void validate_rows_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                     int64_t n_rows, int64_t row_begin, int64_t n_cols, unsigned long long *err);
__global__ void cast_rows_f32_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                     int64_t n_rows, int64_t row_begin, float *out, unsigned long long *err);
__global__ void row_len_max_kernel(const int64_t *rowptr, int64_t n_rows, unsigned long long *out);
__global__ void symmetry_kernel(const int64_t *rowptr, const int32_t *col, const double *val, int64_t base,
                                int64_t n_rows, int64_t row_begin, unsigned long long *err);
cudaError_t exclusive_scan(const int32_t *in, int64_t n, int64_t *out, int64_t *tmp_tiles, cudaStream_t st,
                           int64_t *launches);
int64_t scan_tmp_elems(int64_t n);
__global__ void fill_rows_kernel(int64_t n_rows, const int32_t *scol, const double *sval, int32_t stride,
                                 const int64_t *rowptr, int32_t *col, double *val);
__global__ void count_cols_kernel(int64_t nnz, const int32_t *col, int64_t col_lo, int64_t n_out, int32_t *cnt);
__global__ void scatter_t_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                                 int64_t row_begin, int64_t col_lo, int64_t n_out, const int64_t *t_rowptr,
                                 int32_t *cursor, int32_t *t_col, double *t_val);
// sort every row of a scattered G^T by source row (C10); in_* is clobbered
void sort_gt_rows(int64_t n_rows, const int64_t *rowptr, int32_t *in_col, double *in_val, int32_t *out_col,
                  double *out_val, int grid, cudaStream_t st, int64_t *launches);
// G^T (columns [col_lo, col_lo + n_out) of G) by a stable LSD radix sort of G's entries by
// column: writes t_col (source rows) and t_val in G^T's CSR order (t_rowptr from the
// column counts).  tmp: radix_tmp_bytes(nnz, n_out) bytes of device scratch.
int64_t radix_tmp_bytes(int64_t nnz, int64_t n_out);
cudaError_t transpose_radix(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                            int64_t nnz, int64_t col_lo, int64_t n_out, int64_t row_begin, char *tmp,
                            int32_t *t_col, double *t_val, int grid, cudaStream_t st, int64_t *launches);
__global__ void row_lengths_kernel(const int64_t *rowptr, int64_t n_rows, int32_t *len);
__global__ void g_triples_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                                 int64_t row_begin, int32_t *tc, int32_t *tr, double *tv);
__global__ void count_dest_kernel(int64_t nnz, const int32_t *tc, const int64_t *bounds, int nranks,
                                  unsigned long long *cnt);
__global__ void scatter_dest_kernel(int64_t nnz, const int32_t *tc, const int32_t *tr, const double *tv,
                                    const int64_t *bounds, int nranks, const unsigned long long *off,
                                    unsigned long long *cur, int32_t *oc, int32_t *orow, double *ov);
__global__ void band_count_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, int64_t lo, int64_t hi,
                                  int32_t *cnt);
__global__ void band_fill_kernel(int64_t n_rows, const int64_t *rowptr, const int32_t *col, const double *val,
                                 int64_t row_begin, int64_t lo, int64_t hi, const int64_t *off, int32_t *tc,
                                 int32_t *tr, double *tv);
__global__ void count_triples_kernel(int64_t nnz, const int32_t *tc, int64_t col_lo, int64_t n_out, int32_t *cnt);
__global__ void scatter_triples_kernel(int64_t nnz, const int32_t *tc, const int32_t *tr, const double *tv,
                                       int64_t col_lo, int64_t n_out, const int64_t *t_rowptr, int32_t *cursor,
                                       int32_t *t_col, double *t_val);
}  // namespace afsai
