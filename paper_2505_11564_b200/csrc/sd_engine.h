// Internal interfaces shared by the translation units of libspecden_b200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "specden_b200.h"

namespace sd {
void probe_fill(void* x, uint64_t begin, uint64_t end, uint64_t seed, int dist, uint64_t one_hot, int prec,
                cudaStream_t s);
void axpy_dot(const void* x, void* y, const void* z, const double* coef, uint64_t begin, uint64_t end, uint64_t total,
              int prec, double* partial, cudaStream_t s);
void cgs(const void* Q, uint64_t ldq, uint64_t j, void* r, const double* coef, int mode, uint64_t begin, uint64_t end,
         uint64_t total, int prec, double* partials, uint64_t pstride, cudaStream_t s);
void combine_device(uint64_t nranks, const uint64_t* begins, const uint64_t* ends, uint64_t total, uint64_t m,
                    uint64_t plen_max, const double* partials, double* out, cudaStream_t s, int post_sqrt);
void scale(const void* x, void* out, uint64_t n, const double* c, int recip, int prec, cudaStream_t s);
void axpy(const void* x, void* y, uint64_t n, const double* alpha, double sign, int prec, cudaStream_t s);
void dense_apply(const double* a, uint64_t n, const void* xf, void* y, uint64_t rb, uint64_t re, int prec,
                 cudaStream_t s);
void diag_apply(const void* d, const void* x, void* y, uint64_t n, int prec, cudaStream_t s);
void comm_allgather(sd_comm c, const void* send, void* recv, uint64_t bytes, cudaStream_t s);
void comm_allreduce_f32(sd_comm c, float* buf, uint64_t n, cudaStream_t s);
void comm_reducescatter_f32(sd_comm c, const float* send, float* recv, uint64_t n, cudaStream_t s);
// variable-length slices [rb[r], re[r]) of a full-length vector (the Lanczos
// ShardLayout): all-gather of each rank's slice into `full`, and the
// rank-ordered sum of every rank's `full` over this rank's slice into `mine`
void comm_allgatherv_f32(sd_comm c, const float* mine, float* full, const uint64_t* rb, const uint64_t* re,
                         cudaStream_t s);
void comm_reducescatterv_f32(sd_comm c, const float* full, float* mine, const uint64_t* rb, const uint64_t* re,
                             cudaStream_t s);
void comm_send_f32(sd_comm c, const float* buf, uint64_t n, int peer, cudaStream_t s);
void comm_recv_f32(sd_comm c, float* buf, uint64_t n, int peer, cudaStream_t s);
void comm_group_begin(sd_comm c);
void comm_group_end(sd_comm c, cudaStream_t s);
// stream wait that surfaces NCCL async errors / timeouts as SD_NCCL_ERROR
void comm_wait(sd_comm c, cudaStream_t s);
int comm_rank(sd_comm c);
int comm_size(sd_comm c);
void operator_apply(sd_operator op, const void* x, void* y, int prec, cudaStream_t s, uint64_t row_begin,
                    uint64_t row_end, const void* x_full);
bool operator_needs_full(sd_operator op);
// tree-mode Lanczos passes (sd_lanczos_tree.cu): mode 0 = single-column
// axpy update + dots over jb columns, 1 = GEMV update + dots, 2 = GEMV update +
// norm; the per-CTA partial rows live in `part` (tree_part_bytes(n) bytes,
// followed by the counter the last CTA resets)
uint64_t tree_part_bytes(uint64_t n);
void tree_pass(int prec, int mode, const void* Q, uint64_t ldq, int jb, void* r, uint64_t n, const double* coef,
               int ucol, int xcol, double* part, unsigned* counter, double* out, double* alpha_out, int alpha_col,
               int post_sqrt, cudaStream_t s);
void tree_rank_fold(const double* recv, int nranks, int m, double* out, int post_sqrt, double* alpha_out,
                    int alpha_col, cudaStream_t s);
// ctx release on sd_operator_destroy (operators the engines create around their contexts)
void operator_set_dtor(sd_operator op, void (*dtor)(void*));
}  // namespace sd
