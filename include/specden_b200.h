/*
 * specden_b200.h — C-ABI of the B200-native SLQ hot path (HessFormer, arxiv
 * 2505.11564). Implemented by paper_2505_11564_b200/libspecden_b200.so
 * (hand-written sm_100a CUDA kernels + a C++ host engine).
 *
 * Conventions
 *  - Every entry point returns sd_status; on failure sd_last_error() holds a
 *    thread-local message. Codes 1-6 are the six classes of
 *    proj/include/specden/errors.hpp:13-41; 7/8 are CUDA / NCCL failures.
 *  - Device buffers are CALLER-OWNED (plain pointers + element counts).
 *    Launchers ("sd_k_*") never allocate, never synchronise, and are ordered
 *    on the caller's stream. Engine calls that need scratch take a caller
 *    workspace sized by a matching *_workspace_bytes query.
 *  - prec: SD_F32 (float* storage) or SD_F64 (double* storage), the
 *    Precision of proj/include/specden/precision.hpp:15-19. Scalars (dots,
 *    alpha, beta) are always f64 (precision.hpp:9-14).
 *  - Shards: a rank owns [begin, end) of a logical vector of length `total`
 *    (ShardLayout, proj/include/specden/layout.hpp:12-72); pointers passed
 *    for a shard point at its first owned element.
 */
#ifndef SPECDEN_B200_H
#define SPECDEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sd_stream; /* == cudaStream_t */

typedef enum {
  SD_OK = 0,
  SD_CONFIG_ERROR = 1,    /* config_error   errors.hpp:13-17 */
  SD_LAYOUT_ERROR = 2,    /* layout_error   errors.hpp:19-22 */
  SD_ARGUMENT_ERROR = 3,  /* argument_error errors.hpp:24-27 */
  SD_NUMERICAL_ERROR = 4, /* numerical_error errors.hpp:29-32 */
  SD_STATE_ERROR = 5,     /* state_error    errors.hpp:34-38 */
  SD_PROTOCOL_ERROR = 6,  /* protocol_error errors.hpp:40-43 */
  SD_CUDA_ERROR = 7,
  SD_NCCL_ERROR = 8
} sd_status;

enum { SD_F32 = 0, SD_F64 = 1 };
/* ProbeDist, sharded.hpp:34. SD_GAUSSIAN is bit-exact with the reference
 * (drawn with glibc's log/cos on the host, uploaded; the fill synchronises);
 * SD_GAUSSIAN_DEVICE draws on the device with CUDA's log/cos (within 1-2 ulp). */
enum { SD_GAUSSIAN = 0, SD_RADEMACHER = 1, SD_ONE_HOT = 2, SD_GAUSSIAN_DEVICE = 3 };
enum { SD_REORTH_NONE = 0, SD_REORTH_FULL = 1, SD_REORTH_SELECTIVE = 2 };

const char* sd_last_error(void);
int sd_abi_version(void);
/* number of CUDA kernels this library has launched in this process */
uint64_t sd_launch_count(void);

/* ---------------------------------------------------------------- RNG (host)
 * Replaces mix64/keyed_counter/uniform01/gaussian/rademacher/uniform_index,
 * proj/include/specden/rng.hpp:17-52 (host copies for bookkeeping/tests). */
uint64_t sd_keyed_counter(uint64_t seed, uint64_t counter);
double sd_rademacher(uint64_t seed, uint64_t i);
uint64_t sd_uniform_index(uint64_t seed, uint64_t i, uint64_t n);

/* ------------------------------------------------------------- layout (host)
 * split_evenly (layout.hpp:59-72), validate_layout (layout.hpp:45-55),
 * ShardLayout::owner (layout.hpp:28-32). `begins/ends` hold >= n entries. */
sd_status sd_split_evenly(uint64_t dim, uint64_t n, uint64_t* begins, uint64_t* ends, uint64_t* count);
/* 1F1B pipeline schedule of one stage (host only): *count (kind, micro-batch)
 * int pairs in ops[2*i], ops[2*i+1]; GROUP_BEGIN/END bracket exchanges that
 * must progress together. ops == NULL returns the count only. */
enum { SD_PIPE_F = 0, SD_PIPE_B = 1, SD_PIPE_SEND_F = 2, SD_PIPE_RECV_F = 3, SD_PIPE_SEND_B = 4, SD_PIPE_RECV_B = 5,
       SD_PIPE_GROUP_BEGIN = 6, SD_PIPE_GROUP_END = 7 };
sd_status sd_pipeline_schedule(int n_stages, int stage, int n_micro, int* ops, uint64_t cap, uint64_t* count);
sd_status sd_validate_layout(uint64_t total, uint64_t n, const uint64_t* begins, const uint64_t* ends);
sd_status sd_layout_owner(uint64_t n, const uint64_t* ends, uint64_t i, uint64_t* owner);

/* ------------------------------------------------- blocked partials (host)
 * Shape of one rank's BlockedPartial (reduction.hpp:40-71) on the fixed
 * 1024-block global grid: n_head raw terms, n_sums block folds, n_tail raw
 * terms. Device partial buffers store them contiguously as f64
 * [head | sums | tail]; sd_partial_len = n_head + n_sums + n_tail. */
sd_status sd_partial_shape(uint64_t begin, uint64_t end, uint64_t total, uint64_t* n_head, uint64_t* n_sums,
                           uint64_t* n_tail);
uint64_t sd_partial_len(uint64_t begin, uint64_t end, uint64_t total);
/* Host fold of per-rank partials in rank order (combine_blocked,
 * reduction.hpp:76-107): parts[r] points at rank r's [head|sums|tail]. */
sd_status sd_combine_partials_host(uint64_t nranks, const uint64_t* begins, const uint64_t* ends, uint64_t total,
                                   const double* const* parts, double* out);

/* ----------------------------------------------------- vector kernels (GPU)
 * draw_probe fill (sharded.cpp:59-76, unnormalised): x[i-begin] =
 * round(dist(seed, i)) for i in [begin, end). SD_GAUSSIAN: host-drawn and
 * uploaded through pinned staging (synchronises the stream). */
sd_status sd_k_probe_fill(void* x, uint64_t begin, uint64_t end, uint64_t seed, int dist, uint64_t one_hot_index,
                          int prec, sd_stream s);
/* Blocked dot partial of a[i]*b[i] over this rank's shard (dot, sharded.cpp:85-100). */
sd_status sd_k_dot_partial(const void* a, const void* b, uint64_t begin, uint64_t end, uint64_t total, int prec,
                           double* partial, sd_stream s);
/* m independent partial sets folded in rank order on the device:
 * partials laid out [rank][seq][plen_r]; out[seq] = combine_blocked. */
sd_status sd_k_combine(uint64_t nranks, const uint64_t* begins, const uint64_t* ends, uint64_t total, uint64_t m,
                       const double* partials, double* out, sd_stream s);
/* y = round(y + alpha*x) with alpha = sign * (*alpha_dev) (axpy, sharded.cpp:106-118). */
sd_status sd_k_axpy(const void* x, void* y, uint64_t n, const double* alpha_dev, double sign, int prec, sd_stream s);
/* out = round(c*x), c = (*c_dev) or, with reciprocal, 1.0/(*c_dev) (scale, sharded.cpp:120-130). */
sd_status sd_k_scale(const void* x, void* out, uint64_t n, const double* c_dev, int reciprocal, int prec,
                     sd_stream s);
/* Fused recurrence pass: y = round(y - (*coef)*x) (skipped if x == NULL),
 * then the blocked partial of dot(z, y) (z == NULL: dot(y, y)). */
sd_status sd_k_axpy_dot(const void* x, void* y, const void* z, const double* coef, uint64_t begin, uint64_t end,
                        uint64_t total, int prec, double* partial, sd_stream s);
/* Classical Gram-Schmidt pass over j stored columns Q[i] = Q + i*ldq:
 *   if coef: r = round(...round(r - coef[0] Q[0]) ... - coef[j-1] Q[j-1]) per element,
 *   then mode 0: no dots, 1: partials of dot(Q[i], r) for all i ([i][plen]),
 *   2: partial of dot(r, r). */
sd_status sd_k_cgs(const void* Q, uint64_t ldq, uint64_t j, void* r, const double* coef, int mode, uint64_t begin,
                   uint64_t end, uint64_t total, int prec, double* partials, sd_stream s);
/* Dense symmetric apply (dense_operator, operators.cpp:26-48): row i of this
 * shard = round(sum_j a[i*n+j] * x_full[j]), serial f64 fold; a is row-major
 * n x n f64 on device; rows [row_begin, row_end). */
sd_status sd_k_dense_apply(const double* a, uint64_t n, const void* x_full, void* y, uint64_t row_begin,
                           uint64_t row_end, int prec, sd_stream s);
/* column_report statistics of one shard (SPEC.md column_probe module):
 * counts[t] = #{i : |x_i| < thresholds[t]} (strict, <= 32 thresholds) and
 * max_abs = max |x_i|; then the histogram of |x| over [0, max_abs] in `bins`
 * uniform bins, bin = min(bins-1, floor(|x|/max_abs*bins)) in f64 (all in bin
 * 0 when max_abs == 0). Host outputs; both calls synchronise the stream.
 * Across shards: max of maxima, sums of counts (integer, layout-invariant). */
sd_status sd_k_abs_stats(const void* x, uint64_t n, int prec, const double* thresholds, int n_thresholds,
                         uint64_t* counts, double* max_abs, sd_stream s);
sd_status sd_k_abs_histogram(const void* x, uint64_t n, int prec, double max_abs, int bins, uint64_t* counts,
                             sd_stream s);

/* ------------------------------------------------------- quadrature (host)
 * ritz_decompose: implicit-shift QL, f64. values ascending;
 * weights = squared first eigenvector components. resid (optional) receives
 * max_i ||T y_i - theta_i y_i|| / ||T||. */
sd_status sd_ritz_decompose(uint64_t k, const double* alphas, const double* betas, double* values, double* weights,
                            double* resid);
/* smooth_density; sigma <= 0 selects (max-min)/100. */
sd_status sd_smooth_density(uint64_t k, const double* values, const double* weights, double sigma, uint64_t npts,
                            double* grid, double* density, double* sigma_used);

/* Dense test operators built on the host (wigner_dense / spiked_dense,
 * operators.cpp:50-102); out is row-major n x n f64. */
sd_status sd_wigner_dense(uint64_t n, double sigma, uint64_t seed, double* out);
sd_status sd_spiked_dense(uint64_t n, double sigma, const double* spikes, uint64_t n_spikes, uint64_t seed,
                          double* out);

/* ------------------------------------------------------ communication
 * One process per GPU. An sd_comm carries the rank/size and the collectives
 * the engine needs; sd_comm_nccl_* builds one over NCCL (NVLink/NVSwitch). */
typedef struct sd_comm_s* sd_comm;
sd_status sd_nccl_unique_id(unsigned char out_id[128]);
sd_status sd_comm_nccl_create(const unsigned char id[128], int nranks, int rank, sd_comm* out);
sd_status sd_comm_destroy(sd_comm c);
/* n in-process workers on one device (the reference's WorkerPool model): out[r]
 * is worker r's communicator, driven by its own host thread and stream; the
 * collectives synchronise the caller's stream, meet at a host barrier and
 * exchange by device copies (rank-ordered sums); point-to-point sends complete
 * when the receiver has copied them, groups batch them like NCCL groups. */
sd_status sd_comm_local_create(int nranks, sd_comm* out);
/* a failing in-process worker aborts its group: the others' pending and
 * future collectives fail with SD_PROTOCOL_ERROR instead of waiting forever;
 * on an NCCL communicator: ncclCommAbort */
sd_status sd_comm_abort(sd_comm c);
/* stream wait that, over NCCL, polls ncclCommGetAsyncError and aborts the
 * communicator on an asynchronous error or after SD_NCCL_TIMEOUT_S (default
 * 1800 s): SD_NCCL_ERROR instead of a hang when a peer fails. The Lanczos
 * engine waits this way once per step. Reductions over NCCL are rank-ordered
 * (grouped send/recv + ascending-rank sum, bitwise equal to in-process
 * workers); SD_NCCL_ORDERED=0 selects ncclReduceScatter / ncclAllReduce. */
sd_status sd_comm_wait(sd_comm c, sd_stream s);
/* In-place sum all-reduce of n floats (data-sharded HVP, C1 of SURVEY §2.1). */
sd_status sd_comm_allreduce_f32(sd_comm c, float* buf, uint64_t n, sd_stream s);
/* All-gather of `bytes` per rank (ordered scalar partial exchange). */
sd_status sd_comm_allgather(sd_comm c, const void* send, void* recv, uint64_t bytes, sd_stream s);

/* ------------------------------------------------------------- GEMM
 * C[z] = alpha * op(A[z]) . op(B[z]) + beta * C[z] on tcgen05 tensor cores,
 * fp32 in/out. 3xTF32 when a_small and b_small are given (x_small =
 * x - trunc_tf32(x), see sd_split_tf32), else 1xTF32. a_mn = 0: A row-major
 * m x k, 1: row-major k x m; b_mn = 0: B row-major n x k, 1: row-major k x n.
 * Batch z = z1 + Z1*z2 with element strides per operand. Leading dimensions
 * and strides must be multiples of 4 elements (16 B, TMA). */
typedef struct {
  int m, n, k;
  const float* a;
  const float* a_small;
  long long lda;
  int a_mn;
  const float* b;
  const float* b_small;
  long long ldb;
  int b_mn;
  float* c;
  long long ldc;
  float alpha, beta;
  int z1, z2;
  long long sa1, sa2, sb1, sb2, sc1, sc2;
} sd_gemm_desc;
sd_status sd_gemm_tf32(const sd_gemm_desc* d, sd_stream s);
/* Dual source: C = alpha (op(A1) op(B1) + op(A2) op(B2)) + beta C in one
 * accumulation (the tangent products of the HVP). d1 carries the shape, C,
 * alpha/beta and the first pair; d2 only its a/b operands, lds and strides
 * (m, n, k, majors and precision must match d1). */
sd_status sd_gemm_tf32_dual(const sd_gemm_desc* d1, const sd_gemm_desc* d2, sd_stream s);
/* General form: d2 optional (dual source); flags SD_GEMM_ONCHIP_RESIDUAL =
 * 3xTF32 with the tf32 residuals of the raw operand tiles computed in shared
 * memory (a_small/b_small ignored; same result bits as passing
 * sd_split_tf32(mode 0) residuals, half the operand traffic). */
/* SD_GEMM_B_EXACT / SD_GEMM_B2_EXACT: B (B2) holds tf32-exact values (e.g.
 * bf16-valued weights): b_small may be NULL and the A.B_lo product is skipped
 * (2 MMAs instead of 3; bit-identical to passing its all-zero residual). */
enum { SD_GEMM_ONCHIP_RESIDUAL = 1, SD_GEMM_B_EXACT = 2, SD_GEMM_B2_EXACT = 4 };
sd_status sd_gemm_tf32_ex(const sd_gemm_desc* d1, const sd_gemm_desc* d2, int flags, sd_stream s);
/* small[i] = x[i] - hi(x[i]); mode 0: hi = trunc_tf32 (what the MMA reads),
 * mode 1: hi = round-to-nearest-away tf32. */
sd_status sd_split_tf32(const float* x, float* small, uint64_t n, int mode, sd_stream s);
/* CUDA-event timing of every GEMM launch between begin and end (end syncs):
 * summed kernel ms, algorithmic flops (2*m*n*k*batch), launch count. */
sd_status sd_gemm_profile_begin(void);
sd_status sd_gemm_profile_end(double* ms, double* flops, uint64_t* launches);

/* ---------------------------------------------------------- GPT HVP engine
 * Hessian-vector product of a GPT-2-style decoder (pre-LN, fused QKV, causal
 * softmax attention, GELU-tanh MLP, tied embeddings, mean next-token
 * cross-entropy) by forward-over-reverse: PAPER.md Alg. 1 / SPEC.md:193-210
 * (hvp, batched_hvp) for the SPEC's attention_block model family. Flat
 * parameter order = declaration order, row-major. */
typedef struct {
  int n_layer, d, n_head, ff, vocab, ctx;
  int arch;        /* SD_ARCH_GPT2 (pre-LN, biases, GELU, learned positions, tied head) or
                      SD_ARCH_LLAMA (RMSNorm, RoPE, SwiGLU, no biases, untied head) */
  float rope_base; /* RoPE base (SD_ARCH_LLAMA), e.g. 10000 */
  int n_kv_head;   /* SD_ARCH_LLAMA grouped-query attention: key/value heads (0 = n_head) */
  int bf16_weights; /* parameters are bf16-valued (BASELINE C5 "bf16 weights"): exact in tf32, so the
                       engine keeps no weight residuals and the weight products run 2 MMAs, not 3;
                       sd_gpt_init_params rounds to bf16, sd_gpt_create checks */
} sd_gpt_config;
enum { SD_ARCH_GPT2 = 0, SD_ARCH_LLAMA = 1 };
typedef struct sd_gpt_s* sd_gpt;
uint64_t sd_gpt_param_count(const sd_gpt_config* c);
sd_status sd_gpt_param_layout(const sd_gpt_config* c, uint64_t* offsets, uint64_t* rows, uint64_t* cols, int* kinds,
                              uint64_t* count);
/* synthetic init: matrices 0.02*N(0,1), LN gains 1 + gain_scale*N, biases
 * bias_scale*N, N = gaussian(seed, flat index) (rng.hpp:37-41) */
sd_status sd_gpt_init_params(const sd_gpt_config* c, uint64_t seed, double gain_scale, double bias_scale,
                             float* theta, sd_stream s);
/* the same values for the flat range [begin, end) only: theta_slice[i - begin] */
sd_status sd_gpt_init_params_range(const sd_gpt_config* c, uint64_t seed, double gain_scale, double bias_scale,
                                   uint64_t begin, uint64_t end, float* theta_slice, sd_stream s);
uint64_t sd_gpt_workspace_bytes(const sd_gpt_config* c, int batch, int seq);
/* theta: caller-owned device parameters (P floats), must outlive the engine */
sd_status sd_gpt_create(const sd_gpt_config* c, int batch, int seq, const float* theta, void* workspace,
                        uint64_t workspace_bytes, sd_stream s, sd_gpt* out);
/* host int32 tokens/targets (batch*seq each); Hv is scaled by loss_scale/1
 * relative to the per-token SUM (loss_scale = 1/global_tokens for the mean) */
sd_status sd_gpt_set_batch(sd_gpt g, const int* tokens, const int* targets, float loss_scale, sd_stream s);
/* Pipeline stages (SD_ARCH_LLAMA; PAPER.md:95-96,121-125 place contiguous
 * layers per device): a stage owns layers [layer_begin, layer_end), the token
 * embedding if layer_begin == 0, the final norm + head + loss if layer_end ==
 * n_layer; its parameters are the contiguous slice sd_gpt_stage_params of the
 * flat layout (theta_stage, v and Hv are that slice). n_micro micro-batches
 * of micro_batch x seq tokens (set_batch takes all of them) run through
 * n_sets activation sets (micro-batch m uses set m % n_sets). The whole model
 * with n_micro > 1 is a memory-bounded single-device HVP. */
/* engine flags (SD_ARCH_LLAMA): SD_GPT_RECOMPUTE keeps only each layer's input
 * per in-flight micro-batch and re-runs the layer in the backward (bit-identical
 * Hv, one extra layer forward); SD_GPT_NO_PROBE_RESIDUAL keeps no tf32 residual
 * of v (the tangent products form it on chip). Together with bf16_weights they
 * take the per-stage memory of BASELINE C5 under 180 GB. */
enum { SD_GPT_RECOMPUTE = 1, SD_GPT_NO_PROBE_RESIDUAL = 2 };
uint64_t sd_gpt_stage_workspace_bytes(const sd_gpt_config* c, int micro_batch, int seq, int n_micro, int layer_begin,
                                      int layer_end, int n_sets, int flags);
sd_status sd_gpt_stage_params(const sd_gpt_config* c, int layer_begin, int layer_end, uint64_t* begin, uint64_t* end);
sd_status sd_gpt_stage_create(const sd_gpt_config* c, int micro_batch, int seq, int n_micro, int layer_begin,
                              int layer_end, int n_sets, int flags, const float* theta_stage, void* workspace,
                              uint64_t workspace_bytes, sd_stream s, sd_gpt* out);
/* one Hv pass: begin (v, Hv = stage slices), then forward/backward per
 * micro-batch in a 1F1B order; Hv of micro-batches after the first accumulates */
sd_status sd_gpt_stage_begin(sd_gpt g, const float* v_stage, float* hv_stage, sd_stream s);
sd_status sd_gpt_stage_forward(sd_gpt g, int m, const float* x_in, const float* dx_in, float* x_out, float* dx_out,
                               sd_stream s);
sd_status sd_gpt_stage_backward(sd_gpt g, int m, const float* gx_in, const float* gdx_in, float* gx_out,
                                float* gdx_out, sd_stream s);
/* whole-model Hv = H v on stream s. v is first copied into an engine-owned
 * buffer; from the second call with the same hv pointer and loss scale the
 * HVP's kernels replay as one CUDA graph (SD_GPT_GRAPH=0: always launched
 * one by one); results are bit-identical either way */
sd_status sd_gpt_hvp(sd_gpt g, const float* v, float* hv, sd_stream s);
sd_status sd_gpt_last_loss(sd_gpt g, double* loss, sd_stream s);
sd_status sd_gpt_destroy(sd_gpt g);

/* ---------------------------------------------------------- MLP HVP engine
 * SPEC.md:179 mlp(layer_widths): tanh hidden layers, linear output, mse
 * loss; flat parameters W_0 [w0 x w1] row-major, b_0 [w1], W_1, b_1, ...
 * (declaration order). Same forward-over-reverse HVP as the GPT
 * engine; the engine owns its (small) device workspace. */
typedef struct sd_mlp_s* sd_mlp;
uint64_t sd_mlp_param_count(const uint64_t* widths, int n_widths);
/* theta: caller-owned device parameters (P floats); n_max: batch capacity */
sd_status sd_mlp_create(const uint64_t* widths, int n_widths, int n_max, const float* theta, sd_stream s,
                        sd_mlp* out);
/* host f32 features [n x w0] and targets [n x w_last], row-major; Hv is
 * scaled by loss_scale relative to the SUM of squared errors
 * (loss_scale = 1/(n*w_last) for the mean of SPEC's mse) */
sd_status sd_mlp_set_batch(sd_mlp m, const float* x, const float* y, int n, float loss_scale, sd_stream s);
sd_status sd_mlp_hvp(sd_mlp m, const float* v, float* hv, sd_stream s);
sd_status sd_mlp_last_loss(sd_mlp m, double* loss);
sd_status sd_mlp_destroy(sd_mlp m);

/* ------------------------------------------------------------ operators
 * OperatorHandle (operators.hpp:15-21): apply(x, y) on this rank's shard.
 * x_full is the gathered logical vector when the operator needs it. */
typedef sd_status (*sd_apply_fn)(void* ctx, const void* x, void* y, sd_stream s);
typedef struct sd_operator_s* sd_operator;
sd_status sd_operator_custom(uint64_t dim, sd_apply_fn fn, void* ctx, sd_operator* out);
/* dense_operator (operators.cpp:26-48); `a` host row-major n x n f64, uploaded. */
sd_status sd_operator_dense(uint64_t n, const double* a_host, sd_operator* out);
/* Diagonal test operator y = round(d * x); d is caller-owned device memory
 * holding this rank's shard of the diagonal (prec storage). */
sd_status sd_operator_diag(uint64_t dim, const void* d_dev, int prec, sd_operator* out);
/* Lanczos operator y = H x of a GPT engine; with comm, per-rank Hv over
 * data-sharded batches are summed with an NCCL all-reduce (Alg. 1). */
sd_status sd_operator_gpt(sd_gpt g, sd_comm comm, sd_operator* out);
/* Parameter-sharded form: the Lanczos vectors are split over
 * the comm's ranks by (begins, ends); apply() all-gathers x, runs this
 * rank's batch HVP on the full vector and reduce-scatters Hv into y (f32). */
/* Pipeline-parallel operator: comm rank r runs stage r (engine built by
 * sd_gpt_stage_create with rank r's layers); the Lanczos vectors are sharded
 * by the stages' parameter slices, so x/y are this stage's slice and only the
 * stage-boundary activations (primal|tangent, adjoint|adjoint tangent) move,
 * by NCCL send/recv along the 1F1B schedule. */
sd_status sd_operator_gpt_pipeline(sd_gpt g, sd_comm comm, sd_operator* out);
sd_status sd_operator_gpt_sharded(sd_gpt g, sd_comm comm, const uint64_t* begins, const uint64_t* ends,
                                  sd_operator* out);
/* Lanczos operator y = H x of an MLP engine (all-reduced over comm if given) */
sd_status sd_operator_mlp(sd_mlp m, sd_comm comm, sd_operator* out);
sd_status sd_operator_apply(sd_operator op, const void* x, void* y, int prec, sd_stream s);
uint64_t sd_operator_dim(sd_operator op);
sd_status sd_operator_destroy(sd_operator op);

/* -------------------------------------------------------------- Lanczos
 * lanczos_run (Alg. 2) on device. Vectors are this
 * rank's shard [begin,end) of `total`; scalar partials are exchanged through
 * `comm` (NULL: single rank) and folded in rank order, so alpha/beta are
 * bit-identical to the reference fold for any rank count. Full reorth = two
 * classical Gram-Schmidt passes over all stored columns. */
typedef struct {
  uint64_t k_max;
  double eps; /* <= 0: 1e-12 (f64) / 1e-7 (f32) */
  int reorth; /* SD_REORTH_* */
  int prec;
  uint64_t probe_seed;
  int probe_dist;
  uint64_t selective_window; /* SD_REORTH_SELECTIVE: columns kept (most recent) */
  int reduction; /* SD_REDUCE_ORDERED (default): the reference's fixed 1024-block fold, bitwise
                    (reduction.hpp:30-107); SD_REDUCE_TREE: fused GEMV passes with warp-shuffle +
                    block reductions in a fixed order (deterministic, tolerance parity; <= 256
                    stored basis columns) -- the mode for HVP operators */
} sd_lanczos_config;
enum { SD_REDUCE_ORDERED = 0, SD_REDUCE_TREE = 1 };

typedef struct {
  uint64_t n_alpha, n_beta;
  int breakdown;         /* beta < eps: benign truncation */
  int numerical_failure; /* non-finite alpha/beta: partial T returned */
  double ms_apply, ms_recurrence, ms_reorth, ms_comm; /* CUDA-event phase times */
} sd_lanczos_info;

/* Layout: begins/ends hold every rank's shard (comm size entries; NULL comm =
 * one rank), this rank = comm rank. */
uint64_t sd_lanczos_workspace_bytes(const uint64_t* begins, const uint64_t* ends, uint64_t total,
                                    const sd_lanczos_config* cfg, int nranks, int rank);
/* alphas/betas: host arrays of k_max. */
sd_status sd_lanczos_run(sd_operator op, sd_comm comm, const uint64_t* begins, const uint64_t* ends, uint64_t total,
                         const sd_lanczos_config* cfg, void* workspace, uint64_t workspace_bytes, double* alphas,
                         double* betas, sd_lanczos_info* info, sd_stream s);

/* Step-level engine (what bench.py times): state lives in the workspace. */
typedef struct sd_lanczos_s* sd_lanczos;
sd_status sd_lanczos_begin(sd_operator op, sd_comm comm, const uint64_t* begins, const uint64_t* ends, uint64_t total,
                           const sd_lanczos_config* cfg, void* workspace, uint64_t workspace_bytes, sd_stream s,
                           sd_lanczos* out);
/* One Lanczos step (apply + recurrence + reorth). *done = 1 once the run
 * stopped (k_max reached, benign breakdown, or numerical failure). */
sd_status sd_lanczos_step(sd_lanczos L, int* done);
sd_status sd_lanczos_result(sd_lanczos L, double* alphas, double* betas, sd_lanczos_info* info);
/* Device pointers: current Lanczos vector q_k and the stored basis
 * (column-major, column stride sd_lanczos_basis_ld elements = the shard length
 * rounded up to 32 so that every column is 128-byte aligned for TMA; *ncols
 * columns; NULL if not stored). */
const void* sd_lanczos_current(sd_lanczos L);
sd_status sd_lanczos_basis(sd_lanczos L, const void** basis, uint64_t* ncols);
uint64_t sd_lanczos_basis_ld(sd_lanczos L);
/* loss_of_orthogonality: max_{i!=j} |q_i^T q_j| over the
 * stored basis (full reorth only; state error otherwise), reference dots. */
sd_status sd_lanczos_orthogonality(sd_lanczos L, double* out);
sd_status sd_lanczos_end(sd_lanczos L);

#ifdef __cplusplus
}
#endif
#endif /* SPECDEN_B200_H */
