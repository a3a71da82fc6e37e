/*
 * dbp_b200.h -- C ABI of libdbp_b200.so, the sm_100a (B200) implementation of
 * the decentralized feedforward equalization path of arXiv 1808.04473.
 *
 * Boundary: the reference (`dbp` Python package, /root/reference/pkg) has no
 * FFI; its only plugin seam is `dbp.kernels` (kernels.py:13-19,41-50) and its
 * operator API is the public functions of dbp.equalize / dbp.fusion.  Each
 * entry point below replaces one of those functions (cited per entry) and is
 * bound from Python with ctypes by paper_1808_04473_b200/_lib.py.
 *
 * Conventions
 *  - Every data pointer is a DEVICE pointer (cudaMalloc / torch tensor
 *    data_ptr()).  Complex numbers are interleaved float pairs (complex64).
 *    Small parameter arrays marked "host" are read synchronously.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *    asynchronous on it.  Calls are reentrant.
 *  - Return value: DBP_OK, or a negative DBP_E_* code with a message from
 *    dbp_last_error() (thread-local).
 *  - Numerical faults are reported per item in `status` (int32, one per
 *    item), the batched form of the reference's exceptions:
 *       DBP_ST_SINGULAR   -> SingularGramError   (Cholesky pivot <= 0 /
 *                            relative fp32 tolerance; MRC diag <= 0; L-MMSE
 *                            signal gain <= 0)
 *       DBP_ST_NEGVAR     -> NegativeVarianceError
 *       DBP_ST_DIVERGED   -> DivergenceError, iteration in `iters`
 *       DBP_ST_BADVAR     -> ConfigError (fusion weights need sigma2 > 0)
 *
 * Layouts (row-major):
 *   H      [n][B][u_stride]   channel per item (item = (frame, subcarrier)),
 *                             u_stride even, columns >= u ignored
 *   Y      [n][T][B]          T receive vectors per item (channel constant
 *                             over T)
 *   stats  [n][ncl][u*u + T*u]  Gram G (u x u, full Hermitian) then the
 *                             matched filter ymrc [T][u]
 *   xhat   [n][T][u]          estimates;  dec [n][T][u] uint8 symbol index
 *   sigma2 [n][u] (MRC/ZF/L-MMSE) or [n][T] (LAMA: tau broadcast over u)
 *   nu     [n][C][u] (linear FD) or [n][C][T] (LAMA FD)
 *
 * Limits: u <= 64, T <= 16, C <= 16, cluster row counts and B even, at most
 * 64 row chunks of 32 per item (B <= 2048).
 */
#ifndef DBP_B200_H
#define DBP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBP_ABI_VERSION 1

#define DBP_OK 0
#define DBP_E_ARG (-1)
#define DBP_E_CUDA (-2)
#define DBP_E_UNSUPPORTED (-3)

#define DBP_ST_OK 0
#define DBP_ST_SINGULAR 1
#define DBP_ST_NEGVAR 2
#define DBP_ST_DIVERGED 3
#define DBP_ST_BADVAR 4

/* equalizer kinds: equalize.py:27-31 (Equalizer enum) */
#define DBP_MRC 0
#define DBP_ZF 1
#define DBP_LMMSE 2
#define DBP_LAMA 3

/* architectures: model.py:20-27 (Architecture enum) plus the multi-GPU
 * FD partial-sum mode */
#define DBP_ARCH_PD 1
#define DBP_ARCH_FD 2
#define DBP_ARCH_FD_PARTIAL 3

int dbp_abi_version(void);
const char* dbp_last_error(void);
/* Which fused kernel the calling thread's last dbp_equalize / dbp_gram_mrc
 * launched (DBP_KERNEL_*; 0 = none).  Introspection only (tests and
 * benchmarks); no reference counterpart. */
#define DBP_KERNEL_AUTO 0
#define DBP_KERNEL_SIMT 1     /* FP32-SIMT streaming kernel (ragged clusters, LAMA at u <= 16) */
#define DBP_KERNEL_TC_TF32 2  /* 3xTF32 tensor-core kernel (U <= 32; LAMA 16 < u <= 32: statistics + lama_kernel) */
#define DBP_KERNEL_TC_BF16 3  /* split-bf16 tensor-core streaming kernel (U <= 16 linear / statistics) */
int dbp_last_kernel(void);

/* Process-wide options for tests and A/B studies; all default to 0
 * (automatic).  Returns the previous value (or DBP_E_ARG).  Nothing in the
 * library reads the environment. */
#define DBP_OPT_KERNEL 0      /* force a DBP_KERNEL_* (it must cover the geometry) */
#define DBP_OPT_TC_SMAX_KB 1  /* tf32 kernel: max stage size (KB) */
#define DBP_OPT_TC_NS 2       /* tensor-core kernels: stage ring depth (cap) */
#define DBP_OPT_TC_PAIR 3     /* tf32 kernel: units per operand tile (1, 2) */
#define DBP_OPT_TC_NSOLV 4    /* tf32 kernel: solver warps */
#define DBP_OPT_SIMT_NS 5     /* SIMT kernel: stage ring depth */
#define DBP_OPT_NO_WIDE 6     /* U = 64: SIMT statistics instead of the tensor cores */
#define DBP_OPT_T2_NSPLIT 7   /* split-bf16 kernel: bf16 parts per operand (2, 3) */
#define DBP_OPT_T2_QUAD 8     /* split-bf16 kernel, u <= 8: 2 = two units per solver pass instead of four */
#define DBP_OPT_WIDE_CHUNK 9  /* FD, U = 64: items per statistics chunk (default ~3 GB of records) */
#define DBP_OPT_LAMA_KERNEL 10 /* LAMA, u <= 32: 1 = the recursion inside the streaming / statistics kernels */
#define DBP_OPT_COUNT 11
int dbp_set_option(int key, int value);
int dbp_device_query(int* sm_count, int* cc_major, int* cc_minor, long long* l2_bytes);

/* Per-cluster Gram + matched filter.  Replaces local_preprocess
 * (equalize.py:85-93); with sum_clusters=1 also fuse_partials
 * (equalize.py:96-107) / centralized_stats (:110-112).
 * offsets: host int32[C+1] row offsets (even).  stats: [n][sum?1:C][...]. */
int dbp_gram_mrc(const void* H, const void* Y, int64_t n_items, int B, int u,
                 int u_stride, int T, int C, const int32_t* offsets,
                 int sum_clusters, void* stats, void* stream);
/* dbp_gram_mrc with the split-bf16 part count of the tensor-core statistics
 * kernels chosen by the caller: 0 = the default (3 parts, ~3xTF32), 2 = two
 * parts (~2^-17 per Gram entry) -- for statistics that feed a well-conditioned
 * PD solve (B >= 4 u), as the multi-GPU PD path uses it (the fused
 * single-GPU PD kernel makes the same choice itself).  No reference
 * counterpart beyond local_preprocess / centralized_stats (equalize.py:85-112). */
int dbp_gram_mrc_parts(const void* H, const void* Y, int64_t n_items, int B, int u,
                       int u_stride, int T, int C, const int32_t* offsets,
                       int sum_clusters, int bf16_parts, void* stats, void* stream);

/* Central equalization from fused statistics.  Replaces linear_equalize
 * (equalize.py:130-176) + unbiased_output (:179-195) for kind MRC/ZF/LMMSE,
 * and lama_equalize (:208-259) for kind LAMA (beta, t_max, damping; the
 * statistics and N0 are multiplied by lama_scale, as cluster_equalize does
 * with 1/w_c, fusion.py:66-68).  Noise: item i uses n0_dev[i / n0_group]
 * when n0_dev != NULL, else n0.  Constellation: square-QAM PAM levels
 * (host float[L], ascending; L=0 for a generic set) and the symbol set
 * (host float[2*M]).  unbias: write z/c and the unbiased sigma2 (L-MMSE);
 * gain (nullable) receives c.  dec (nullable): nearest-symbol indices.
 * tr_* (nullable, LAMA): per-iteration z/s/v [n][t_max][T][u] and
 * phi [n][t_max][T]. */
int dbp_equalize_stats(const void* stats, int64_t n_items, int u, int T,
                       int kind, float n0, const float* n0_dev,
                       int64_t n0_group, float es, int unbias, float beta,
                       float lama_scale, int t_max, float damping,
                       const float* levels, int L, const float* symbols, int M,
                       void* xhat, float* sigma2, float* gain, uint8_t* dec,
                       int32_t* status, int32_t* iters, void* tr_z, void* tr_s,
                       void* tr_v, float* tr_phi, void* stream);

/* Fused single-pass pipeline from (H, Y) to estimates and decisions; the
 * Gram, matched filter and all per-cluster intermediates stay on chip.
 *  arch PD: montecarlo.py:131-145 -- sum of all clusters' statistics, then
 *           the central equalizer (LAMA with beta, lama_scale as above).
 *  arch FD: fd_equalize (fusion.py:127-154) -- per cluster equalization
 *           (LAMA on the rescaled system with beta_c = u/B_c, w_c =
 *           B_c/B_total), unbiasing, inverse-variance (MRC: Gram-diagonal)
 *           weights, fusion; nu receives the weights.
 *  arch FD_PARTIAL: as FD but writes the un-normalised fusion sums
 *           fd_acc [n][2*T*u + 2*wdim] = {sum_c w z, sum_c w, sum_c 1/s2}
 *           and the raw weights fd_wraw [n][C][wdim] (wdim = u, or T for
 *           LAMA) for a cross-GPU sum (dbp_fd_finalize / dbp_fd_weights).
 *  real_counts (host int32[C], nullable): true antenna counts per cluster
 *  when the rows were zero-padded to even counts; B_total = sum of them. */
int dbp_equalize(int arch, int kind, const void* H, const void* Y,
                 int64_t n_items, int B, int u, int u_stride, int T, int C,
                 const int32_t* offsets, const int32_t* real_counts,
                 int B_total, float n0, const float* n0_dev, int64_t n0_group,
                 float es, int unbias, float beta, float lama_scale, int t_max,
                 float damping, const float* levels, int L,
                 const float* symbols, int M, void* xhat, float* sigma2,
                 float* gain, float* nu, uint8_t* dec, int32_t* status,
                 int32_t* iters, float* fd_acc, float* fd_wraw, void* stream);

/* Finish an FD fusion from summed partials (fuse_estimates,
 * fusion.py:108-124): xhat = sum w z / sum w, sigma2 = 1 / sum 1/s2. */
int dbp_fd_finalize(const float* fd_acc, int64_t n_items, int u, int T,
                    int wdim, const float* levels, int L, const float* symbols,
                    int M, void* xhat, float* sigma2, uint8_t* dec,
                    void* stream);

/* nu[n][c][k] = wraw[n][c][k] / den[n][k]  (optimal_fusion_weights,
 * fusion.py:96-105, with the denominator summed over all GPUs). */
int dbp_fd_weights(const float* wraw, const float* den, int64_t n_items,
                   int C, int wdim, float* nu, void* stream);

/* Discrete-posterior mean/variance (kernels.posterior_mean_var,
 * kernels.py:41-50 -> _kernels.pyx:19-71) for n complex entries. */
int dbp_posterior(const void* z, int64_t n, float tau, const float* symbols,
                  int M, void* f_out, float* g_out, void* stream);

/* Nearest-symbol decision, ties to the lowest index (hard_detect,
 * equalize.py:262-268). */
int dbp_hard_detect(const void* z, int64_t n, const float* symbols, int M,
                    int32_t* idx_out, void* stream);

/* fuse_partials (equalize.py:96-107): out[e] = sum_p parts[p*count + e]
 * over `count` complex entries (P stacked statistics records). */
int dbp_stats_sum(const void* parts, int P, int64_t count, void* out, void* stream);

/* unbiased_output (equalize.py:179-195) for z [n][T][u], s2/gain [n][u]:
 * z/c and (s2 - (1-c)^2 Es)/c^2 (clamped at 0); status per item. */
int dbp_unbias(const void* z, const float* s2, const float* gain, int64_t n, int T, int u, float es, void* z_out,
               float* s2_out, int32_t* status, void* stream);

/* optimal_fusion_weights (fusion.py:96-105) for s2 [n][C][u] -> nu [n][C][u];
 * status DBP_ST_BADVAR where some s2 <= 0. */
int dbp_fusion_weights(const float* s2, int64_t n, int C, int u, float* nu, int32_t* status, void* stream);

/* fuse_estimates (fusion.py:108-124) over z, s2, nu [C][count]:
 * z_out = sum_c nu z, s2_out = 1 / sum_c 1/max(s2, 1e-15). */
int dbp_fuse_estimates(const void* z, const float* s2, const float* nu, int C, int64_t count, void* z_out,
                       float* s2_out, void* stream);

/* On-device input synthesis.  Replaces the draws of
 * run_trial / sample_rayleigh_channel / sample_symbols / transmit
 * (montecarlo.py:154-160, model.py:207-236) for whole batches on the GPU:
 * H [n][B][u] ~ CN(0, 1/B), symbol indices [n][T][u] uniform over the M
 * symbols (complex pairs), Y [n][T][B] = H s + CN(0, N0), N0 = n0 or
 * n0_dev[(item0 + i) / n0_group].  Counter-based Philox4x32-10 keyed by seed
 * and the global item index (counter mapping in csrc/dbp_synth.cuh), so any
 * item range is reproducible independently.  sym may be NULL.  B and u even. */
int dbp_synthesize(uint64_t seed, int64_t n_items, int64_t item0, int B, int u, int T, const float* symbols, int M,
                   float n0, const float* n0_dev, int64_t n0_group, void* H, void* Y, uint8_t* sym, void* stream);

/* Soft outputs (no reference counterpart: the
 * reference stops at hard_detect, equalize.py:262-268).  Gray-labelled bit
 * LLRs llr [n][T][u][2 log2 L] (log P(b=0)/P(b=1), bits MSB first, label of
 * symbol k = i L + j is (gray(i) << log2 L) | gray(j), model.gray_labels)
 * from x-hat [n][T][u] under x = s + CN(0, sigma2); sigma2 is [n][u] or, with
 * s2_per_symbol, [n][T] (LAMA).  exact = 0: max-log; 1: log-sum-exp. */
int dbp_llr(const void* xhat, const float* sigma2, int64_t n, int T, int u, int s2_per_symbol, const float* levels,
            int L, int exact, float* llr, void* stream);

/* Hard Gray bits (the north star's "hard decisions as indices plus Gray
 * bits"; SURVEY.md 8(b) dbp_demap bits_out): bits [n][2 log2 L], one byte per
 * bit, MSB first, of symbol indices idx [n] (uint8 decisions when
 * idx_bytes = 1, int32 hard_detect indices when 4); label as in dbp_llr. */
int dbp_gray_bits(const void* idx, int idx_bytes, int64_t n, int L, uint8_t* bits, void* stream);

/* Gauss-Hermite quadratures of the large-system analysis (SURVEY.md 8(f)
 * rank 4; replaces kernels.lama_mse_pam / lama_mse / mi_awgn,
 * _kernels.pyx:74-158), fp64, one value per point x[n] (device): kind 0 =
 * PAM posterior-mean MSE (values = M real levels), 1 = 2-D MSE, 2 = AWGN
 * mutual information in bits (values = M complex symbols interleaved re/im,
 * host); x = sigma^2 (MSE) or the noise variance (MI); nodes / weights = the
 * q-point rule for exp(-x^2) (device); out[n] (device). */
int dbp_quadrature(int kind, const double* x, int64_t n, const double* values, int M, const double* nodes,
                   const double* weights, int q, double* out, void* stream);


/* Batched state evolution of the message-passing equalizer: for each of P
 * points the largest (start = (N0 + beta Es)/w) or smallest (start just above
 * N0/w) solution of w sigma2 = N0 + beta Psi(sigma2), Psi the posterior-mean
 * MSE by the dbp_quadrature rule of kind 0 (PAM levels) or 1 (2-D symbols).
 * Replaces solve_fixed_point / fixed_point_multiplicity
 * (asymptotics.py:75-129) for a whole grid in one launch.  All arrays device
 * (values host as in dbp_quadrature); iters[p] < 0: no convergence. */
int dbp_fixed_point(int kind, const double* n0, const double* beta, const double* w, const double* start, int64_t P,
                    const double* values, int M, const double* nodes, const double* weights, int q, double tol,
                    int max_iter, double* sigma2, int32_t* iters, void* stream);

/* ---- multi-GPU fusion over NCCL (one process per GPU) -------------------
 * The path's one exchange step (the paper fuses one cluster
 * per GPU with ncclReduce to a master; the reference runs its clusters
 * sequentially, fusion.py:141-146, montecarlo.py:132-135), as a sum
 * reduce-scatter by item block so every rank finishes n / nranks items:
 *   PD: sum over clusters of {G_c, y_c^mrc}   -> fuse_partials (equalize.py:96-107)
 *   FD: sum over clusters of {w z, w, 1/s2}   -> fuse_estimates (fusion.py:108-124)
 * plus the all-reduce of the FD weight sums behind nu
 * (optimal_fusion_weights, fusion.py:96-105).  NCCL is loaded at run time
 * (dlopen libnccl.so.2).  Calls are asynchronous on `stream`. */
typedef struct dbp_comm* dbp_comm_t;
/* ncclGetUniqueId: 128 bytes for rank 0 to share with the group */
int dbp_comm_unique_id(void* id128);
/* ncclCommInitRank (collective over the group's ranks) */
int dbp_comm_init(const void* id128, int nranks, int rank, dbp_comm_t* comm);
int dbp_comm_destroy(dbp_comm_t comm);
/* stats_send [nranks * items_per_rank][u*u + T*u] complex64 (this rank's
 * cluster sums, dbp_gram_mrc with sum_clusters = 1) -> stats_recv
 * [items_per_rank][u*u + T*u]: the group sum of items
 * [rank * items_per_rank, (rank + 1) * items_per_rank). */
int dbp_pd_reduce_scatter(dbp_comm_t comm, const void* stats_send, void* stats_recv, int64_t items_per_rank, int u,
                          int T, void* stream);
/* acc_send [nranks * items_per_rank][2*T*u + 2*wdim] float (DBP_ARCH_FD_PARTIAL
 * sums of dbp_equalize) -> acc_recv [items_per_rank][...], then
 * dbp_fd_finalize on the received block. */
int dbp_fd_reduce_scatter(dbp_comm_t comm, const float* acc_send, float* acc_recv, int64_t items_per_rank, int u,
                          int T, int wdim, void* stream);
/* in-place sum over the group (FD weight denominators for dbp_fd_weights) */
int dbp_allreduce_sum(dbp_comm_t comm, float* buf, int64_t count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DBP_B200_H */
