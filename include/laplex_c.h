/*
 * laplex_c.h -- C-ABI of the B200-native LAPLEX hot path (liblaplex_b200.so).
 *
 * Plain pointers and sizes only.  Each entry replaces one reference C++ call
 * (paths under /root/reference/proj/include/laplex/):
 *
 *   laplex_plan_create[_dev]   LaplexOperator(a, b, t[, phi, psi])      operator.hpp:77-137
 *   laplex_plan_transposed     LaplexOperator::transposed()             operator.hpp:157-159
 *   laplex_plan_shape          n() k() temperature() has_phases()       operator.hpp:139-142
 *   laplex_plan_sorted         sorted_rows() / sorted_cols()            operator.hpp:151-152
 *   laplex_plan_ranks          row_buckets() / col_buckets()            operator.hpp:153-154,110-120
 *   laplex_apply[_dev]         matvec / batch_matvec / matvec_transpose operator.hpp:162-188
 *                              / phased_matvec                          operator.hpp:197-213
 *   laplex_backward[_dev]      matvec_vjp / phased_matvec_vjp           gradients.hpp:110-184
 *   laplex_gram[_dev]          weighted_gram / phased_gram              operator.hpp:191-248,371-415
 *   laplex_gram_vjp_weights    gram_vjp_weights                         gradients.hpp:190-219
 *   laplex_sort                sort_anchors                             scan.hpp:27-46
 *   laplex_scan                prefix_decay_scan / suffix_decay_scan    scan.hpp:50-73
 *
 * Errors: every call returns 0 or one of the LAPLEX_E_* codes below, which
 * map 1:1 onto the reference exception types (errors.hpp:8-50); the message
 * of the last failure on the calling thread is laplex_last_error().  Host
 * entry points validate in the reference's order (e.g. phase presence, then
 * lengths, then finiteness) so a C++ wrapper can rethrow the same type.
 *
 * Memory: host entry points take host pointers and return once results are
 * in host memory.  *_dev entry points take device pointers and a
 * cudaStream_t (as void*, NULL = legacy default stream); they are
 * stream-ordered and do not synchronise, except laplex_plan_create_dev which
 * synchronises once to report non-finite anchors synchronously (the _async
 * variant does not).
 *
 * Layout: batches are row-major (rows x cols, leading dimension = cols).
 * Permutations/ranks are returned as uint64 (the reference's size_t).
 * Limits: n, k < 2^31.
 */
#ifndef LAPLEX_C_H
#define LAPLEX_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAPLEX_ABI_VERSION 1

/* dtype tags */
#define LAPLEX_F32 0
#define LAPLEX_F64 1

/* sides */
#define LAPLEX_ROWS 0 /* anchors a, length n (outputs of apply) */
#define LAPLEX_COLS 1 /* anchors b, length k (inputs of apply) */

/* apply / backward / gram flags */
#define LAPLEX_TRANSPOSE 1u /* apply: y = A^T g (matvec_transpose) */
#define LAPLEX_PHASED 2u    /* phased_matvec / phased_matvec_vjp / phased_gram */
/* laplex_apply[_dev]: keep the forward's sorted x (and its tile aggregates) in
 * the plan for the backward -- the autograd "save for backward" of x; one x
 * per plan, replaced by the next save, released when consumed.  The host-
 * pointer laplex_apply keys the saved x by the caller's host pointer. */
#define LAPLEX_SAVE_X 8u
/* laplex_backward[_dev] / laplex_sharded_backward_dev: reuse the x saved by the
 * preceding forward (same X pointer, rows and orientation; the caller asserts X
 * is unchanged) instead of gathering it again -- for the host-pointer
 * laplex_backward, x is then neither uploaded nor re-checked.  Results are
 * bitwise identical; a non-matching X is simply gathered (and uploaded). */
#define LAPLEX_REUSE_X 4u

/* error codes (reference exception types) */
#define LAPLEX_OK 0
#define LAPLEX_E_EMPTY_INPUT 1          /* laplex::EmptyInput */
#define LAPLEX_E_NON_FINITE 2           /* laplex::NonFinite */
#define LAPLEX_E_DIMENSION_MISMATCH 3   /* laplex::DimensionMismatch */
#define LAPLEX_E_PHASE_PRESENT 4        /* laplex::PhasePresent */
#define LAPLEX_E_PHASE_ABSENT 5         /* laplex::PhaseAbsent */
#define LAPLEX_E_ASYMMETRIC_COTANGENT 6 /* laplex::AsymmetricCotangent */
#define LAPLEX_E_INVALID_SIZE 7         /* laplex::InvalidSize (n or k >= 2^31) */
#define LAPLEX_E_INVALID_ARGUMENT 8     /* bad handle / dtype / flag combination */
#define LAPLEX_E_CUDA 100               /* CUDA runtime failure (message in laplex_last_error) */

typedef struct laplex_plan_s* laplex_plan;

int laplex_abi_version(void);
const char* laplex_last_error(void);

/* Plan = the reference constructor: validate, scale by 1/t, stable-sort both
 * anchor sets on the device, merge-path partition.  phi/psi both NULL
 * (unphased) or both non-NULL (lengths n and k). */
int laplex_plan_create(int dtype, const void* a, size_t n, const void* b, size_t k, double t,
                       const void* phi, const void* psi, laplex_plan* out);
int laplex_plan_create_dev(int dtype, const void* a, size_t n, const void* b, size_t k, double t,
                           const void* phi, const void* psi, void* stream, laplex_plan* out);
/* Same as laplex_plan_create_dev without its one host synchronisation (for
 * training loops that build a plan per step): non-finite anchors / phases are
 * then reported by laplex_plan_check (which waits for the build), in the
 * reference's order; the products of a plan with non-finite anchors are
 * undefined.  All other argument errors are still returned immediately. */
int laplex_plan_create_dev_async(int dtype, const void* a, size_t n, const void* b, size_t k, double t,
                                 const void* phi, const void* psi, void* stream, laplex_plan* out);
int laplex_plan_check(laplex_plan plan);
/* Device memory: temporaries and plans come from the library's own
 * stream-ordered pool per device (a caching allocator, separate from the
 * device's default pool): freed blocks stay with it for reuse until
 * laplex_pool_trim, which synchronises the device and returns every unused
 * byte (the analogue of torch.cuda.empty_cache).  LAPLEX_POOL_RESERVE_GB
 * (env) sizes the up-front working-set reservation of large plans (0
 * disables). */
int laplex_pool_trim(void);
/* Reference counting (plans are immutable and shareable across threads and
 * streams; release is stream-ordered after every stream that used the plan
 * and never blocks the host). */
int laplex_plan_retain(laplex_plan plan);
int laplex_plan_release(laplex_plan plan);
/* Role-swapped view sharing the sorted anchors (no re-sort). */
int laplex_plan_transposed(laplex_plan plan, laplex_plan* out);
int laplex_plan_shape(laplex_plan plan, size_t* n, size_t* k, double* t, int* has_phases, int* dtype);
/* Sorted, temperature-scaled anchors of one side (host outputs, any may be
 * NULL): values[m], perm[m] (sorted -> caller index), decays[m-1]. */
int laplex_plan_sorted(laplex_plan plan, int side, void* values, uint64_t* perm, void* decays);
/* Co-ranks (host output):
 *   side ROWS: strict=0 -> j_of_row = #{j : B_j <= A_i}, strict=1 -> #{j : B_j < A_i}
 *   side COLS: strict=0 -> r_of_col = #{i : A_i <= B_j}, strict=1 -> #{i : A_i < B_j}
 * indexed by sorted position, exactly as operator.hpp:110-120. */
int laplex_plan_ranks(laplex_plan plan, int side, int strict, uint64_t* ranks);

/* Y = A X (rows x k -> rows x n), or with LAPLEX_TRANSPOSE Y = A^T X
 * (rows x n -> rows x k), or with LAPLEX_PHASED the phased product.
 * `cols` is the caller's row length (checked -> DimensionMismatch). */
int laplex_apply(laplex_plan plan, unsigned flags, const void* X, size_t rows, size_t cols, void* Y);
int laplex_apply_dev(laplex_plan plan, unsigned flags, const void* X, size_t rows, void* Y, void* stream);

/* Gram-vector product Y = A^T (A X) (rows x k -> rows x k) of an unphased
 * plan: the composition matvec_transpose(matvec(x)) of SPEC.md:187
 * (operator.hpp:162-172) in one call, with A X kept in sorted-row order on
 * the device; bitwise equal to the two-call composition.  Errors as matvec. */
int laplex_gram_apply(laplex_plan plan, const void* X, size_t rows, size_t cols, void* Y);
int laplex_gram_apply_dev(laplex_plan plan, const void* X, size_t rows, void* Y, void* stream);

/* Cotangents of L = sum_r G_r^T A X_r: x_bar (rows x k), a_bar (n) and
 * b_bar (k) summed over rows; with LAPLEX_PHASED also phi_bar (n), psi_bar (k). */
int laplex_backward(laplex_plan plan, unsigned flags, const void* X, size_t rows, size_t xcols,
                    const void* G, size_t gcols, void* x_bar, void* a_bar, void* b_bar, void* phi_bar,
                    void* psi_bar);
int laplex_backward_dev(laplex_plan plan, unsigned flags, const void* X, const void* G, size_t rows,
                        void* x_bar, void* a_bar, void* b_bar, void* phi_bar, void* psi_bar,
                        void* stream);

/* M = A diag(D) A^T (n x n, bit-exactly symmetric); LAPLEX_PHASED: phased_gram. */
int laplex_gram(laplex_plan plan, unsigned flags, const void* D, size_t dlen, void* M);
int laplex_gram_dev(laplex_plan plan, unsigned flags, const void* D, void* M, void* stream);
/* D_bar_t = sum_i K_it (G_bar A)_it for symmetric G_bar (n x n). */
int laplex_gram_vjp_weights(laplex_plan plan, const void* D, size_t dlen, const void* G_bar, size_t grows,
                            size_t gcols, void* D_bar);

/* Device variant: G_bar (n x n) and D_bar (k) are device pointers.  The
 * finiteness / symmetry checks of gradients.hpp:196-205 run on the device and
 * the call synchronises once to report them. */
int laplex_gram_vjp_weights_dev(laplex_plan plan, const void* G_bar, void* D_bar, void* stream);

/* Free functions of scan.hpp: sort_anchors (scan.hpp:27-46) and
 * prefix/suffix_decay_scan (scan.hpp:50-73) on sorted values. */
int laplex_sort(int dtype, const void* raw, size_t m, void* values, uint64_t* perm, void* decays);
int laplex_scan(int dtype, const void* sorted_values, size_t m, const void* payload, void* prefix,
                void* suffix);
/* Device variants.  laplex_sort_dev: values[m], perm[m] (uint32, the device
 * layout), decays[m-1] (may be NULL); with nonfinite == NULL it synchronises
 * once to return NonFinite, else *nonfinite (device int) is set instead and
 * the call is stream-ordered.  laplex_scan_dev: prefix / suffix may be NULL. */
int laplex_sort_dev(int dtype, const void* raw, size_t m, void* values, uint32_t* perm, void* decays,
                    int* nonfinite, void* stream);
int laplex_scan_dev(int dtype, const void* sorted_values, size_t m, const void* payload, void* prefix,
                    void* suffix, void* stream);

/* ---- range-sharded operator (multi-GPU) ----------------------
 * A long vector is split over ranks by VALUE: shard(v) = #{splitters < v} with
 * splitters shared by a and b (equal-value runs never straddle shards).  The
 * caller (paper_2605_24584_b200/sharded.py) moves data with NCCL; these entry
 * points are the per-rank device work.  All device pointers, stream-ordered. */
typedef struct laplex_work_s* laplex_work;
/* Stable partition of raw/t by shard: counts[s] = elements of shard s
 * (s = 0..nsplit), perm[j] = local index of the j-th element in shard order. */
int laplex_shard_partition_dev(int dtype, const void* raw, size_t m, double t, const void* splitters,
                               int nsplit, uint32_t* perm, uint32_t* counts, void* stream);
/* dst[r][j] = src[r*ld_src + idx[j]]  /  dst[r*ld_dst + idx[j]] = src[r][j] */
int laplex_gather_dev(int dtype, const void* src, size_t ld_src, const uint32_t* idx, size_t m, size_t rows,
                      void* dst, void* stream);
int laplex_scatter_dev(int dtype, const void* src, const uint32_t* idx, size_t m, size_t rows, void* dst,
                       size_t ld_dst, void* stream);
/* Plan of one shard's received anchors; one side may be empty (n + k >= 1). */
int laplex_shard_plan_create_dev(int dtype, const void* a, size_t n, const void* b, size_t k, double t,
                                 const void* phi, const void* psi, void* stream, laplex_plan* out);
/* Entries (Real) of a totals / ext array: 3 + 2 * slots * rows, slots = 2 * channels. */
int laplex_shard_totals_count(laplex_plan plan, unsigned flags, int backward, size_t rows, size_t* count);
/* begin: local tile aggregates + carries; writes this shard's totals
 *   [0] last anchor, [1] first anchor, [2] 1, prefix totals [slot][rows], suffix totals [slot][rows].
 * end: folds the external carries ext (same layout; [0] prefix anchor, [1]
 * suffix anchor, [2] flags 1|2 = prefix|suffix present; NULL = none) and
 * writes the outputs (in this shard's received order); releases work. */
int laplex_shard_apply_begin(laplex_plan plan, unsigned flags, const void* X, size_t rows, void* totals,
                             laplex_work* work, void* stream);
int laplex_shard_apply_end(laplex_work work, const void* ext, void* Y, void* stream);
int laplex_shard_backward_begin(laplex_plan plan, unsigned flags, const void* X, const void* G, size_t rows,
                                void* totals, laplex_work* work, void* stream);
int laplex_shard_backward_end(laplex_work work, const void* ext, void* x_bar, void* a_bar, void* b_bar,
                              void* phi_bar, void* psi_bar, void* stream);
int laplex_work_release(laplex_work work);

/* ---- multi-GPU host layer, C++ in the library ---------------
 * Communicators: NCCL (libnccl.so.2 resolved at run time; rank 0 makes the
 * 128-byte id, the caller broadcasts it, every rank calls
 * laplex_comm_init_nccl on its device) or "local" (ranks are threads of one
 * process sharing `key`, e.g. N shards on one GPU).  Collectives are
 * stream-ordered on the stream each call is given. */
typedef struct laplex_comm_s* laplex_comm;
int laplex_nccl_unique_id(void* id128);
int laplex_comm_init_nccl(const void* id128, int world, int rank, laplex_comm* out);
int laplex_comm_init_local(uint64_t key, int world, int rank, laplex_comm* out);
int laplex_comm_destroy(laplex_comm comm);

/* Range-sharded operator over one long vector (B rows): rank r holds caller
 * slices a_r (n_local), b_r (k_local) and passes x_r / g_r / outputs in the
 * same slice order.  Creation = splitters from all-gathered samples, stable
 * partition by value, all-to-all of the anchors, local plan (one host
 * synchronisation: the exchange counts).  apply / backward: payload
 * all-to-alls, one all-gather of the shards' totals folded into external
 * carries on the device, outputs routed back; no host synchronisation.
 * LAPLEX_REUSE_X: backward reuses the x routed by the preceding apply. */
typedef struct laplex_sharded_s* laplex_sharded;
int laplex_sharded_create_dev(laplex_comm comm, int dtype, const void* a, size_t n_local, const void* b,
                              size_t k_local, double t, void* stream, laplex_sharded* out);
int laplex_sharded_shape(laplex_sharded s, size_t* n_recv, size_t* k_recv);
int laplex_sharded_apply_dev(laplex_sharded s, const void* x, size_t rows, void* y, void* stream);
int laplex_sharded_backward_dev(laplex_sharded s, unsigned flags, const void* x, const void* g, size_t rows,
                                void* x_bar, void* a_bar, void* b_bar, void* stream);
int laplex_sharded_release(laplex_sharded s);

/* Batch replicas (C2-C4 on N GPUs): each rank runs laplex_backward_dev on its
 * own rows over a replicated plan; a_bar / b_bar (/ phi_bar / psi_bar), sums
 * over ALL ranks' rows (gradients.hpp:122-133), are combined by an all-gather
 * of the per-rank partials summed in rank order: deterministic, identical on
 * every rank. */
int laplex_replica_backward_dev(laplex_plan plan, laplex_comm comm, unsigned flags, const void* X, const void* G,
                                size_t rows, void* x_bar, void* a_bar, void* b_bar, void* phi_bar, void* psi_bar,
                                void* stream);

/* Number of CUDA kernels this library launched on the calling process
 * (instrumentation for the benchmark's gpu_launches count). */
uint64_t laplex_kernel_launches(void);

/* Optional per-kernel CUDA-event timing: while enabled every kernel launch is
 * bracketed by two events on its stream; laplex_profile_dump synchronises
 * them and writes {"kernel": {"launches": L, "ms": T}, ...} (JSON) into buf,
 * then clears the records. */
int laplex_profile_enable(int on);
int laplex_profile_dump(char* buf, size_t cap);

#ifdef __cplusplus
}
#endif

#endif /* LAPLEX_C_H */
