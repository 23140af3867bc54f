// lx_scan.cuh -- merge-path tiles + bidirectional anchored linear-recurrence
// scans: the LAPLEX forward (matvec), transpose and backward (matvec_vjp).
//
// Reference algorithm being replaced (paths under /root/reference/proj):
//   matvec branch A/B           include/laplex/operator.hpp:319-369
//   prefix/suffix_decay_scan    include/laplex/scan.hpp:50-73
//   co-ranks r_of_col/j_of_row  include/laplex/operator.hpp:110-120
//   row/col split sums (VJP)    include/laplex/gradients.hpp:33-103,110-135
//
// B200 formulation.  Sorted rows A (n) and sorted cols Bh (k) are merged
// (rows first on ties: A_i <= Bh_j puts row i first).  The merged sequence is
// cut into fixed tiles of kTile elements by merge path (lx_partition), so a
// tile needs no co-rank arrays at all.  Inside a tile every element carries an
// anchor s and per-channel payloads (x on column elements, g on row elements);
// one pass computes, per channel,
//   prefix  P_p = sum_{e<=p} exp(s_e - s_p) pay_e
//   suffix  Q_p = sum_{e>=p} exp(s_p - s_e) pay_e
// and the "strict" variants (only elements with a different anchor), which
// give the tie handling of the reference VJP without its O(run) tie walks.
// Forward:  y_i  = P^x(A_i) + Q^x(A_i)                (cols before row i are < A_i,
//                                                    the rest >= A_i)
// Transpose: xb_j = P^g(B_j) + Q^g(B_j)
// VJP:  b_bar_j = x_j/t (Q^g(B_j) - Pstrict^g(B_j)),   a_bar_i = g_i/t (Qstrict^x(A_i) - P^x(A_i))
//
// Numerics: a carry is ALWAYS applied as exp(anchor
// difference) taken from the anchors themselves -- never as a product of
// per-step decays -- except inside one thread's kItems consecutive elements.
// Tile carries are scanned in fp64.
//
// Carries across tiles are lazy: the main kernel writes tile-local results and
// per-tile aggregates; lx_carry scans the aggregates (both directions, fp64);
// the fix-up kernel folds the two carries in with two exps per element and
// scatters to the caller's order.  No inter-CTA waiting in the main pass.
#pragma once

#include "lx_common.cuh"

namespace lx {
namespace ms {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef LX_TILE_ITEMS
#define LX_TILE_ITEMS 8
#endif
constexpr int kItems = LX_TILE_ITEMS;  // kTile = kThreads * kItems merged elements per tile
constexpr int kTile = kThreads * kItems;  // merged elements per tile
constexpr int kFixThreads = 256;

// ---------------------------------------------------------------------------
// merge path
// ---------------------------------------------------------------------------
// Number of A elements among the first `diag` merged elements.  AFIRST:
// A_i precedes B_j iff A_i <= B_j (rows first on ties); otherwise iff A_i < B_j.
template <bool AFIRST, class R, class I>
__device__ __forceinline__ I merge_path(const R* a, I na, const R* b, I nb, I diag) {
    I lo = diag > nb ? diag - nb : 0;
    I hi = diag < na ? diag : na;
    while (lo < hi) {
        const I mid = (lo + hi) >> 1;
        const R av = a[mid];
        const R bv = b[diag - 1 - mid];
        const bool take = AFIRST ? (av <= bv) : (av < bv);
        if (take)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Merge path restricted to A indices [lo, hi) (the answer must lie there).
template <bool AFIRST, class R, class I>
__device__ __forceinline__ I merge_path_in(const R* a, const R* b, I diag, I lo, I hi) {
    while (lo < hi) {
        const I mid = (lo + hi) >> 1;
        const bool take = AFIRST ? (a[mid] <= b[diag - 1 - mid]) : (a[mid] < b[diag - 1 - mid]);
        if (take)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Two-level: the first and last boundary of a block's 256 tiles are searched
// over the whole sequence, then every boundary between them inside that
// bracket (merge path is monotone in the diagonal), so most probes are short
// and hit data the block already touched.  blockDim.x == 256.
template <class R, bool AFIRST>
__global__ void lx_partition(const R* __restrict__ A, uint32_t n, const R* __restrict__ B, uint32_t k,
                             uint32_t* __restrict__ part, uint32_t T) {
    using I = unsigned long long;
    __shared__ I bracket[2];
    const I total = (I)n + k;
    auto diag_of = [&](uint32_t t) { return min((I)t * kTile, total); };
    const uint32_t t0 = blockIdx.x * blockDim.x;
    const uint32_t tl = min(t0 + blockDim.x - 1, T);
    if (threadIdx.x < 2) bracket[threadIdx.x] = merge_path<AFIRST, R, I>(A, n, B, k, diag_of(threadIdx.x ? tl : t0));
    __syncthreads();
    const uint32_t t = t0 + threadIdx.x;
    if (t > T) return;
    const I diag = diag_of(t);
    const I lo = max(bracket[0], diag > k ? diag - k : (I)0);
    const I hi = min(bracket[1], min(diag, (I)n));
    part[t] = (uint32_t)merge_path_in<AFIRST, R, I>(A, B, diag, lo, hi);
}

// Per-tile descriptor, built once per plan orientation: the tile's row/col
// offsets and the anchors of its first and last merged element (the carries'
// reference points).  desc[T] = {n, k} is the sentinel.
template <class R>
struct TileDesc {
    uint32_t a0, b0;
    R s_first, s_last;
};

template <class R>
__global__ void lx_tiledesc(const R* __restrict__ A, uint32_t n, const R* __restrict__ B, uint32_t k,
                            const uint32_t* __restrict__ part, uint32_t T, TileDesc<R>* __restrict__ desc,
                            R* __restrict__ s_first, R* __restrict__ s_last) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > T) return;
    TileDesc<R> d;
    if (t == T) {
        d.a0 = n;
        d.b0 = k;
        d.s_first = d.s_last = R(0);
        desc[t] = d;
        return;
    }
    const uint32_t a0 = part[t], a1 = part[t + 1];
    const unsigned long long d0 = (unsigned long long)t * kTile;
    const unsigned long long total = (unsigned long long)n + k;
    const unsigned long long d1 = d0 + kTile < total ? d0 + kTile : total;
    const uint32_t b0 = (uint32_t)(d0 - a0), b1 = (uint32_t)(d1 - a1);
    d.a0 = a0;
    d.b0 = b0;
    if (a1 == a0) {
        d.s_first = B[b0];
        d.s_last = B[b1 - 1];
    } else if (b1 == b0) {
        d.s_first = A[a0];
        d.s_last = A[a1 - 1];
    } else {
        d.s_first = A[a0] < B[b0] ? A[a0] : B[b0];
        d.s_last = A[a1 - 1] > B[b1 - 1] ? A[a1 - 1] : B[b1 - 1];
    }
    desc[t] = d;
    s_first[t] = d.s_first;
    s_last[t] = d.s_last;
}

// ---------------------------------------------------------------------------
// Merge words (built by lx_group_plan, once per plan orientation): word g of a
// tile covers merged elements [16g, 16g + 16) (rows first on ties, the order
// lx_main consumes); bit q = element 16g + q is a row, bits 16..31 = rows of
// the tile before element 16g.  The main pass then reads its elements' anchors
// with independent shared-memory loads instead of a merge-path search and a
// serial merge.
// ---------------------------------------------------------------------------
constexpr int kMergeGroup = 16;
constexpr int kMergeWords = kTile / kMergeGroup;  // words per tile
static_assert(kItems * 2 == kMergeGroup, "two merge threads per word");

// ---------------------------------------------------------------------------
// co-ranks (accessor path): AFIRST gives J<[i] and R<=[j]; !AFIRST gives
// J<=[i] and R<[j]  (operator.hpp:110-120 are the two tie-inclusive ones).
// ---------------------------------------------------------------------------
template <class R, bool AFIRST>
__global__ void __launch_bounds__(kThreads) lx_coranks(const R* __restrict__ A, uint32_t n,
                                                      const R* __restrict__ B, uint32_t k,
                                                      const uint32_t* __restrict__ part,
                                                      uint32_t* __restrict__ rank_rows,
                                                      uint32_t* __restrict__ rank_cols) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    R* sAB = reinterpret_cast<R*>(smem_raw);
    const uint32_t t = blockIdx.x;
    const uint32_t a0 = part[t], a1 = part[t + 1];
    const unsigned long long d0 = (unsigned long long)t * kTile;
    const unsigned long long total = (unsigned long long)n + k;
    const unsigned long long d1 = d0 + kTile < total ? d0 + kTile : total;
    const uint32_t b0 = (uint32_t)(d0 - a0), b1 = (uint32_t)(d1 - a1);
    const int na = (int)(a1 - a0), nb = (int)(b1 - b0), len = na + nb;
    for (int i = threadIdx.x; i < na; i += kThreads) sAB[i] = A[a0 + i];
    for (int i = threadIdx.x; i < nb; i += kThreads) sAB[na + i] = B[b0 + i];
    __syncthreads();
    const R* sA = sAB;
    const R* sB = sAB + na;
    const int dd = min((int)threadIdx.x * kItems, len);
    int ia = merge_path<AFIRST, R, int>(sA, na, sB, nb, dd);
    int ib = dd - ia;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        if (dd + q < len) {
            const bool takeA = ib >= nb || (ia < na && (AFIRST ? sA[ia] <= sB[ib] : sA[ia] < sB[ib]));
            if (takeA) {
                rank_rows[a0 + ia] = b0 + ib;
                ++ia;
            } else {
                rank_cols[b0 + ib] = a0 + ia;
                ++ib;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// main pass
// ---------------------------------------------------------------------------
template <class R>
struct MainArgs {
    const R* A;
    const uint32_t* perm_a;
    const R* B;
    const uint32_t* perm_b;
    const uint32_t* part;  // T+1 row offsets of the merged tiles
    uint32_t* tile_ctr;    // zeroed tile counter (lx_main's in-order tile schedule)
    // per-tile store order (lx_group_plan): gmt[t * kTile + k] = row-local index
    // of the k-th tile row in output-bucket order (k < na), then the cols
    const uint16_t* gmt;
    const TileDesc<R>* desc;  // T+1 tile descriptors
    const uint32_t* mwords;   // merge words (lx_group_plan): kMergeWords per tile (null: single-sequence SEQ pass)
    uint32_t n, k, T;
    int rows;
    // payloads in SORTED order (lx_gather_agg output), rows x ld (ld % (16/sizeof(R)) == 0)
    const R* Gs;
    size_t ldgs;
    const R* Xs;
    size_t ldxs;
    // payloads are read as X[r*ldx + perm_b[j]] / G[r*ldg + perm_a[i]]: either
    // the caller's arrays with the true permutations, or (large sides) the
    // bucket-staged copies with the plan's pos[] tables (lx_perm_stage_gather)
    const R* X;
    size_t ldx;
    const R* G;
    size_t ldg;
    const R* cpsi;  // phase modulation cos/sin, SORTED order, phased only
    const R* spsi;
    const R* cphi;
    const R* sphi;
    const R* s_last;   // [T] anchor of each tile's last merged element
    const R* s_first;  // [T] anchor of each tile's first merged element
    const R* cp;  // inclusive tile carries (lx_carry), [slot][rows][T]
    const R* cq;
    // external carries from other range shards (multi-GPU): the combined
    // prefix of all lower shards (anchor = their last element, <= every local
    // anchor) and suffix of all higher shards; [slot][rows] like one carry tile
    // device layout: [0] prefix anchor, [1] suffix anchor, [2] flags (1: prefix
    // present, 2: suffix present), then prefix values [slot][rows] and suffix
    // values [slot][rows]; null when the operator is not sharded
    const R* ext;
    R inv_t;
    // final outputs, written at index perm_a[i] / perm_b[j] (caller order, or
    // the bucket-staged position when perm_* holds a plan's pos[] table)
    R* y;       // forward: rows x ldy (row side);  transpose: rows x ldy (col side)
    size_t ldy;
    R* xbar;    // backward: rows x ldxb (col side)
    size_t ldxb;
    R* abar;    // backward: n, summed over rows
    R* bbar;    // backward: k
    R* phibar;  // phased backward
    R* psibar;
    R* pre;     // SEQ: inclusive prefix / suffix, sorted order
    R* suf;
    // row split (batches over few tiles): work item i = (tile i / rsplit, rows
    // [c * rchunk, min(rows, (c + 1) * rchunk)) with c = i % rsplit); the
    // row-summed cotangents of chunk c go to abar/phibar + c * ldpa and
    // bbar/psibar + c * ldpb (summed over chunks by lx_chunk_sum).  rsplit = 1:
    // one item per tile, every row
    uint32_t rsplit;
    int rchunk;
    size_t ldpa, ldpb;
};

// Channel layout: g channels first (c < NG), then x channels.  Strict prefix
// variants exist for g channels and strict suffix variants for x channels, in
// the backward (BWD) configuration only.
template <int NG, int NX, bool BWD>
struct Ch {
    static constexpr int NC = NG + NX;
    static __host__ __device__ constexpr bool pst(int c) { return BWD && c < NG; }
    static __host__ __device__ constexpr bool qst(int c) { return BWD && c >= NG; }
};

constexpr int kGroupBuckets = 256;

// barrier among the TPB consumer threads (named barrier 1; the producer warp is not part of it)
template <int TPB>
__device__ __forceinline__ void cbar() {
    asm volatile("bar.sync 1, %0;" ::"n"(TPB) : "memory");
}

// Plan-time per-tile data consumed by lx_main, built once per plan orientation
// (it depends only on the plan): the store order of both sides (grouping by
// output bucket) and the tile's merge words (see above).
// Shared memory of lx_group_plan: both sides' output positions and anchors
// arrive by TMA (each range at a 16-byte aligned-down start), the store order
// is built in one per-tile array [rows | cols] and leaves with 16-byte stores.
template <class R>
struct GroupSmem {
    static constexpr int kPadU = 4, kPadR = 16 / sizeof(R);
    unsigned long long bar;
    uint32_t gcnt[2][kGroupBuckets];
    uint32_t gwarp[2][kGroupBuckets / 32];
    alignas(16) uint32_t sA[kTile + 2 * kPadU], sB[kTile + 2 * kPadU];
    alignas(16) R mA[kTile + 2 * kPadR], mB[kTile + 2 * kPadR];  // + room for the +inf sentinels
    alignas(16) uint16_t gm[kTile];
};
template <class R>
constexpr size_t group_plan_smem() {
    return sizeof(GroupSmem<R>);
}

// Per merge tile: the merge words and the store order of both sides.  The
// store order lives in a per-tile slot gm[t * kTile + e]: the tile's rows at
// e < na (row-local indices ranked by output bucket), its cols at na + k.
template <class R>
__global__ void __launch_bounds__(kGroupBuckets) lx_group_plan(const TileDesc<R>* __restrict__ desc, uint32_t T,
                                                               const uint32_t* __restrict__ posA, int shA,
                                                               const uint32_t* __restrict__ posB, int shB,
                                                               uint16_t* __restrict__ gmt, const R* __restrict__ A,
                                                               const R* __restrict__ B, uint32_t* __restrict__ words) {
    constexpr int TPB = kGroupBuckets, NW = TPB / 32;
    static_assert(TPB == kThreads, "one merge thread per grouping thread");
    using SM = GroupSmem<R>;
    extern __shared__ __align__(16) unsigned char smem_group[];  // dynamic: > 48 KB
    SM& sm = *reinterpret_cast<SM*>(smem_group);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = blockIdx.x;
    const TileDesc<R> dt = desc[t], dn = desc[t + 1];
    const uint32_t a0 = dt.a0, b0 = dt.b0;
    const int na = (int)(dn.a0 - a0), nb = (int)(dn.b0 - b0), len = na + nb;
    // 16-byte aligned-down starts of the four ranges
    const int oPA = (int)(a0 & (SM::kPadU - 1)), oPB = (int)(b0 & (SM::kPadU - 1));
    const int oMA = (int)(a0 & (SM::kPadR - 1)), oMB = (int)(b0 & (SM::kPadR - 1));
    auto rb = [](int off, int cnt, int esz) { return cnt ? (uint32_t)(((off + cnt) * esz + 15) & ~15) : 0u; };
    const uint32_t bPA = rb(oPA, na, 4), bPB = rb(oPB, nb, 4);
    const uint32_t bMA = rb(oMA, na, (int)sizeof(R)), bMB = rb(oMB, nb, (int)sizeof(R));
    if (tid == 0) {
        mbar_init(&sm.bar, 1);
        fence_mbar_init();
        mbar_expect_tx(&sm.bar, bPA + bPB + bMA + bMB);
        if (bPA) bulk_g2s(sm.sA, posA + (a0 - oPA), bPA, &sm.bar);
        if (bPB) bulk_g2s(sm.sB, posB + (b0 - oPB), bPB, &sm.bar);
        if (bMA) bulk_g2s(sm.mA, A + (a0 - oMA), bMA, &sm.bar);
        if (bMB) bulk_g2s(sm.mB, B + (b0 - oMB), bMB, &sm.bar);
    }
    sm.gcnt[0][tid] = 0u;
    sm.gcnt[1][tid] = 0u;
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(&sm.bar, 0);
    const uint32_t* sA = sm.sA + oPA;
    const uint32_t* sB = sm.sB + oPB;
    R* mA = sm.mA + oMA;
    R* mB = sm.mB + oMB;
    if (tid == 0) {  // +inf behind both ranges: the merge reads past an exhausted side
        const R inf = R(__int_as_float(0x7f800000));
        mA[na] = inf;
        mB[nb] = inf;
    }
    __syncthreads();
    {   // merge words (rows first on ties), kItems merged elements per thread
        const int dd = min(tid * kItems, len);
        const int nval = min(kItems, len - dd);
        int ia = merge_path<true, R, int>(mA, na, mB, nb, dd), ib = dd - ia;
        const int ia0 = ia;
        uint32_t m = 0;
        R av = mA[ia], bv = mB[ib];
        for (int q = 0; q < nval; ++q) {
            const bool takeA = av <= bv;
            m |= (uint32_t)takeA << q;
            if (takeA)
                av = mA[++ia];
            else
                bv = mB[++ib];
        }
        const uint32_t hi = __shfl_down_sync(FULL, m, 1);
        if ((tid & 1) == 0) words[(size_t)t * kMergeWords + tid / 2] = m | (hi << kItems) | ((uint32_t)ia0 << 16);
    }
    // store order: counting sort of each side's elements by output bucket
    for (int li = tid; li < na; li += TPB) atomicAdd(&sm.gcnt[0][sA[li] >> shA], 1u);
    for (int li = tid; li < nb; li += TPB) atomicAdd(&sm.gcnt[1][sB[li] >> shB], 1u);
    __syncthreads();
    {
        const uint32_t c0 = sm.gcnt[0][tid], c1 = sm.gcnt[1][tid];
        uint32_t x0 = c0, x1 = c1;  // inclusive warp scans
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y0 = __shfl_up_sync(FULL, x0, o), y1 = __shfl_up_sync(FULL, x1, o);
            if (lane >= o) {
                x0 += y0;
                x1 += y1;
            }
        }
        if (lane == 31) {
            sm.gwarp[0][warp] = x0;
            sm.gwarp[1][warp] = x1;
        }
        __syncthreads();
        uint32_t w0 = 0, w1 = (uint32_t)na;  // the cols follow the rows in the tile's slot
#pragma unroll
        for (int w = 0; w < NW; ++w)
            if (w < warp) {
                w0 += sm.gwarp[0][w];
                w1 += sm.gwarp[1][w];
            }
        sm.gcnt[0][tid] = w0 + x0 - c0;  // exclusive offsets
        sm.gcnt[1][tid] = w1 + x1 - c1;
    }
    __syncthreads();
    for (int li = tid; li < na; li += TPB) sm.gm[atomicAdd(&sm.gcnt[0][sA[li] >> shA], 1u)] = (uint16_t)li;
    for (int li = tid; li < nb; li += TPB) sm.gm[atomicAdd(&sm.gcnt[1][sB[li] >> shB], 1u)] = (uint16_t)li;
    __syncthreads();
    // the whole slot, 8 entries per 16-byte store (entries past len are don't-care)
    for (int v = tid; v * 8 < len; v += TPB)
        reinterpret_cast<uint4*>(gmt + (size_t)t * kTile)[v] = reinterpret_cast<const uint4*>(sm.gm)[v];
}

// ---------------------------------------------------------------------------
// gather + tile aggregates (one pass per payload side).  For every merge tile
// and row it (1) gathers the side's payload into SORTED order (written
// contiguous, so the main kernel loads it with TMA), and (2) sums per channel
//   prefix  sum_e exp(s_e - S_last) pay_e     (+ strict: only s_e < S_last)
//   suffix  sum_e exp(S_first - s_e) pay_e    (+ strict: only s_e > S_first)
// directly (every term one exp of an anchor difference) in a fixed order
// (thread-strided partials, then a fixed tree): deterministic and independent
// of the batch size.  Rows carry the g channels (prefix-strict in the VJP),
// cols the x channels (suffix-strict in the VJP).
// ---------------------------------------------------------------------------
#ifndef LX_AGG_THREADS
#define LX_AGG_THREADS 256
#endif
constexpr int kAggThreads = LX_AGG_THREADS;

template <class R>
struct GatherAggArgs {
    const TileDesc<R>* desc;
    uint32_t T;
    int rows;
    const R* V;           // this side's sorted anchors
    const uint32_t* idx;  // sorted -> source index (perm or plan pos); null: source already sorted
    const R* src;         // payload source, rows x ld_src
    size_t ld_src;
    R* out;               // payload in sorted order, rows x ld_out
    size_t ld_out;
    const R* cph;         // sorted-order phases (2 channels)
    const R* sph;
    R* aggp;              // [slot][rows][T]
    R* aggq;
    int cbase;            // first channel index of this side
    int rows_per_cta;     // batch rows per CTA (grid.y = row groups)
};

// SIDE_A: the tile range is the rows range; GFORM: g-channel formulas (prefix
// strict) vs x-channel formulas (suffix strict).
// One CTA covers kAggTiles consecutive merge tiles (about kTile elements of
// this side), so every thread has ~kTile/kAggThreads useful loads in flight
// per round trip (the chain is descriptors -> indices/anchors -> payload).
#ifndef LX_AGG_TILES
#define LX_AGG_TILES 4
#endif
// resident CTAs per SM the register budget targets for the two-channel
// (phased) pass, which is latency-bound at 3 (C3: 3.54 -> 2.52 ms at 4); the
// one-channel pass keeps its 74-register, 3-CTA form (a 64-register budget
// spilled and measured 1% slower at 2^30)
#ifndef LX_AGG_CTAS
#define LX_AGG_CTAS 4
#endif
#ifndef LX_AGG1_CTAS
#define LX_AGG1_CTAS 3  // 4 (62 registers, no spills) measured slower: C5 14.6 -> 16.7 ms
#endif
constexpr int kAggTiles = LX_AGG_TILES;

template <class R, int NCH, bool SIDE_A, bool GFORM, bool STRICT>
__global__ void __launch_bounds__(kAggThreads, NCH == 2 ? LX_AGG_CTAS : LX_AGG1_CTAS) lx_gather_agg(GatherAggArgs<R> g) {
    constexpr int NW = kAggThreads / 32;
    constexpr int NT = kAggTiles;
    constexpr int kGI = kTile * NT / 2 / kAggThreads;  // slots for ~the side's share of NT tiles
    constexpr int kSpan = kGI * kAggThreads;
    const uint32_t t0 = blockIdx.x * NT;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t T = g.T;
    const int nt = (int)min((uint32_t)NT, T - t0);  // tiles of this CTA
    uint32_t sb[NT + 1];                             // side offsets of the tiles (+ end)
    R Sf[NT], Sl[NT];
#pragma unroll
    for (int j = 0; j <= NT; ++j) {
        const TileDesc<R> d = g.desc[min(t0 + j, T)];
        sb[j] = SIDE_A ? d.a0 : d.b0;
        if (j < NT) {
            Sf[j] = d.s_first;
            Sl[j] = d.s_last;
        }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j)
        if (j >= nt) sb[j + 1] = sb[j];
    const uint32_t s0 = sb[0];
    const int ns = (int)(sb[NT] - s0);
    const uint32_t* __restrict__ idx = g.idx;
    const R* __restrict__ src = g.src;
    const R* __restrict__ V = g.V;
    R* __restrict__ out = g.out;
    __shared__ R red[NT][4 * NCH][NW];
    // The plan positions of the CTA's range arrive by one TMA bulk copy (16-byte
    // aligned-down start), so the gathers depend on a shared load instead of
    // a per-thread global load, and batch rows reuse them.
    constexpr int kIdxCap = NT * kTile + 8;
    __shared__ alignas(16) uint32_t six[kIdxCap];
    __shared__ unsigned long long ibar;
    const int oI = (int)(s0 & 3u);
    const bool tma_idx = idx != nullptr && ns > 0;
    if (tma_idx) {
        if (tid == 0) {
            mbar_init(&ibar, 1);
            fence_mbar_init();
            const uint32_t bytes = (uint32_t)(((oI + ns) * 4 + 15) & ~15);
            mbar_expect_tx(&ibar, bytes);
            bulk_g2s(six, idx + (s0 - (uint32_t)oI), bytes, &ibar);
        }
        __syncthreads();  // barrier initialised before anyone waits on it
        mbar_wait(&ibar, 0);
    }
    const uint32_t* __restrict__ sx = six + oI;
    // batch rows are split over blockIdx.y (row groups of g.rows_per_cta)
    const int r_lo = (int)blockIdx.y * g.rows_per_cta, r_hi = min(g.rows, r_lo + g.rows_per_cta);
    for (int r = r_lo; r < r_hi; ++r) {
        R pi[NT][NCH], ps[NT][NCH], qi[NT][NCH], qs[NT][NCH];
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int c = 0; c < NCH; ++c) pi[j][c] = ps[j][c] = qi[j][c] = qs[j][c] = R(0);
        // row / range base pointers: 32-bit element offsets below
        const R* __restrict__ srow = src + (size_t)r * g.ld_src;
        R* __restrict__ orow = out + (size_t)r * g.ld_out + s0;
        const R* __restrict__ Vs = V + s0;
        for (int base = 0; base < ns; base += kSpan) {  // one round unless the side dominates
            // all loads of the thread's (up to) kGI elements are issued before use
            R v[kGI], sv[kGI];
#pragma unroll
            for (int q = 0; q < kGI; ++q) {
                const int i = base + tid + q * kAggThreads;
                const uint32_t x = i < ns ? (tma_idx ? sx[i] : s0 + (uint32_t)i) : 0u;
                v[q] = i < ns ? srow[x] : R(0);
                sv[q] = i < ns ? Vs[i] : R(0);
            }
#pragma unroll
            for (int q = 0; q < kGI; ++q) {
                const int i = base + tid + q * kAggThreads;
                if (i >= ns) continue;
                const uint32_t e = s0 + (uint32_t)i;
                orow[i] = v[q];
                const R s = sv[q];
                // the element's tile: one branch target per tile (static
                // accumulator registers, one exp pair per element; the tile of
                // an element is uniform across a warp except at tile edges)
                int jj = 0;
#pragma unroll
                for (int j = 1; j < NT; ++j) jj += e >= sb[j];
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    if (j != jj) continue;  // element of tile t0 + j
                    const R S_first = Sf[j], S_last = Sl[j];
                    const R e1 = xexp(xsub(s, S_last)), e2 = xexp(xsub(S_first, s));
                    R pay[NCH];
                    if constexpr (NCH == 2) {
                        pay[0] = xmul(g.cph[e], v[q]);
                        pay[1] = xmul(g.sph[e], v[q]);
                    } else {
                        pay[0] = v[q];
                    }
#pragma unroll
                    for (int c = 0; c < NCH; ++c) {
                        if constexpr (GFORM) {
                            const R pe = xmul(e1, pay[c]);
                            pi[j][c] = xadd(pi[j][c], pe);
                            if (STRICT && s < S_last) ps[j][c] = xadd(ps[j][c], pe);
                            qi[j][c] = xfma(e2, pay[c], qi[j][c]);
                        } else {
                            pi[j][c] = xfma(e1, pay[c], pi[j][c]);
                            const R qe = xmul(e2, pay[c]);
                            qi[j][c] = xadd(qi[j][c], qe);
                            if (STRICT && S_first < s) qs[j][c] = xadd(qs[j][c], qe);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    pi[j][c] = xadd(pi[j][c], __shfl_xor_sync(FULL, pi[j][c], off));
                    ps[j][c] = xadd(ps[j][c], __shfl_xor_sync(FULL, ps[j][c], off));
                    qi[j][c] = xadd(qi[j][c], __shfl_xor_sync(FULL, qi[j][c], off));
                    qs[j][c] = xadd(qs[j][c], __shfl_xor_sync(FULL, qs[j][c], off));
                }
                if (lane == 0) {
                    red[j][4 * c + 0][warp] = pi[j][c];
                    red[j][4 * c + 1][warp] = ps[j][c];
                    red[j][4 * c + 2][warp] = qi[j][c];
                    red[j][4 * c + 3][warp] = qs[j][c];
                }
            }
        __syncthreads();
        if (tid < NT * 4 * NCH) {
            const int j = tid / (4 * NCH), k = tid % (4 * NCH);
            if (j < nt) {
                R a = red[j][k][0];
#pragma unroll
                for (int w = 1; w < NW; ++w) a = xadd(a, red[j][k][w]);
                const int c = g.cbase + (k >> 2), kind = k & 3;
                const size_t TT = T, t = t0 + j;
                if (kind == 0) g.aggp[((size_t)(2 * c) * g.rows + r) * TT + t] = a;
                if (kind == 1 && STRICT && GFORM) g.aggp[((size_t)(2 * c + 1) * g.rows + r) * TT + t] = a;
                if (kind == 2) g.aggq[((size_t)(2 * c) * g.rows + r) * TT + t] = a;
                if (kind == 3 && STRICT && !GFORM) g.aggq[((size_t)(2 * c + 1) * g.rows + r) * TT + t] = a;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// tile-carry scan (fp64), both directions: grid (rows, 2, blocks)
// out = inclusive scan over tiles; fix-up of tile t reads prefix[t-1], suffix[t+1]
//
// MODE 0: one CTA scans all T elements of a (row, direction).
// MODE 1: CTA z reduces elements [z*chunk, (z+1)*chunk) to one block
//         aggregate (written to bagg*, anchors to bS*).
// MODE 2: like MODE 0 on block z's range, seeded with the inclusive carry of
//         the neighbouring block (bcarry*, produced by MODE 0 over the block
//         aggregates).  MODE 1 -> 0 -> 2 is a reduce-then-scan with every
//         carry applied as exp(anchor difference).
// ---------------------------------------------------------------------------
constexpr int kCarryThreads = 1024;
constexpr uint32_t kCarryBlock = 16384;  // tiles per CTA in the multi-CTA path

template <class R, int NC>
struct CarryArgs {
    const R* aggp;
    const R* aggq;
    R* outp;
    R* outq;
    const R* s_last;
    const R* s_first;
    uint32_t T;
    int rows;
    unsigned pst_mask, qst_mask;
    uint32_t chunk;  // elements per CTA (MODE 1/2)
    uint32_t NB;     // number of CTAs along z
    R* baggp;        // MODE 1 outputs [slot][rows][NB]
    R* baggq;
    R* bs_last;      // [NB]
    R* bs_first;
    const R* bcp;    // MODE 2 inputs: inclusive block carries [slot][rows][NB]
    const R* bcq;
};

template <class R, int NC, int MODE>
__global__ void __launch_bounds__(kCarryThreads) lx_carry(CarryArgs<R, NC> a) {
    const int r = blockIdx.x;
    const bool suffix = blockIdx.y == 1;
    const uint32_t z = blockIdx.z;
    const R* agg = suffix ? a.aggq : a.aggp;
    const R* S = suffix ? a.s_first : a.s_last;
    const unsigned stm = suffix ? a.qst_mask : a.pst_mask;
    const int rows = a.rows;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kCarryThreads / 32;
    const uint32_t lo = MODE == 0 ? 0 : z * a.chunk;
    const uint32_t hi = MODE == 0 ? a.T : min(a.T, lo + a.chunk);
    const uint32_t cnt = hi - lo;
    const size_t TT = a.T;
    const uint32_t per = (cnt + kCarryThreads - 1) / kCarryThreads;
    // scan order q -> array position
    auto pos = [&](uint32_t q) -> uint32_t { return suffix ? hi - 1 - q : lo + q; };
    const uint32_t q0 = (uint32_t)tid * per;
    const uint32_t q1 = min(q0 + per, cnt);
    auto at = [&](int c, int st, uint32_t u) -> double { return (double)agg[((size_t)(2 * c + st) * rows + r) * TT + u]; };
    // combine "state (sa, v, w)" with element at anchor su (scan order: state precedes element)
    auto step = [&](double& sa, double* v, double* w, bool& has, double su, const double* ev, const double* ew) {
        if (!has) {
            for (int c = 0; c < NC; ++c) {
                v[c] = ev[c];
                w[c] = ew[c];
            }
            has = true;
        } else {
            const double e = suffix ? exp(su - sa) : exp(sa - su);
            const bool lt = suffix ? su < sa : sa < su;
            for (int c = 0; c < NC; ++c) {
                if ((stm >> c) & 1) w[c] = ew[c] + (lt ? e * v[c] : w[c]);
                v[c] = fma(e, v[c], ev[c]);
            }
        }
        sa = su;
    };
    // pass 1: per-thread chunk aggregate
    double v[NC], w[NC];
    double sa = (double)S[suffix ? lo : hi - 1];  // identity padding at the far end of the scan
    bool has = false;
    for (int c = 0; c < NC; ++c) v[c] = w[c] = 0.0;
    for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t u = pos(q);
        double ev[NC], ew[NC];
        for (int c = 0; c < NC; ++c) {
            ev[c] = at(c, 0, u);
            ew[c] = ((stm >> c) & 1) ? at(c, 1, u) : 0.0;
        }
        step(sa, v, w, has, (double)S[u], ev, ew);
    }
    // warp-level inclusive Kogge-Stone over thread aggregates
    double kv[NC], kw[NC];
    for (int c = 0; c < NC; ++c) {
        kv[c] = v[c];
        kw[c] = w[c];
    }
    for (int j = 0; j < 5; ++j) {
        const int off = 1 << j;
        const double so = __shfl_up_sync(FULL, sa, off);
        const double e = exp(suffix ? sa - so : so - sa);
        const bool lt = suffix ? sa < so : so < sa;
        for (int c = 0; c < NC; ++c) {
            const double vo = __shfl_up_sync(FULL, kv[c], off);
            const double wo = __shfl_up_sync(FULL, kw[c], off);
            if (lane >= off) {
                if ((stm >> c) & 1) kw[c] = kw[c] + (lt ? e * vo : wo);
                kv[c] = fma(e, vo, kv[c]);
            }
        }
    }
    __shared__ double w_sa[NW], w_v[NC][NW], w_w[NC][NW];
    __shared__ double x_sa[NW], x_v[NC][NW], x_w[NC][NW];
    __shared__ int x_has[NW];
    if (lane == 31) {
        w_sa[warp] = sa;
        for (int c = 0; c < NC; ++c) {
            w_v[c][warp] = kv[c];
            w_w[c][warp] = kw[c];
        }
    }
    __syncthreads();
    if (tid == 0) {
        double ca = 0.0, cv[NC], cw[NC];
        bool ch = false;
        for (int c = 0; c < NC; ++c) cv[c] = cw[c] = 0.0;
        if (MODE == 2) {
            // seed with the inclusive carry of the neighbouring block in scan order
            const bool hasn = suffix ? (z + 1 < a.NB) : (z > 0);
            if (hasn) {
                const uint32_t nb = suffix ? z + 1 : z - 1;
                const R* bc = suffix ? a.bcq : a.bcp;
                const R* bS = suffix ? a.s_first : a.s_last;
                // anchor of that carry = anchor of the neighbouring block's edge element
                ca = (double)bS[suffix ? (nb * a.chunk) : min(a.T, (nb + 1) * a.chunk) - 1];
                for (int c = 0; c < NC; ++c) {
                    cv[c] = (double)bc[((size_t)(2 * c) * rows + r) * a.NB + nb];
                    cw[c] = ((stm >> c) & 1) ? (double)bc[((size_t)(2 * c + 1) * rows + r) * a.NB + nb] : 0.0;
                }
                ch = true;
            }
        }
        for (int u = 0; u < NW; ++u) {
            x_has[u] = ch;
            x_sa[u] = ca;
            for (int c = 0; c < NC; ++c) {
                x_v[c][u] = cv[c];
                x_w[c][u] = cw[c];
            }
            double ev[NC], ew[NC];
            for (int c = 0; c < NC; ++c) {
                ev[c] = w_v[c][u];
                ew[c] = w_w[c][u];
            }
            step(ca, cv, cw, ch, w_sa[u], ev, ew);
        }
        if (MODE == 1) {
            R* bo = suffix ? a.baggq : a.baggp;
            for (int c = 0; c < NC; ++c) {
                bo[((size_t)(2 * c) * rows + r) * a.NB + z] = (R)cv[c];
                if ((stm >> c) & 1) bo[((size_t)(2 * c + 1) * rows + r) * a.NB + z] = (R)cw[c];
            }
            if (r == 0) {
                if (suffix)
                    a.bs_first[z] = S[lo];
                else
                    a.bs_last[z] = S[hi - 1];
            }
        }
    }
    if (MODE == 1) return;
    __syncthreads();
    // exclusive carry-in for this thread: warp exclusive (+) lane exclusive
    bool hin = x_has[warp] != 0;
    double ia = x_sa[warp], iv[NC], iw[NC];
    for (int c = 0; c < NC; ++c) {
        iv[c] = x_v[c][warp];
        iw[c] = x_w[c][warp];
    }
    {
        const double la = __shfl_up_sync(FULL, sa, 1);
        double lv[NC], lw[NC];
        for (int c = 0; c < NC; ++c) {
            lv[c] = __shfl_up_sync(FULL, kv[c], 1);
            lw[c] = __shfl_up_sync(FULL, kw[c], 1);
        }
        if (lane > 0) {
            if (hin) {
                const double e = exp(suffix ? la - ia : ia - la);
                const bool lt = suffix ? la < ia : ia < la;
                for (int c = 0; c < NC; ++c) {
                    if ((stm >> c) & 1) lw[c] = lw[c] + (lt ? e * iv[c] : iw[c]);
                    lv[c] = fma(e, iv[c], lv[c]);
                }
            }
            hin = true;
            ia = la;
            for (int c = 0; c < NC; ++c) {
                iv[c] = lv[c];
                iw[c] = lw[c];
            }
        }
    }
    // pass 2: rescan the chunk with the carry-in and write inclusive values
    R* out = suffix ? a.outq : a.outp;
    for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t u = pos(q);
        double ev[NC], ew[NC];
        for (int c = 0; c < NC; ++c) {
            ev[c] = at(c, 0, u);
            ew[c] = ((stm >> c) & 1) ? at(c, 1, u) : 0.0;
        }
        step(ia, iv, iw, hin, (double)S[u], ev, ew);
        for (int c = 0; c < NC; ++c) {
            out[((size_t)(2 * c) * rows + r) * TT + u] = (R)iv[c];
            if ((stm >> c) & 1) out[((size_t)(2 * c + 1) * rows + r) * TT + u] = (R)iw[c];
        }
    }
}

__global__ void lx_seq_partition(uint32_t n, uint32_t* __restrict__ part, uint32_t T) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > T) return;
    const unsigned long long d = (unsigned long long)t * kTile;
    part[t] = (uint32_t)(d < n ? d : n);
}

// ---------------------------------------------------------------------------
// single-sequence scans on already-sorted anchors (prefix_decay_scan,
// suffix_decay_scan; scan.hpp:50-73): the merged machinery with every element
// a "row" carrying its own payload.  Implemented as a merged pass with k = 0
// in which row elements carry x payload -- see lx_seq_* in lx_capi.cu.
// ---------------------------------------------------------------------------

}  // namespace ms
}  // namespace lx
