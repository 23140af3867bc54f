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
constexpr int kItems = 8;
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

template <class R, bool AFIRST>
__global__ void lx_partition(const R* __restrict__ A, uint32_t n, const R* __restrict__ B, uint32_t k,
                             uint32_t* __restrict__ part, uint32_t T) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > T) return;
    const unsigned long long total = (unsigned long long)n + k;
    unsigned long long diag = (unsigned long long)t * kTile;
    if (diag > total) diag = total;
    part[t] = (uint32_t)merge_path<AFIRST, R, unsigned long long>(A, n, B, k, diag);
}

// Per-thread merge of kItems consecutive merged positions of one tile held in
// shared memory (sA = tile rows, sB = tile cols).
template <bool AFIRST, class R>
struct TileMerge {
    int ia, ib;  // counters at the thread's first item
};

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
    uint32_t n, k, T;
    int rows;
    const R* X;  // payload on columns, rows x ldx, caller order
    size_t ldx;
    const R* G;  // payload on rows, rows x ldg, caller order
    size_t ldg;
    const R* cpsi;  // phase modulation (caller order), phased only
    const R* spsi;
    const R* cphi;
    const R* sphi;
    R* wa[2];   // row-side outputs per x channel, [rows][n] sorted order
    R* wa2[2];  // phased backward: P^x + Q^x at rows
    R* wb[2];   // col-side outputs per g channel, [rows][k] sorted order
    R* wb2[2];  // backward: Q^g - Pstrict^g at cols
    R* gsave;   // backward: gathered g, [rows][n] sorted order
    R* xsave;   // backward: gathered x, [rows][k] sorted order
    R* aggp;    // [slot][rows][T] prefix tile aggregates, slot = 2*c + strict
    R* aggq;    // suffix tile aggregates
    R* s_last;  // [T] anchor of each tile's last merged element
    R* s_first; // [T] anchor of each tile's first merged element
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

template <class R, int NG, int NX>
struct MainSmem {
    static constexpr int NC = NG + NX;
    R wsl[kWarps];  // warp last anchors
    R wsf[kWarps];  // warp first anchors
    R pv[NC][kWarps], pw[NC][kWarps];  // warp prefix totals (inclusive, strict)
    R qv[NC][kWarps], qw[NC][kWarps];  // warp suffix totals
    R xpv[NC][kWarps], xpw[NC][kWarps];  // warp exclusive prefix
    R xqv[NC][kWarps], xqw[NC][kWarps];  // warp exclusive suffix
};

// SEQ: single sorted sequence (k = 0, part[t] = t*kTile): every element is a
// "row" carrying its own payload X[r][i] (sorted order) and receiving both the
// inclusive prefix (wa[0]) and inclusive suffix (wa2[0]) -- the free functions
// prefix_decay_scan / suffix_decay_scan of scan.hpp:50-73.
template <class R, int NG, int NX, bool BWD, bool SEQ = false>
__global__ void __launch_bounds__(kThreads, 2) lx_main(MainArgs<R> p) {
    using C = Ch<NG, NX, BWD>;
    constexpr int NC = C::NC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MainSmem<R, NG, NX>& sm = *reinterpret_cast<MainSmem<R, NG, NX>*>(smem_raw);
    R* sAB = reinterpret_cast<R*>(smem_raw + ((sizeof(MainSmem<R, NG, NX>) + 15) & ~size_t(15)));

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t t = blockIdx.x;
    const uint32_t a0 = p.part[t], a1 = p.part[t + 1];
    const unsigned long long d0 = (unsigned long long)t * kTile;
    const unsigned long long total = (unsigned long long)p.n + p.k;
    const unsigned long long d1 = d0 + kTile < total ? d0 + kTile : total;
    const uint32_t b0 = (uint32_t)(d0 - a0), b1 = (uint32_t)(d1 - a1);
    const int na = (int)(a1 - a0), nb = (int)(b1 - b0), len = na + nb;

    for (int i = tid; i < na; i += kThreads) sAB[i] = p.A[a0 + i];
    for (int i = tid; i < nb; i += kThreads) sAB[na + i] = p.B[b0 + i];
    __syncthreads();
    const R* sA = sAB;
    const R* sB = sAB + na;
    // anchor of the tile's last merged element (pads trailing empty slots)
    R s_end;
    if (na == 0)
        s_end = sB[nb - 1];
    else if (nb == 0)
        s_end = sA[na - 1];
    else
        s_end = sA[na - 1] > sB[nb - 1] ? sA[na - 1] : sB[nb - 1];

    // ---- per-thread merge: anchors, kind, local index ----
    R s[kItems];
    uint32_t code[kItems];  // bit31 row element, bit30 valid, low bits local index
    {
        const int dd = min(tid * kItems, len);
        int ia = merge_path<true, R, int>(sA, na, sB, nb, dd);
        int ib = dd - ia;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            if (dd + q < len) {
                const bool takeA = ib >= nb || (ia < na && sA[ia] <= sB[ib]);
                if (takeA) {
                    s[q] = sA[ia];
                    code[q] = 0xC0000000u | (uint32_t)ia;
                    ++ia;
                } else {
                    s[q] = sB[ib];
                    code[q] = 0x40000000u | (uint32_t)ib;
                    ++ib;
                }
            } else {
                s[q] = s_end;
                code[q] = 0;
            }
        }
    }

    // ---- row-independent geometry: all exps are taken from anchor differences ----
    R E[kItems];  // E[q] = exp(s[q-1] - s[q])
    E[0] = R(0);
#pragma unroll
    for (int q = 1; q < kItems; ++q) E[q] = xexp(xsub(s[q - 1], s[q]));
    const R sl = s[kItems - 1], sf = s[0];
    R eP[5], eQ[5];
    unsigned ltP = 0, ltQ = 0;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int off = 1 << j;
        const R so = shfl_up(sl, off);
        const R sq = shfl_down(sf, off);
        eP[j] = lane >= off ? xexp(xsub(so, sl)) : R(0);
        if (lane >= off && so < sl) ltP |= 1u << j;
        eQ[j] = lane + off < 32 ? xexp(xsub(sf, sq)) : R(0);
        if (lane + off < 32 && sf < sq) ltQ |= 1u << j;
    }
    if (lane == 31) sm.wsl[warp] = sl;
    if (lane == 0) sm.wsf[warp] = sf;
    const R S1 = shfl_up(sl, 1);   // previous lane's last anchor
    const R S1q = shfl_down(sf, 1);  // next lane's first anchor
    __syncthreads();
    // warp-0 geometry for the scan over warp totals
    R eBP[5], eBQ[5];
    unsigned ltBP = 0, ltBQ = 0;
    if (warp == 0) {
        const R wl = lane < kWarps ? sm.wsl[lane] : sm.wsl[kWarps - 1];
        const R wf = lane < kWarps ? sm.wsf[lane] : sm.wsf[kWarps - 1];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int off = 1 << j;
            const R so = shfl_up(wl, off);
            const R sq = shfl_down(wf, off);
            eBP[j] = lane >= off ? xexp(xsub(so, wl)) : R(0);
            if (lane >= off && so < wl) ltBP |= 1u << j;
            eBQ[j] = lane + off < 32 ? xexp(xsub(wf, sq)) : R(0);
            if (lane + off < 32 && wf < sq) ltBQ |= 1u << j;
        }
    }
    // thread-exclusive anchors and the exps that fold them into each item
    const bool hasP = tid > 0, hasQ = tid < kThreads - 1;
    const R SW = warp > 0 ? sm.wsl[warp - 1] : sf;          // prev warp's last anchor
    const R SWq = warp < kWarps - 1 ? sm.wsf[warp + 1] : sl;  // next warp's first anchor
    const R eTW = (lane > 0 && warp > 0) ? xexp(xsub(SW, S1)) : R(0);
    const bool ltTW = SW < S1;
    const R eTWq = (lane < 31 && warp < kWarps - 1) ? xexp(xsub(S1q, SWq)) : R(0);
    const bool ltTWq = S1q < SWq;
    const R SE = lane > 0 ? S1 : SW;
    const R SEq = lane < 31 ? S1q : SWq;
    R eI[kItems], eIq[kItems];
    unsigned ltI = 0, ltIq = 0;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        eI[q] = hasP ? xexp(xsub(SE, s[q])) : R(0);
        if (SE < s[q]) ltI |= 1u << q;
        eIq[q] = hasQ ? xexp(xsub(s[q], SEq)) : R(0);
        if (s[q] < SEq) ltIq |= 1u << q;
    }

    const R* cphi = p.cphi;
    const R* sphi = p.sphi;
    const R* cpsi = p.cpsi;
    const R* spsi = p.spsi;
    const size_t T = p.T;

    for (int r = 0; r < p.rows; ++r) {
        // ---- payloads ----
        R pay[NC][kItems];
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
#pragma unroll
            for (int c = 0; c < NC; ++c) pay[c][q] = R(0);
            const uint32_t cd = code[q];
            if (!(cd & 0x40000000u)) continue;
            const uint32_t li = cd & 0x3fffffffu;
            if (cd & 0x80000000u) {
                if constexpr (SEQ) {
                    pay[0][q] = p.X[(size_t)r * p.ldx + a0 + li];
                } else if constexpr (NG > 0) {
                    const uint32_t u = p.perm_a[a0 + li];
                    const R g = p.G[(size_t)r * p.ldg + u];
                    if constexpr (BWD) p.gsave[(size_t)r * p.n + a0 + li] = g;
                    if constexpr (NG == 2) {
                        pay[0][q] = xmul(cphi[u], g);
                        pay[1][q] = xmul(sphi[u], g);
                    } else {
                        pay[0][q] = g;
                    }
                }
            } else {
                if constexpr (NX > 0) {
                    const uint32_t u = p.perm_b[b0 + li];
                    const R x = p.X[(size_t)r * p.ldx + u];
                    if constexpr (BWD) p.xsave[(size_t)r * p.k + b0 + li] = x;
                    if constexpr (NX == 2) {
                        pay[NG][q] = xmul(cpsi[u], x);
                        pay[NG + 1][q] = xmul(spsi[u], x);
                    } else {
                        pay[NG][q] = x;
                    }
                }
            }
        }

        // ---- prefix: thread-serial, warp Kogge-Stone, block ----
        R pi[NC][kItems], ps[NC][kItems];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            pi[c][0] = pay[c][0];
            ps[c][0] = R(0);
#pragma unroll
            for (int q = 1; q < kItems; ++q) {
                if (C::pst(c)) ps[c][q] = (s[q - 1] < s[q]) ? xmul(E[q], pi[c][q - 1]) : ps[c][q - 1];
                pi[c][q] = xfma(E[q], pi[c][q - 1], pay[c][q]);
            }
        }
        R v[NC], w[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            v[c] = pi[c][kItems - 1];
            w[c] = C::pst(c) ? ps[c][kItems - 1] : R(0);
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int off = 1 << j;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const R vo = shfl_up(v[c], off);
                if (C::pst(c)) {
                    const R wo = shfl_up(w[c], off);
                    if (lane >= off) w[c] = xadd(w[c], ((ltP >> j) & 1) ? xmul(eP[j], vo) : wo);
                }
                if (lane >= off) v[c] = xfma(eP[j], vo, v[c]);
            }
        }
        // ---- suffix: thread-serial, warp Kogge-Stone ----
        R qi[NC][kItems], qs[NC][kItems];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            qi[c][kItems - 1] = pay[c][kItems - 1];
            qs[c][kItems - 1] = R(0);
#pragma unroll
            for (int q = kItems - 2; q >= 0; --q) {
                if (C::qst(c)) qs[c][q] = (s[q] < s[q + 1]) ? xmul(E[q + 1], qi[c][q + 1]) : qs[c][q + 1];
                qi[c][q] = xfma(E[q + 1], qi[c][q + 1], pay[c][q]);
            }
        }
        R vq[NC], wq[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            vq[c] = qi[c][0];
            wq[c] = C::qst(c) ? qs[c][0] : R(0);
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int off = 1 << j;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const R vo = shfl_down(vq[c], off);
                if (C::qst(c)) {
                    const R wo = shfl_down(wq[c], off);
                    if (lane + off < 32) wq[c] = xadd(wq[c], ((ltQ >> j) & 1) ? xmul(eQ[j], vo) : wo);
                }
                if (lane + off < 32) vq[c] = xfma(eQ[j], vo, vq[c]);
            }
        }
        // ---- warp totals -> block scan in warp 0 ----
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (lane == 31) {
                sm.pv[c][warp] = v[c];
                sm.pw[c][warp] = w[c];
            }
            if (lane == 0) {
                sm.qv[c][warp] = vq[c];
                sm.qw[c][warp] = wq[c];
            }
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                R bv = lane < kWarps ? sm.pv[c][lane] : R(0);
                R bw = lane < kWarps ? sm.pw[c][lane] : R(0);
                R cv = lane < kWarps ? sm.qv[c][lane] : R(0);
                R cw = lane < kWarps ? sm.qw[c][lane] : R(0);
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    const int off = 1 << j;
                    const R vo = shfl_up(bv, off);
                    const R wo = shfl_up(bw, off);
                    const R vqo = shfl_down(cv, off);
                    const R wqo = shfl_down(cw, off);
                    if (lane >= off) {
                        if (C::pst(c)) bw = xadd(bw, ((ltBP >> j) & 1) ? xmul(eBP[j], vo) : wo);
                        bv = xfma(eBP[j], vo, bv);
                    }
                    if (lane + off < 32) {
                        if (C::qst(c)) cw = xadd(cw, ((ltBQ >> j) & 1) ? xmul(eBQ[j], vqo) : wqo);
                        cv = xfma(eBQ[j], vqo, cv);
                    }
                }
                // exclusive per warp (prefix from lane-1, suffix from lane+1)
                const R xv = shfl_up(bv, 1), xw = shfl_up(bw, 1);
                const R yv = shfl_down(cv, 1), yw = shfl_down(cw, 1);
                if (lane < kWarps) {
                    sm.xpv[c][lane] = xv;
                    sm.xpw[c][lane] = xw;
                    sm.xqv[c][lane] = yv;
                    sm.xqw[c][lane] = yw;
                }
                // tile aggregates (inclusive over the whole tile)
                if (lane == kWarps - 1) {
                    p.aggp[((size_t)(2 * c) * p.rows + r) * T + t] = bv;
                    if (C::pst(c)) p.aggp[((size_t)(2 * c + 1) * p.rows + r) * T + t] = bw;
                }
                if (lane == 0) {
                    p.aggq[((size_t)(2 * c) * p.rows + r) * T + t] = cv;
                    if (C::qst(c)) p.aggq[((size_t)(2 * c + 1) * p.rows + r) * T + t] = cw;
                }
            }
        }
        // lane-exclusive values within the warp
        R V1[NC], W1[NC], V1q[NC], W1q[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            V1[c] = shfl_up(v[c], 1);
            W1[c] = shfl_up(w[c], 1);
            V1q[c] = shfl_down(vq[c], 1);
            W1q[c] = shfl_down(wq[c], 1);
        }
        __syncthreads();

        // ---- thread-exclusive carries, item finals ----
        R fp[NC][kItems], fps[NC][kItems], fq[NC][kItems], fqs[NC][kItems];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            R VE = R(0), WE = R(0), VEq = R(0), WEq = R(0);
            if (lane > 0) {
                VE = V1[c];
                WE = W1[c];
                if (warp > 0) {
                    const R VW = sm.xpv[c][warp], WW = sm.xpw[c][warp];
                    if (C::pst(c)) WE = xadd(W1[c], ltTW ? xmul(eTW, VW) : WW);
                    VE = xfma(eTW, VW, V1[c]);
                }
            } else if (warp > 0) {
                VE = sm.xpv[c][warp];
                WE = sm.xpw[c][warp];
            }
            if (lane < 31) {
                VEq = V1q[c];
                WEq = W1q[c];
                if (warp < kWarps - 1) {
                    const R VW = sm.xqv[c][warp], WW = sm.xqw[c][warp];
                    if (C::qst(c)) WEq = xadd(W1q[c], ltTWq ? xmul(eTWq, VW) : WW);
                    VEq = xfma(eTWq, VW, V1q[c]);
                }
            } else if (warp < kWarps - 1) {
                VEq = sm.xqv[c][warp];
                WEq = sm.xqw[c][warp];
            }
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                fp[c][q] = xfma(eI[q], VE, pi[c][q]);
                if (C::pst(c)) fps[c][q] = xadd(ps[c][q], ((ltI >> q) & 1) ? xmul(eI[q], VE) : WE);
                fq[c][q] = xfma(eIq[q], VEq, qi[c][q]);
                if (C::qst(c)) fqs[c][q] = xadd(qs[c][q], ((ltIq >> q) & 1) ? xmul(eIq[q], VEq) : WEq);
            }
        }

        // ---- outputs (sorted order; the fix-up pass scatters) ----
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const uint32_t cd = code[q];
            if (!(cd & 0x40000000u)) continue;
            const uint32_t li = cd & 0x3fffffffu;
            if (cd & 0x80000000u) {
                const size_t o = (size_t)r * p.n + a0 + li;
                if constexpr (SEQ) {
                    p.wa[0][o] = fp[0][q];
                    p.wa2[0][o] = fq[0][q];
                    continue;
                }
#pragma unroll
                for (int c = NG; c < NC; ++c) {
                    if constexpr (BWD) {
                        p.wa[c - NG][o] = xsub(fqs[c][q], fp[c][q]);
                        if constexpr (NX == 2) p.wa2[c - NG][o] = xadd(fp[c][q], fq[c][q]);
                    } else {
                        p.wa[c - NG][o] = xadd(fp[c][q], fq[c][q]);
                    }
                }
            } else {
                const size_t o = (size_t)r * p.k + b0 + li;
#pragma unroll
                for (int c = 0; c < NG; ++c) {
                    p.wb[c][o] = xadd(fp[c][q], fq[c][q]);
                    if constexpr (BWD) p.wb2[c][o] = xsub(fq[c][q], fps[c][q]);
                }
            }
        }
    }
    if (tid == 0) {
        p.s_last[t] = s_end;
        p.s_first[t] = na == 0 ? sB[0] : (nb == 0 ? sA[0] : (sA[0] < sB[0] ? sA[0] : sB[0]));
    }
}

// ---------------------------------------------------------------------------
// tile-carry scan (fp64), both directions: grid (rows, 2)
// out = inclusive scan over tiles; fix-up of tile t reads prefix[t-1], suffix[t+1]
// ---------------------------------------------------------------------------
constexpr int kCarryThreads = 1024;

template <class R, int NC>
__global__ void __launch_bounds__(kCarryThreads) lx_carry(const R* __restrict__ aggp, const R* __restrict__ aggq,
                                                         R* __restrict__ cp, R* __restrict__ cq,
                                                         const R* __restrict__ s_last,
                                                         const R* __restrict__ s_first, uint32_t T, int rows,
                                                         unsigned pst_mask, unsigned qst_mask) {
    const int r = blockIdx.x;
    const bool suffix = blockIdx.y == 1;
    const R* agg = suffix ? aggq : aggp;
    R* out = suffix ? cq : cp;
    const R* S = suffix ? s_first : s_last;
    const unsigned stm = suffix ? qst_mask : pst_mask;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kCarryThreads / 32;
    const uint32_t chunk = (T + kCarryThreads - 1) / kCarryThreads;
    // suffix direction: thread tid owns the chunk counted from the right
    auto pos = [&](uint32_t q) -> uint32_t { return suffix ? T - 1 - q : q; };
    const uint32_t q0 = (uint32_t)tid * chunk;
    const uint32_t q1 = min(q0 + chunk, T);
    auto at = [&](int c, int st, uint32_t u) -> double {
        return (double)agg[((size_t)(2 * c + st) * rows + r) * T + u];
    };
    // pass 1: chunk aggregate (anchor = last element of the chunk in scan order)
    double v[NC], w[NC];
    double sa;  // anchor of running aggregate
    for (int c = 0; c < NC; ++c) v[c] = w[c] = 0.0;
    sa = (double)S[pos(T - 1)];  // identity padding (never ahead of real elements)
    bool has = false;
    for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t u = pos(q);
        const double su = (double)S[u];
        if (!has) {
            for (int c = 0; c < NC; ++c) {
                v[c] = at(c, 0, u);
                w[c] = ((stm >> c) & 1) ? at(c, 1, u) : 0.0;
            }
            has = true;
        } else {
            const double e = suffix ? exp(su - sa) : exp(sa - su);
            const bool lt = suffix ? su < sa : sa < su;
            for (int c = 0; c < NC; ++c) {
                if ((stm >> c) & 1) w[c] = at(c, 1, u) + (lt ? e * v[c] : w[c]);
                v[c] = fma(e, v[c], at(c, 0, u));
            }
        }
        sa = su;
    }
    // block exclusive scan of chunk aggregates (sequential in warp 0 over warps)
    __shared__ double s_sa[kCarryThreads];
    __shared__ double s_v[NC][kCarryThreads];
    __shared__ double s_w[NC][kCarryThreads];
    s_sa[tid] = sa;
    for (int c = 0; c < NC; ++c) {
        s_v[c][tid] = v[c];
        s_w[c][tid] = w[c];
    }
    __syncthreads();
    // warp-level inclusive KS over thread aggregates
    double kv[NC], kw[NC];
    for (int c = 0; c < NC; ++c) {
        kv[c] = v[c];
        kw[c] = w[c];
    }
    for (int j = 0; j < 5; ++j) {
        const int off = 1 << j;
        const double so = __shfl_up_sync(FULL, sa, off);
        const double e = exp(suffix ? sa - so : so - sa);  // partner precedes in scan order
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
        for (int u = 0; u < NW; ++u) {
            x_has[u] = ch;
            x_sa[u] = ca;
            for (int c = 0; c < NC; ++c) {
                x_v[c][u] = cv[c];
                x_w[c][u] = cw[c];
            }
            const double su = w_sa[u];
            if (!ch) {
                for (int c = 0; c < NC; ++c) {
                    cv[c] = w_v[c][u];
                    cw[c] = w_w[c][u];
                }
                ch = true;
            } else {
                const double e = exp(suffix ? su - ca : ca - su);
                const bool lt = suffix ? su < ca : ca < su;
                for (int c = 0; c < NC; ++c) {
                    if ((stm >> c) & 1) cw[c] = w_w[c][u] + (lt ? e * cv[c] : cw[c]);
                    cv[c] = fma(e, cv[c], w_v[c][u]);
                }
            }
            ca = su;
        }
    }
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
    for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t u = pos(q);
        const double su = (double)S[u];
        if (!hin) {
            for (int c = 0; c < NC; ++c) {
                iv[c] = at(c, 0, u);
                iw[c] = ((stm >> c) & 1) ? at(c, 1, u) : 0.0;
            }
            hin = true;
        } else {
            const double e = suffix ? exp(su - ia) : exp(ia - su);
            const bool lt = suffix ? su < ia : ia < su;
            for (int c = 0; c < NC; ++c) {
                if ((stm >> c) & 1) iw[c] = at(c, 1, u) + (lt ? e * iv[c] : iw[c]);
                iv[c] = fma(e, iv[c], at(c, 0, u));
            }
        }
        ia = su;
        for (int c = 0; c < NC; ++c) {
            out[((size_t)(2 * c) * rows + r) * T + u] = (R)iv[c];
            if ((stm >> c) & 1) out[((size_t)(2 * c + 1) * rows + r) * T + u] = (R)iw[c];
        }
    }
}

// ---------------------------------------------------------------------------
// fix-up passes: fold the tile carries in, apply phases, scatter to caller order
// ---------------------------------------------------------------------------
template <class R>
struct FixArgs {
    const R* A;
    const uint32_t* perm_a;
    const R* B;
    const uint32_t* perm_b;
    const uint32_t* part;
    uint32_t n, k, T;
    int rows;
    R inv_t;
    const R* cp;  // carries, [slot][rows][T]
    const R* cq;
    const R* s_last;
    const R* s_first;
    const R* wa[2];
    const R* wa2[2];
    const R* wb[2];
    const R* wb2[2];
    const R* gsave;
    const R* xsave;
    const R* cpsi;
    const R* spsi;
    const R* cphi;
    const R* sphi;
    R* y;  // forward: rows x ldy (caller row order); transpose: rows x ldy over cols
    size_t ldy;
    R* xbar;  // backward
    size_t ldxb;
    R* abar;
    R* bbar;
    R* phibar;
    R* psibar;
};

// shared: tile-carry lookups (value of channel-slot at tile t-1 / t+1 for row r)
template <class R>
__device__ __forceinline__ R carry_at(const R* c, int slot, int rows, int r, size_t T, size_t t) {
    return c[((size_t)slot * rows + r) * T + t];
}

// Forward fix-up (NG == 0): outputs at row elements.
template <class R, int NX>
__global__ void __launch_bounds__(kFixThreads) lx_fix_fwd(FixArgs<R> p) {
    const uint32_t t = blockIdx.x;
    const size_t T = p.T;
    const uint32_t a0 = p.part[t], a1 = p.part[t + 1];
    const bool hl = t > 0, hr = t + 1 < p.T;
    const R SL = hl ? p.s_last[t - 1] : R(0);
    const R SR = hr ? p.s_first[t + 1] : R(0);
    for (uint32_t i = a0 + threadIdx.x; i < a1; i += kFixThreads) {
        const R s = p.A[i];
        const R eL = hl ? xexp(xsub(SL, s)) : R(0);
        const R eR = hr ? xexp(xsub(s, SR)) : R(0);
        const uint32_t u = p.perm_a[i];
        for (int r = 0; r < p.rows; ++r) {
            R val[2];
#pragma unroll
            for (int c = 0; c < NX; ++c) {
                const R cpv = hl ? carry_at(p.cp, 2 * c, p.rows, r, T, t - 1) : R(0);
                const R cqv = hr ? carry_at(p.cq, 2 * c, p.rows, r, T, t + 1) : R(0);
                val[c] = xfma(eR, cqv, xfma(eL, cpv, p.wa[c][(size_t)r * p.n + i]));
            }
            R out = val[0];
            if constexpr (NX == 2) out = xadd(xmul(p.cphi[u], val[0]), xmul(p.sphi[u], val[1]));
            p.y[(size_t)r * p.ldy + u] = out;
        }
    }
}

// x_bar at one column element for g channel c (shared by transpose and VJP so
// both produce bit-identical x_bar).
template <class R>
__device__ __forceinline__ R xbar_value(R wb, R eL, R cpv, R eR, R cqv) {
    return xfma(eR, cqv, xfma(eL, cpv, wb));
}

// Transpose fix-up (NX == 0, NG == 1): outputs at column elements.
template <class R>
__global__ void __launch_bounds__(kFixThreads) lx_fix_trn(FixArgs<R> p) {
    const uint32_t t = blockIdx.x;
    const size_t T = p.T;
    const uint32_t a0 = p.part[t], a1 = p.part[t + 1];
    const unsigned long long d0 = (unsigned long long)t * kTile;
    const unsigned long long total = (unsigned long long)p.n + p.k;
    const unsigned long long d1 = d0 + kTile < total ? d0 + kTile : total;
    const uint32_t b0 = (uint32_t)(d0 - a0), b1 = (uint32_t)(d1 - a1);
    const bool hl = t > 0, hr = t + 1 < p.T;
    const R SL = hl ? p.s_last[t - 1] : R(0);
    const R SR = hr ? p.s_first[t + 1] : R(0);
    for (uint32_t j = b0 + threadIdx.x; j < b1; j += kFixThreads) {
        const R s = p.B[j];
        const R eL = hl ? xexp(xsub(SL, s)) : R(0);
        const R eR = hr ? xexp(xsub(s, SR)) : R(0);
        const uint32_t u = p.perm_b[j];
        for (int r = 0; r < p.rows; ++r) {
            const R cpv = hl ? carry_at(p.cp, 0, p.rows, r, T, t - 1) : R(0);
            const R cqv = hr ? carry_at(p.cq, 0, p.rows, r, T, t + 1) : R(0);
            p.y[(size_t)r * p.ldy + u] = xbar_value(p.wb[0][(size_t)r * p.k + j], eL, cpv, eR, cqv);
        }
    }
}

// Backward fix-up: x_bar (per row), b_bar / psi_bar (summed over rows) at
// column elements; a_bar / phi_bar (summed over rows) at row elements.
template <class R, int NCH>
__global__ void __launch_bounds__(kFixThreads) lx_fix_bwd(FixArgs<R> p) {
    // channels: g = 0..NCH-1, x = NCH..2*NCH-1
    const uint32_t t = blockIdx.x;
    const size_t T = p.T;
    const uint32_t a0 = p.part[t], a1 = p.part[t + 1];
    const unsigned long long d0 = (unsigned long long)t * kTile;
    const unsigned long long total = (unsigned long long)p.n + p.k;
    const unsigned long long d1 = d0 + kTile < total ? d0 + kTile : total;
    const uint32_t b0 = (uint32_t)(d0 - a0), b1 = (uint32_t)(d1 - a1);
    const bool hl = t > 0, hr = t + 1 < p.T;
    const R SL = hl ? p.s_last[t - 1] : R(0);
    const R SR = hr ? p.s_first[t + 1] : R(0);
    const int rows = p.rows;
    // column side
    for (uint32_t j = b0 + threadIdx.x; j < b1; j += kFixThreads) {
        const R s = p.B[j];
        const R eL = hl ? xexp(xsub(SL, s)) : R(0);
        const R eR = hr ? xexp(xsub(s, SR)) : R(0);
        const bool ltL = SL < s;
        const uint32_t u = p.perm_b[j];
        R m0 = R(1), m1 = R(0);
        if constexpr (NCH == 2) {
            m0 = p.cpsi[u];
            m1 = p.spsi[u];
        }
        R acc_b = R(0), acc_psi = R(0);
        for (int r = 0; r < rows; ++r) {
            R xb[NCH], inner[NCH];
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const R cpv = hl ? carry_at(p.cp, 2 * c, rows, r, T, t - 1) : R(0);
                const R cps = hl ? carry_at(p.cp, 2 * c + 1, rows, r, T, t - 1) : R(0);
                const R cqv = hr ? carry_at(p.cq, 2 * c, rows, r, T, t + 1) : R(0);
                xb[c] = xbar_value(p.wb[c][(size_t)r * p.k + j], eL, cpv, eR, cqv);
                const R strict_left = hl ? (ltL ? xmul(eL, cpv) : cps) : R(0);
                inner[c] = xsub(xfma(eR, cqv, p.wb2[c][(size_t)r * p.k + j]), strict_left);
            }
            const R xr = p.xsave[(size_t)r * p.k + j];
            if constexpr (NCH == 2) {
                p.xbar[(size_t)r * p.ldxb + u] = xadd(xmul(m0, xb[0]), xmul(m1, xb[1]));
                acc_psi = xfma(xr, xadd(xmul(-m1, xb[0]), xmul(m0, xb[1])), acc_psi);
                acc_b = xfma(xmul(xmul(m0, xr), p.inv_t), inner[0], acc_b);
                acc_b = xfma(xmul(xmul(m1, xr), p.inv_t), inner[1], acc_b);
            } else {
                p.xbar[(size_t)r * p.ldxb + u] = xb[0];
                acc_b = xfma(xmul(xr, p.inv_t), inner[0], acc_b);
            }
        }
        p.bbar[u] = acc_b;
        if constexpr (NCH == 2) p.psibar[u] = acc_psi;
    }
    // row side
    for (uint32_t i = a0 + threadIdx.x; i < a1; i += kFixThreads) {
        const R s = p.A[i];
        const R eL = hl ? xexp(xsub(SL, s)) : R(0);
        const R eR = hr ? xexp(xsub(s, SR)) : R(0);
        const bool ltR = s < SR;
        const uint32_t u = p.perm_a[i];
        R m0 = R(1), m1 = R(0);
        if constexpr (NCH == 2) {
            m0 = p.cphi[u];
            m1 = p.sphi[u];
        }
        R acc_a = R(0), acc_phi = R(0);
        for (int r = 0; r < rows; ++r) {
            R inner[NCH], pq[NCH];
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const int cc = NCH + c;
                const R cpv = hl ? carry_at(p.cp, 2 * cc, rows, r, T, t - 1) : R(0);
                const R cqv = hr ? carry_at(p.cq, 2 * cc, rows, r, T, t + 1) : R(0);
                const R cqs = hr ? carry_at(p.cq, 2 * cc + 1, rows, r, T, t + 1) : R(0);
                const R strict_right = hr ? (ltR ? xmul(eR, cqv) : cqs) : R(0);
                inner[c] = xsub(xadd(p.wa[c][(size_t)r * p.n + i], strict_right), xmul(eL, cpv));
                if constexpr (NCH == 2)
                    pq[c] = xfma(eR, cqv, xfma(eL, cpv, p.wa2[c][(size_t)r * p.n + i]));
                else
                    pq[c] = R(0);
            }
            const R gr = p.gsave[(size_t)r * p.n + i];
            if constexpr (NCH == 2) {
                acc_a = xfma(xmul(xmul(m0, gr), p.inv_t), inner[0], acc_a);
                acc_a = xfma(xmul(xmul(m1, gr), p.inv_t), inner[1], acc_a);
                acc_phi = xfma(gr, xadd(xmul(-m1, pq[0]), xmul(m0, pq[1])), acc_phi);
            } else {
                acc_a = xfma(xmul(gr, p.inv_t), inner[0], acc_a);
            }
        }
        p.abar[u] = acc_a;
        if constexpr (NCH == 2) p.phibar[u] = acc_phi;
    }
}


// SEQ fix-up: prefix/suffix in sorted order (no permutation).
template <class R>
__global__ void __launch_bounds__(kFixThreads) lx_fix_seq(FixArgs<R> p, R* pre, R* suf) {
    const uint32_t t = blockIdx.x;
    const size_t T = p.T;
    const uint32_t a0 = p.part[t], a1 = p.part[t + 1];
    const bool hl = t > 0, hr = t + 1 < p.T;
    const R SL = hl ? p.s_last[t - 1] : R(0);
    const R SR = hr ? p.s_first[t + 1] : R(0);
    for (uint32_t i = a0 + threadIdx.x; i < a1; i += kFixThreads) {
        const R s = p.A[i];
        const R eL = hl ? xexp(xsub(SL, s)) : R(0);
        const R eR = hr ? xexp(xsub(s, SR)) : R(0);
        for (int r = 0; r < p.rows; ++r) {
            const R cpv = hl ? carry_at(p.cp, 0, p.rows, r, T, t - 1) : R(0);
            const R cqv = hr ? carry_at(p.cq, 0, p.rows, r, T, t + 1) : R(0);
            const size_t o = (size_t)r * p.n + i;
            if (pre) pre[o] = xfma(eL, cpv, p.wa[0][o]);
            if (suf) suf[o] = xfma(eR, cqv, p.wa2[0][o]);
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
