// lx_main.cuh -- the main merged-tile scan pass (forward, transpose, backward,
// single-sequence scans) as a persistent, double-buffered sm_100a kernel.
//
// Reference algorithm being replaced (paths under /root/reference/proj):
//   matvec branch A/B           include/laplex/operator.hpp:319-369
//   prefix/suffix_decay_scan    include/laplex/scan.hpp:50-73
//   row/col split sums (VJP)    include/laplex/gradients.hpp:33-103,110-135
//
// One CTA per SM slot walks the merge tiles t = blockIdx.x, +gridDim.x, ...
// Each tile's inputs (the two anchor ranges, the output-index ranges and the
// row-0 payload ranges) arrive by TMA bulk copy into one of two shared-memory
// stages; the copy for the CTA's next tile is issued before the current tile
// is computed, so the loads overlap the scan.
//
// Per tile and batch row (merged order, rows first on ties; see lx_scan.cuh):
//   1. merge the two anchor ranges (merge path), IPT consecutive merged
//      elements per thread; anchors, kinds and payloads go to registers;
//   2. thread-local totals of the prefix and suffix recurrences (+ strict);
//   3. warp Kogge-Stone over the thread totals, block totals over warps in
//      every warp (one barrier), tile carries and shard carries folded in:
//      each thread gets its exclusive carry from the left and from the right;
//   4. the thread re-runs its IPT-element recurrences seeded with those
//      carries (suffix first, recording what the outputs need, then prefix)
//      and writes each output into a shared-memory staging row indexed by
//      the element's side-local index;
//   5. the staged outputs are stored side by side (one side at a time, no
//      divergence) to perm / plan position.
// Numerics: every carry that crosses a thread is applied as one exp of an
// anchor difference; within a thread's IPT consecutive elements carries are
// products of per-step decays (the exception DESIGN.md section 4 allows).
#pragma once

#include "lx_scan.cuh"

namespace lx {
namespace ms {

template <class R, int NC>
struct MainStage {
    static constexpr int kPad = 16 / sizeof(R);
    unsigned long long bar;    // "full": header, anchors + output indices (producer -> consumers)
    unsigned long long barp;   // payloads (one completion per batch row)
    unsigned long long empty;  // consumers -> producer: the stage may be refilled
    R c0[4][NC];               // row-0 tile carries: prefix, strict prefix, suffix, strict suffix
    uint32_t t;  // tile index staged here (>= T: no more tiles)
    uint32_t a0, b0;
    int na, nb;
    R s_last, SL, SR;  // tile's last anchor, previous tile's last, next tile's first
    // A range at [offA], then a 16-byte gap, B range at [baseB]; the gap and the
    // tail leave room for the +inf sentinels behind each range (merge)
    alignas(16) R anch[kTile + 8 * kPad];
    alignas(16) R pay[kTile + 8 * kPad];  // row payloads, same layout
    alignas(16) uint32_t oidx[kTile + 16];  // output index ranges: A at [offIA], B at [baseIB + offIB]
    alignas(16) uint16_t gm[kTile];         // store order (lx_group_plan): rows at [0, na), cols at [na, len)
    alignas(16) uint32_t mw[kMergeWords];   // the tile's merge words (lx_group_plan)
    int r0;  // first batch row of the work item (row split, see MainArgs::rsplit; last: the header layout above is shared)
};

#ifndef LX_MAIN_STAGES
#define LX_MAIN_STAGES 2
#endif
constexpr int kMainStages = LX_MAIN_STAGES;

template <class R, int NC, int NW, int NACC, int NOS, int NMC = 0>
struct MainShared {
    MainStage<R, NC> st[kMainStages];
    // phased fp32: each thread's cos / sin of its elements' phases for the
    // current tile, [q][thread] (row-invariant values that would otherwise stay
    // live in registers across the batch-row loop and spill; C3 main kernels
    // 5.77 -> 5.43 ms.  The in-thread decays there as well measured slower)
    R mcs[NMC > 0 ? NMC : 1];
    // suffix values recorded between the two re-scans, [k][q][thread] (fp32
    // unphased backward: saves 8 registers where the kernel would spill)
    R os[NOS > 0 ? NOS : 1];
    // backward: a_bar at [li], b_bar at [na + li] (and phi_bar / psi_bar),
    // accumulated over the batch rows by the element's owning thread
    R acc[NACC > 0 ? NACC : 1][kTile];
    R wsl[NW], wsf[NW];                 // warp last / first anchors (per tile)
    R cr[2][4][NC];                     // tile carries of batch rows >= 1 (prefetched a row ahead)
    R pv[NC][NW], pw[NC][NW];           // warp prefix totals (inclusive, strict)
    R qv[NC][NW], qw[NC][NW];           // warp suffix totals
};

// Geometry of one staged tile, derived from its header.
template <class R>
struct TileGeom {
    uint32_t a0, b0;
    int na, nb;
    int offA, baseB, offIA, baseIB;  // element offsets inside anch/pay, oidx
    uint32_t bytesA, bytesB, ibytesA, ibytesB, gbytes;
    uint32_t a0al, b0al, a0i, b0i;
    __device__ __forceinline__ void init(uint32_t a0_, uint32_t b0_, int na_, int nb_, bool outA, bool outB) {
        constexpr int kPad = 16 / sizeof(R);
        a0 = a0_;
        b0 = b0_;
        na = na_;
        nb = nb_;
        a0al = a0 & ~uint32_t(kPad - 1);
        b0al = b0 & ~uint32_t(kPad - 1);
        offA = (int)(a0 - a0al);
        const int offB = (int)(b0 - b0al);
        bytesA = na ? (uint32_t)(((offA + na + kPad - 1) / kPad) * 16) : 0u;
        bytesB = nb ? (uint32_t)(((offB + nb + kPad - 1) / kPad) * 16) : 0u;
        baseB = (int)(bytesA / sizeof(R)) + kPad + offB;  // B region after a 16-byte gap
        a0i = a0 & ~3u;
        b0i = b0 & ~3u;
        offIA = (int)(a0 - a0i);
        const int offIB = (int)(b0 - b0i);
        ibytesA = (outA && na) ? (uint32_t)(((offIA + na + 3) / 4) * 16) : 0u;
        ibytesB = (outB && nb) ? (uint32_t)(((offIB + nb + 3) / 4) * 16) : 0u;
        baseIB = (int)(ibytesA / 4) + offIB;
        // the tile's store-order slot (16-byte aligned): rows then cols
        gbytes = (outA || outB) ? (uint32_t)(((na + nb + 7) / 8) * 16) : 0u;
    }
};

// Producer lane: stage tile t (header, row-0 carries, anchors, output
// indices, row-0 payloads) and arm the stage's barriers.  t >= T stages the
// end-of-work sentinel (header only).
template <class R, int NC, bool SEQ, bool PAY_A, bool PAY_B, bool OUT_A, bool OUT_B, class CH, bool SPLIT>
__device__ __forceinline__ void issue_tile(MainStage<R, NC>& S, const MainArgs<R>& p, uint32_t t, int r0,
                                           const TileDesc<R>& dt, const TileDesc<R>& dn, R SL) {
    S.t = t;
    if constexpr (SPLIT) S.r0 = r0;
    else r0 = 0;
    if (t >= p.T) {
        mbar_expect_tx(&S.bar, 0u);
        return;
    }
    const size_t T = p.T, rows = p.rows;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const size_t sl0 = (size_t)(2 * c) * rows + r0, sl1 = (size_t)(2 * c + 1) * rows + r0;
        S.c0[0][c] = t > 0 ? p.cp[sl0 * T + t - 1] : R(0);
        S.c0[1][c] = (t > 0 && CH::pst(c)) ? p.cp[sl1 * T + t - 1] : R(0);
        S.c0[2][c] = t + 1 < T ? p.cq[sl0 * T + t + 1] : R(0);
        S.c0[3][c] = (t + 1 < T && CH::qst(c)) ? p.cq[sl1 * T + t + 1] : R(0);
    }
    TileGeom<R> g;
    g.init(dt.a0, dt.b0, (int)(dn.a0 - dt.a0), (int)(dn.b0 - dt.b0), OUT_A, OUT_B);
    S.a0 = dt.a0;
    S.b0 = dt.b0;
    S.na = g.na;
    S.nb = g.nb;
    S.s_last = dt.s_last;
    S.SL = SL;
    S.SR = dn.s_first;
    constexpr uint32_t kMW = SEQ ? 0u : (uint32_t)(kMergeWords * 4);
    mbar_expect_tx(&S.bar, g.bytesA + g.bytesB + g.ibytesA + g.ibytesB + g.gbytes + kMW);
    if (kMW) bulk_g2s(S.mw, p.mwords + (size_t)t * kMergeWords, kMW, &S.bar);
    if (g.bytesA) bulk_g2s(S.anch, p.A + g.a0al, g.bytesA, &S.bar);
    if (g.bytesB) bulk_g2s(S.anch + (g.bytesA / sizeof(R)) + MainStage<R, NC>::kPad, p.B + g.b0al, g.bytesB, &S.bar);
    if (g.ibytesA) bulk_g2s(S.oidx, p.perm_a + g.a0i, g.ibytesA, &S.bar);
    if (g.ibytesB) bulk_g2s(S.oidx + g.ibytesA / 4, p.perm_b + g.b0i, g.ibytesB, &S.bar);
    if (g.gbytes) bulk_g2s(S.gm, p.gmt + (size_t)t * kTile, g.gbytes, &S.bar);
    const R* srcA = (SEQ ? p.Xs : p.Gs) + (size_t)r0 * (SEQ ? p.ldxs : p.ldgs);
    mbar_expect_tx(&S.barp, (PAY_A ? g.bytesA : 0u) + (PAY_B ? g.bytesB : 0u));
    if (PAY_A && g.bytesA) bulk_g2s(S.pay, srcA + g.a0al, g.bytesA, &S.barp);
    if (PAY_B && g.bytesB)
        bulk_g2s(S.pay + (g.bytesA / sizeof(R)) + MainStage<R, NC>::kPad, p.Xs + (size_t)r0 * p.ldxs + g.b0al,
                 g.bytesB, &S.barp);
}

// Diagnostics only (LX_DIAG_CONTIG): write outputs at the sorted position
// instead of the perm / plan position, to isolate the cost of the stores.
#ifdef LX_DIAG_CONTIG
#define LXO(perm_pos, sorted_pos) (sorted_pos)
#else
#define LXO(perm_pos, sorted_pos) (perm_pos)
#endif

// Resident consumer threads per SM the register budget targets (fp32): for
// the 128-thread unphased shape 3 forward / transpose CTAs and 2 backward
// CTAs; for the 256-thread phased shape 3 and 2 as well (measured best).
#ifndef LX_MAIN_CTAS
#define LX_MAIN_CTAS 384
#endif
#ifndef LX_BWD_CTAS
#define LX_BWD_CTAS 256
#endif
// fp32 unphased backward: suffix values between the two re-scans in shared
// memory (1) or registers (0)
#ifndef LX_OS_SMEM
#define LX_OS_SMEM 0
#endif
#ifndef LX_PH_MC_SMEM
#define LX_PH_MC_SMEM 1
#endif
// phased (256-thread) kernels: resident CTAs per SM the register budget targets
#ifndef LX_PH_FWD_CTAS
#define LX_PH_FWD_CTAS 2  // 3 spilled (72 registers): C3 forward 3.37 -> 2.42 ms with 2
#endif
#ifndef LX_PH_BWD_CTAS
#define LX_PH_BWD_CTAS 2
#endif
template <class R, bool BWD, int TPB>
constexpr int main_min_blocks() {
    return sizeof(R) != 4 ? 1
           : TPB == 256   ? (BWD ? LX_PH_BWD_CTAS : LX_PH_FWD_CTAS)
                          : (BWD ? LX_BWD_CTAS : LX_MAIN_CTAS) / TPB;
}

// Channel layout: g channels first (c < NG), then x channels.  Strict prefix
// variants for g channels and strict suffix variants for x channels, in the
// backward (BWD) configuration only.  SEQ: one x channel carried by rows.
// MB: CTAs per SM the register budget targets, 0 = main_min_blocks (the
// batched unphased backward runs a 3-CTA instantiation, see launch_main)
template <class R, int NG, int NX, bool BWD, bool SEQ, int TPB, int IPT, int MB = 0>
__global__ void __launch_bounds__(TPB + 32, MB ? MB : main_min_blocks<R, BWD, TPB>()) lx_main(MainArgs<R> p) {
    static_assert(TPB * IPT == kTile, "a CTA covers one merge tile");
    constexpr int NW = TPB / 32;
    static_assert(NW <= 32 && (NW & (NW - 1)) == 0, "warps per CTA: power of two");
    constexpr int LOGW = NW <= 1 ? 0 : NW <= 2 ? 1 : NW <= 4 ? 2 : NW <= 8 ? 3 : NW <= 16 ? 4 : 5;
    using C = Ch<NG, NX, BWD>;
    constexpr int NC = C::NC;
    constexpr bool PHASED = (NG == 2 || NX == 2);
    constexpr int NP = PHASED ? 2 : 1;  // modulated payload channels per element
    constexpr bool PAY_A = SEQ || NG > 0;
    constexpr bool PAY_B = !SEQ && NX > 0;
    constexpr bool OUT_A = !SEQ && (BWD || NX > 0);  // row-side outputs
    constexpr bool OUT_B = !SEQ && NG > 0;           // col-side outputs
    // suffix values recorded per element for the outputs
    constexpr int KS = SEQ ? 1 : (!BWD ? (NG > 0 ? NG : NX) : (PHASED ? 4 : 1));
    constexpr int NACC = BWD ? (PHASED ? 2 : 1) : 0;
    constexpr bool OS_SMEM = LX_OS_SMEM && BWD && !PHASED && sizeof(R) == 4;
    constexpr bool MC_SMEM = LX_PH_MC_SMEM && PHASED && sizeof(R) == 4;
    using SM = MainShared<R, NC, NW, NACC, OS_SMEM ? KS * kTile : 0, MC_SMEM ? 2 * kTile : 0>;
    extern __shared__ __align__(16) unsigned char smem_main[];
    SM& sm = *reinterpret_cast<SM*>(smem_main);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t T = p.T;
    const int rows = p.rows;
    const int ext_flags = p.ext ? (int)p.ext[2] : 0;
    const bool has_ext_p = ext_flags & 1, has_ext_q = ext_flags & 2;
    const R ext_pa = has_ext_p ? p.ext[0] : R(0), ext_qa = has_ext_q ? p.ext[1] : R(0);
    const R* ext_pv = p.ext ? p.ext + 3 : nullptr;
    const R* ext_qv = p.ext ? p.ext + 3 + (size_t)2 * NC * rows : nullptr;
    const R* cphi = p.cphi;
    const R* sphi = p.sphi;
    const R* cpsi = p.cpsi;
    const R* spsi = p.spsi;

    // row split (MainArgs::rsplit) only in the phased kernels (C3's head: a
    // large batch over few tiles); in the unphased kernels its registers and
    // producer arithmetic measured slower (C2 +1.3 ms, C5 forward +0.25 ms)
    constexpr bool SPLIT = PHASED;

    // ---- tile schedule: one producer warp, TPB consumer threads ----
    // Tiles are claimed in increasing order from a global counter, so the
    // tiles in flight stay a compact window of the merged sequence (the
    // staged output writes of neighbouring tiles then combine in L2).  Lane 0
    // of the producer warp claims a tile, loads its descriptors, waits for a
    // free stage and stages the tile by TMA; its latencies never stall the
    // consumers, which synchronise among themselves on named barrier 1.
    if (tid == 0) {
        for (int s = 0; s < kMainStages; ++s) {
            mbar_init(&sm.st[s].bar, 1);
            mbar_init(&sm.st[s].barp, 1);
            mbar_init(&sm.st[s].empty, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NW) {
        if (lane == 0) {
            const uint32_t RS = SPLIT ? p.rsplit : 1u;
            auto claim = [&](uint32_t& tt, int& r0, TileDesc<R>& d0, TileDesc<R>& d1, R& sl) {
                const uint32_t item = atomicAdd(p.tile_ctr, 1u);
                tt = SPLIT ? item / RS : item;
                r0 = SPLIT ? (int)(item - tt * RS) * p.rchunk : 0;
                if (tt < T) {
                    d0 = p.desc[tt];
                    d1 = p.desc[tt + 1];
                    sl = tt > 0 ? p.s_last[tt - 1] : R(0);
                }
            };
            uint32_t tc;
            int r0;
            TileDesc<R> d0, d1;
            R sl = R(0);
            claim(tc, r0, d0, d1, sl);
            for (int it = 0;; ++it) {
                const int s = it % kMainStages;
                const uint32_t use = (uint32_t)(it / kMainStages);
                if (it >= kMainStages) mbar_wait_sleep(&sm.st[s].empty, (use - 1u) & 1u);
                issue_tile<R, NC, SEQ, PAY_A, PAY_B, OUT_A, OUT_B, C, SPLIT>(sm.st[s], p, tc, r0, d0, d1, sl);
                if (tc >= T) break;
                claim(tc, r0, d0, d1, sl);
            }
        }
        return;
    }

    unsigned pph = 0;  // SPLIT: bit s = phase of stage s's payload barrier
    for (int it = 0;; ++it) {
        const int sidx = it % kMainStages;
        auto& S = sm.st[sidx];
        const uint32_t use = (uint32_t)(it / kMainStages);  // completions of this stage's barriers so far
        mbar_wait(&S.bar, use & 1u);
        const uint32_t t = S.t;
        if (t >= T) break;
        const int r0 = SPLIT ? S.r0 : 0, r1 = SPLIT ? min(rows, r0 + p.rchunk) : rows;  // this item's batch rows
        TileGeom<R> g;
        g.init(S.a0, S.b0, S.na, S.nb, OUT_A, OUT_B);
        const int na = g.na, nb = g.nb, len = na + nb;
        const R s_end = S.s_last;
        const bool hl = t > 0 || has_ext_p, hr = t + 1 < T || has_ext_q;
        const R SL = t > 0 ? S.SL : ext_pa;
        const R SR = t + 1 < T ? S.SR : ext_qa;
        R* sA = S.anch + g.offA;
        R* sB = S.anch + g.baseB;
        const R* pA = S.pay + g.offA;
        const R* pB = S.pay + g.baseB;
        const uint32_t* iA = S.oidx + g.offIA;
        const uint32_t* iB = S.oidx + g.baseIB;
        const uint16_t* gmA = S.gm;  // store order of the tile rows / cols
        const uint16_t* gmB = S.gm + na;

        // ---- this thread's IPT merged elements: kinds from the plan's merge
        // words, anchors by independent shared-memory loads ----
        static_assert(kMergeGroup % IPT == 0, "a thread's elements lie in one merge word");
        R s[IPT];
        unsigned rowm;  // bit q: element q is a row
        int ia0, ib0, nval;
        {
            const int dd = min(tid * IPT, len);
            nval = min(IPT, len - dd);
            int ia;
            if constexpr (SEQ) {  // one sequence: every element is a "row"
                rowm = (1u << IPT) - 1u;
                ia = dd;
            } else {
                const uint32_t w = S.mw[(tid * IPT) / kMergeGroup];
                const int sh = (tid * IPT) % kMergeGroup;
                rowm = (w >> sh) & ((1u << IPT) - 1u);
                ia = (int)(w >> 16) + __popc(w & ((1u << sh) - 1u));
            }
            int ib = dd - ia;
            ia0 = ia;
            ib0 = ib;
#pragma unroll
            for (int q = 0; q < IPT; ++q) {
                const bool r = (rowm >> q) & 1u;
                s[q] = r ? sA[ia] : sB[ib];  // past the tile end: stale, replaced below
                ia += r;
                ib += !r;
            }
#pragma unroll
            for (int q = 0; q < IPT; ++q)
                if (q >= nval) s[q] = s_end;
        }
        const unsigned valm = (1u << nval) - 1u;

        // ---- row-independent geometry: every exp is taken from an anchor difference ----
        R E[IPT];  // E[q] = exp(s[q-1] - s[q])
        E[0] = R(0);
#pragma unroll
        for (int q = 1; q < IPT; ++q) E[q] = xexp(xsub(s[q - 1], s[q]));
        unsigned ltE = 0;  // bit q: s[q-1] < s[q]
#pragma unroll
        for (int q = 1; q < IPT; ++q)
            if (s[q - 1] < s[q]) ltE |= 1u << q;
        const R sl = s[IPT - 1], sf = s[0];
        if (lane == 31) sm.wsl[warp] = sl;
        if (lane == 0) sm.wsf[warp] = sf;
        const R S1 = shfl_up(sl, 1);     // previous lane's last anchor
        const R S1q = shfl_down(sf, 1);  // next lane's first anchor

        const bool first_t = tid == 0, last_t = tid == TPB - 1;

        // phased: cos / sin of each element's phase (rows: phi, cols: psi),
        // loaded once per tile instead of once per batch row and use
        R mcr[PHASED && !MC_SMEM ? IPT : 1], msr[PHASED && !MC_SMEM ? IPT : 1];
        auto MCw = [&](int q) -> R& { if constexpr (MC_SMEM) return sm.mcs[q * TPB + tid]; else return mcr[q]; };
        auto MSw = [&](int q) -> R& { if constexpr (MC_SMEM) return sm.mcs[(IPT + q) * TPB + tid]; else return msr[q]; };
        if constexpr (PHASED) {
            int ia = ia0, ib = ib0;
#pragma unroll
            for (int q = 0; q < IPT; ++q) {
                const bool isr = (rowm >> q) & 1, val = (valm >> q) & 1;
                const R* cs = isr ? cphi + g.a0 + ia : cpsi + g.b0 + ib;
                const R* sn = isr ? sphi + g.a0 + ia : spsi + g.b0 + ib;
                const bool has = val && (isr ? (NG == 2 || !BWD) : NX == 2);
                MCw(q) = has ? *cs : R(1);
                MSw(q) = has ? *sn : R(0);
                ia += isr;
                ib += !isr;
            }
        }

        for (int r = r0; r < r1; ++r) {
            if constexpr (SPLIT) {
                mbar_wait(&S.barp, (pph >> sidx) & 1u);
                pph ^= 1u << sidx;
            } else {
                mbar_wait(&S.barp, (use * (uint32_t)rows + (uint32_t)r) & 1u);
            }
            // phased kernels: the next batch row's tile carries are copied
            // global -> shared asynchronously now and read after barrier (A)
            // of that row (row 0's come with the producer's staging; C3 bwd
            // 5.43 -> 4.71 ms).  The unphased kernels load them at use: the
            // prefetch's registers cost the single-row C5 kernels more than
            // it saves the batched C2 ones.
            constexpr bool PF = PHASED || MB != 0;  // MB != 0: the batched unphased backward
            const bool pf = PF && r + 1 < r1 && tid < 4 * NC;
            if (pf) {
                const int c = tid % NC, kind = tid / NC;  // kind: prefix, strict prefix, suffix, strict suffix
                const bool strict = kind & 1;
                const size_t sl = ((size_t)(2 * c + (strict ? 1 : 0)) * rows + r + 1);
                const bool ok = (kind < 2 ? t > 0 : t + 1 < T) && (!strict || (kind < 2 ? C::pst(c) : C::qst(c)));
                R* d = &sm.cr[(r + 1) & 1][kind][c];
                if (ok) {
                    const R* src = kind < 2 ? p.cp + sl * T + t - 1 : p.cq + sl * T + t + 1;
                    if constexpr (sizeof(R) == 4)
                        cp_async4(d, src);
                    else
                        cp_async8(d, src);
                } else {
                    *d = R(0);
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            // ---- payloads: modulated channel values of each element ----
            R pay[NP][IPT];
            R raw[PHASED ? IPT : 1];
            {
                int ia = ia0, ib = ib0;
#pragma unroll
                for (int q = 0; q < IPT; ++q) {
                    const bool isr = (rowm >> q) & 1, val = (valm >> q) & 1;
                    const int li = isr ? ia : ib;
                    ia += isr;
                    ib += !isr;
                    R v = R(0);
                    if constexpr (PAY_A && PAY_B) {
                        v = val ? (isr ? pA : pB)[li] : R(0);
                    } else if constexpr (PAY_A) {
                        v = (val && isr) ? pA[li] : R(0);
                    } else {
                        v = (val && !isr) ? pB[li] : R(0);
                    }
                    if constexpr (PHASED) {
                        // payload channels: the side's own modulation (rows: phi in the
                        // backward; cols: psi); the forward's rows carry no payload
                        const bool mod = isr ? NG == 2 : NX == 2;
                        raw[q] = v;
                        pay[0][q] = mod ? xmul(MCw(q), v) : v;
                        pay[1][q] = mod ? xmul(MSw(q), v) : R(0);
                    } else {
                        pay[0][q] = v;
                    }
                }
            }
            // payload of channel c at element q
            auto chp = [&](int c, int q) -> R {
                const bool isr = (rowm >> q) & 1;
                if constexpr (SEQ) {
                    return pay[0][q];
                } else {
                    if (c < NG) return isr ? pay[NG == 2 ? c : 0][q] : R(0);
                    return isr ? R(0) : pay[NX == 2 ? c - NG : 0][q];
                }
            };

            // ---- 2. thread-local totals ----
            R v[NC], w[NC], vq[NC], wq[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                R a = chp(c, 0), b = R(0);
#pragma unroll
                for (int q = 1; q < IPT; ++q) {
                    if (C::pst(c)) b = ((ltE >> q) & 1) ? xmul(E[q], a) : b;
                    a = xfma(E[q], a, chp(c, q));
                }
                v[c] = a;
                w[c] = b;
                R u = chp(c, IPT - 1), z = R(0);
#pragma unroll
                for (int q = IPT - 2; q >= 0; --q) {
                    if (C::qst(c)) z = ((ltE >> (q + 1)) & 1) ? xmul(E[q + 1], u) : z;
                    u = xfma(E[q + 1], u, chp(c, q));
                }
                vq[c] = u;
                wq[c] = z;
            }
            // ---- 3a. warp Kogge-Stone (prefix from lower lanes, suffix from upper) ----
            // (geometry recomputed per batch row: short live ranges beat reuse)
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
                    const R uo = shfl_down(vq[c], off);
                    if (C::qst(c)) {
                        const R zo = shfl_down(wq[c], off);
                        if (lane + off < 32) wq[c] = xadd(wq[c], ((ltQ >> j) & 1) ? xmul(eQ[j], uo) : zo);
                    }
                    if (lane + off < 32) vq[c] = xfma(eQ[j], uo, vq[c]);
                }
            }
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
            if (PF && r > r0 && tid < 4 * NC) {  // this row's prefetched carries have landed
                if (pf)
                    asm volatile("cp.async.wait_group 1;" ::: "memory");
                else
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            cbar<TPB>();  // (A) warp totals; every merge of this tile is done; row carries in shared memory
            if (tid == 0 && r + 1 < r1) {  // next batch row's payloads into this stage
                const R* srcA = SEQ ? p.Xs : p.Gs;
                const size_t ldA = SEQ ? p.ldxs : p.ldgs;
                mbar_expect_tx(&S.barp, (PAY_A ? g.bytesA : 0u) + (PAY_B ? g.bytesB : 0u));
                if (PAY_A && g.bytesA) bulk_g2s(S.pay, srcA + (size_t)(r + 1) * ldA + g.a0al, g.bytesA, &S.barp);
                if (PAY_B && g.bytesB)
                    bulk_g2s(S.pay + (g.bytesA / sizeof(R)) + MainStage<R, NC>::kPad,
                             p.Xs + (size_t)(r + 1) * p.ldxs + g.b0al, g.bytesB,
                             &S.barp);
            }
            // block-level geometry (warp anchors stay in shared memory for the whole tile)
            R eBP[LOGW > 0 ? LOGW : 1], eBQ[LOGW > 0 ? LOGW : 1];
            unsigned ltBP = 0, ltBQ = 0;
            {
                const R wl = lane < NW ? sm.wsl[lane] : sm.wsl[NW - 1];
                const R wf = lane < NW ? sm.wsf[lane] : sm.wsf[NW - 1];
#pragma unroll
                for (int j = 0; j < LOGW; ++j) {
                    const int off = 1 << j;
                    const R so = shfl_up(wl, off);
                    const R sq = shfl_down(wf, off);
                    eBP[j] = lane >= off ? xexp(xsub(so, wl)) : R(0);
                    if (lane >= off && so < wl) ltBP |= 1u << j;
                    eBQ[j] = lane + off < NW ? xexp(xsub(wf, sq)) : R(0);
                    if (lane + off < NW && wf < sq) ltBQ |= 1u << j;
                }
            }
            // thread-exclusive anchors: the first thread's left neighbour is the
            // previous tile's last element (SL), the last thread's right
            // neighbour is the next tile's first element (SR)
            const R SW = warp > 0 ? sm.wsl[warp - 1] : sf;       // previous warp's last anchor
            const R SWq = warp < NW - 1 ? sm.wsf[warp + 1] : sl;  // next warp's first anchor
            const R eTW = (lane > 0 && warp > 0) ? xexp(xsub(SW, S1)) : R(0);
            const bool ltTW = SW < S1;
            const R eTWq = (lane < 31 && warp < NW - 1) ? xexp(xsub(S1q, SWq)) : R(0);
            const bool ltTWq = S1q < SWq;
            const R SE = first_t ? SL : (lane > 0 ? S1 : SW);
            const R SEq = last_t ? SR : (lane < 31 ? S1q : SWq);
            const bool hasP = first_t ? hl : true;
            const bool hasQ = last_t ? hr : true;
            const R eTL = (!first_t && hl) ? xexp(xsub(SL, SE)) : R(0);
            const bool ltTL = SL < SE;
            const R eTR = (!last_t && hr) ? xexp(xsub(SEq, SR)) : R(0);
            const bool ltTR = SEq < SR;
            const R eL0 = hasP ? xexp(xsub(SE, sf)) : R(0);
            const bool ltL0 = SE < sf;
            const R eRq = hasQ ? xexp(xsub(sl, SEq)) : R(0);
            const bool ltRq = sl < SEq;
            // ---- 3b. block totals over warps (every warp), exclusive per warp ----
            R XV[NC], XW[NC], YV[NC], YW[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                R bv = lane < NW ? sm.pv[c][lane] : R(0);
                R bw = lane < NW ? sm.pw[c][lane] : R(0);
                R cv = lane < NW ? sm.qv[c][lane] : R(0);
                R cw = lane < NW ? sm.qw[c][lane] : R(0);
#pragma unroll
                for (int j = 0; j < LOGW; ++j) {
                    const int off = 1 << j;
                    const R vo = shfl_up(bv, off);
                    const R wo = shfl_up(bw, off);
                    const R vqo = shfl_down(cv, off);
                    const R wqo = shfl_down(cw, off);
                    if (lane >= off) {
                        if (C::pst(c)) bw = xadd(bw, ((ltBP >> j) & 1) ? xmul(eBP[j], vo) : wo);
                        bv = xfma(eBP[j], vo, bv);
                    }
                    if (lane + off < NW) {
                        if (C::qst(c)) cw = xadd(cw, ((ltBQ >> j) & 1) ? xmul(eBQ[j], vqo) : wqo);
                        cv = xfma(eBQ[j], vqo, cv);
                    }
                }
                const int lp = warp > 0 ? warp - 1 : 0, lq = warp < NW - 1 ? warp + 1 : NW - 1;
                XV[c] = __shfl_sync(FULL, bv, lp);
                XW[c] = __shfl_sync(FULL, bw, lp);
                YV[c] = __shfl_sync(FULL, cv, lq);
                YW[c] = __shfl_sync(FULL, cw, lq);
            }
            // tile carries of this row, combined with the external shard carries:
            // ext (+) tiles<t  and  tiles>t (+) ext
            R cpv[NC], cps[NC], cqv[NC], cqs[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const size_t sl0 = ((size_t)(2 * c) * rows + r), sl1 = ((size_t)(2 * c + 1) * rows + r);
                if (r == r0) {  // staged by the producer
                    cpv[c] = S.c0[0][c];
                    cps[c] = S.c0[1][c];
                    cqv[c] = S.c0[2][c];
                    cqs[c] = S.c0[3][c];
                } else if constexpr (PF) {
                    cpv[c] = sm.cr[r & 1][0][c];
                    cps[c] = sm.cr[r & 1][1][c];
                    cqv[c] = sm.cr[r & 1][2][c];
                    cqs[c] = sm.cr[r & 1][3][c];
                } else {
                    cpv[c] = t > 0 ? p.cp[sl0 * T + t - 1] : R(0);
                    cps[c] = (t > 0 && C::pst(c)) ? p.cp[sl1 * T + t - 1] : R(0);
                    cqv[c] = t + 1 < T ? p.cq[sl0 * T + t + 1] : R(0);
                    cqs[c] = (t + 1 < T && C::qst(c)) ? p.cq[sl1 * T + t + 1] : R(0);
                }
                if (has_ext_p) {
                    const R ev = ext_pv[sl0], es = C::pst(c) ? ext_pv[sl1] : R(0);
                    if (t > 0) {  // (ext_anchor, ev, es) then (SL, cpv, cps)
                        const R e = xexp(xsub(ext_pa, SL));
                        if (C::pst(c)) cps[c] = xadd(cps[c], ext_pa < SL ? xmul(e, ev) : es);
                        cpv[c] = xfma(e, ev, cpv[c]);
                    } else {
                        cpv[c] = ev;
                        cps[c] = es;
                    }
                }
                if (has_ext_q) {
                    const R ev = ext_qv[sl0], es = C::qst(c) ? ext_qv[sl1] : R(0);
                    if (t + 1 < T) {  // (SR, cqv, cqs) then (ext_anchor, ev, es)
                        const R e = xexp(xsub(SR, ext_qa));
                        if (C::qst(c)) cqs[c] = xadd(cqs[c], SR < ext_qa ? xmul(e, ev) : es);
                        cqv[c] = xfma(e, ev, cqv[c]);
                    } else {
                        cqv[c] = ev;
                        cqs[c] = es;
                    }
                }
            }
            // ---- 3c. thread-exclusive carries (+ tile carries) ----
            R VE[NC], WE[NC], VEq[NC], WEq[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const R V1 = shfl_up(v[c], 1), W1 = shfl_up(w[c], 1);
                const R V1q = shfl_down(vq[c], 1), W1q = shfl_down(wq[c], 1);
                R a = R(0), b = R(0), aq = R(0), bq = R(0);
                if (first_t) {
                    a = cpv[c];
                    b = cps[c];
                } else {
                    if (lane > 0) {
                        a = V1;
                        b = W1;
                        if (warp > 0) {
                            if (C::pst(c)) b = xadd(W1, ltTW ? xmul(eTW, XV[c]) : XW[c]);
                            a = xfma(eTW, XV[c], V1);
                        }
                    } else {
                        a = XV[c];
                        b = XW[c];
                    }
                    if (hl) {  // previous tiles, anchored at SL <= SE
                        if (C::pst(c)) b = xadd(b, ltTL ? xmul(eTL, cpv[c]) : cps[c]);
                        a = xfma(eTL, cpv[c], a);
                    }
                }
                if (last_t) {
                    aq = cqv[c];
                    bq = cqs[c];
                } else {
                    if (lane < 31) {
                        aq = V1q;
                        bq = W1q;
                        if (warp < NW - 1) {
                            if (C::qst(c)) bq = xadd(W1q, ltTWq ? xmul(eTWq, YV[c]) : YW[c]);
                            aq = xfma(eTWq, YV[c], V1q);
                        }
                    } else {
                        aq = YV[c];
                        bq = YW[c];
                    }
                    if (hr) {  // following tiles, anchored at SR >= SEq
                        if (C::qst(c)) bq = xadd(bq, ltTR ? xmul(eTR, cqv[c]) : cqs[c]);
                        aq = xfma(eTR, cqv[c], aq);
                    }
                }
                VE[c] = a;
                WE[c] = b;
                VEq[c] = aq;
                WEq[c] = bq;
            }

            // ---- 4a. suffix re-scan seeded with the right carry; record what outputs need ----
            R osr[OS_SMEM ? 1 : KS][IPT];
            auto OS = [&](int k, int q) -> R& {
                if constexpr (OS_SMEM)
                    return sm.os[(k * IPT + q) * TPB + tid];
                else
                    return osr[k][q];
            };
            {
                R u[NC], z[NC];
#pragma unroll
                for (int q = IPT - 1; q >= 0; --q) {
                    const R e = q == IPT - 1 ? eRq : E[q + 1];
                    const bool lt = q == IPT - 1 ? ltRq : (bool)((ltE >> (q + 1)) & 1);
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        const R prevu = q == IPT - 1 ? VEq[c] : u[c];
                        if (C::qst(c)) z[c] = lt ? xmul(e, prevu) : (q == IPT - 1 ? WEq[c] : z[c]);
                        u[c] = xfma(e, prevu, chp(c, q));
                    }
                    const bool isr = (rowm >> q) & 1;
                    if constexpr (SEQ) {
                        OS(0, q) = u[0];
                    } else if constexpr (!BWD) {
                        if constexpr (NG > 0) {
#pragma unroll
                            for (int c = 0; c < NG; ++c) OS(c, q) = u[c];
                        } else {
#pragma unroll
                            for (int c = 0; c < NX; ++c) OS(c, q) = u[c];
                        }
                    } else if constexpr (!PHASED) {
                        OS(0, q) = isr ? z[1] : u[0];  // rows: strict suffix of x; cols: suffix of g
                    } else {
                        // rows: Q and strict Q of the two x channels; cols: Q of the two g channels
                        OS(0, q) = isr ? u[2] : u[0];
                        OS(1, q) = isr ? u[3] : u[1];
                        OS(2, q) = z[2];
                        OS(3, q) = z[3];
                    }
                }
            }
            // ---- 4b. prefix re-scan seeded with the left carry; outputs ----
            R* stg = S.anch;  // staging row (anchors are no longer needed after (A))
            {
                R a[NC], b[NC];
                int ia = ia0, ib = ib0;
#pragma unroll
                for (int q = 0; q < IPT; ++q) {
                    const R e = q == 0 ? eL0 : E[q];
                    const bool lt = q == 0 ? ltL0 : (bool)((ltE >> q) & 1);
#pragma unroll
                    for (int c = 0; c < NC; ++c) {
                        const R preva = q == 0 ? VE[c] : a[c];
                        if (C::pst(c)) b[c] = lt ? xmul(e, preva) : (q == 0 ? WE[c] : b[c]);
                        a[c] = xfma(e, preva, chp(c, q));
                    }
                    if (!((valm >> q) & 1)) continue;
                    const bool isr = (rowm >> q) & 1;
                    // backward accumulators of this element (shared memory, summed over rows)
                    R* acp1 = &sm.acc[0][isr ? ia : na + ib];
                    R* acp2 = &sm.acc[NACC > 1 ? 1 : 0][isr ? ia : na + ib];
                    R acc1 = R(0), acc2 = R(0);
                    if constexpr (BWD) {
                        if (r > r0) {
                            acc1 = *acp1;
                            if constexpr (PHASED) acc2 = *acp2;
                        }
                    }
                    if constexpr (SEQ) {
                        const uint32_t i = g.a0 + ia;
                        p.pre[(size_t)r * p.n + i] = a[0];
                        p.suf[(size_t)r * p.n + i] = OS(0, q);
                        ++ia;
                    } else if (isr) {
                        const int li = ia++;
                        if constexpr (!BWD && NX > 0) {
                            R out = xadd(a[0], OS(0, q));
                            if constexpr (NX == 2) out = xadd(xmul(MCw(q), out), xmul(MSw(q), xadd(a[1], OS(1, q))));
                            stg[li] = out;
                        } else if constexpr (BWD) {
                            if constexpr (!PHASED) {
                                const R gg = pay[0][q];
                                acc1 = xfma(xmul(gg, p.inv_t), xsub(OS(0, q), a[1]), acc1);
                            } else {
                                const R gg = raw[q];
                                const R m0 = MCw(q), m1 = MSw(q);
                                const R in0 = xsub(OS(2, q), a[NG]);  // sum_{b>a} - sum_{b<a}
                                const R in1 = xsub(OS(3, q), a[NG + 1]);
                                acc1 = xfma(xmul(xmul(m0, gg), p.inv_t), in0, acc1);
                                acc1 = xfma(xmul(xmul(m1, gg), p.inv_t), in1, acc1);
                                const R p0 = xadd(a[NG], OS(0, q)), p1 = xadd(a[NG + 1], OS(1, q));
                                acc2 = xfma(gg, xadd(xmul(-m1, p0), xmul(m0, p1)), acc2);
                            }
                        }
                    } else {
                        const int li = ib++;
                        if constexpr (NG > 0) {
                            const R xb0 = xadd(a[0], OS(0, q));  // x_bar: identical in transpose and VJP
                            if constexpr (!BWD) {
                                stg[li] = xb0;
                            } else if constexpr (!PHASED) {
                                stg[li] = xb0;
                                const R x = pay[0][q];
                                acc1 = xfma(xmul(x, p.inv_t), xsub(OS(0, q), b[0]), acc1);
                            } else {
                                const R x = raw[q];
                                const R m0 = MCw(q), m1 = MSw(q);
                                const R xb1 = xadd(a[1], OS(1, q));
                                stg[li] = xadd(xmul(m0, xb0), xmul(m1, xb1));
                                acc2 = xfma(x, xadd(xmul(-m1, xb0), xmul(m0, xb1)), acc2);
                                acc1 = xfma(xmul(xmul(m0, x), p.inv_t), xsub(OS(0, q), b[0]), acc1);
                                acc1 = xfma(xmul(xmul(m1, x), p.inv_t), xsub(OS(1, q), b[1]), acc1);
                            }
                        }
                    }
                    if constexpr (BWD) {
                        *acp1 = acc1;
                        if constexpr (PHASED) *acp2 = acc2;
                    }
                }
            }
            // ---- 5. staged per-row outputs -> perm / plan position ----
            if constexpr (!SEQ && ((!BWD && NX > 0) || NG > 0)) {
                cbar<TPB>();  // (B) staging row complete
                if constexpr (!BWD && NX > 0) {
                    R* y = p.y + (size_t)r * p.ldy;
                    for (int k = tid; k < na; k += TPB) {
                        const int li = gmA[k];
                        y[LXO(iA[li], g.a0 + li)] = stg[li];
                    }
                } else if constexpr (!BWD) {
                    R* y = p.y + (size_t)r * p.ldy;
                    for (int k = tid; k < nb; k += TPB) {
                        const int li = gmB[k];
                        y[LXO(iB[li], g.b0 + li)] = stg[li];
                    }
                } else {
                    R* xb = p.xbar + (size_t)r * p.ldxb;
                    if (r + 1 < r1) {
                        for (int k = tid; k < nb; k += TPB) {
                            const int li = gmB[k];
                            xb[LXO(iB[li], g.b0 + li)] = stg[li];
                        }
                    } else {  // last row: the column cotangents (summed over rows in 4b) are complete
                        for (int k = tid; k < nb; k += TPB) {
                            const int li = gmB[k];
                            const uint32_t u = LXO(iB[li], g.b0 + li);
                            xb[u] = stg[li];
                            const size_t cu = SPLIT ? (size_t)(r0 / p.rchunk) * p.ldpb + u : u;  // row chunk's partial
                            p.bbar[cu] = sm.acc[0][na + li];
                            if constexpr (PHASED) p.psibar[cu] = sm.acc[NACC - 1][na + li];
                        }
                    }
                }
            }
            fence_proxy_async_smem();  // staging writes before any TMA refill of this stage
            cbar<TPB>();  // (C) staging row and warp totals free for the next row / tile
        }
        if constexpr (BWD) {  // row cotangents summed over rows (complete after (C)); the
                              // column ones went out with the last row's x_bar
            const uint32_t* iA = S.oidx + g.offIA;
            for (int k = tid; k < na; k += TPB) {
                const int li = gmA[k];
                const uint32_t u = LXO(iA[li], g.a0 + li);
                const size_t cu = SPLIT ? (size_t)(r0 / p.rchunk) * p.ldpa + u : u;  // row chunk's partial
                p.abar[cu] = sm.acc[0][li];
                if constexpr (PHASED) p.phibar[cu] = sm.acc[NACC - 1][li];
            }
            cbar<TPB>();
        }
        if (tid == 0) mbar_arrive(&S.empty);  // the stage may be refilled
    }
}

// Row split: out[i] = sum over the C row chunks of part[c * m + i], chunks in
// order (deterministic; the unsplit kernel sums the same rows in row order)
template <class R>
__global__ void __launch_bounds__(256) lx_chunk_sum(const R* __restrict__ part, int C, size_t m, R* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
        R v = part[i];
        for (int c = 1; c < C; ++c) v = xadd(v, part[(size_t)c * m + i]);
        out[i] = v;
    }
}

}  // namespace ms
}  // namespace lx
