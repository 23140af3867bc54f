// lx_sort.cuh -- onesweep LSD radix sort of temperature-scaled anchors.
//
// Replaces sort_anchors (reference scan.hpp:27-46, std::stable_sort by value)
// inside the LaplexOperator constructor (operator.hpp:103-107).
//
//   key    = radix_key(raw[i] / t)   (IEEE division, -0 canonicalised)
//   payload= i | (raw[i]/t is -0) << 31
//
// Structure (Merrill & Adinets "onesweep"):
//   1. lx_sort_hist     one read of the keys -> all digit histograms
//                       (per-warp shared-memory sub-histograms)
//   2. lx_sort_bases    exclusive scan of each pass's 256 counts
//   3. lx_sort_pass x P one kernel per 8-bit digit; each CTA takes a dynamic
//                       tile id, counts its digits (smem atomics) and publishes
//                       them at once, ranks its keys stably (warp multi-split:
//                       8 ballots give each key's peer mask), then resolves
//                       its global offsets by DECOUPLED LOOK-BACK over the
//                       tiles before it (by then usually one probe) and
//                       scatters through shared memory so global writes are
//                       digit-contiguous runs.
// LSD with stable passes == std::stable_sort on the IEEE order; the last pass
// writes the sorted Real values (sign of zero restored) and the u32 perm.
#pragma once

#include <type_traits>

#include "lx_common.cuh"

namespace lx {
namespace sort {

constexpr int kBits = 8;
constexpr int kRadix = 256;
constexpr int kThreads = 256;  // == kRadix: one look-back lane per digit
constexpr int kWarps = kThreads / 32;
// keys per thread: 24 measured best at 2^30 (sort + counts + plan pass: 16:
// 65.3 ms, 20: 62.4, 24: 60.8, 28: 62.1, 32: 63.1) -- larger tiles shrink the
// per-tile count tables and overheads until registers spill
#ifndef LX_SORT_ITEMS
#define LX_SORT_ITEMS 24
#endif
constexpr int kItems = LX_SORT_ITEMS;
constexpr int kTile = kThreads * kItems;  // 6144 keys per tile

// look-back status word: [63:62] flag (1 aggregate, 2 inclusive prefix),
// [61:32] pass epoch, [31:0] count
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;

__device__ __forceinline__ unsigned long long status(unsigned long long flag, uint32_t epoch, uint32_t c) {
    return flag | ((unsigned long long)(epoch & 0x3fffffffu) << 32) | c;
}

// Upfront digit histograms of all passes in one read of the keys.  Each warp
// owns a private sub-histogram in shared memory (no cross-warp contention);
// each thread keeps kHistItems independent loads in flight.
constexpr int kHistThreads = 512;
constexpr int kHistItems = 8;
#ifndef LX_HIST_SUB
#define LX_HIST_SUB 4
#endif
constexpr int kHistSub = LX_HIST_SUB;

template <class R>
__global__ void __launch_bounds__(kHistThreads) lx_sort_hist(const R* __restrict__ raw, size_t n, R t,
                                                            uint32_t* __restrict__ hist, int* __restrict__ bad) {
    using K = typename Traits<R>::Key;
    constexpr int P = Traits<R>::kPasses;
    constexpr int W = kHistThreads / 32;
    constexpr int SUB = kHistSub;  // sub-histograms per block (warp % SUB)
    extern __shared__ uint32_t shh[];  // [SUB][P][kRadix]
    for (int i = threadIdx.x; i < SUB * P * kRadix; i += kHistThreads) shh[i] = 0;
    __syncthreads();
    uint32_t* mine = shh + ((threadIdx.x >> 5) % SUB) * P * kRadix;
    (void)W;
    int any_bad = 0;
    const size_t per_block = (size_t)kHistThreads * kHistItems;
    for (size_t base = (size_t)blockIdx.x * per_block; base < n; base += (size_t)gridDim.x * per_block) {
        R v[kHistItems];
#pragma unroll
        for (int q = 0; q < kHistItems; ++q) {
            const size_t i = base + (size_t)q * kHistThreads + threadIdx.x;
            v[q] = i < n ? raw[i] : R(0);
        }
#pragma unroll
        for (int q = 0; q < kHistItems; ++q) {
            const size_t i = base + (size_t)q * kHistThreads + threadIdx.x;
            if (i < n) {
                if (!isfinite(v[q])) any_bad = 1;
                const K key = radix_key<R>(xdiv(v[q], t));
#pragma unroll
                for (int p = 0; p < P; ++p) atomicAdd(&mine[p * kRadix + (int)((key >> (p * kBits)) & (kRadix - 1))], 1u);
            }
        }
    }
    if (any_bad) atomicOr(bad, 1);
    __syncthreads();
    for (int i = threadIdx.x; i < P * kRadix; i += kHistThreads) {
        uint32_t c = 0;
#pragma unroll
        for (int sub = 0; sub < SUB; ++sub) c += shh[sub * P * kRadix + i];
        if (c) atomicAdd(&hist[i], c);
    }
}

// Reduce-then-scan form of the histogram: the same single read of the raw
// keys also yields pass 1's per-tile digit counts (its tiles are the raw
// order), so pass 1 needs no count kernel.  Up to kHistTilesPerCta consecutive
// pass tiles per CTA (8 measured best at 2^30: 1 -> 2.37 ms, 8 -> 2.11, 64 ->
// 2.32 for both sides); small inputs take fewer per CTA so that every SM gets
// work (2^20 keys: 171 tiles).
#ifndef LX_HIST_TILES
#define LX_HIST_TILES 8
#endif
constexpr int kHistTilesPerCta = LX_HIST_TILES;

// HIST = false: only pass 1's per-tile counts (and the finiteness flag); the
// global digit bases then come from the per-digit totals of lx_sort_scan.
template <class R, bool HIST = true>
__global__ void __launch_bounds__(kThreads, 4) lx_sort_hist_count0(const R* __restrict__ raw, size_t n, R t,
                                                               uint32_t* __restrict__ hist, int* __restrict__ bad,
                                                               uint32_t* __restrict__ cnt, uint32_t tiles,
                                                               uint32_t tiles_per_cta) {
    using K = typename Traits<R>::Key;
    constexpr int P = Traits<R>::kPasses;
    constexpr int SUB = 4;
    __shared__ uint32_t wt[kWarps][kRadix];        // this tile's digit-0 counts per warp
    __shared__ uint32_t gh[SUB][P][kRadix];        // this CTA's histograms of every digit
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < kWarps * kRadix; i += kThreads) (&wt[0][0])[i] = 0;
    for (int i = tid; i < SUB * P * kRadix; i += kThreads) (&gh[0][0][0])[i] = 0;
    __syncthreads();
    uint32_t* mine = &gh[warp % SUB][0][0];
    int any_bad = 0;
    const uint32_t t_lo = blockIdx.x * tiles_per_cta;
    const uint32_t t_hi = min(tiles, t_lo + tiles_per_cta);
    for (uint32_t tile = t_lo; tile < t_hi; ++tile) {
        const size_t base = (size_t)tile * kTile;
        R v[kItems];
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const size_t i = base + (size_t)q * kThreads + tid;
            v[q] = i < n ? raw[i] : R(0);
        }
        auto count = [&](auto unit_t) {  // unit_t: t == 1, where raw / t == raw exactly
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                const size_t i = base + (size_t)q * kThreads + tid;
                if (i >= n) continue;
                if (!isfinite(v[q])) any_bad = 1;
                const K key = radix_key<R>(decltype(unit_t)::value ? v[q] : xdiv(v[q], t));
                atomicAdd(&wt[warp][(int)(key & (kRadix - 1))], 1u);
                if constexpr (HIST) {
#pragma unroll
                    for (int p = 0; p < P; ++p)
                        atomicAdd(&mine[p * kRadix + (int)((key >> (p * kBits)) & (kRadix - 1))], 1u);
                }
            }
        };
        if (t == R(1))
            count(std::true_type{});
        else
            count(std::false_type{});
        __syncthreads();
        if (tid < kRadix) {
            uint32_t c = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                c += wt[w][tid];
                wt[w][tid] = 0;
            }
            cnt[(size_t)tid * tiles + tile] = c;
        }
        __syncthreads();
    }
    if (any_bad) atomicOr(bad, 1);
    if constexpr (HIST) {
        for (int i = tid; i < P * kRadix; i += kThreads) {
            uint32_t c = 0;
#pragma unroll
            for (int sub = 0; sub < SUB; ++sub) c += (&gh[sub][0][0])[i];
            if (c) atomicAdd(&hist[i], c);
        }
    }
}

// Exclusive scan of each pass's digit counts -> global bucket bases.
template <int P>
__global__ void __launch_bounds__(kRadix) lx_sort_bases(const uint32_t* __restrict__ hist,
                                                        uint32_t* __restrict__ bases) {
    __shared__ uint32_t s[kRadix];
    const int p = blockIdx.x;
    const int d = threadIdx.x;
    s[d] = hist[p * kRadix + d];
    __syncthreads();
    for (int off = 1; off < kRadix; off <<= 1) {
        const uint32_t v = d >= off ? s[d - off] : 0;
        __syncthreads();
        s[d] += v;
        __syncthreads();
    }
    bases[p * kRadix + d] = s[d] - hist[p * kRadix + d];
}

// Digit of a key in this pass.  Sort passes take whole bytes (one PRMT for
// 32-bit keys); the permutation-plan pass (SPLAN) takes 8 bits at any shift.
template <bool SPLAN, class K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift) {
    if constexpr (!SPLAN && sizeof(K) == 4)
        return __byte_perm((uint32_t)key, 0u, 0x4440u | (uint32_t)(shift >> 3));
    else
        return (uint32_t)(key >> shift) & (kRadix - 1);
}

// Lanes of the warp whose 8-bit digit equals this lane's, within `peers`:
// per bit one predicate (LOP3), one ballot, one select and one LOP3.
__device__ __forceinline__ unsigned match_digit8(unsigned peers, uint32_t dk) {
    static_assert(kBits == 8, "match_digit8 covers 8 digit bits");
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t, m, s;\n\t"
            "and.b32 t, %1, 1;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 2;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 4;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 8;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 16;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 32;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 64;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "and.b32 t, %1, 128;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 m, p, 0xffffffff;\n\t"
            "selp.b32 s, 0, -1, p;\n\t"
            "xor.b32 m, m, s;\n\t"
            "and.b32 %0, %0, m;\n\t"
            "}"
            : "+r"(peers)
            : "r"(dk));
    return peers;
}

template <class R>
struct PassSmem {
    using K = typename Traits<R>::Key;
    unsigned long long bar;
    uint32_t whist[kWarps][kRadix];  // per-warp digit cursors, then per-warp digit starts
    uint32_t gbase[kRadix];
    uint32_t scan[kWarps];
    uint32_t tscan[kWarps];
    uint32_t tile;
    // the input tile; reordered in place into digit order before the global
    // writes (keys, then payload, each through registers)
    alignas(16) K ik[kTile];
    alignas(16) uint32_t iv[kTile];
};

// CTAs per SM the 32-bit-key pass is built for: 3 (80 registers, ~58 KB of
// shared memory with 24 keys per thread; at 16 keys, 4 CTAs at 64 registers
// measured 2% faster than 3).  A persistent double-buffered form (next tile's
// TMA in flight during ranking) measured 7% slower.
#ifndef LX_SORT_CTAS
#define LX_SORT_CTAS 3
#endif
template <class R>
constexpr int sort_min_blocks() { return sizeof(typename Traits<R>::Key) == 4 ? LX_SORT_CTAS : 2; }

// One digit pass.  FIRST reads the raw anchors and builds keys+payload on the
// fly; LAST writes sorted values (Real) and perm (u32) instead of key/payload.
// SPLAN is the same machinery run once over a permutation P (sorted -> caller
// index) with digit = P[i] >> shift: it writes pos[i] = o (the stable position
// of i in caller-index-bucket order, out_vals) and dst[o] = P[i] (out_keys);
// the bucket bases are d << shift (a permutation fills every bucket exactly).
// That is the B200 form of the reference's cache-blocked ScatterPlan
// (operator.hpp:26-60,130-136).
//
// The tile (keys, payload) arrives in shared memory by TMA bulk copy; keys are
// then read from shared memory where needed, so no thread holds its 16 keys
// across the load latency (register pressure, hence occupancy).
// UNIT (first pass with t == 1, where raw / t == raw bitwise): the raw values
// are turned into radix keys where they are read (ranking, reorder) instead of
// in a separate shared-memory pass; the payload's -0 flags ride in a register
// mask (first pass 5.9 ms -> see DESIGN.md 3).
template <class R, bool FIRST, bool LAST, bool SPLAN = false, bool UNIT = false>
__global__ void __launch_bounds__(kThreads, sort_min_blocks<R>()) lx_sort_pass(const void* __restrict__ in_keys,
                                                        const uint32_t* __restrict__ in_vals,
                                                        void* __restrict__ out_keys,
                                                        uint32_t* __restrict__ out_vals, size_t n, R t,
                                                        int shift, const uint32_t* __restrict__ bases,
                                                        unsigned long long* __restrict__ lookback,
                                                        uint32_t* __restrict__ tile_counter, uint32_t epoch,
                                                        const uint32_t* __restrict__ offs = nullptr,
                                                        const uint32_t* __restrict__ totals = nullptr) {
    using K = typename Traits<R>::Key;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PassSmem<R>& sm = *reinterpret_cast<PassSmem<R>*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    constexpr bool HAS_VALS = !FIRST && !SPLAN;

    // offs (reduce-then-scan mode): global output offset of every (digit, tile),
    // digit-major [kRadix][gridDim.x], from lx_sort_count + lx_sort_scan; the
    // tile is then blockIdx.x and there is no look-back
    if (tid == 0) {
        sm.tile = offs ? blockIdx.x : atomicAdd(tile_counter, 1u);
        mbar_init(&sm.bar, 1);
        fence_mbar_init();
    }
    for (int i = tid; i < kWarps * kRadix; i += kThreads) (&sm.whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = sm.tile;
    const size_t tile_start = (size_t)tile * kTile;
    const int tile_n = (int)min((size_t)kTile, n - tile_start);

    // ---- TMA the tile; a ragged tail (< 16 bytes) is loaded by threads ----
    const K* gk = reinterpret_cast<const K*>(in_keys) + tile_start;
    const uint32_t* gv = HAS_VALS ? in_vals + tile_start : nullptr;
    const bool tma_ok = ((reinterpret_cast<uintptr_t>(gk) & 15) == 0) &&
                        (!HAS_VALS || (reinterpret_cast<uintptr_t>(gv) & 15) == 0);
    const uint32_t kbytes = tma_ok ? ((uint32_t)(tile_n * sizeof(K)) & ~15u) : 0u;
    const uint32_t vbytes = (tma_ok && HAS_VALS) ? ((uint32_t)(tile_n * 4) & ~15u) : 0u;
    if (tid == 0) {
        mbar_expect_tx(&sm.bar, kbytes + vbytes);
        if (kbytes) bulk_g2s(sm.ik, gk, kbytes, &sm.bar);
        if (vbytes) bulk_g2s(sm.iv, gv, vbytes, &sm.bar);
    }
    for (int i = (int)(kbytes / sizeof(K)) + tid; i < tile_n; i += kThreads) sm.ik[i] = gk[i];
    if constexpr (HAS_VALS)
        for (int i = (int)(vbytes / 4) + tid; i < tile_n; i += kThreads) sm.iv[i] = gv[i];
    mbar_wait(&sm.bar, 0);
    __syncthreads();
    static_assert(!UNIT || FIRST, "UNIT is a first-pass form");
    static_assert(!UNIT || kItems <= 32, "the -0 flags live in one 32-bit mask");
    if constexpr (FIRST && !UNIT) {  // raw/t -> radix key, payload = index | (-0 flag)
        // t == 1 (the API default): raw / t == raw bitwise in IEEE arithmetic,
        // so the division (~10 instructions per key) is skipped
        auto convert = [&](auto unit_t) {
            for (int i = tid; i < tile_n; i += kThreads) {
                const R raw = from_bits(sm.ik[i], R(0));
                const R sv = decltype(unit_t)::value ? raw : xdiv(raw, t);
                const bool nz = as_bits(sv) == Traits<R>::kSign;
                sm.ik[i] = radix_key<R>(sv);
                sm.iv[i] = (uint32_t)(tile_start + i) | (nz ? 0x80000000u : 0u);
            }
        };
        if (t == R(1))
            convert(std::true_type{});
        else
            convert(std::false_type{});
        __syncthreads();
    }
    // warp-striped item layout: item k of lane l is tile element w*32*kItems + k*32 + l
    const int wbase = warp * 32 * kItems;
    const bool full = tile_n == kTile;  // every tile but the last: no bounds checks
    const int d = tid;                  // kThreads == kRadix
    // digit totals of the whole pass (reduce-then-scan without upfront histogram)
    const uint32_t tot = (offs && totals) ? totals[d] : 0u;
    unsigned long long* my_status = lookback + (size_t)tile * kRadix + d;

    // ---- stable in-warp ranks.  Per item: the mask of lanes holding the same
    // digit (8 ballots), rank = the warp's running cursor of the digit + lower
    // peers.  All peers read the cursor (one warp-wide LDS) and the highest
    // peer advances it.  Rank and digit stay packed in one register per item.
    uint32_t rd[kItems];  // rank | digit << 16
    const unsigned lt = lanemask_lt();
    uint32_t* wh = sm.whist[warp];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int li = wbase + k * 32 + lane;
        const bool valid = full || li < tile_n;
        K key = sm.ik[li];
        if constexpr (UNIT) key = radix_key<R>(from_bits(key, R(0)));
        const uint32_t dk = digit_of<SPLAN>(key, shift);  // tail slots: stale, masked
        // invalid tail lanes sit above every valid lane of the item: they are
        // masked out of the peers and never advance a cursor
        const unsigned peers = match_digit8(full ? FULL : __ballot_sync(FULL, valid), dk);
        const uint32_t cnt = wh[dk];
        const uint32_t r = cnt + __popc(peers & lt);
        __syncwarp();
        if (valid && (peers >> lane) == 1u) wh[dk] = r + 1u;
        rd[k] = r | (dk << 16);
        __syncwarp();
    }
    __syncthreads();
    uint32_t count = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) count += sm.whist[w][d];
    if (!offs) st_relaxed_u64(my_status, status(tile == 0 ? kFlagInc : kFlagAgg, epoch, count));

    // block exclusive scan of counts over digits -> shared-memory positions
    uint32_t incl = count, tincl = tot;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, off);
        const uint32_t tv = __shfl_up_sync(FULL, tincl, off);
        if (lane >= off) incl += v, tincl += tv;
    }
    if (lane == 31) sm.scan[warp] = incl, sm.tscan[warp] = tincl;
    __syncthreads();
    uint32_t wpre = 0, tpre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
        if (w < warp) wpre += sm.scan[w], tpre += sm.tscan[w];
    const uint32_t dstart = wpre + incl - count;
    const uint32_t dbase = tpre + tincl - tot;  // global start of digit d (0 without totals)
    {   // per (warp, digit): shared-memory start of the warp's keys of the digit
        uint32_t run = dstart;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = sm.whist[w][d];
            sm.whist[w][d] = run;
            run += c;
        }
    }

    if (offs) {  // reduce-then-scan: the offset is known
        sm.gbase[d] = dbase + offs[(size_t)d * gridDim.x + tile] - dstart;
        __syncthreads();
        goto scatter;
    }
    {
    // ---- decoupled look-back (one lane per digit) ----
    uint32_t excl = 0;
    if (tile > 0) {
        uint32_t j = tile - 1;
        while (true) {
            const unsigned long long st = ld_relaxed_u64(lookback + (size_t)j * kRadix + d);
            const uint32_t e = (uint32_t)(st >> 32) & 0x3fffffffu;
            const unsigned long long f = st & (3ull << 62);
            if (f == 0 || e != (epoch & 0x3fffffffu)) continue;  // predecessor not published yet
            excl += (uint32_t)st;
            if (f == kFlagInc) break;
            --j;
        }
        st_relaxed_u64(my_status, status(kFlagInc, epoch, excl + count));
    }
    if constexpr (SPLAN)
        sm.gbase[d] = ((uint32_t)d << shift) + excl - dstart;
    else
        sm.gbase[d] = bases[d] + excl - dstart;
    __syncthreads();
    }
scatter:

    // ---- reorder the tile in place into digit order: keys, then payload ----
    uint32_t nzm = 0;  // UNIT: bit k = item k is -0 (the payload's flag)
    {
        K kv[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const int li = wbase + k * 32 + lane;
            kv[k] = sm.ik[li];  // tail slots: stale, never stored
            if constexpr (UNIT) {
                nzm |= (uint32_t)(kv[k] == Traits<R>::kSign) << k;
                kv[k] = radix_key<R>(from_bits(kv[k], R(0)));
            }
            rd[k] = (wh[rd[k] >> 16] + (rd[k] & 0xffffu)) | (rd[k] & 0xffff0000u);  // shared position | digit
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const int li = wbase + k * 32 + lane;
            if (full || li < tile_n) {
                const uint32_t pos = rd[k] & 0xffffu;
                sm.ik[pos] = kv[k];
                if constexpr (SPLAN) out_vals[tile_start + li] = sm.gbase[rd[k] >> 16] + pos;
            }
        }
    }
    if constexpr (!SPLAN) {
        uint32_t vv[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const int li = wbase + k * 32 + lane;
            if constexpr (UNIT)
                vv[k] = (uint32_t)(tile_start + li) | (((nzm >> k) & 1u) << 31);
            else
                vv[k] = sm.iv[li];
        }
        if constexpr (!UNIT) __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const int li = wbase + k * 32 + lane;
            if (full || li < tile_n) sm.iv[rd[k] & 0xffffu] = vv[k];
        }
    }
    __syncthreads();

    // ---- digit-contiguous global writes ----
    auto put = [&](int i) {
        const K kk = sm.ik[i];
        const uint32_t o = sm.gbase[digit_of<SPLAN>(kk, shift)] + (uint32_t)i;
        if constexpr (SPLAN) {
            reinterpret_cast<K*>(out_keys)[o] = kk;
        } else if constexpr (LAST) {
            const uint32_t v = sm.iv[i];
            reinterpret_cast<R*>(out_keys)[o] = radix_value<R>(kk, (v >> 31) != 0);
            out_vals[o] = v & 0x7fffffffu;
        } else {
            reinterpret_cast<K*>(out_keys)[o] = kk;
            out_vals[o] = sm.iv[i];
        }
    };
    if (full) {
#pragma unroll
        for (int j = 0; j < kItems; ++j) put(j * kThreads + tid);
    } else {
        for (int i = tid; i < tile_n; i += kThreads) put(i);
    }
}

// ---- reduce-then-scan form of a pass (no look-back) --------------------------
// lx_sort_count: per-tile digit counts of the pass (the same tiles and digit
// function as lx_sort_pass), digit-major cnt[d * tiles + tile].
// kCountTiles pass tiles per CTA, all their loads issued up front (more bytes
// in flight per round trip), each tile counted into its own column.
#ifndef LX_COUNT_TILES
#define LX_COUNT_TILES 2
#endif
constexpr int kCountTiles = LX_COUNT_TILES;

template <class R, bool FIRST, bool SPLAN>
__global__ void __launch_bounds__(kThreads) lx_sort_count(const void* __restrict__ in_keys, size_t n, R t, int shift,
                                                         uint32_t* __restrict__ cnt, uint32_t tiles) {
    using K = typename Traits<R>::Key;
    __shared__ uint32_t wh[kCountTiles][kWarps][kRadix];
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < kCountTiles * kWarps * kRadix; i += kThreads) (&wh[0][0][0])[i] = 0;
    __syncthreads();
    const K* gk = reinterpret_cast<const K*>(in_keys);
    constexpr int kV = 16 / sizeof(K);  // keys per 16-byte vector
    constexpr int kVec = kItems / kV;   // vectors per thread per tile
    const uint32_t tile0 = blockIdx.x * kCountTiles;
    const size_t start = (size_t)tile0 * kTile;
    const bool full = start + (size_t)kCountTiles * kTile <= n && (reinterpret_cast<uintptr_t>(gk) & 15) == 0;
    auto count = [&](int j, K key) {
        if constexpr (FIRST) key = radix_key<R>(xdiv(from_bits(key, R(0)), t));
        atomicAdd(&wh[j][warp][(int)((key >> shift) & (kRadix - 1))], 1u);
    };
    if (full) {
        uint4 q4[kCountTiles][kVec];
#pragma unroll
        for (int j = 0; j < kCountTiles; ++j)
#pragma unroll
            for (int v = 0; v < kVec; ++v)
                q4[j][v] = reinterpret_cast<const uint4*>(gk + start + (size_t)j * kTile)[(size_t)v * kThreads + tid];
#pragma unroll
        for (int j = 0; j < kCountTiles; ++j)
#pragma unroll
            for (int v = 0; v < kVec; ++v) {
                const K* kk = reinterpret_cast<const K*>(&q4[j][v]);
#pragma unroll
                for (int e = 0; e < kV; ++e) count(j, kk[e]);
            }
    } else {
        for (int j = 0; j < kCountTiles; ++j)
            for (int q = 0; q < kItems; ++q) {
                const size_t i = start + (size_t)j * kTile + (size_t)q * kThreads + tid;
                if (i < n) count(j, gk[i]);
            }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kCountTiles; ++j) {
        if (tile0 + j >= tiles) break;
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) c += wh[j][w][tid];
        cnt[(size_t)tid * tiles + tile0 + j] = c;
    }
}

// lx_sort_scan: one CTA per digit; offs[d][tile] = base[d] + sum of the
// digit's counts in earlier tiles (in place over cnt).  base = bases[d], or
// d << shift for the plan pass (every caller bucket holds exactly 2^shift).
// Coalesced: the CTA walks the digit's row in chunks of 4 * kScanThreads.
constexpr int kScanThreads = 1024;
// With bases == nullptr and shift < 0 the offsets are relative to the digit's
// own start and the digit's total goes to totals[d]; the pass adds the global
// base (the exclusive scan of the totals, formed in every pass CTA), so no
// upfront histogram of the keys is needed.
__global__ void __launch_bounds__(kScanThreads) lx_sort_scan(uint32_t* __restrict__ cnt, uint32_t tiles,
                                                            const uint32_t* __restrict__ bases, int shift,
                                                            uint32_t* __restrict__ totals = nullptr) {
    constexpr int NW = kScanThreads / 32;
    __shared__ uint32_t ws[NW];
    __shared__ uint32_t carry;
    const int d = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t* c = cnt + (size_t)d * tiles;
    if (tid == 0) carry = bases ? bases[d] : (shift >= 0 ? ((uint32_t)d << shift) : 0u);
    __syncthreads();
    for (uint32_t base = 0; base < tiles; base += 4 * kScanThreads) {
        const uint32_t i0 = base + 4 * (uint32_t)tid;
        uint32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = i0 + j < tiles ? c[i0 + j] : 0u;
        const uint32_t sum = v[0] + v[1] + v[2] + v[3];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) ws[warp] = incl;
        __syncthreads();
        uint32_t before = carry;
        for (int w = 0; w < warp; ++w) before += ws[w];
        uint32_t run = before + incl - sum;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i0 + j < tiles) c[i0 + j] = run;
            run += v[j];
        }
        __syncthreads();  // everyone has read carry and ws
        if (tid == kScanThreads - 1) carry = run;
        __syncthreads();
    }
    if (totals && tid == 0) totals[d] = carry;
}

// ---- permutation plans: the two L2-window passes --------------------------
// Blocks cover contiguous, launch-ordered chunks of the bucketed index q, so
// the resident blocks always sit in one or two caller-index buckets and the
// random side of each pass stays inside an L2-resident window.
constexpr int kPermThreads = 256;
// items per thread: the gather half keeps more independent random reads in
// flight (16: 4.69 -> 4.58 ms per 2^30 launch against 8).  The scatter half
// writes at random inside one caller window, and the entries in flight across
// the GPU (resident threads x items) decide how many windows are live in L2 at
// once: a single row takes 1 item per thread (7.73 ms at 8 -> 7.45 at 4 ->
// 7.02 at 2 -> 6.95 at 1 per 2^30 launch); batched calls, whose grid walks
// the rows, take 4 (C2: 11.2 ms at 4, 12.1 at 2).
#ifndef LX_PERM_GATHER_ITEMS
#define LX_PERM_GATHER_ITEMS 16
#endif
constexpr int kGatherItems = LX_PERM_GATHER_ITEMS;
constexpr int kGatherChunk = kPermThreads * kGatherItems;
constexpr int kScatterItemsRow = 1;    // single-row scatters
constexpr int kScatterItemsBatch = 4;  // batched scatters

// gather (caller order -> sorted order), first half: stage[r][q] = src[r][dst[q]];
// the consumer then reads stage[r][pos[i]].  grid: (chunks, rows)
template <class R>
__global__ void __launch_bounds__(kPermThreads) lx_perm_stage_gather(const R* __restrict__ src, size_t ld_src,
                                                                    const uint32_t* __restrict__ dst, uint32_t m,
                                                                    R* __restrict__ stage) {
    const size_t r = blockIdx.y;
    const size_t q0 = (size_t)blockIdx.x * kGatherChunk + threadIdx.x;
    uint32_t u[kGatherItems];
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
        const size_t q = q0 + (size_t)j * kPermThreads;
        u[j] = q < m ? dst[q] : 0u;
    }
    R v[kGatherItems];
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
        const size_t q = q0 + (size_t)j * kPermThreads;
        v[j] = q < m ? src[r * ld_src + u[j]] : R(0);
    }
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
        const size_t q = q0 + (size_t)j * kPermThreads;
        if (q < m) stage[r * m + q] = v[j];
    }
}

// scatter (sorted order -> caller order), second half: out[r][dst[q]] = stage[r][q]
// for up to three arrays sharing the permutation (s2/s3 may be null, row 0
// only).  One batch row per blockIdx.y: CTAs launch row by row, so the random
// writes in flight stay inside one row's caller window (a CTA looping over 64
// rows kept 64 windows -- 1 GB at n = 2^24 -- live in the 126 MB L2 and ran at
// a third of the single-row rate).  dst is re-read per row (+4 B/element-row).
template <class R, int ITEMS>
__global__ void __launch_bounds__(kPermThreads) lx_perm_stage_scatter(const uint32_t* __restrict__ dst, uint32_t m,
                                                                     const R* __restrict__ s1, R* __restrict__ o1,
                                                                     size_t ld1, int rows1, const R* __restrict__ s2,
                                                                     R* __restrict__ o2, const R* __restrict__ s3,
                                                                     R* __restrict__ o3, uint32_t block0) {
    const size_t q0 = (size_t)(blockIdx.x + block0) * (kPermThreads * ITEMS) + threadIdx.x;
    const size_t r = blockIdx.y;
    uint32_t u[ITEMS];
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const size_t q = q0 + (size_t)j * kPermThreads;
        u[j] = q < m ? dst[q] : 0u;
    }
    R v[ITEMS];  // all loads in flight before the random stores
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const size_t q = q0 + (size_t)j * kPermThreads;
        v[j] = q < m ? s1[r * m + q] : R(0);
    }
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const size_t q = q0 + (size_t)j * kPermThreads;
        if (q < m) o1[r * ld1 + u[j]] = v[j];
    }
    (void)rows1;
    if (r == 0) {
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const size_t q = q0 + (size_t)j * kPermThreads;
            if (q < m) {
                if (s2) o2[u[j]] = s2[q];
                if (s3) o3[u[j]] = s3[q];
            }
        }
    }
}

// gather of a per-element caller-order vector into sorted order (plan build)
template <class R>
__global__ void lx_gather_sorted(const R* __restrict__ src, const uint32_t* __restrict__ perm, uint32_t m,
                                 R* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = src[perm[i]];
}

// Neighbour decays of the sorted values: decays[i] = exp(v_i - v_{i+1})
// (scan.hpp:44-45); only needed by the sorted_rows()/sorted_cols() accessor.
template <class R>
__global__ void lx_decays(const R* __restrict__ v, size_t m, R* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 < m) out[i] = xexp(xsub(v[i], v[i + 1]));
}

}  // namespace sort
}  // namespace lx
