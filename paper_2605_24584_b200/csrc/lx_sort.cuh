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
//                       (warp-aggregated via match.any, then smem atomics)
//   2. lx_sort_bases    exclusive scan of each pass's 256 counts
//   3. lx_sort_pass x P one kernel per 8-bit digit; each CTA takes a dynamic
//                       tile id, ranks its keys stably (warp multi-split with
//                       match.any), publishes per-digit counts and resolves
//                       its global offsets by DECOUPLED LOOK-BACK over the
//                       tiles before it, then scatters through shared memory
//                       so global writes are digit-contiguous runs.
// LSD with stable passes == std::stable_sort on the IEEE order; the last pass
// writes the sorted Real values (sign of zero restored) and the u32 perm.
#pragma once

#include "lx_common.cuh"

namespace lx {
namespace sort {

constexpr int kBits = 8;
constexpr int kRadix = 256;
constexpr int kThreads = 256;  // == kRadix: one look-back lane per digit
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per tile

// look-back status word: [63:62] flag (1 aggregate, 2 inclusive prefix),
// [61:32] pass epoch, [31:0] count
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;

__device__ __forceinline__ unsigned long long status(unsigned long long flag, uint32_t epoch, uint32_t c) {
    return flag | ((unsigned long long)(epoch & 0x3fffffffu) << 32) | c;
}

template <class R>
__global__ void __launch_bounds__(kThreads) lx_sort_hist(const R* __restrict__ raw, size_t n, R t,
                                                        uint32_t* __restrict__ hist, int* __restrict__ bad) {
    using K = typename Traits<R>::Key;
    constexpr int P = Traits<R>::kPasses;
    __shared__ uint32_t sh[P][kRadix];
    for (int i = threadIdx.x; i < P * kRadix; i += kThreads) (&sh[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int any_bad = 0;
    const size_t stride = (size_t)gridDim.x * kThreads;
    for (size_t base = (size_t)blockIdx.x * kThreads; base < n; base += stride) {
        const size_t i = base + threadIdx.x;
        const bool valid = i < n;
        K key = 0;
        if (valid) {
            const R v = raw[i];
            if (!isfinite(v)) any_bad = 1;
            key = radix_key<R>(xdiv(v, t));
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int d = valid ? (int)((key >> (p * kBits)) & (kRadix - 1)) : kRadix;
            const unsigned peers = __match_any_sync(FULL, d);
            if (d < kRadix && lane == __ffs(peers) - 1) atomicAdd(&sh[p][d], (uint32_t)__popc(peers));
        }
    }
    if (any_bad) atomicOr(bad, 1);
    __syncthreads();
    for (int i = threadIdx.x; i < P * kRadix; i += kThreads) {
        const uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
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

template <class R>
struct PassSmem {
    using K = typename Traits<R>::Key;
    uint32_t whist[kWarps][kRadix];
    uint32_t dstart[kRadix];
    uint32_t gbase[kRadix];
    uint32_t scan[kWarps];
    uint32_t tile;
    K keys[kTile];
    uint32_t vals[kTile];
};

// One digit pass.  FIRST reads the raw anchors and builds keys+payload on the
// fly; LAST writes sorted values (Real) and perm (u32) instead of key/payload.
template <class R, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kThreads) lx_sort_pass(const void* __restrict__ in_keys,
                                                        const uint32_t* __restrict__ in_vals,
                                                        void* __restrict__ out_keys,
                                                        uint32_t* __restrict__ out_vals, size_t n, R t,
                                                        int shift, const uint32_t* __restrict__ bases,
                                                        unsigned long long* __restrict__ lookback,
                                                        uint32_t* __restrict__ tile_counter, uint32_t epoch) {
    using K = typename Traits<R>::Key;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem<R>& sm = *reinterpret_cast<PassSmem<R>*>(smem_raw);
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    if (tid == 0) sm.tile = atomicAdd(tile_counter, 1u);
    for (int i = tid; i < kWarps * kRadix; i += kThreads) (&sm.whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = sm.tile;
    const size_t tile_start = (size_t)tile * kTile;
    const int tile_n = (int)min((size_t)kTile, n - tile_start);

    // ---- load (warp-striped: item k of lane l is element base + k*32 + l) ----
    K key[kItems];
    uint32_t val[kItems];
    const size_t wbase = tile_start + (size_t)warp * 32 * kItems;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const size_t i = wbase + (size_t)k * 32 + lane;
        if (i < n) {
            if constexpr (FIRST) {
                const R s = xdiv(reinterpret_cast<const R*>(in_keys)[i], t);
                const bool nz = as_bits(s) == Traits<R>::kSign;
                key[k] = radix_key<R>(s);
                val[k] = (uint32_t)i | (nz ? 0x80000000u : 0u);
            } else {
                key[k] = reinterpret_cast<const K*>(in_keys)[i];
                val[k] = in_vals[i];
            }
        } else {
            key[k] = 0;
            val[k] = 0;
        }
    }

    // ---- stable warp multi-split ranking ----
    uint32_t rank[kItems];
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const size_t i = wbase + (size_t)k * 32 + lane;
        const int d = i < n ? (int)((key[k] >> shift) & (kRadix - 1)) : kRadix;
        const unsigned peers = __match_any_sync(FULL, d);
        const int leader = __ffs(peers) - 1;
        uint32_t cnt = 0;
        if (d < kRadix && lane == leader) cnt = sm.whist[warp][d];
        cnt = __shfl_sync(FULL, cnt, leader);
        if (d < kRadix && lane == leader) sm.whist[warp][d] = cnt + __popc(peers);
        rank[k] = cnt + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // ---- per digit: warp-exclusive offsets, tile count ----
    const int d = tid;  // kThreads == kRadix
    uint32_t count = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = sm.whist[w][d];
        sm.whist[w][d] = count;
        count += c;
    }
    unsigned long long* my_status = lookback + (size_t)tile * kRadix + d;
    if (tile == 0)
        st_relaxed_u64(my_status, status(kFlagInc, epoch, count));
    else
        st_relaxed_u64(my_status, status(kFlagAgg, epoch, count));

    // block exclusive scan of counts over digits -> shared-memory positions
    uint32_t incl = count;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) sm.scan[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
        if (w < warp) wpre += sm.scan[w];
    const uint32_t dstart = wpre + incl - count;

    // ---- decoupled look-back (one lane per digit) ----
    uint32_t excl = 0;
    if (tile > 0) {
        uint32_t j = tile - 1;
        while (true) {
            const unsigned long long s = ld_relaxed_u64(lookback + (size_t)j * kRadix + d);
            const uint32_t e = (uint32_t)(s >> 32) & 0x3fffffffu;
            const unsigned long long f = s & (3ull << 62);
            if (f == 0 || e != (epoch & 0x3fffffffu)) continue;  // predecessor not published yet
            excl += (uint32_t)s;
            if (f == kFlagInc) break;
            --j;
        }
        st_relaxed_u64(my_status, status(kFlagInc, epoch, excl + count));
    }
    sm.dstart[d] = dstart;
    sm.gbase[d] = bases[d] + excl - dstart;
    __syncthreads();

    // ---- scatter into shared memory in digit order ----
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const size_t i = wbase + (size_t)k * 32 + lane;
        if (i < n) {
            const int dk = (int)((key[k] >> shift) & (kRadix - 1));
            const uint32_t pos = sm.dstart[dk] + sm.whist[warp][dk] + rank[k];
            sm.keys[pos] = key[k];
            sm.vals[pos] = val[k];
        }
    }
    __syncthreads();

    // ---- digit-contiguous global writes ----
    for (int i = tid; i < tile_n; i += kThreads) {
        const K kk = sm.keys[i];
        const uint32_t v = sm.vals[i];
        const int dk = (int)((kk >> shift) & (kRadix - 1));
        const uint32_t o = sm.gbase[dk] + (uint32_t)i;
        if constexpr (LAST) {
            reinterpret_cast<R*>(out_keys)[o] = radix_value<R>(kk, (v >> 31) != 0);
            out_vals[o] = v & 0x7fffffffu;
        } else {
            reinterpret_cast<K*>(out_keys)[o] = kk;
            out_vals[o] = v;
        }
    }
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
