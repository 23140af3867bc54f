// lx_shard.cuh -- building blocks of the range-sharded (multi-GPU) operator.
//
// a single long vector is split into contiguous SORTED ranges,
// one per GPU.  Splitters are VALUES shared by a and b and an element goes to
// shard #{splitters < value}, so a run of equal values never straddles two
// shards (the tie-inclusive co-ranks stay shard-local).  These kernels:
//   lx_shard_count / lx_shard_totals / lx_shard_scan / lx_shard_scatter
//       stable partition of raw/t by shard: counts per shard and the local
//       index of every element in shard order (what goes into the all-to-all);
//   lx_collect_totals
//       per-shard totals of the tile-carry scan (prefix inclusive at the last
//       tile, suffix inclusive at the first) -- what the all-gather exchanges;
//   lx_gather_idx / lx_scatter_idx
//       payload routing by those index lists.
#pragma once

#include "lx_common.cuh"

namespace lx {
namespace shard {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;
constexpr int kMaxShards = 64;

template <class R>
__device__ __forceinline__ int shard_of(R v, const R* spl, int nspl) {
    int s = 0;
    for (int i = 0; i < nspl; ++i) s += spl[i] < v ? 1 : 0;
    return s;
}

// per-tile shard counts: cnt[tile * kMaxShards + s]
template <class R>
__global__ void __launch_bounds__(kThreads) lx_shard_count(const R* __restrict__ raw, size_t m, R t,
                                                          const R* __restrict__ spl, int nspl,
                                                          uint32_t* __restrict__ cnt) {
    __shared__ uint32_t sc[kMaxShards];
    __shared__ R ss[kMaxShards];
    if (threadIdx.x < kMaxShards) sc[threadIdx.x] = 0;
    if (threadIdx.x < nspl) ss[threadIdx.x] = spl[threadIdx.x];
    __syncthreads();
    const size_t base = (size_t)blockIdx.x * kTile;
    for (int q = 0; q < kItems; ++q) {
        const size_t i = base + (size_t)q * kThreads + threadIdx.x;
        if (i < m) atomicAdd(&sc[shard_of(xdiv(raw[i], t), ss, nspl)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < kMaxShards) cnt[(size_t)blockIdx.x * kMaxShards + threadIdx.x] = sc[threadIdx.x];
}

// Exclusive offsets off[tile][s] = sum_{s' < s} total[s'] + sum_{tile' < tile}
// cnt[tile'][s], one CTA per shard (a serial one-block walk took ~1.7 ms per
// call at 2^27 elements): lx_shard_totals sums each shard's column (counts[s]),
// lx_shard_scan turns it into offsets seeded with the lower shards' totals.
constexpr int kOffThreads = 1024;

__global__ void __launch_bounds__(kOffThreads) lx_shard_totals(const uint32_t* __restrict__ cnt, uint32_t tiles,
                                                              uint32_t* __restrict__ counts) {
    __shared__ uint32_t ws[kOffThreads / 32];
    const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t sum = 0;
    for (uint32_t t = tid; t < tiles; t += kOffThreads) sum += cnt[(size_t)t * kMaxShards + s];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    if (lane == 0) ws[warp] = sum;
    __syncthreads();
    if (tid == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < kOffThreads / 32; ++w) tot += ws[w];
        counts[s] = tot;
    }
}

__global__ void __launch_bounds__(kOffThreads) lx_shard_scan(uint32_t* __restrict__ cnt, uint32_t tiles,
                                                            const uint32_t* __restrict__ counts) {
    constexpr int NW = kOffThreads / 32;
    __shared__ uint32_t ws[NW];
    __shared__ uint32_t carry;
    const int s = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        uint32_t b = 0;
        for (int q = 0; q < s; ++q) b += counts[q];
        carry = b;
    }
    __syncthreads();
    for (uint32_t base = 0; base < tiles; base += kOffThreads) {
        const uint32_t t = base + tid;
        const uint32_t v = t < tiles ? cnt[(size_t)t * kMaxShards + s] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) ws[warp] = incl;
        __syncthreads();
        uint32_t before = carry;
        for (int w = 0; w < warp; ++w) before += ws[w];
        if (t < tiles) cnt[(size_t)t * kMaxShards + s] = before + incl - v;
        __syncthreads();
        if (tid == kOffThreads - 1) carry = before + incl;
        __syncthreads();
    }
}

// stable scatter of local indices into shard order (ranks by ballots over the
// shard id bits, warp order = input order)
template <class R>
__global__ void __launch_bounds__(kThreads) lx_shard_scatter(const R* __restrict__ raw, size_t m, R t,
                                                            const R* __restrict__ spl, int nspl,
                                                            const uint32_t* __restrict__ off,
                                                            uint32_t* __restrict__ perm) {
    constexpr int W = kThreads / 32;
    __shared__ uint32_t wc[W][kMaxShards];
    __shared__ R ss[kMaxShards];
    for (int i = threadIdx.x; i < W * kMaxShards; i += kThreads) (&wc[0][0])[i] = 0;
    if (threadIdx.x < nspl) ss[threadIdx.x] = spl[threadIdx.x];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t base = (size_t)blockIdx.x * kTile + (size_t)warp * 32 * kItems;
    int sh[kItems];
    uint32_t rk[kItems];
    const unsigned lt = lanemask_lt();
    for (int q = 0; q < kItems; ++q) {
        const size_t i = base + (size_t)q * 32 + lane;
        const bool valid = i < m;
        const int d = valid ? shard_of(xdiv(raw[i], t), ss, nspl) : kMaxShards - 1;
        unsigned peers = __ballot_sync(FULL, valid);
        if (!valid) peers = ~peers;
        for (int b = 0; b < 6; ++b) {
            const bool bit = (d >> b) & 1;
            const unsigned mk = __ballot_sync(FULL, bit);
            peers &= bit ? mk : ~mk;
        }
        const int leader = __ffs(peers) - 1;
        uint32_t c = 0;
        if (lane == leader) c = wc[warp][d];
        c = __shfl_sync(FULL, c, leader);
        if (lane == leader && valid) wc[warp][d] = c + __popc(peers);
        sh[q] = d;
        rk[q] = c + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    // warp-exclusive offsets per shard
    if (threadIdx.x < kMaxShards) {
        uint32_t run = 0;
        for (int w = 0; w < W; ++w) {
            const uint32_t c = wc[w][threadIdx.x];
            wc[w][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int q = 0; q < kItems; ++q) {
        const size_t i = base + (size_t)q * 32 + lane;
        if (i < m) perm[off[(size_t)blockIdx.x * kMaxShards + sh[q]] + wc[warp][sh[q]] + rk[q]] = (uint32_t)i;
    }
}

// totals layout (R): [0] prefix anchor (last merged element), [1] suffix anchor
// (first merged element), [2] 1 if the shard has elements, then prefix totals
// [slot][rows] and suffix totals [slot][rows] (slots = 2 * channels).
template <class R>
__global__ void lx_collect_totals(const R* __restrict__ cp, const R* __restrict__ cq, const R* __restrict__ s_last,
                                  const R* __restrict__ s_first, uint32_t T, int rows, int slots,
                                  R* __restrict__ out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int per = slots * rows;
    if (e == 0) {
        out[0] = s_last[T - 1];
        out[1] = s_first[0];
        out[2] = R(1);
    }
    if (e < per) {
        out[3 + e] = cp[(size_t)e * T + T - 1];
        out[3 + per + e] = cq[(size_t)e * T + 0];
    }
}

// Routing by index list (partition order <-> caller order).  The index list
// of a stable partition is a few increasing runs (one per destination shard),
// so blocks take contiguous chunks of the partition order in launch order:
// the runs then advance together through the caller array and every region of
// it is read (or written) by all runs within a short window -- L2-resident --
// instead of grid-strided positions spread over the whole array (measured on
// the simulated 8-rank step at 2^27 per rank: 65 ms -> see DESIGN.md 7).
// grid: (chunks, rows of this launch)
constexpr int kRouteThreads = 256;
constexpr int kRouteItems = 8;
constexpr int kRouteChunk = kRouteThreads * kRouteItems;

template <class R>
__global__ void __launch_bounds__(kRouteThreads) lx_gather_idx(const R* __restrict__ src, size_t ld_src,
                                                              const uint32_t* __restrict__ idx, size_t m,
                                                              R* __restrict__ dst) {
    const size_t r = blockIdx.y;
    const size_t p0 = (size_t)blockIdx.x * kRouteChunk + threadIdx.x;
    uint32_t u[kRouteItems];
#pragma unroll
    for (int q = 0; q < kRouteItems; ++q) {
        const size_t p = p0 + (size_t)q * kRouteThreads;
        u[q] = p < m ? idx[p] : 0u;
    }
    R v[kRouteItems];
#pragma unroll
    for (int q = 0; q < kRouteItems; ++q) {
        const size_t p = p0 + (size_t)q * kRouteThreads;
        v[q] = p < m ? src[r * ld_src + u[q]] : R(0);
    }
#pragma unroll
    for (int q = 0; q < kRouteItems; ++q) {
        const size_t p = p0 + (size_t)q * kRouteThreads;
        if (p < m) dst[r * m + p] = v[q];
    }
}

template <class R>
__global__ void __launch_bounds__(kRouteThreads) lx_scatter_idx(const R* __restrict__ src,
                                                               const uint32_t* __restrict__ idx, size_t m,
                                                               R* __restrict__ dst, size_t ld_dst) {
    const size_t r = blockIdx.y;
    const size_t p0 = (size_t)blockIdx.x * kRouteChunk + threadIdx.x;
    uint32_t u[kRouteItems];
    R v[kRouteItems];
#pragma unroll
    for (int q = 0; q < kRouteItems; ++q) {
        const size_t p = p0 + (size_t)q * kRouteThreads;
        u[q] = p < m ? idx[p] : 0u;
        v[q] = p < m ? src[r * m + p] : R(0);
    }
#pragma unroll
    for (int q = 0; q < kRouteItems; ++q) {
        const size_t p = p0 + (size_t)q * kRouteThreads;
        if (p < m) dst[r * ld_dst + u[q]] = v[q];
    }
}

}  // namespace shard
}  // namespace lx
