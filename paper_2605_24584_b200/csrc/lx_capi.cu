// lx_capi.cu -- the C-ABI (include/laplex_c.h) over the sm_100a kernels.
//
// A plan is the device-resident image of the reference LaplexOperator
// (operator.hpp:75-437): sorted scaled anchors + permutations of both sides,
// cos/sin of the phases, and the merge-path tile partition.  It is immutable
// after creation; lazily-built extras (role-swapped partition, co-rank arrays)
// are guarded by a mutex.  Temporaries come from the stream-ordered memory
// pool (cudaMallocAsync) so per-call allocation is free after warm-up.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <utility>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/laplex_c.h"
#include "lx_common.cuh"
#include "lx_gram.cuh"
#include "lx_main.cuh"
#include "lx_scan.cuh"
#include "lx_shard.cuh"
#include "lx_sort.cuh"

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

struct Fail {
    int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
    g_last_error = msg;
    throw Fail{code};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(LAPLEX_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void ck_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    ck(cudaGetLastError(), what);
}

// ---- optional per-kernel CUDA-event timing (laplex_profile_*) ----
std::atomic<bool> g_prof{false};
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_recs;

// Launch wrapper: every kernel goes through here, so the launch counter and
// the optional event bracketing see all of them.
template <class F>
void launch(const char* name, cudaStream_t st, F&& f) {
    const bool prof = g_prof.load(std::memory_order_relaxed);
    ProfRec r{name, nullptr, nullptr};
    if (prof) {
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        cudaEventRecord(r.a, st);
    }
    f();
    ck_launch(name);
    if (prof) {
        cudaEventRecord(r.b, st);
        std::lock_guard<std::mutex> g(g_prof_mu);
        g_prof_recs.push_back(r);
    }
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return LAPLEX_OK;
    } catch (const Fail& e) {
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return LAPLEX_E_CUDA;
    }
}

// ---- per-device state ---------------------------------------------------------
// Everything cached per process is keyed by device, so one process may drive
// several GPUs (one thread per device, or switching with cudaSetDevice).
constexpr int kMaxDevices = 64;

int current_device() {
    int d = 0;
    ck(cudaGetDevice(&d), "cudaGetDevice");
    if (d < 0 || d >= kMaxDevices) fail(LAPLEX_E_INVALID_ARGUMENT, "device ordinal out of range");
    return d;
}

// The library's own stream-ordered memory pool per device (not the device's
// default pool), a caching allocator like torch's: freed blocks are kept for
// reuse until laplex_pool_trim() (the analogue of torch.cuda.empty_cache())
// returns them.  A training loop that builds a plan per step must not re-map
// its working set every step: measured +450 ms per C5 step when the pool was
// trimmed on each plan release, and +190 ms (C2) / +200 ms (C4) per step with
// a 1 GiB release threshold, which re-maps at every synchronisation.
struct DevState {
    std::once_flag init;
    cudaMemPool_t pool = nullptr;
    int sms = 148;
    std::mutex mu;
    size_t reserved = 0;  // working-set reservation currently held by the pool
    int live_plans = 0;
    cudaStream_t release = nullptr;  // plan buffers are freed here, after every user stream
};
DevState g_dev[kMaxDevices];

DevState& dev_state(int d = -1) {
    if (d < 0) d = current_device();
    DevState& s = g_dev[d];
    std::call_once(s.init, [&] {
        cudaMemPoolProps props;
        std::memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = d;
        ck(cudaMemPoolCreate(&s.pool, &props), "cudaMemPoolCreate");
        uint64_t thr = UINT64_MAX;
        ck(cudaMemPoolSetAttribute(s.pool, cudaMemPoolAttrReleaseThreshold, &thr), "cudaMemPoolSetAttribute");
        cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, d);
        ck(cudaStreamCreateWithFlags(&s.release, cudaStreamNonBlocking), "cudaStreamCreate");
    });
    return s;
}

int num_sms() { return dev_state().sms; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device)
template <class K>
void smem_attr(K kern, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, int>> done;
    const int d = current_device();
    const void* key = reinterpret_cast<const void*>(kern);
    std::lock_guard<std::mutex> g(mu);
    for (auto& e : done)
        if (e.first == key && e.second == d) return;
    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "cudaFuncSetAttribute");
    done.emplace_back(key, d);
}

// resident CTAs per SM of a kernel (after smem_attr), cached per (kernel, device)
template <class K>
int occupancy(K kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> done;
    const int d = current_device();
    const void* key = reinterpret_cast<const void*>(kern);
    std::lock_guard<std::mutex> g(mu);
    for (auto& e : done)
        if (e.first.first == key && e.first.second == d) return e.second;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    per_sm = std::max(per_sm, 1);
    done.push_back({{key, d}, per_sm});
    return per_sm;
}

// Working-set reservation.  The stream-ordered pool maps physical memory on
// demand; at 2^30 it otherwise kept growing in some runs well after warm-up
// (fragmentation), and each growth stalled the enqueue thread (measured:
// 1 run in 4 with 10-60 ms/step of GPU idle).  A plan of m = n + k elements
// reserves its working set once, as one block that the pool then
// sub-allocates: 36 B per element for device-pointer plans (the step peaks
// at 28 B per element), 48 B for host-pointer plans (which add the uploaded
// inputs and outputs).  LAPLEX_POOL_RESERVE_GB overrides the size (0
// disables).
void reserve_pool(size_t m, size_t rsz, size_t per_elem, cudaStream_t st) {
    DevState& ds = dev_state();
    size_t bytes = m * per_elem * (rsz / 4);
    if (const char* e = std::getenv("LAPLEX_POOL_RESERVE_GB")) bytes = (size_t)(std::atof(e) * (double)(1ull << 30));
    if (bytes < (size_t(1) << 31)) return;  // small problems: on-demand growth is cheap
    std::lock_guard<std::mutex> g(ds.mu);
    if (bytes <= ds.reserved) return;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return;
    bytes = std::min(bytes, free_b - std::min(free_b, size_t(4) << 30));  // leave headroom
    void* q = nullptr;
    if (bytes > ds.reserved && cudaMallocFromPoolAsync(&q, bytes, ds.pool, st) == cudaSuccess) {
        cudaFreeAsync(q, st);
        ds.reserved = bytes;
    }
    cudaGetLastError();
}

void plan_born(int d) {
    DevState& ds = dev_state(d);
    std::lock_guard<std::mutex> g(ds.mu);
    ++ds.live_plans;
}

void plan_died(int d) {
    DevState& ds = dev_state(d);
    std::lock_guard<std::mutex> g(ds.mu);
    --ds.live_plans;
}

// stream-ordered device buffer from the library's pool
struct DBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    DBuf() = default;
    DBuf(size_t bytes, cudaStream_t s) : st(s) {
        if (bytes) ck(cudaMallocFromPoolAsync(&p, bytes, dev_state().pool, s), "cudaMallocFromPoolAsync");
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
    DBuf& operator=(DBuf&& o) noexcept {
        release();
        p = o.p;
        st = o.st;
        o.p = nullptr;
        return *this;
    }
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
    }
    template <class T>
    T* as() const {
        return reinterpret_cast<T*>(p);
    }
};

size_t rsize(int dtype) { return dtype == LAPLEX_F64 ? 8 : 4; }

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
struct Side {
    DBuf vals;  // sorted scaled anchors
    DBuf perm;  // u32 sorted -> caller index
    DBuf cph, sph;  // cos/sin of this side's phases, SORTED order
    // permutation plan (large sides): pos[i] = bucketed position of sorted i,
    // dst[q] = caller index at bucketed position q (caller-index buckets of
    // 2^shift elements, so each bucket's caller range is an L2-sized window)
    DBuf spos, sdst;
    bool staged = false;     // large side: every call permutes through the plan
    bool has_splan = false;  // spos / sdst exist (large side, or built for a large batch)
    uint32_t m = 0;
};

// Plans up to this many anchors (n + k) build their two sides concurrently
// (device API; see the core build).  C1 (2^20 + 2^20): 0.338 -> 0.271 ms; at
// C4's 2 x 3 * 2^20 the forked build measured slower and erratic (3.14 ->
// 3.29 / 4.40 ms: the side stream cannot reuse pool blocks freed on the other)
constexpr size_t kForkSidesMax = size_t(1) << 21;

// a second, non-blocking stream of the calling thread on the current device
cudaStream_t side_stream() {
    thread_local cudaStream_t ss[64] = {};
    const int d = current_device();
    if (d < 0 || d >= 64) fail(LAPLEX_E_CUDA, "device index");
    if (!ss[d]) ck(cudaStreamCreateWithFlags(&ss[d], cudaStreamNonBlocking), "cudaStreamCreate");
    return ss[d];
}

// Sides up to this many elements permute directly (the whole vector is
// L2-resident, 126 MB); larger ones go through the two-pass plan.
constexpr uint32_t kDirectMax = 1u << 22;
#ifndef LX_FWD_TPB
#define LX_FWD_TPB 128
#endif
#ifndef LX_BWD_TPB
#define LX_BWD_TPB 128
#endif
constexpr size_t kTmaPad = 64;  // slack after anchor arrays for 16-byte TMA rounding

struct Core {
    int dtype = LAPLEX_F32;
    int device = 0;
    double t = 1.0;
    bool phased = false;
    Side side[2];  // [ROWS], [COLS]
    std::mutex mu;
    DBuf part[2];  // merge-path tiles with side 0 (resp. 1) as the "A" operand, A-first
    DBuf desc[2], sfirst[2], slast[2];  // per-tile descriptors and edge anchors
    DBuf gmt[2];      // per orientation: store order of both sides, one kTile slot per tile (lx_group_plan)
    DBuf mwd[2];      // per orientation: merge words of every tile (lx_group_plan)
    uint32_t T[2] = {0, 0};
    DBuf ranks[4];  // [side*2 + strict]
    bool has_ranks[4] = {false, false, false, false};
    cudaEvent_t built[2] = {nullptr, nullptr};  // [0]: plan created; [1]: role-swapped data (lazy)
    cudaEvent_t splan_ev[2] = {nullptr, nullptr};  // permutation plan of a small side built for a batch
    // x of the last forward kept for its backward (LAPLEX_SAVE_X / LAPLEX_REUSE_X):
    // the sorted payload and its tile aggregates (inclusive + strict), i.e.
    // exactly what the backward's x gather would recompute
    struct SavedX {
        const void* X = nullptr;  // device pointer, or the caller's host pointer (host API)
        size_t rows = 0;
        bool swapped = false, phased = false, host = false;
        DBuf xs, aggp, aggq;
        size_t ldxs = 0, agg_count = 0;
        cudaEvent_t ready = nullptr;
    } saved;
    std::mutex saved_mu;
    int bad_host[4] = {0, 0, 0, 0};
    // Streams that used the plan, each with an event after its last use.  The
    // buffers are freed on the device's release stream once it has waited
    // for all of them: stream-ordered, and the releasing host thread never blocks.
    std::mutex use_mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
    template <class F>
    void for_each_buf(F&& f) {
        for (Side& sd : side)
            for (DBuf* b : {&sd.vals, &sd.perm, &sd.cph, &sd.sph, &sd.spos, &sd.sdst}) f(*b);
        for (int o = 0; o < 2; ++o)
            for (DBuf* b : {&part[o], &desc[o], &sfirst[o], &slast[o], &gmt[o], &mwd[o]}) f(*b);
        for (DBuf& b : ranks) f(b);
        f(saved.xs), f(saved.aggp), f(saved.aggq);
    }
    ~Core() {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        // one stream used the plan (the common case): free on it, behind its
        // work; several: on the release stream, after every one of them
        cudaStream_t rel = uses.size() == 1 ? uses[0].first : dev_state(device).release;
        for (auto& u : uses) {
            if (rel != u.first) cudaStreamWaitEvent(rel, u.second, 0);
            cudaEventDestroy(u.second);
        }
        for (cudaEvent_t e : {built[0], built[1], saved.ready, splan_ev[0], splan_ev[1]})
            if (e) {
                if (uses.size() != 1) cudaStreamWaitEvent(rel, e, 0);
                cudaEventDestroy(e);
            }
        for_each_buf([&](DBuf& b) {
            b.st = rel;
            b.release();
        });
        plan_died(device);
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

struct laplex_plan_s {
    std::shared_ptr<Core> core;
    bool swapped = false;
    std::atomic<int> refs{1};
};

struct laplex_work_s;  // defined after the staged helpers

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

laplex_plan_s* check_plan(laplex_plan p) {
    if (!p || !p->core) fail(LAPLEX_E_INVALID_ARGUMENT, "invalid plan handle");
    return p;
}

// Orientation-resolved view: A = output side of apply, B = input side.
template <class R>
struct View {
    const R* A;
    const uint32_t* pa;
    uint32_t n;
    const R* B;
    const uint32_t* pb;
    uint32_t k;
    const R *cphi, *sphi, *cpsi, *spsi;
    const uint32_t* part;
    const lx::ms::TileDesc<R>* desc;
    const R* s_first;
    const R* s_last;
    uint32_t T;
    R inv_t;
    const uint32_t *pos_a, *dst_a, *pos_b, *dst_b;  // null = direct permutation
    const uint16_t* gmt;                              // per-tile store order (lx_group_plan)
    const uint32_t* mw;                               // per-tile merge words (lx_group_plan)
};

// ≤256 caller-index buckets of 2^shift elements (permutation plans, store grouping)
int bucket_shift(uint32_t m) {
    int bits = 0;
    while ((1ull << bits) < m) ++bits;
    return bits > 8 ? bits - 8 : 0;
}

uint32_t tiles_for(uint64_t total) { return (uint32_t)((total + lx::ms::kTile - 1) / lx::ms::kTile); }

template <class R>
void build_partition(Core& c, int which, cudaStream_t st) {
    const Side& a = c.side[which];
    const Side& b = c.side[1 - which];
    const uint32_t T = tiles_for((uint64_t)a.m + b.m);
    c.part[which] = DBuf((size_t)(T + 1) * 4, st);
    c.desc[which] = DBuf((size_t)(T + 1) * sizeof(lx::ms::TileDesc<R>), st);
    c.sfirst[which] = DBuf((size_t)T * sizeof(R), st);
    c.slast[which] = DBuf((size_t)T * sizeof(R), st);
    launch("lx_partition", st, [&] {
        lx::ms::lx_partition<R, true><<<(T + 1 + 255) / 256, 256, 0, st>>>(
            a.vals.as<R>(), a.m, b.vals.as<R>(), b.m, c.part[which].as<uint32_t>(), T);
    });
    launch("lx_tiledesc", st, [&] {
        lx::ms::lx_tiledesc<R><<<(T + 1 + 255) / 256, 256, 0, st>>>(
            a.vals.as<R>(), a.m, b.vals.as<R>(), b.m, c.part[which].as<uint32_t>(), T,
            c.desc[which].as<lx::ms::TileDesc<R>>(), c.sfirst[which].as<R>(), c.slast[which].as<R>());
    });
    c.T[which] = T;
    c.mwd[which] = DBuf((size_t)T * lx::ms::kMergeWords * 4 + 16, st);
    // per-tile store order of both sides (output positions: plan pos or perm)
    const uint32_t* pa = a.staged ? a.spos.as<uint32_t>() : a.perm.as<uint32_t>();
    const uint32_t* pb = b.staged ? b.spos.as<uint32_t>() : b.perm.as<uint32_t>();
    c.gmt[which] = DBuf((size_t)T * lx::ms::kTile * 2 + 16, st);
    const size_t gsm = lx::ms::group_plan_smem<R>();
    smem_attr(lx::ms::lx_group_plan<R>, gsm);
    if (T)
        launch("lx_group_plan", st, [&] {
            lx::ms::lx_group_plan<R><<<T, lx::ms::kGroupBuckets, gsm, st>>>(
                c.desc[which].as<lx::ms::TileDesc<R>>(), T, pa, bucket_shift(a.m), pb, bucket_shift(b.m),
                c.gmt[which].as<uint16_t>(), a.vals.as<R>(), b.vals.as<R>(), c.mwd[which].as<uint32_t>());
        });
}

void build_splan(Side& sd, cudaStream_t st);

// Batches whose rows x side footprint exceeds this permute a small side (one
// that fits L2 and is permuted directly for single rows) through its plan too:
// the main pass stores a row's outputs at perm positions, and with many rows
// those random stores span rows x m elements, far beyond L2 (measured: the C4
// transpose, 32 rows x 3.1M, at 0.23 TB/s writing direct).
constexpr size_t kBatchStageBytes = size_t(48) << 20;

// rows: batch rows of the call the view is for (selects the batch staging).
template <class R>
View<R> view(Core& c, bool swapped, cudaStream_t st, size_t rows = 1) {
    const int ia = swapped ? 1 : 0;
    bool use[2];
    for (int sd = 0; sd < 2; ++sd) {
        const Side& x = c.side[sd];
        use[sd] = x.staged || (rows > 1 && x.m > (1u << 16) && rows * x.m * sizeof(R) > kBatchStageBytes);
    }
    {
        // The role-swapped orientation is built on first use, on the first
        // caller's stream; every caller (any stream) orders itself after it.
        std::lock_guard<std::mutex> g(c.mu);
        if (!c.part[ia].p) {
            build_partition<R>(c, ia, st);
            if (!c.built[ia]) ck(cudaEventCreateWithFlags(&c.built[ia], cudaEventDisableTiming), "cudaEventCreate");
            ck(cudaEventRecord(c.built[ia], st), "cudaEventRecord");
        }
        if (c.built[0]) ck(cudaStreamWaitEvent(st, c.built[0], 0), "cudaStreamWaitEvent");
        if (ia && c.built[1]) ck(cudaStreamWaitEvent(st, c.built[1], 0), "cudaStreamWaitEvent");
        for (int sd = 0; sd < 2; ++sd) {
            if (use[sd] && !c.side[sd].has_splan) {  // lazily, once per side, on this stream
                build_splan(c.side[sd], st);
                if (!c.splan_ev[sd]) ck(cudaEventCreateWithFlags(&c.splan_ev[sd], cudaEventDisableTiming), "cudaEventCreate");
                ck(cudaEventRecord(c.splan_ev[sd], st), "cudaEventRecord");
            }
            if (use[sd] && c.splan_ev[sd]) ck(cudaStreamWaitEvent(st, c.splan_ev[sd], 0), "cudaStreamWaitEvent");
        }
    }
    View<R> v;
    const Side& a = c.side[ia];
    const Side& b = c.side[1 - ia];
    v.A = a.vals.as<R>();
    v.pa = a.perm.as<uint32_t>();
    v.n = a.m;
    v.B = b.vals.as<R>();
    v.pb = b.perm.as<uint32_t>();
    v.k = b.m;
    v.cphi = a.cph.as<R>();
    v.sphi = a.sph.as<R>();
    v.cpsi = b.cph.as<R>();
    v.spsi = b.sph.as<R>();
    v.part = c.part[ia].as<uint32_t>();
    v.desc = c.desc[ia].as<lx::ms::TileDesc<R>>();
    v.s_first = c.sfirst[ia].as<R>();
    v.s_last = c.slast[ia].as<R>();
    v.T = c.T[ia];
    v.inv_t = R(1) / R(c.t);
    v.pos_a = use[ia] ? a.spos.as<uint32_t>() : nullptr;
    v.dst_a = use[ia] ? a.sdst.as<uint32_t>() : nullptr;
    v.pos_b = use[1 - ia] ? b.spos.as<uint32_t>() : nullptr;
    v.dst_b = use[1 - ia] ? b.sdst.as<uint32_t>() : nullptr;
    v.gmt = c.gmt[ia].as<uint16_t>();
    v.mw = c.mwd[ia].as<uint32_t>();
    return v;
}

// ---- sort -------------------------------------------------------------------
// Pass structure: reduce-then-scan (count kernel + per-digit tile scan, then a
// pass with known offsets) unless LX_SORT_LOOKBACK selects onesweep's
// decoupled look-back.
#ifdef LX_SORT_LOOKBACK
constexpr bool kSortRts = false;
#else
constexpr bool kSortRts = true;
#endif
// after_hist: enqueued right behind the histogram kernel (whose read of the
// raw keys sets the finiteness flag)
template <class R>
void radix_sort(const R* raw, uint32_t m, R t, R* vals_out, uint32_t* perm_out, int* bad, cudaStream_t st,
                const std::function<void()>& after_hist = {}) {
    using namespace lx::sort;
    using K = typename lx::Traits<R>::Key;
    constexpr int P = lx::Traits<R>::kPasses;
    const uint32_t tiles = (m + kTile - 1) / kTile;
    DBuf hist((size_t)P * kRadix * 4, st), bases((size_t)P * kRadix * 4, st);
    DBuf counters((size_t)P * 4, st);
    DBuf keys0((size_t)m * sizeof(K), st), keys1((size_t)m * sizeof(K), st);
    DBuf v0((size_t)m * 4, st), v1((size_t)m * 4, st);
    DBuf look(kSortRts ? 8 : (size_t)tiles * kRadix * 8, st);
    DBuf cnt(kSortRts ? (size_t)tiles * kRadix * 4 : 4, st);
    DBuf totals(kSortRts ? (size_t)P * kRadix * 4 : 4, st);
    if (!kSortRts) ck(cudaMemsetAsync(hist.p, 0, (size_t)P * kRadix * 4, st), "memset");
    ck(cudaMemsetAsync(counters.p, 0, (size_t)P * 4, st), "memset");
    if (!kSortRts) ck(cudaMemsetAsync(look.p, 0, (size_t)tiles * kRadix * 8, st), "memset");
    const int sms = num_sms();
    const uint32_t per_block = kHistThreads * kHistItems;
    const uint32_t hgrid = std::max(1u, std::min<uint32_t>((m + per_block - 1) / per_block, (uint32_t)sms * 4));
    const size_t hsmem = (size_t)kHistSub * P * kRadix * sizeof(uint32_t);
    if (kSortRts) {  // pass 1's per-tile counts (and the finiteness check) in one read of the keys;
                     // the digit bases of every pass come from the scans' totals
        const uint32_t tpc = std::max<uint32_t>(
            1u, std::min<uint32_t>(kHistTilesPerCta, tiles / (uint32_t)(num_sms() * 4)));
        const uint32_t g0 = (tiles + tpc - 1) / tpc;
        launch("lx_sort_hist", st, [&] {
            lx_sort_hist_count0<R, false><<<g0, kThreads, 0, st>>>(raw, m, t, hist.as<uint32_t>(), bad,
                                                                   cnt.as<uint32_t>(), tiles, tpc);
        });
        if (after_hist) after_hist();
    } else {
        launch("lx_sort_hist", st, [&] {
            lx_sort_hist<R><<<hgrid, kHistThreads, hsmem, st>>>(raw, m, t, hist.as<uint32_t>(), bad);
        });
        launch("lx_sort_bases", st, [&] {
            lx_sort_bases<P><<<P, kRadix, 0, st>>>(hist.as<uint32_t>(), bases.as<uint32_t>());
        });
    }
    const size_t smem = sizeof(PassSmem<R>);
    smem_attr(lx_sort_pass<R, true, false>, smem);
    smem_attr(lx_sort_pass<R, true, false, false, true>, smem);
    smem_attr(lx_sort_pass<R, false, false>, smem);
    smem_attr(lx_sort_pass<R, false, true>, smem);
    const void* in = raw;
    const uint32_t* inv = nullptr;
    for (int pass = 0; pass < P; ++pass) {
        const bool last = pass == P - 1;
        void* out = last ? (void*)vals_out : (pass % 2 == 0 ? keys0.p : keys1.p);
        uint32_t* outv = last ? perm_out : (pass % 2 == 0 ? v0.as<uint32_t>() : v1.as<uint32_t>());
        const uint32_t* bptr = bases.as<uint32_t>() + pass * kRadix;
        uint32_t* ctr = counters.as<uint32_t>() + pass;
        unsigned long long* lb = look.as<unsigned long long>();
        const uint32_t epoch = (uint32_t)pass + 1;
        const uint32_t* offs = nullptr;
        if (kSortRts) {  // per-(digit, tile) offsets first: the pass needs no look-back
            const uint32_t cgrid = (tiles + kCountTiles - 1) / kCountTiles;
            if (pass > 0)  // pass 1's counts came with the histograms
                launch("lx_sort_count", st, [&] {
                    lx_sort_count<R, false, false><<<cgrid, kThreads, 0, st>>>(in, m, t, pass * kBits,
                                                                               cnt.as<uint32_t>(), tiles);
                });
            launch("lx_sort_scan", st, [&] {
                lx_sort_scan<<<kRadix, kScanThreads, 0, st>>>(cnt.as<uint32_t>(), tiles, nullptr, -1,
                                                              totals.as<uint32_t>() + pass * kRadix);
            });
            offs = cnt.as<uint32_t>();
        }
        const uint32_t* tots = kSortRts ? totals.as<uint32_t>() + pass * kRadix : nullptr;
        launch("lx_sort_pass", st, [&] {
            if (pass == 0 && t == R(1))
                lx_sort_pass<R, true, false, false, true><<<tiles, kThreads, smem, st>>>(
                    in, inv, out, outv, m, t, pass * kBits, bptr, lb, ctr, epoch, offs, tots);
            else if (pass == 0)
                lx_sort_pass<R, true, false><<<tiles, kThreads, smem, st>>>(in, inv, out, outv, m, t, pass * kBits,
                                                                           bptr, lb, ctr, epoch, offs, tots);
            else if (!last)
                lx_sort_pass<R, false, false><<<tiles, kThreads, smem, st>>>(in, inv, out, outv, m, t, pass * kBits,
                                                                            bptr, lb, ctr, epoch, offs, tots);
            else
                lx_sort_pass<R, false, true><<<tiles, kThreads, smem, st>>>(in, inv, out, outv, m, t, pass * kBits,
                                                                           bptr, lb, ctr, epoch, offs, tots);
        });
        in = out;
        inv = outv;
    }
}

template <class R>
__global__ void cos_sin_kernel(const R* __restrict__ ph, uint32_t m, R* __restrict__ c, R* __restrict__ s) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        c[i] = lx::xcos(ph[i]);
        s[i] = lx::xsin(ph[i]);
    }
}

void build_splan(Side& sd, cudaStream_t st) {
    using namespace lx::sort;
    const uint32_t m = sd.m;
    const int shift = bucket_shift(m);
    const uint32_t tiles = (m + kTile - 1) / kTile;
    sd.spos = DBuf((size_t)m * 4 + 16, st);  // + slack: the main kernel TMA-reads it in 16-byte units
    sd.sdst = DBuf((size_t)m * 4, st);
    DBuf look(kSortRts ? 8 : (size_t)tiles * kRadix * 8, st), ctr(4, st);
    DBuf cnt(kSortRts ? (size_t)tiles * kRadix * 4 : 4, st);
    if (!kSortRts) ck(cudaMemsetAsync(look.p, 0, (size_t)tiles * kRadix * 8, st), "memset");
    ck(cudaMemsetAsync(ctr.p, 0, 4, st), "memset");
    const uint32_t* offs = nullptr;
    if (kSortRts) {
        launch("lx_splan_count", st, [&] {
            lx_sort_count<float, false, true><<<(tiles + kCountTiles - 1) / kCountTiles, kThreads, 0, st>>>(
                sd.perm.p, m, 1.0f, shift, cnt.as<uint32_t>(), tiles);
        });
        launch("lx_sort_scan", st, [&] {
            lx_sort_scan<<<kRadix, kScanThreads, 0, st>>>(cnt.as<uint32_t>(), tiles, nullptr, shift);
        });
        offs = cnt.as<uint32_t>();
    }
    const size_t smem = sizeof(PassSmem<float>);
    smem_attr(lx_sort_pass<float, false, false, true>, smem);
    launch("lx_splan", st, [&] {
        lx_sort_pass<float, false, false, true><<<tiles, kThreads, smem, st>>>(
            sd.perm.p, nullptr, sd.sdst.p, sd.spos.as<uint32_t>(), m, 1.0f, shift, nullptr,
            look.as<unsigned long long>(), ctr.as<uint32_t>(), 1u, offs);
    });
    sd.has_splan = true;
}

template <class R>
void build_side(Side& sd, const R* raw, uint32_t m, R t, const R* phase, int* bad, cudaStream_t st,
                const std::function<void()>& after_hist = {}) {
    sd.m = m;
    sd.vals = DBuf((size_t)m * sizeof(R) + kTmaPad, st);  // TMA reads round up to 16 B
    sd.perm = DBuf((size_t)m * 4 + 16, st);
    if (m == 0) {  // empty side of a range shard
        if (after_hist) after_hist();
        return;
    }
    radix_sort<R>(raw, m, t, sd.vals.as<R>(), sd.perm.as<uint32_t>(), bad, st, after_hist);
    if (phase) {
        DBuf ph((size_t)m * sizeof(R), st);
        launch("lx_gather_sorted", st, [&] {
            lx::sort::lx_gather_sorted<R><<<(m + 255) / 256, 256, 0, st>>>(phase, sd.perm.as<uint32_t>(), m,
                                                                           ph.as<R>());
        });
        sd.cph = DBuf((size_t)m * sizeof(R), st);
        sd.sph = DBuf((size_t)m * sizeof(R), st);
        launch("cos_sin", st, [&] {
            cos_sin_kernel<R><<<(m + 255) / 256, 256, 0, st>>>(ph.as<R>(), m, sd.cph.as<R>(), sd.sph.as<R>());
        });
    }
    if (m > kDirectMax) {
        build_splan(sd, st);
        sd.staged = true;
    }
}

// ---- permutation application ------------------------------------------------
int grid_for(size_t work) {
    const int sms = num_sms();
    const size_t blocks = (work + 255) / 256;
    return (int)std::max<size_t>(1, std::min<size_t>(blocks, (size_t)sms * 16));
}

// caller-order rows x m -> bucket-staged copy (consumer reads stage[pos[i]])
template <class R>
DBuf stage_gather(const R* src, size_t ld, const uint32_t* dst, uint32_t m, int rows, cudaStream_t st) {
    DBuf out((size_t)rows * m * sizeof(R), st);
    using namespace lx::sort;
    const uint32_t chunks = (m + kGatherChunk - 1) / kGatherChunk;
    launch("lx_perm_gather", st, [&] {
        lx_perm_stage_gather<R><<<dim3(chunks, rows), kPermThreads, 0, st>>>(src, ld, dst, m, out.as<R>());
    });
    return out;
}

// Host-pointer API: finished caller-order output ranges are handed to this
// hook as the scatter completes them, so their device->host copies overlap
// the rest of the scatter (and of the call).  Set per thread by the host API.
struct OutHook {
    std::function<void(const void* dev, size_t u0, size_t u1, int rows, size_t ld, cudaStream_t st)> fn;
};
thread_local OutHook* g_out_hook = nullptr;

// One launch per output array: with two arrays in one pass the random writes of
// both windows thrash L2 (measured at 2^30: 17.5 ms for x_bar + b_bar together
// vs 7.2 ms for one array, with ~60% DRAM read/write amplification).
template <class R, int ITEMS>
void stage_scatter_one_t(const uint32_t* dst, uint32_t m, const R* s1, R* o1, size_t ld1, int rows1, cudaStream_t st) {
    using namespace lx::sort;
    constexpr uint32_t kChunk = kPermThreads * ITEMS;
    const uint32_t chunks = (m + kChunk - 1) / kChunk;
    if (!g_out_hook) {
        launch("lx_perm_scatter", st, [&] {
            lx_perm_stage_scatter<R, ITEMS><<<dim3(chunks, rows1), kPermThreads, 0, st>>>(dst, m, s1, o1, ld1, rows1, nullptr,
                                                                                 nullptr, nullptr, nullptr, 0u);
        });
        return;
    }
    // groups of whole caller windows (bucket w holds exactly the caller
    // indices [w << shift, (w + 1) << shift), at the same bucketed positions)
    const int shift = bucket_shift(m);
    const uint32_t W = (uint32_t)(((uint64_t)m + (1ull << shift) - 1) >> shift);
    const uint32_t G = std::min<uint32_t>(W, 16u);  // 16 groups: the last download tail is 1/16 of the array
    for (uint32_t gi = 0; gi < G; ++gi) {
        const uint64_t u0 = ((uint64_t)(gi * W / G)) << shift;
        const uint64_t u1 = std::min<uint64_t>(((uint64_t)((gi + 1) * W / G)) << shift, m);
        if (u1 <= u0) continue;
        const uint32_t b0 = (uint32_t)(u0 / kChunk), b1 = (uint32_t)((u1 + kChunk - 1) / kChunk);
        launch("lx_perm_scatter", st, [&] {
            lx_perm_stage_scatter<R, ITEMS><<<dim3(b1 - b0, rows1), kPermThreads, 0, st>>>(dst, m, s1, o1, ld1, rows1,
                                                                                  nullptr, nullptr, nullptr, nullptr,
                                                                                  b0);
        });
        g_out_hook->fn(o1, u0, u1, rows1, ld1, st);
    }
}

template <class R>
void stage_scatter_one(const uint32_t* dst, uint32_t m, const R* s1, R* o1, size_t ld1, int rows1, cudaStream_t st) {
    if (rows1 == 1)
        stage_scatter_one_t<R, lx::sort::kScatterItemsRow>(dst, m, s1, o1, ld1, rows1, st);
    else
        stage_scatter_one_t<R, lx::sort::kScatterItemsBatch>(dst, m, s1, o1, ld1, rows1, st);
}

template <class R>
void stage_scatter(const uint32_t* dst, uint32_t m, const R* s1, R* o1, size_t ld1, int rows1, const R* s2, R* o2,
                   const R* s3, R* o3, cudaStream_t st) {
    stage_scatter_one<R>(dst, m, s1, o1, ld1, rows1, st);
    if (s2) stage_scatter_one<R>(dst, m, s2, o2, m, 1, st);
    if (s3) stage_scatter_one<R>(dst, m, s3, o3, m, 1, st);
}

// any non-finite entry of v[0, m) sets *bad (host-pointer API validation,
// run on the device after the upload instead of a host pass over the input)
template <class R>
__global__ void finite_check(const R* __restrict__ v, size_t m, int* __restrict__ bad) {
    constexpr int kV = 16 / sizeof(R);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t i0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    // v is a pool allocation (256-byte aligned): 16-byte vectors, then the tail
    const size_t nv = m / kV;
    int b = 0;
    for (size_t i = i0; i < nv; i += stride) {
        if constexpr (kV == 4) {
            const float4 q = reinterpret_cast<const float4*>(v)[i];
            b |= !isfinite(q.x) | !isfinite(q.y) | !isfinite(q.z) | !isfinite(q.w);
        } else {
            const double2 q = reinterpret_cast<const double2*>(v)[i];
            b |= !isfinite(q.x) | !isfinite(q.y);
        }
    }
    for (size_t i = nv * kV + i0; i < m; i += stride) b |= !isfinite(v[i]);
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

template <class R>
void launch_finite(const R* v, size_t m, int* bad, cudaStream_t st) {
    if (!m) return;
    const int sms = num_sms();
    const size_t blocks = std::min<size_t>((m + 1023) / 1024, (size_t)sms * 8);
    launch("finite_check", st, [&] { finite_check<R><<<(unsigned)blocks, 256, 0, st>>>(v, m, bad); });
}

// Record the end of this call's work on st (see Core::uses).
void touch(Core& c, cudaStream_t st) {
    std::lock_guard<std::mutex> g(c.use_mu);
    for (auto& u : c.uses)
        if (u.first == st) {
            ck(cudaEventRecord(u.second, st), "cudaEventRecord");
            return;
        }
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(e, st), "cudaEventRecord");
    c.uses.emplace_back(st, e);
}

// NonFinite of the anchors / phases found by the plan build, in the
// reference's check order (operator.hpp:88-101); the flags must be on the host.
void raise_bad(const Core& c) {
    if (c.bad_host[0]) fail(LAPLEX_E_NON_FINITE, "LaplexOperator row anchors: non-finite entry");
    if (c.bad_host[1]) fail(LAPLEX_E_NON_FINITE, "LaplexOperator col anchors: non-finite entry");
    if (c.bad_host[2]) fail(LAPLEX_E_NON_FINITE, "LaplexOperator phases: non-finite entry");
}

// ready[s]: optional event the build of side s waits for (host-pointer API:
// side 1 is still uploading while side 0 sorts).  Non-finite anchors (found by
// the histogram pass) and phases raise NonFinite after the one synchronisation,
// in the reference's check order (operator.hpp:88-101).
// sync = false (laplex_plan_create_dev_async): no host synchronisation; the
// finiteness flags land in the plan and laplex_plan_check reports them.
template <class R>
laplex_plan create_plan(const R* a, uint32_t n, const R* b, uint32_t k, double t, const R* phi, const R* psi,
                        cudaStream_t st, const cudaEvent_t* ready = nullptr, bool sync = true) {
    reserve_pool((size_t)n + k, sizeof(R), ready ? 48 : 36, st);
    auto core = std::make_shared<Core>();
    core->dtype = sizeof(R) == 8 ? LAPLEX_F64 : LAPLEX_F32;
    core->device = current_device();
    plan_born(core->device);
    core->t = t;
    core->phased = phi != nullptr;
    DBuf bad(sizeof(int) * 4, st);
    ck(cudaMemsetAsync(bad.p, 0, sizeof(int) * 4, st), "memset");
    // Host-pointer API (ready != null): the call returns as soon as the
    // finiteness flags are known -- right behind the histogram of the second
    // side -- and the rest of the build runs on behind it, overlapping the
    // next call's upload (its kernels queue behind the build on the same
    // stream).  NonFinite is still raised synchronously, in the reference's order.
    const bool early = ready && sync;
    thread_local int* hflags = [] {
        int* q = nullptr;
        ck(cudaMallocHost(&q, 4 * sizeof(int)), "cudaMallocHost");
        return q;
    }();
    cudaEvent_t fev = nullptr;
    auto flags_out = [&] {
        if (phi) {
            launch_finite<R>(phi, n, bad.as<int>() + 2, st);
            launch_finite<R>(psi, k, bad.as<int>() + 2, st);
        }
        ck(cudaMemcpyAsync(hflags, bad.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaEventCreateWithFlags(&fev, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(fev, st), "cudaEventRecord");
    };
    // Device API, small plans: the two sides' sorts are short launches that
    // fill a fraction of the GPU (2^20 keys = 171 tiles for 444 CTA slots), so
    // side a is built on a second stream, concurrently with side b.  Its
    // buffers are handed back to `st` (freed there) after the join.
    const bool fork = !ready && n > 0 && k > 0 && (size_t)n + k <= kForkSidesMax;
    cudaStream_t st0 = fork ? side_stream() : st;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    if (fork) {
        ck(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(ev_fork, st), "cudaEventRecord");
        ck(cudaStreamWaitEvent(st0, ev_fork, 0), "cudaStreamWaitEvent");
    }
    if (ready) ck(cudaStreamWaitEvent(st, ready[0], 0), "cudaStreamWaitEvent");
    build_side<R>(core->side[0], a, n, R(t), phi, bad.as<int>() + 0, st0);
    if (ready) ck(cudaStreamWaitEvent(st, ready[1], 0), "cudaStreamWaitEvent");
    build_side<R>(core->side[1], b, k, R(t), psi, bad.as<int>() + 1, st,
                  early ? std::function<void()>(flags_out) : std::function<void()>());
    if (fork) {
        ck(cudaEventRecord(ev_join, st0), "cudaEventRecord");
        ck(cudaStreamWaitEvent(st, ev_join, 0), "cudaStreamWaitEvent");
        cudaEventDestroy(ev_fork);
        cudaEventDestroy(ev_join);
        Side& s0 = core->side[0];
        for (DBuf* d : {&s0.vals, &s0.perm, &s0.cph, &s0.sph, &s0.spos, &s0.sdst}) d->st = st;
    }
    if (!early && phi) {
        launch_finite<R>(phi, n, bad.as<int>() + 2, st);
        launch_finite<R>(psi, k, bad.as<int>() + 2, st);
    }
    build_partition<R>(*core, 0, st);
    if (!early)
        ck(cudaMemcpyAsync(core->bad_host, bad.p, sizeof(core->bad_host), cudaMemcpyDeviceToHost, st),
           "cudaMemcpyAsync");
    touch(*core, st);
    ck(cudaEventCreateWithFlags(&core->built[0], cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(core->built[0], st), "cudaEventRecord");
    if (early) {
        ck(cudaEventSynchronize(fev), "cudaEventSynchronize");
        cudaEventDestroy(fev);
        std::memcpy(core->bad_host, hflags, sizeof(core->bad_host));
        raise_bad(*core);  // the plan (released) still frees its buffers behind the build
    } else if (sync) {
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        raise_bad(*core);
    }
    auto* p = new laplex_plan_s;
    p->core = core;
    return p;
}


// ---- apply --------------------------------------------------------------------
template <class R>
lx::ms::MainArgs<R> main_args(const View<R>& v, int rows) {
    lx::ms::MainArgs<R> a;
    std::memset(&a, 0, sizeof(a));
    a.A = v.A;
    a.perm_a = v.pa;
    a.B = v.B;
    a.perm_b = v.pb;
    a.part = v.part;
    a.desc = v.desc;
    a.mwords = v.mw;
    a.s_last = v.s_last;
    a.s_first = v.s_first;
    a.n = v.n;
    a.k = v.k;
    a.T = v.T;
    a.rows = rows;
    a.cphi = v.cphi;
    a.sphi = v.sphi;
    a.cpsi = v.cpsi;
    a.spsi = v.spsi;
    a.inv_t = v.inv_t;
    a.gmt = v.gmt;
    return a;
}

// Main-kernel shape: consumer threads per CTA x items per thread (= one 2048
// element merge tile).  Unphased kernels run 128 x 16 (fewer per-thread
// overheads per element; measured best at 2^30); the phased kernels carry
// twice the channels and keep 256 x 8.  The transpose and the backward share
// a shape, so x_bar of the VJP is bitwise the transpose.
template <bool GCH, bool PHASED>  // GCH: the kernel carries g channels (transpose, backward)
struct MainShape {
    static constexpr int TPB = PHASED ? 256 : (GCH ? LX_BWD_TPB : LX_FWD_TPB);
    static constexpr int IPT = lx::ms::kTile / TPB;
};

template <class R, int NG, int NX, bool BWD, bool SEQ = false, int MB = 0>
void launch_main_mb(const char* name, const lx::ms::MainArgs<R>& a, cudaStream_t st) {
    using namespace lx::ms;
    constexpr int TPB = MainShape<(NG > 0), (NG == 2 || NX == 2)>::TPB, IPT = MainShape<(NG > 0), (NG == 2 || NX == 2)>::IPT;
    auto kern = lx_main<R, NG, NX, BWD, SEQ, TPB, IPT, MB>;
    constexpr bool os_smem = LX_OS_SMEM && BWD && NG != 2 && sizeof(R) == 4;
    constexpr bool mc_smem = LX_PH_MC_SMEM && (NG == 2 || NX == 2) && sizeof(R) == 4;
    const size_t smem = sizeof(MainShared<R, NG + NX, TPB / 32, BWD ? (NG == 2 ? 2 : 1) : 0, os_smem ? kTile : 0,
                                          mc_smem ? 2 * kTile : 0>);
    smem_attr(kern, smem);
    const int per_sm = occupancy(kern, TPB + 32, smem), sms = num_sms();
    const uint32_t slots = (uint32_t)(sms * per_sm);
    lx::ms::MainArgs<R> b = a;
    // Row split: a batch over fewer tiles than a few rounds of the resident
    // CTAs leaves slots idle in the last round (C3: 513 tiles of 256 rows on
    // 296 slots = 2 rounds for 1.73 of work).  Items of (tile, row chunk)
    // even that out: the chunk count minimising rounds / chunks.
    uint32_t rc = 1;
    constexpr bool can_split = NG == 2 || NX == 2;  // lx_main's SPLIT
    if (can_split && !SEQ && a.rows >= 16 && a.T < 4 * slots) {
        double best = std::ceil((double)a.T / slots);
        for (uint32_t c = 2; c <= 8 && (int)c * 4 <= a.rows; ++c) {
            const double m = std::ceil((double)a.T * c / slots) / c;
            if (m < best - 1e-9) best = m, rc = c;
        }
    }
    b.rchunk = (a.rows + (int)rc - 1) / (int)rc;
    b.rsplit = (uint32_t)((a.rows + b.rchunk - 1) / b.rchunk);  // every chunk non-empty
    DBuf pa, pb;  // per-chunk partial row / column cotangents (backward)
    if (BWD && b.rsplit > 1) {
        constexpr int nacc = NG == 2 ? 2 : 1;
        b.ldpa = a.n;
        b.ldpb = a.k;
        pa = DBuf((size_t)nacc * b.rsplit * a.n * sizeof(R), st);
        pb = DBuf((size_t)nacc * b.rsplit * a.k * sizeof(R), st);
        b.abar = pa.as<R>();
        b.phibar = nacc == 2 ? pa.as<R>() + (size_t)b.rsplit * a.n : nullptr;
        b.bbar = pb.as<R>();
        b.psibar = nacc == 2 ? pb.as<R>() + (size_t)b.rsplit * a.k : nullptr;
    }
    // persistent: one CTA per resident slot, work items claimed in order
    const uint32_t grid = std::max<uint32_t>(1u, std::min<uint32_t>(a.T * b.rsplit, slots));
    DBuf ctr(4, st);
    ck(cudaMemsetAsync(ctr.p, 0, 4, st), "memset");
    b.tile_ctr = ctr.as<uint32_t>();
    launch(name, st, [&] { kern<<<grid, TPB + 32, smem, st>>>(b); });  // + producer warp
    if (BWD && b.rsplit > 1) {
        auto sum = [&](const R* part, size_t m, R* out) {
            if (!m || !out) return;
            const unsigned g = (unsigned)std::min<size_t>((m + 255) / 256, (size_t)sms * 8);
            launch("lx_chunk_sum", st, [&] { lx::ms::lx_chunk_sum<R><<<g, 256, 0, st>>>(part, (int)b.rsplit, m, out); });
        };
        sum(b.abar, a.n, a.abar);
        sum(b.bbar, a.k, a.bbar);
        if (NG == 2) {
            sum(b.phibar, a.n, a.phibar);
            sum(b.psibar, a.k, a.psibar);
        }
    }
}

// The unphased fp32 backward: 2 CTAs/SM (168 registers) for single rows, 3
// (128 registers, some spills) for batches, where every tile walks many rows
// and the extra warps hide more latency than the spills cost (C2 backward
// 14.9 -> 13.8 ms; C5 20.7 -> 24.2 ms with 3).  Same arithmetic either way.
// (The forward / transpose gain nothing from it: C2 forward 5.9 -> 7.6 ms at
// 4 CTAs, 8.2 at 2.)
template <class R, int NG, int NX, bool BWD, bool SEQ = false>
void launch_main(const char* name, const lx::ms::MainArgs<R>& a, cudaStream_t st) {
    if constexpr (BWD && NG == 1 && NX == 1 && sizeof(R) == 4) {
        if (a.rows > 1) {
            launch_main_mb<R, NG, NX, BWD, SEQ, 3>(name, a, st);
            return;
        }
    }
    // batched unphased forward / transpose: the same 3-CTA budget as the
    // single-row kernel, instantiated apart so that it prefetches the next
    // row's tile carries (MB != 0 in lx_main)
    if constexpr (!BWD && !SEQ && NG + NX == 1 && sizeof(R) == 4 && LX_MAIN_CTAS / MainShape<(NG > 0), false>::TPB == 3) {
        if (a.rows > 1) {
            launch_main_mb<R, NG, NX, BWD, SEQ, 3>(name, a, st);
            return;
        }
    }

    launch_main_mb<R, NG, NX, BWD, SEQ, 0>(name, a, st);
}

template <class R, int NC>
void launch_carry(const R* aggp, const R* aggq, R* cp, R* cq, const R* sl, const R* sf, uint32_t T, int rows,
                  unsigned pm, unsigned qm, cudaStream_t st) {
    using namespace lx::ms;
    CarryArgs<R, NC> a;
    std::memset(&a, 0, sizeof(a));
    a.aggp = aggp;
    a.aggq = aggq;
    a.outp = cp;
    a.outq = cq;
    a.s_last = sl;
    a.s_first = sf;
    a.T = T;
    a.rows = rows;
    a.pst_mask = pm;
    a.qst_mask = qm;
    if (T <= kCarryBlock) {
        launch("lx_carry", st, [&] { lx_carry<R, NC, 0><<<dim3(rows, 2, 1), kCarryThreads, 0, st>>>(a); });
        return;
    }
    // reduce -> spine -> apply
    const uint32_t NB = (T + kCarryBlock - 1) / kCarryBlock;
    const size_t slots = 2 * NC;
    DBuf bagp(slots * rows * NB * sizeof(R), st), bagq(slots * rows * NB * sizeof(R), st);
    DBuf bcp(slots * rows * NB * sizeof(R), st), bcq(slots * rows * NB * sizeof(R), st);
    DBuf bsl(NB * sizeof(R), st), bsf(NB * sizeof(R), st);
    a.chunk = kCarryBlock;
    a.NB = NB;
    a.baggp = bagp.as<R>();
    a.baggq = bagq.as<R>();
    a.bs_last = bsl.as<R>();
    a.bs_first = bsf.as<R>();
    launch("lx_carry", st, [&] { lx_carry<R, NC, 1><<<dim3(rows, 2, NB), kCarryThreads, 0, st>>>(a); });
    CarryArgs<R, NC> sp = a;
    sp.aggp = bagp.as<R>();
    sp.aggq = bagq.as<R>();
    sp.outp = bcp.as<R>();
    sp.outq = bcq.as<R>();
    sp.s_last = bsl.as<R>();
    sp.s_first = bsf.as<R>();
    sp.T = NB;
    sp.NB = 1;
    launch("lx_carry", st, [&] { lx_carry<R, NC, 0><<<dim3(rows, 2, 1), kCarryThreads, 0, st>>>(sp); });
    a.bcp = bcp.as<R>();
    a.bcq = bcq.as<R>();
    launch("lx_carry", st, [&] { lx_carry<R, NC, 2><<<dim3(rows, 2, NB), kCarryThreads, 0, st>>>(a); });
}

// sorted-payload row stride: 16-byte multiple so every row start is TMA-aligned
size_t padded_ld(uint32_t m) { return ((size_t)m + 3) & ~size_t(3); }

struct Scratch {
    DBuf aggp, aggq, cp, cq;
    Scratch(size_t slots, int rows, uint32_t T, size_t rs, cudaStream_t st)
        : aggp(slots * rows * T * rs, st), aggq(slots * rows * T * rs, st), cp(slots * rows * T * rs, st),
          cq(slots * rows * T * rs, st) {}
};

// Gather one payload side into sorted order (through the side's permutation
// plan when it has one) and compute its tile aggregates in the same pass.
template <class R, int NCH, bool SIDE_A, bool GFORM, bool STRICT>
DBuf sorted_payload(const View<R>& v, int rows, const R* user, const Scratch& sc, int cbase, size_t& ld_out,
                    cudaStream_t st, bool already_sorted = false) {
    const uint32_t m = SIDE_A ? v.n : v.k;
    const uint32_t* dst = SIDE_A ? v.dst_a : v.dst_b;
    const uint32_t* pos = SIDE_A ? v.pos_a : v.pos_b;
    const uint32_t* perm = SIDE_A ? v.pa : v.pb;
    ld_out = padded_ld(m);
    DBuf out((size_t)rows * ld_out * sizeof(R) + kTmaPad, st);
    DBuf stg;
    lx::ms::GatherAggArgs<R> g;
    std::memset(&g, 0, sizeof(g));
    g.desc = v.desc;
    g.T = v.T;
    g.rows = rows;
    g.V = SIDE_A ? v.A : v.B;
    g.out = out.as<R>();
    g.ld_out = ld_out;
    g.cph = SIDE_A ? v.cphi : v.cpsi;
    g.sph = SIDE_A ? v.sphi : v.spsi;
    g.aggp = sc.aggp.as<R>();
    g.aggq = sc.aggq.as<R>();
    g.cbase = cbase;
    g.ld_src = m;
    if (already_sorted) {
        g.src = user;
        g.idx = nullptr;
    } else if (dst) {
        stg = stage_gather<R>(user, m, dst, m, rows, st);
        g.src = stg.as<R>();
        g.idx = pos;
    } else {
        g.src = user;
        g.idx = perm;
    }
    launch("lx_gather_agg", st, [&] {
        const uint32_t grid = (v.T + lx::ms::kAggTiles - 1) / lx::ms::kAggTiles;
        // few tiles and many rows (batched calls): split the rows over CTAs too,
        // rows per CTA chosen to minimise waves x (rows per CTA + a per-CTA
        // overhead of ~2 rows) over the resident slots (4 per SM): C3's 129
        // CTAs x 256 rows went out as 645 CTAs of 52 rows = 2 waves for 1.09
        uint32_t rpc = (uint32_t)std::max(rows, 1);
        if (rows > 1) {
            const double slots = 4.0 * num_sms();
            double best = 1e300;
            for (uint32_t r = 1; r <= (uint32_t)rows; ++r) {
                const uint32_t gy_r = ((uint32_t)rows + r - 1) / r;
                if (r > 1 && ((uint32_t)rows + r - 2) / (r - 1) == gy_r) continue;  // same split, fewer rows per CTA
                const double cost = std::ceil((double)grid * gy_r / slots) * (r + 2.0);
                if (cost < best - 1e-9) best = cost, rpc = r;
            }
        }
        g.rows_per_cta = (int)rpc;
        const uint32_t gy = (uint32_t)std::max(1, (rows + g.rows_per_cta - 1) / g.rows_per_cta);
        lx::ms::lx_gather_agg<R, NCH, SIDE_A, GFORM, STRICT><<<dim3(grid, gy), lx::ms::kAggThreads, 0, st>>>(g);
    });
    return out;
}

template <class R, int NC>
void scan_carries(const View<R>& v, const Scratch& sc, int rows, unsigned pm, unsigned qm, cudaStream_t st) {
    launch_carry<R, NC>(sc.aggp.as<R>(), sc.aggq.as<R>(), sc.cp.as<R>(), sc.cq.as<R>(), v.s_last, v.s_first, v.T,
                        rows, pm, qm, st);
}

// ---- staged forward / backward (begin: aggregates + local carries; end:
// optional external shard carries -> outputs).  The unsharded calls run both
// halves back to back; the range-sharded operator exchanges the shard totals
// between them. ----
struct WorkBase {
    virtual ~WorkBase() = default;
    std::shared_ptr<Core> keep;  // the plan outlives the work
    size_t total_count = 0;      // Real entries of the totals / ext arrays
};

template <class R>
void collect_totals(const View<R>& v, const Scratch& sc, int rows, int slots, R* out, cudaStream_t st) {
    const int per = slots * rows;
    launch("lx_collect_totals", st, [&] {
        lx::shard::lx_collect_totals<R><<<(per + 255) / 256, 256, 0, st>>>(
            sc.cp.as<R>(), sc.cq.as<R>(), v.s_last, v.s_first, v.T, rows, slots, out);
    });
}

template <class R, int NX>
struct FwdWork : WorkBase {
    View<R> v;
    lx::ms::MainArgs<R> a;
    Scratch sc;
    DBuf xs;
    int rows;
    FwdWork(const View<R>& v_, int rows_, cudaStream_t st) : v(v_), sc(2 * NX, rows_, v_.T, sizeof(R), st), rows(rows_) {}
};

// STRICT: also the strict aggregates of x (unused by the forward; computed when
// the sorted x is kept for the backward, whose x channel needs them)
template <class R, int NX, bool STRICT = false>
std::unique_ptr<FwdWork<R, NX>> fwd_begin(const View<R>& v, const R* X, int rows, cudaStream_t st) {
    auto w = std::make_unique<FwdWork<R, NX>>(v, rows, st);
    w->a = main_args(v, rows);
    w->xs = sorted_payload<R, NX, false, false, STRICT>(v, rows, X, w->sc, 0, w->a.ldxs, st);
    w->a.Xs = w->xs.template as<R>();
    scan_carries<R, NX>(v, w->sc, rows, 0u, 0u, st);
    w->a.cp = w->sc.cp.template as<R>();
    w->a.cq = w->sc.cq.template as<R>();
    w->total_count = 3 + 2 * (size_t)(2 * NX) * rows;
    return w;
}

template <class R, int NX>
void fwd_end(FwdWork<R, NX>& w, const R* ext, R* Y, cudaStream_t st, bool keep_xs = false) {
    const View<R>& v = w.v;
    auto& a = w.a;
    a.ext = ext;
    DBuf yst;
    if (v.dst_a) {  // write bucket-staged, then scatter through the rows plan
        yst = DBuf((size_t)w.rows * v.n * sizeof(R), st);
        a.y = yst.as<R>();
        a.perm_a = v.pos_a;
    } else {
        a.y = Y;
    }
    a.ldy = v.n;
    if (v.n) launch_main<R, 0, NX, false>(NX == 2 ? "lx_main_fwd_phased" : "lx_main_fwd", a, st);
    if (!keep_xs) w.xs.release();
    if (v.dst_a)
        stage_scatter<R>(v.dst_a, v.n, yst.as<R>(), Y, v.n, w.rows, nullptr, nullptr, nullptr, nullptr, st);
}

}  // namespace
struct laplex_work_s {
    std::unique_ptr<WorkBase> impl;
    int dtype = LAPLEX_F32;
    bool backward = false;
    bool phased = false;
};
namespace {

template <class R, int NX>
void apply_fwd(const View<R>& v, const R* X, int rows, R* Y, cudaStream_t st, Core* save = nullptr,
               bool swapped = false) {
    if (!save) {
        auto w = fwd_begin<R, NX>(v, X, rows, st);
        fwd_end<R, NX>(*w, nullptr, Y, st);
        return;
    }
    auto w = fwd_begin<R, NX, true>(v, X, rows, st);
    fwd_end<R, NX>(*w, nullptr, Y, st, true);
    std::lock_guard<std::mutex> g(save->saved_mu);
    auto& sv = save->saved;
    sv.X = X;
    sv.host = false;
    sv.rows = (size_t)rows;
    sv.swapped = swapped;
    sv.phased = NX == 2;
    sv.xs = std::move(w->xs);
    sv.ldxs = w->a.ldxs;
    sv.aggp = std::move(w->sc.aggp);
    sv.aggq = std::move(w->sc.aggq);
    sv.agg_count = (size_t)2 * NX * rows * v.T;
    if (!sv.ready) ck(cudaEventCreateWithFlags(&sv.ready, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventRecord(sv.ready, st), "cudaEventRecord");
}

template <class R>
void apply_trn(const View<R>& v, const R* G, int rows, R* Y, cudaStream_t st) {
    auto a = main_args(v, rows);
    Scratch sc(2, rows, v.T, sizeof(R), st);
    DBuf gs = sorted_payload<R, 1, true, true, false>(v, rows, G, sc, 0, a.ldgs, st);
    a.Gs = gs.as<R>();
    scan_carries<R, 1>(v, sc, rows, 0u, 0u, st);
    a.cp = sc.cp.as<R>();
    a.cq = sc.cq.as<R>();
    DBuf yst;
    if (v.dst_b) {
        yst = DBuf((size_t)rows * v.k * sizeof(R), st);
        a.y = yst.as<R>();
        a.perm_b = v.pos_b;
    } else {
        a.y = Y;
    }
    a.ldy = v.k;
    launch_main<R, 1, 0, false>("lx_main_trn", a, st);
    gs.release();
    if (v.dst_b)
        stage_scatter<R>(v.dst_b, v.k, yst.as<R>(), Y, v.k, rows, nullptr, nullptr, nullptr, nullptr, st);
}

template <class R, int NCH>
struct BwdWork : WorkBase {
    View<R> v;
    lx::ms::MainArgs<R> a;
    Scratch sc;
    DBuf gs, xs;
    int rows;
    BwdWork(const View<R>& v_, int rows_, cudaStream_t st)
        : v(v_), sc(2 * 2 * NCH, rows_, v_.T, sizeof(R), st), rows(rows_) {}
};

// reuse: the Core whose saved forward x (LAPLEX_REUSE_X) matches X / rows /
// orientation, or null.  The saved sorted x and aggregates replace the x gather.
template <class R, int NCH>
std::unique_ptr<BwdWork<R, NCH>> bwd_begin(const View<R>& v, const R* X, const R* G, int rows, cudaStream_t st,
                                           const std::function<void()>& before_g = {}, Core* reuse = nullptr) {
    constexpr int NC = 2 * NCH;
    auto w = std::make_unique<BwdWork<R, NCH>>(v, rows, st);
    auto& a = w->a;
    a = main_args(v, rows);
    if (reuse) {
        auto& sv = reuse->saved;
        ck(cudaStreamWaitEvent(st, sv.ready, 0), "cudaStreamWaitEvent");
        w->xs = std::move(sv.xs);
        w->xs.st = st;  // read and freed on this stream from now on
        a.ldxs = sv.ldxs;
        const size_t off = (size_t)2 * NCH * rows * v.T * sizeof(R);  // x channels follow the g channels
        ck(cudaMemcpyAsync(w->sc.aggp.template as<char>() + off, sv.aggp.p, sv.agg_count * sizeof(R),
                           cudaMemcpyDeviceToDevice, st), "D2D");
        ck(cudaMemcpyAsync(w->sc.aggq.template as<char>() + off, sv.aggq.p, sv.agg_count * sizeof(R),
                           cudaMemcpyDeviceToDevice, st), "D2D");
        sv.aggp.st = st, sv.aggq.st = st;
        sv.aggp.release(), sv.aggq.release();
        sv.X = nullptr;
    } else {
        w->xs = sorted_payload<R, NCH, false, false, true>(v, rows, X, w->sc, NCH, a.ldxs, st);
    }
    if (before_g) before_g();  // host API: g may still be uploading
    w->gs = sorted_payload<R, NCH, true, true, true>(v, rows, G, w->sc, 0, a.ldgs, st);
    a.Gs = w->gs.template as<R>();
    a.Xs = w->xs.template as<R>();
    const unsigned gmask = (1u << NCH) - 1u;
    scan_carries<R, NC>(v, w->sc, rows, gmask, gmask << NCH, st);
    a.cp = w->sc.cp.template as<R>();
    a.cq = w->sc.cq.template as<R>();
    w->total_count = 3 + 2 * (size_t)(2 * NC) * rows;
    return w;
}

template <class R, int NCH>
void bwd_end(BwdWork<R, NCH>& w, const R* ext, R* xbar, R* abar, R* bbar, R* phibar, R* psibar, cudaStream_t st) {
    const View<R>& v = w.v;
    auto& a = w.a;
    const int rows = w.rows;
    const size_t rs = sizeof(R);
    a.ext = ext;
    DBuf sxb, sbb, sqb, sab, spb;  // bucket-staged outputs
    if (v.dst_b) {
        sxb = DBuf((size_t)rows * v.k * rs, st);
        sbb = DBuf((size_t)v.k * rs, st);
        if (NCH == 2) sqb = DBuf((size_t)v.k * rs, st);
        a.xbar = sxb.as<R>();
        a.bbar = sbb.as<R>();
        a.psibar = sqb.as<R>();
        a.perm_b = v.pos_b;
    } else {
        a.xbar = xbar;
        a.bbar = bbar;
        a.psibar = psibar;
    }
    if (v.dst_a) {
        sab = DBuf((size_t)v.n * rs, st);
        if (NCH == 2) spb = DBuf((size_t)v.n * rs, st);
        a.abar = sab.as<R>();
        a.phibar = spb.as<R>();
        a.perm_a = v.pos_a;
    } else {
        a.abar = abar;
        a.phibar = phibar;
    }
    a.ldxb = v.k;
    launch_main<R, NCH, NCH, true>(NCH == 2 ? "lx_main_bwd_phased" : "lx_main_bwd", a, st);
    w.gs.release();
    w.xs.release();
    if (v.dst_b)
        stage_scatter<R>(v.dst_b, v.k, sxb.as<R>(), xbar, v.k, rows, sbb.as<R>(), bbar,
                         NCH == 2 ? sqb.as<R>() : nullptr, psibar, st);
    if (v.dst_a)
        stage_scatter<R>(v.dst_a, v.n, sab.as<R>(), abar, v.n, 1, NCH == 2 ? spb.as<R>() : nullptr, phibar, nullptr,
                         nullptr, st);
}

template <class R, int NCH>
void backward_impl(const View<R>& v, const R* X, const R* G, int rows, R* xbar, R* abar, R* bbar, R* phibar,
                   R* psibar, cudaStream_t st, const std::function<void()>& before_g, Core* reuse = nullptr) {
    auto w = bwd_begin<R, NCH>(v, X, G, rows, st, before_g, reuse);
    bwd_end<R, NCH>(*w, nullptr, xbar, abar, bbar, phibar, psibar, st);
}

// Batched calls: the per-call working set grows with rows x (n + k) (sorted
// payloads, bucket-staged copies and outputs, ~24 B per row-element), far
// beyond the plan's per-anchor reservation; without holding it the pool grows
// on demand inside the step (C2 device step 48 -> 83..195 ms in some runs:
// host-side mapping stalls between kernels).
template <class R>
void reserve_batch(const Core& c, size_t rows, cudaStream_t st) {
    if (rows > 1) reserve_pool(((size_t)c.side[0].m + c.side[1].m) * rows, sizeof(R), 24, st);
}

template <class R>
void do_apply(laplex_plan_s* p, unsigned flags, const R* X, size_t rows, R* Y, cudaStream_t st) {
    Core& c = *p->core;
    const bool trn = flags & LAPLEX_TRANSPOSE, ph = flags & LAPLEX_PHASED;
    if (ph && !c.phased) fail(LAPLEX_E_PHASE_ABSENT, "phased_matvec: operator has no phases");
    if (!ph && c.phased) fail(LAPLEX_E_PHASE_PRESENT, "matvec: operator has phases, use phased_matvec");
    if (trn && ph) fail(LAPLEX_E_INVALID_ARGUMENT, "phased transpose is not part of the reference API");
    if (rows == 0) return;
    if (rows > 0x7fffffff) fail(LAPLEX_E_INVALID_SIZE, "too many rows");
    reserve_batch<R>(c, rows, st);
    View<R> v = view<R>(c, p->swapped, st, rows);
    Core* save = (flags & LAPLEX_SAVE_X) && !trn ? &c : nullptr;
    if (trn)
        apply_trn<R>(v, X, (int)rows, Y, st);
    else if (ph)
        apply_fwd<R, 2>(v, X, (int)rows, Y, st, save, p->swapped);
    else
        apply_fwd<R, 1>(v, X, (int)rows, Y, st, save, p->swapped);
    touch(c, st);
}

// host_x: X is the caller's host pointer of a host-API call that reuses the
// x saved by a host-API apply (never dereferenced then).
template <class R>
void do_backward(laplex_plan_s* p, unsigned flags, const R* X, const R* G, size_t rows, R* xbar, R* abar, R* bbar,
                 R* phibar, R* psibar, cudaStream_t st, const std::function<void()>& before_g = {},
                 bool host_x = false) {
    Core& c = *p->core;
    const bool ph = flags & LAPLEX_PHASED;
    if (ph && !c.phased) fail(LAPLEX_E_PHASE_ABSENT, "phased_matvec_vjp: operator has no phases");
    if (!ph && c.phased) fail(LAPLEX_E_PHASE_PRESENT, "matvec_vjp: use phased_matvec_vjp");
    reserve_batch<R>(c, rows, st);
    View<R> v = view<R>(c, p->swapped, st, rows);
    if (rows == 0) {
        if (before_g) before_g();
        ck(cudaMemsetAsync(abar, 0, (size_t)v.n * sizeof(R), st), "memset");
        ck(cudaMemsetAsync(bbar, 0, (size_t)v.k * sizeof(R), st), "memset");
        if (ph && phibar) ck(cudaMemsetAsync(phibar, 0, (size_t)v.n * sizeof(R), st), "memset");
        if (ph && psibar) ck(cudaMemsetAsync(psibar, 0, (size_t)v.k * sizeof(R), st), "memset");
        touch(c, st);
        return;
    }
    // LAPLEX_REUSE_X: the caller asserts X is unchanged since the apply that
    // saved it (LAPLEX_SAVE_X); a saved x that does not match is ignored
    std::unique_lock<std::mutex> lk(c.saved_mu);
    Core* reuse = nullptr;
    if ((flags & LAPLEX_REUSE_X) && c.saved.xs.p && c.saved.X == (const void*)X && c.saved.rows == rows &&
        c.saved.swapped == p->swapped && c.saved.phased == ph && c.saved.host == host_x)
        reuse = &c;
    else
        lk.unlock();
    if (ph)
        backward_impl<R, 2>(v, X, G, (int)rows, xbar, abar, bbar, phibar, psibar, st, before_g, reuse);
    else
        backward_impl<R, 1>(v, X, G, (int)rows, xbar, abar, bbar, nullptr, nullptr, st, before_g, reuse);
    touch(c, st);
}

__global__ void lx_iota(uint32_t* __restrict__ out, uint32_t m) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) out[i] = i;
}

// Gram-vector product Y = A^T (A X) (matvec_transpose(matvec(x)),
// operator.hpp:162-172), one pass pair over the plan.  The intermediate
// Z = A X never leaves sorted-row order: the forward stores it at the sorted
// position (output index = identity) and the transpose reads it as its
// already-sorted payload, so Z pays no scatter and no gather (SURVEY 8(d):
// 84n + 92k + B(8n + 8k) bytes incl. the plan).  Per row, the arithmetic is the
// forward's and the transpose's exactly, so Y is bitwise equal to
// laplex_apply(TRANSPOSE) of laplex_apply(X).
template <class R>
void do_gram_apply(laplex_plan_s* p, const R* X, size_t rows, R* Y, cudaStream_t st) {
    Core& c = *p->core;
    if (c.phased) fail(LAPLEX_E_PHASE_PRESENT, "gram_apply: operator has phases (matvec is unphased)");
    if (rows == 0) return;
    if (rows > 0x7fffffff) fail(LAPLEX_E_INVALID_SIZE, "too many rows");
    View<R> v = view<R>(c, p->swapped, st, rows);
    const int nr = (int)rows;
    DBuf zs((size_t)rows * v.n * sizeof(R) + kTmaPad, st);  // Z in sorted-row order
    {
        DBuf iota((size_t)v.n * 4 + 16, st);
        launch("lx_iota", st, [&] { lx_iota<<<(v.n + 255) / 256, 256, 0, st>>>(iota.as<uint32_t>(), v.n); });
        auto w = fwd_begin<R, 1>(v, X, nr, st);
        auto& a = w->a;
        a.ext = nullptr;
        a.y = zs.as<R>();
        a.perm_a = iota.as<uint32_t>();
        a.ldy = v.n;
        if (v.n) launch_main<R, 0, 1, false>("lx_main_fwd", a, st);
    }
    // Y = A^T Z, Z already sorted (apply_trn with the gather skipped)
    auto a = main_args(v, nr);
    Scratch sc(2, nr, v.T, sizeof(R), st);
    DBuf gs = sorted_payload<R, 1, true, true, false>(v, nr, zs.as<R>(), sc, 0, a.ldgs, st, true);
    zs.release();
    a.Gs = gs.as<R>();
    scan_carries<R, 1>(v, sc, nr, 0u, 0u, st);
    a.cp = sc.cp.as<R>();
    a.cq = sc.cq.as<R>();
    DBuf yst;
    if (v.dst_b) {
        yst = DBuf((size_t)rows * v.k * sizeof(R), st);
        a.y = yst.as<R>();
        a.perm_b = v.pos_b;
    } else {
        a.y = Y;
    }
    a.ldy = v.k;
    launch_main<R, 1, 0, false>("lx_main_trn", a, st);
    gs.release();
    if (v.dst_b) stage_scatter<R>(v.dst_b, v.k, yst.as<R>(), Y, v.k, nr, nullptr, nullptr, nullptr, nullptr, st);
    touch(c, st);
}

template <class R>
void do_gram(laplex_plan_s* p, unsigned flags, const R* D, R* M, cudaStream_t st) {
    Core& c = *p->core;
    const bool ph = flags & LAPLEX_PHASED;
    if (ph && !c.phased) fail(LAPLEX_E_PHASE_ABSENT, "phased_gram: operator has no phases");
    if (!ph && c.phased) fail(LAPLEX_E_PHASE_PRESENT, "weighted_gram: operator has phases");
    View<R> v = view<R>(c, p->swapped, st);
    const int NCH = ph ? 3 : 1;
    const uint32_t n = v.n;
    DBuf ell((size_t)NCH * n * sizeof(R), st), rho((size_t)NCH * n * sizeof(R), st);
    DBuf mass((size_t)NCH * (n + 1) * sizeof(R), st);
    DBuf U((size_t)NCH * n * sizeof(R), st), V((size_t)NCH * n * sizeof(R), st);
    DBuf C((size_t)NCH * (n + 1) * sizeof(R), st);
    DBuf A2((size_t)n * sizeof(R), st), Z((size_t)(n + 1) * sizeof(R), st), dummy((size_t)NCH * (n + 1) * sizeof(R), st);
    const uint32_t warps = n + 1;
    const uint32_t blocks = (warps * 32 + 255) / 256;
    launch("lx_gram_buckets", st, [&] {
        if (ph)
            lx::gram::lx_gram_buckets<R, 3><<<blocks, 256, 0, st>>>(v.A, n, v.B, v.k, v.pb, D, v.cpsi, v.spsi,
                                                                    ell.as<R>(), rho.as<R>(), mass.as<R>());
        else
            lx::gram::lx_gram_buckets<R, 1><<<blocks, 256, 0, st>>>(v.A, n, v.B, v.k, v.pb, D, nullptr, nullptr,
                                                                    ell.as<R>(), rho.as<R>(), mass.as<R>());
    });
    launch("lx_double_anchors", st, [&] {
        lx::gram::lx_double_anchors<R><<<(n + 255) / 256, 256, 0, st>>>(v.A, n, A2.as<R>());
    });
    ck(cudaMemsetAsync(Z.p, 0, (size_t)(n + 1) * sizeof(R), st), "memset");
    // U = prefix scan of ell over anchors 2A; V = suffix scan of rho (channels as rows)
    launch_carry<R, 1>(ell.as<R>(), rho.as<R>(), U.as<R>(), V.as<R>(), A2.as<R>(), A2.as<R>(), n, NCH, 0u, 0u, st);
    // C = cumulative sum of mass (zero anchors -> every decay is exactly 1)
    launch_carry<R, 1>(mass.as<R>(), mass.as<R>(), C.as<R>(), dummy.as<R>(), Z.as<R>(), Z.as<R>(), n + 1, NCH, 0u,
                       0u, st);
    dim3 blk(32, 8), grd((n + 31) / 32, (n + 7) / 8);
    launch("lx_gram_out", st, [&] {
        if (ph)
            lx::gram::lx_gram_out<R, 3><<<grd, blk, 0, st>>>(v.A, n, v.pa, U.as<R>(), V.as<R>(), C.as<R>(), v.cphi,
                                                             v.sphi, M);
        else
            lx::gram::lx_gram_out<R, 1><<<grd, blk, 0, st>>>(v.A, n, v.pa, U.as<R>(), V.as<R>(), C.as<R>(), nullptr,
                                                             nullptr, M);
    });
    touch(c, st);
}

template <class R>
void do_gram_vjp(laplex_plan_s* p, const R* Gbar, R* Dbar, cudaStream_t st) {
    Core& c = *p->core;
    const int ia0 = p->swapped ? 1 : 0;
    View<R> v = view<R>(c, p->swapped, st, c.side[ia0].m);
    DBuf Y((size_t)v.n * v.k * sizeof(R), st);
    apply_trn<R>(v, Gbar, (int)v.n, Y.as<R>(), st);
    DBuf pa((size_t)v.n * 4, st), pb((size_t)v.k * 4, st);
    launch("lx_invert_perm", st, [&] {
        lx::gram::lx_invert_perm<<<(v.n + 255) / 256, 256, 0, st>>>(v.pa, v.n, pa.as<uint32_t>());
    });
    launch("lx_invert_perm", st, [&] {
        lx::gram::lx_invert_perm<<<(v.k + 255) / 256, 256, 0, st>>>(v.pb, v.k, pb.as<uint32_t>());
    });
    launch("lx_gram_vjp_contract", st, [&] {
        lx::gram::lx_gram_vjp_contract<R><<<(v.k + 255) / 256, 256, 0, st>>>(v.A, pa.as<uint32_t>(), v.n, v.B,
                                                                            pb.as<uint32_t>(), v.k, Y.as<R>(), Dbar);
    });
    touch(c, st);
}

template <class R>
void do_ranks(laplex_plan_s* p, int side, int strict, uint64_t* out, cudaStream_t st) {
    Core& c = *p->core;
    // physical side of the request
    const int phys = p->swapped ? 1 - side : side;
    const int slot = phys * 2 + (strict ? 1 : 0);
    std::lock_guard<std::mutex> g(c.mu);
    ck(cudaStreamWaitEvent(st, c.built[0], 0), "cudaStreamWaitEvent");
    if (!c.has_ranks[slot]) {
        // rows = physical side 0, cols = physical side 1.  A-first merge of
        // (rows, cols) gives J<(rows) and R<=(cols); B-first gives J<=, R<.
        const Side& a = c.side[0];
        const Side& b = c.side[1];
        const uint32_t T = tiles_for((uint64_t)a.m + b.m);
        DBuf part((size_t)(T + 1) * 4, st);
        const bool afirst = (phys == 0) ? (strict != 0) : (strict == 0);
        DBuf rr((size_t)a.m * 4, st), rc((size_t)b.m * 4, st);
        const size_t smem = (size_t)lx::ms::kTile * sizeof(R);
        launch("lx_partition", st, [&] {
            if (afirst)
                lx::ms::lx_partition<R, true><<<(T + 256) / 256, 256, 0, st>>>(a.vals.as<R>(), a.m, b.vals.as<R>(),
                                                                              b.m, part.as<uint32_t>(), T);
            else
                lx::ms::lx_partition<R, false><<<(T + 256) / 256, 256, 0, st>>>(a.vals.as<R>(), a.m, b.vals.as<R>(),
                                                                               b.m, part.as<uint32_t>(), T);
        });
        launch("lx_coranks", st, [&] {
            if (afirst)
                lx::ms::lx_coranks<R, true><<<T, lx::ms::kThreads, smem, st>>>(
                    a.vals.as<R>(), a.m, b.vals.as<R>(), b.m, part.as<uint32_t>(), rr.as<uint32_t>(), rc.as<uint32_t>());
            else
                lx::ms::lx_coranks<R, false><<<T, lx::ms::kThreads, smem, st>>>(
                    a.vals.as<R>(), a.m, b.vals.as<R>(), b.m, part.as<uint32_t>(), rr.as<uint32_t>(), rc.as<uint32_t>());
        });
        // A-first: rows get J<, cols get R<= ; B-first: rows J<=, cols R<
        const int rows_slot = 0 * 2 + (afirst ? 1 : 0);
        const int cols_slot = 1 * 2 + (afirst ? 0 : 1);
        c.ranks[rows_slot] = std::move(rr);
        c.ranks[cols_slot] = std::move(rc);
        c.has_ranks[rows_slot] = c.has_ranks[cols_slot] = true;
    }
    const uint32_t m = c.side[phys].m;
    std::vector<uint32_t> h(m);
    ck(cudaMemcpyAsync(h.data(), c.ranks[slot].p, (size_t)m * 4, cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    for (uint32_t i = 0; i < m; ++i) out[i] = h[i];
}

// prefix / suffix decay scans of payload over sorted anchors (scan.hpp:50-73),
// all device pointers; `sorted` must be readable 64 bytes past its end (TMA
// rounding) -- the host entry copies into such a buffer, the device entry
// stages a padded copy when the caller's pointer is not one of its own.
template <class R>
void do_scan_dev(const R* sorted_in, uint32_t m, const R* payload, R* pre, R* suf, cudaStream_t st) {
    using namespace lx::ms;
    const uint32_t T = tiles_for(m);
    DBuf vals((size_t)m * sizeof(R) + kTmaPad, st);
    ck(cudaMemcpyAsync(vals.p, sorted_in, (size_t)m * sizeof(R), cudaMemcpyDeviceToDevice, st), "D2D");
    DBuf part((size_t)(T + 1) * 4, st), desc((size_t)(T + 1) * sizeof(TileDesc<R>), st);
    DBuf sfirst((size_t)T * sizeof(R), st), slast((size_t)T * sizeof(R), st);
    launch("lx_seq_partition", st, [&] {
        lx_seq_partition<<<(T + 256) / 256, 256, 0, st>>>(m, part.as<uint32_t>(), T);
    });
    launch("lx_tiledesc", st, [&] {
        lx_tiledesc<R><<<(T + 1 + 255) / 256, 256, 0, st>>>(vals.as<R>(), m, vals.as<R>(), 0, part.as<uint32_t>(), T,
                                                             desc.as<TileDesc<R>>(), sfirst.as<R>(), slast.as<R>());
    });
    View<R> v;
    std::memset(&v, 0, sizeof(v));
    v.A = vals.as<R>();
    v.n = m;
    v.k = 0;
    v.part = part.as<uint32_t>();
    v.desc = desc.as<TileDesc<R>>();
    v.s_first = sfirst.as<R>();
    v.s_last = slast.as<R>();
    v.T = T;
    DBuf dpre(pre ? 0 : (size_t)m * sizeof(R), st), dsuf(suf ? 0 : (size_t)m * sizeof(R), st);
    auto a = main_args(v, 1);
    Scratch sc(2, 1, T, sizeof(R), st);
    DBuf xs = sorted_payload<R, 1, true, false, false>(v, 1, payload, sc, 0, a.ldxs, st, true);
    a.Xs = xs.as<R>();
    scan_carries<R, 1>(v, sc, 1, 0u, 0u, st);
    a.cp = sc.cp.as<R>();
    a.cq = sc.cq.as<R>();
    a.pre = pre ? pre : dpre.as<R>();
    a.suf = suf ? suf : dsuf.as<R>();
    launch_main<R, 0, 1, false, true>("lx_main_seq", a, st);
}

template <class R>
void do_scan(const R* sorted, uint32_t m, const R* payload, R* pre, R* suf, cudaStream_t st) {
    DBuf vals((size_t)m * sizeof(R), st), pay((size_t)m * sizeof(R), st);
    DBuf dpre((size_t)m * sizeof(R), st), dsuf((size_t)m * sizeof(R), st);
    ck(cudaMemcpyAsync(vals.p, sorted, (size_t)m * sizeof(R), cudaMemcpyHostToDevice, st), "H2D");
    ck(cudaMemcpyAsync(pay.p, payload, (size_t)m * sizeof(R), cudaMemcpyHostToDevice, st), "H2D");
    do_scan_dev<R>(vals.as<R>(), m, pay.as<R>(), dpre.as<R>(), dsuf.as<R>(), st);
    if (pre) ck(cudaMemcpyAsync(pre, dpre.p, (size_t)m * sizeof(R), cudaMemcpyDeviceToHost, st), "D2H");
    if (suf) ck(cudaMemcpyAsync(suf, dsuf.p, (size_t)m * sizeof(R), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

// ---- host helpers ---------------------------------------------------------------
// Host-side require_finite (common.hpp:34-37), split over hardware threads
// for large inputs so the host-buffer API is not bound by one core.
template <class R>
bool host_finite(const R* v, size_t m) {
    auto scan = [v](size_t lo, size_t hi) {
        bool ok = true;
        for (size_t i = lo; i < hi; ++i) ok &= std::isfinite(v[i]);
        return ok;
    };
    const size_t kPar = size_t(1) << 22;
    unsigned nt = std::thread::hardware_concurrency();
    if (m < kPar || nt < 2) return scan(0, m);
    nt = std::min<unsigned>(nt, 32);
    std::vector<std::thread> th;
    std::vector<char> res(nt, 1);
    const size_t chunk = (m + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            const size_t lo = std::min(m, t * chunk), hi = std::min(m, lo + chunk);
            res[t] = scan(lo, hi);
        });
    for (auto& x : th) x.join();
    for (char r : res)
        if (!r) return false;
    return true;
}

// Host -> device upload of one host-pointer argument.  The copy runs on the
// calling thread's upload stream, so the compute stream can start on an
// earlier argument while this one is in flight; the buffer belongs to (and is
// freed on) the compute stream, which must wait() before reading it.
cudaStream_t upload_stream() {
    thread_local cudaStream_t s = [] {
        cudaStream_t x = nullptr;
        ck(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
        return x;
    }();
    return s;
}

// A host buffer uploaded on the per-thread upload stream.  The device copy is
// allocated on the upload stream too, so the copy starts at once, even while
// the consumer stream still runs earlier work (e.g. the tail of a plan build);
// the consumer waits on `done` (wait()) before use and frees the copy in its
// own stream order (the destructor orders the free after the upload).
template <class R>
struct HostUp {
    DBuf d;
    cudaStream_t cons;
    cudaEvent_t done = nullptr;
    HostUp(const void* h, size_t count, cudaStream_t st) : d(count * sizeof(R), upload_stream()), cons(st) {
        if (!count) return;
        ck(cudaMemcpyAsync(d.p, h, count * sizeof(R), cudaMemcpyHostToDevice, d.st), "H2D");
        ck(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventRecord(done, d.st), "cudaEventRecord");
    }
    HostUp(const HostUp&) = delete;
    HostUp& operator=(const HostUp&) = delete;
    ~HostUp() {
        if (done) {
            cudaStreamWaitEvent(cons, done, 0);  // free after the upload, in the consumer's order
            d.st = cons;
            cudaEventDestroy(done);
        }
    }
    void wait(cudaStream_t st) const {
        if (done) ck(cudaStreamWaitEvent(st, done, 0), "cudaStreamWaitEvent");
    }
    R* get() const { return d.as<R>(); }
};

// Device flags of the host-pointer API's finiteness checks (one int each).
// snapshot() copies them to a per-thread pinned buffer behind the checks on
// the stream; wait() blocks only until that copy, not the whole stream.
struct Flags {
    DBuf d;
    int n;
    int* h;
    cudaEvent_t ev = nullptr;
    Flags(int n_, cudaStream_t st) : d(sizeof(int) * n_, st), n(n_) {
        thread_local int* pinned = [] {
            int* q = nullptr;
            ck(cudaMallocHost(&q, 64 * sizeof(int)), "cudaMallocHost");
            return q;
        }();
        h = pinned;
        ck(cudaMemsetAsync(d.p, 0, sizeof(int) * n_, st), "memset");
        ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    }
    Flags(const Flags&) = delete;
    Flags& operator=(const Flags&) = delete;
    ~Flags() {
        if (ev) cudaEventDestroy(ev);
    }
    int* at(int i) const { return d.as<int>() + i; }
    void snapshot(cudaStream_t st) {
        ck(cudaMemcpyAsync(h, d.p, sizeof(int) * n, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaEventRecord(ev, st), "cudaEventRecord");
    }
    const int* wait() const {
        ck(cudaEventSynchronize(ev), "cudaEventSynchronize");
        return h;
    }
    // synchronises st; returns the host copy
    std::vector<int> read(cudaStream_t st) {
        snapshot(st);
        wait();
        return std::vector<int>(h, h + n);
    }
};

// Downloads of the host-pointer API: a per-thread stream, so device->host
// copies of finished output ranges overlap the remaining device work.
cudaStream_t download_stream() {
    thread_local cudaStream_t s = [] {
        cudaStream_t x = nullptr;
        ck(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
        return x;
    }();
    return s;
}

// Routes finished output ranges to the caller's host buffers.  The first
// range waits for the input-finiteness flags (fail() before any host write).
struct Downloader {
    struct Map {
        const void* dev;
        void* host;
        size_t count;  // elements per row
        int rows;
        bool streamed;
    };
    std::vector<Map> maps;
    size_t rsz;
    std::function<void()> check;
    bool checked = false;
    OutHook hook;
    cudaStream_t dl = download_stream();
    std::vector<cudaEvent_t> evs;
    explicit Downloader(size_t rs) : rsz(rs) {
        hook.fn = [this](const void* dev, size_t u0, size_t u1, int rows, size_t ld, cudaStream_t st) {
            copy(dev, u0, u1, rows, ld, st);
        };
    }
    Downloader(const Downloader&) = delete;
    Downloader& operator=(const Downloader&) = delete;
    ~Downloader() {
        for (auto e : evs) cudaEventDestroy(e);
    }
    // device output [rows][count] (row pitch = count) -> host buffer of the same shape
    void add(const void* dev, void* host, size_t count, int rows) {
        if (dev && host && count) maps.push_back({dev, host, count, rows, false});
    }
    void run_check() {
        if (!checked) {
            checked = true;
            if (check) check();
        }
    }
    void copy(const void* dev, size_t u0, size_t u1, int rows, size_t ld, cudaStream_t st) {
        run_check();
        for (Map& mp : maps) {
            if (mp.dev != dev) continue;
            mp.streamed = true;
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            evs.push_back(e);
            ck(cudaEventRecord(e, st), "cudaEventRecord");
            ck(cudaStreamWaitEvent(dl, e, 0), "cudaStreamWaitEvent");
            ck(cudaMemcpy2DAsync((char*)mp.host + u0 * rsz, mp.count * rsz, (const char*)dev + u0 * rsz, ld * rsz,
                                 (u1 - u0) * rsz, (size_t)rows, cudaMemcpyDeviceToHost, dl),
               "D2H");
        }
    }
    // outputs the scatter did not stream (direct permutations): whole copies; then wait
    void finish(cudaStream_t st) {
        run_check();
        for (Map& mp : maps)
            if (!mp.streamed) {
                mp.streamed = true;
                ck(cudaMemcpyAsync(mp.host, mp.dev, mp.count * mp.rows * rsz, cudaMemcpyDeviceToHost, st), "D2H");
            }
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        ck(cudaStreamSynchronize(dl), "cudaStreamSynchronize");
    }
};

struct HookScope {  // installs the downloader's hook for the calling thread
    explicit HookScope(OutHook* h) { g_out_hook = h; }
    ~HookScope() { g_out_hook = nullptr; }
};

cudaStream_t host_stream() { return cudaStreamPerThread; }

template <class R>
void d2h(void* dst, const DBuf& src, size_t count, cudaStream_t st) {
    if (dst && count) ck(cudaMemcpyAsync(dst, src.p, count * sizeof(R), cudaMemcpyDeviceToHost, st), "D2H");
}

int dtype_check(int dtype) {
    if (dtype != LAPLEX_F32 && dtype != LAPLEX_F64) fail(LAPLEX_E_INVALID_ARGUMENT, "dtype must be LAPLEX_F32/F64");
    return dtype;
}

// Inputs up to this many elements are validated on the host (cheaper than a
// device round trip); larger ones on the device after the upload.
constexpr size_t kHostCheckMax = size_t(1) << 20;

// LaplexOperator checks that need no data, in reference order
// (operator.hpp:88-101); anchor / phase finiteness is checked on the device.
struct CreateChecks {
    int code = 0;
    const char* msg = nullptr;
};
CreateChecks create_checks(double t, bool phi, bool psi) {
    CreateChecks c;
    const float tf = (float)t;
    if (!(t > 0.0) || !std::isfinite(t) || !(tf > 0.0f) || !std::isfinite(tf)) {
        c.code = LAPLEX_E_NON_FINITE;
        c.msg = "LaplexOperator: temperature must be positive and finite";
    } else if (phi != psi) {
        c.code = LAPLEX_E_DIMENSION_MISMATCH;
        c.msg = "LaplexOperator: phases must be given for both sides";
    }
    return c;
}

template <class R>
laplex_plan create_from_host(const void* a, size_t n, const void* b, size_t k, double t, const void* phi,
                             const void* psi, cudaStream_t st) {
    if (n == 0 || k == 0) fail(LAPLEX_E_EMPTY_INPUT, "LaplexOperator: empty anchor set");
    if (n >= 0x80000000ull || k >= 0x80000000ull) fail(LAPLEX_E_INVALID_SIZE, "n and k must be < 2^31");
    const CreateChecks cc = create_checks(sizeof(R) == 4 ? (double)(float)t : t, phi != nullptr, psi != nullptr);
    if ((size_t)n + k <= kHostCheckMax) {  // small inputs: the whole check on the host, reference order
        if (!host_finite((const R*)a, n)) fail(LAPLEX_E_NON_FINITE, "LaplexOperator row anchors: non-finite entry");
        if (!host_finite((const R*)b, k)) fail(LAPLEX_E_NON_FINITE, "LaplexOperator col anchors: non-finite entry");
        if (cc.code) fail(cc.code, cc.msg);
        if (phi && (!host_finite((const R*)phi, n) || !host_finite((const R*)psi, k)))
            fail(LAPLEX_E_NON_FINITE, "LaplexOperator phases: non-finite entry");
    }
    // upload order a, phi, b, psi: side 0 sorts while side 1 is in flight
    HostUp<R> da(a, n, st);
    HostUp<R> dp(phi, (phi && !cc.code) ? n : 0, st);
    HostUp<R> db(b, k, st);
    HostUp<R> dq(psi, (psi && !cc.code) ? k : 0, st);
    if (cc.code) {  // the anchors' finiteness is reported before these
        Flags f(2, st);
        da.wait(st);
        launch_finite<R>(da.get(), n, f.at(0), st);
        db.wait(st);
        launch_finite<R>(db.get(), k, f.at(1), st);
        const auto h = f.read(st);
        if (h[0]) fail(LAPLEX_E_NON_FINITE, "LaplexOperator row anchors: non-finite entry");
        if (h[1]) fail(LAPLEX_E_NON_FINITE, "LaplexOperator col anchors: non-finite entry");
        fail(cc.code, cc.msg);
    }
    const cudaEvent_t ready[2] = {phi ? dp.done : da.done, psi ? dq.done : db.done};
    return create_plan<R>(da.get(), (uint32_t)n, db.get(), (uint32_t)k, t, phi ? dp.get() : nullptr,
                          psi ? dq.get() : nullptr, st, ready);
}

}  // namespace

// =============================================================================
// extern "C"
// =============================================================================
extern "C" {

int laplex_abi_version(void) { return LAPLEX_ABI_VERSION; }
const char* laplex_last_error(void) { return g_last_error.c_str(); }
uint64_t laplex_kernel_launches(void) { return g_launches.load(); }

int laplex_profile_enable(int on) {
    g_prof.store(on != 0);
    return LAPLEX_OK;
}

int laplex_profile_dump(char* buf, size_t cap) {
    return guarded([&] {
        std::vector<ProfRec> recs;
        {
            std::lock_guard<std::mutex> g(g_prof_mu);
            recs.swap(g_prof_recs);
        }
        struct Agg {
            std::string name;
            uint64_t count = 0;
            double ms = 0;
        };
        std::vector<Agg> agg;
        for (auto& r : recs) {
            ck(cudaEventSynchronize(r.b), "cudaEventSynchronize");
            float ms = 0;
            cudaEventElapsedTime(&ms, r.a, r.b);
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
            Agg* a = nullptr;
            for (auto& x : agg)
                if (x.name == r.name) a = &x;
            if (!a) {
                agg.push_back({r.name, 0, 0});
                a = &agg.back();
            }
            a->count += 1;
            a->ms += ms;
        }
        std::string js = "{";
        for (size_t i = 0; i < agg.size(); ++i) {
            char tmp[256];
            std::snprintf(tmp, sizeof(tmp), "%s\"%s\": {\"launches\": %llu, \"ms\": %.6f}", i ? ", " : "",
                          agg[i].name.c_str(), (unsigned long long)agg[i].count, agg[i].ms);
            js += tmp;
        }
        js += "}";
        if (buf && cap) {
            std::strncpy(buf, js.c_str(), cap - 1);
            buf[cap - 1] = 0;
        }
        if (js.size() + 1 > cap) fail(LAPLEX_E_INVALID_ARGUMENT, "profile buffer too small");
    });
}

int laplex_plan_create(int dtype, const void* a, size_t n, const void* b, size_t k, double t, const void* phi,
                       const void* psi, laplex_plan* out) {
    return guarded([&] {
        if (!out) fail(LAPLEX_E_INVALID_ARGUMENT, "out is NULL");
        *out = nullptr;
        dtype_check(dtype);
        cudaStream_t st = host_stream();
            if (dtype == LAPLEX_F64)
            *out = create_from_host<double>(a, n, b, k, t, phi, psi, st);
        else
            *out = create_from_host<float>(a, n, b, k, t, phi, psi, st);
    });
}

// Device-pointer plan creation.  `shard`: a range shard may hold no anchors on
// one side.  `sync` false: no host synchronisation (NonFinite anchors are
// reported later by laplex_plan_check).
static int create_dev(int dtype, const void* a, size_t n, const void* b, size_t k, double t, const void* phi,
                      const void* psi, void* stream, laplex_plan* out, bool shard, bool sync) {
    return guarded([&] {
        if (!out) fail(LAPLEX_E_INVALID_ARGUMENT, "out is NULL");
        *out = nullptr;
        dtype_check(dtype);
        if (shard ? n + k == 0 : (n == 0 || k == 0))
            fail(LAPLEX_E_EMPTY_INPUT, shard ? "shard plan: no anchors on this shard" : "LaplexOperator: empty anchor set");
        // t as the plan's Real: an fp32 plan rejects a t that is 0 or inf once rounded
        const CreateChecks cc = create_checks(dtype == LAPLEX_F32 ? (double)(float)t : t, phi != nullptr,
                                              psi != nullptr);
        if (cc.code) fail(cc.code, cc.msg);
        if (n >= 0x80000000ull || k >= 0x80000000ull) fail(LAPLEX_E_INVALID_SIZE, "n and k must be < 2^31");
        cudaStream_t st = as_stream(stream);
        if (dtype == LAPLEX_F64)
            *out = create_plan<double>((const double*)a, (uint32_t)n, (const double*)b, (uint32_t)k, t,
                                       (const double*)phi, (const double*)psi, st, nullptr, sync);
        else
            *out = create_plan<float>((const float*)a, (uint32_t)n, (const float*)b, (uint32_t)k, t,
                                      (const float*)phi, (const float*)psi, st, nullptr, sync);
    });
}

int laplex_plan_create_dev(int dtype, const void* a, size_t n, const void* b, size_t k, double t, const void* phi,
                           const void* psi, void* stream, laplex_plan* out) {
    return create_dev(dtype, a, n, b, k, t, phi, psi, stream, out, false, true);
}

int laplex_plan_create_dev_async(int dtype, const void* a, size_t n, const void* b, size_t k, double t,
                                 const void* phi, const void* psi, void* stream, laplex_plan* out) {
    return create_dev(dtype, a, n, b, k, t, phi, psi, stream, out, false, false);
}

int laplex_plan_check(laplex_plan plan) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        ck(cudaEventSynchronize(c.built[0]), "cudaEventSynchronize");
        raise_bad(c);
    });
}

int laplex_pool_trim(void) {
    return guarded([&] {
        DevState& ds = dev_state();
        ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        std::lock_guard<std::mutex> g(ds.mu);
        ck(cudaMemPoolTrimTo(ds.pool, 0), "cudaMemPoolTrimTo");
        ds.reserved = 0;
    });
}

int laplex_plan_retain(laplex_plan plan) {
    return guarded([&] { check_plan(plan)->refs.fetch_add(1); });
}

int laplex_plan_release(laplex_plan plan) {
    return guarded([&] {
        check_plan(plan);
        if (plan->refs.fetch_sub(1) == 1) delete plan;
    });
}

int laplex_plan_transposed(laplex_plan plan, laplex_plan* out) {
    return guarded([&] {
        check_plan(plan);
        auto* p = new laplex_plan_s;
        p->core = plan->core;
        p->swapped = !plan->swapped;
        *out = p;
    });
}

int laplex_plan_shape(laplex_plan plan, size_t* n, size_t* k, double* t, int* has_phases, int* dtype) {
    return guarded([&] {
        check_plan(plan);
        const Core& c = *plan->core;
        const int ia = plan->swapped ? 1 : 0;
        if (n) *n = c.side[ia].m;
        if (k) *k = c.side[1 - ia].m;
        if (t) *t = c.t;
        if (has_phases) *has_phases = c.phased ? 1 : 0;
        if (dtype) *dtype = c.dtype;
    });
}

int laplex_plan_sorted(laplex_plan plan, int side, void* values, uint64_t* perm, void* decays) {
    return guarded([&] {
        check_plan(plan);
        if (side != LAPLEX_ROWS && side != LAPLEX_COLS) fail(LAPLEX_E_INVALID_ARGUMENT, "side");
        Core& c = *plan->core;
        const int phys = plan->swapped ? 1 - side : side;
        const Side& sd = c.side[phys];
        cudaStream_t st = host_stream();
        ck(cudaStreamWaitEvent(st, c.built[0], 0), "cudaStreamWaitEvent");
        const size_t rs = rsize(c.dtype);
        if (values) ck(cudaMemcpyAsync(values, sd.vals.p, (size_t)sd.m * rs, cudaMemcpyDeviceToHost, st), "D2H");
        std::vector<uint32_t> hp;
        if (perm) {
            hp.resize(sd.m);
            ck(cudaMemcpyAsync(hp.data(), sd.perm.p, (size_t)sd.m * 4, cudaMemcpyDeviceToHost, st), "D2H");
        }
        DBuf dec;
        if (decays && sd.m > 1) {
            dec = DBuf((size_t)(sd.m - 1) * rs, st);
            launch("lx_decays", st, [&] {
                if (c.dtype == LAPLEX_F64)
                    lx::sort::lx_decays<double><<<(sd.m + 255) / 256, 256, 0, st>>>(sd.vals.as<double>(), sd.m,
                                                                                   dec.as<double>());
                else
                    lx::sort::lx_decays<float><<<(sd.m + 255) / 256, 256, 0, st>>>(sd.vals.as<float>(), sd.m,
                                                                                  dec.as<float>());
            });
            ck(cudaMemcpyAsync(decays, dec.p, (size_t)(sd.m - 1) * rs, cudaMemcpyDeviceToHost, st), "D2H");
        }
        ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        if (perm)
            for (uint32_t i = 0; i < sd.m; ++i) perm[i] = hp[i];
    });
}

int laplex_plan_ranks(laplex_plan plan, int side, int strict, uint64_t* ranks) {
    return guarded([&] {
        check_plan(plan);
        if (side != LAPLEX_ROWS && side != LAPLEX_COLS) fail(LAPLEX_E_INVALID_ARGUMENT, "side");
        if (plan->core->dtype == LAPLEX_F64)
            do_ranks<double>(plan, side, strict, ranks, host_stream());
        else
            do_ranks<float>(plan, side, strict, ranks, host_stream());
    });
}

int laplex_apply_dev(laplex_plan plan, unsigned flags, const void* X, size_t rows, void* Y, void* stream) {
    return guarded([&] {
        check_plan(plan);
        if (plan->core->dtype == LAPLEX_F64)
            do_apply<double>(plan, flags, (const double*)X, rows, (double*)Y, as_stream(stream));
        else
            do_apply<float>(plan, flags, (const float*)X, rows, (float*)Y, as_stream(stream));
    });
}

int laplex_apply(laplex_plan plan, unsigned flags, const void* X, size_t rows, size_t cols, void* Y) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const int ia = plan->swapped ? 1 : 0;
        const size_t n = c.side[ia].m, k = c.side[1 - ia].m;
        const bool trn = flags & LAPLEX_TRANSPOSE, ph = flags & LAPLEX_PHASED;
        // operator.hpp:162-165,197-201,255-257: phase checks, length, finiteness
        if (ph && !c.phased) fail(LAPLEX_E_PHASE_ABSENT, "phased_matvec: operator has no phases");
        if (!ph && c.phased) fail(LAPLEX_E_PHASE_PRESENT, "matvec: operator has phases");
        const size_t in_len = trn ? n : k, out_len = trn ? k : n;
        if (cols != in_len) fail(LAPLEX_E_DIMENSION_MISMATCH, "matvec: x length");
        cudaStream_t st = host_stream();
        auto run = [&](auto zero) {
            using R = decltype(zero);
            HostUp<R> dx(X, rows * cols, st);
            DBuf dy(rows * out_len * sizeof(R), st);
            Flags f(1, st);
            dx.wait(st);
            launch_finite<R>(dx.get(), rows * cols, f.at(0), st);
            f.snapshot(st);
            Downloader dl(sizeof(R));
            dl.check = [&] {
                if (f.wait()[0]) fail(LAPLEX_E_NON_FINITE, "matvec x: non-finite entry");
            };
            dl.add(dy.p, Y, out_len, (int)rows);
            {
                HookScope hs(&dl.hook);
                do_apply<R>(plan, flags, dx.get(), rows, dy.as<R>(), st);
            }
            if ((flags & LAPLEX_SAVE_X) && !trn) {  // the saved x is keyed by the caller's host pointer
                std::lock_guard<std::mutex> g(c.saved_mu);
                if (c.saved.X == (const void*)dx.get()) {
                    c.saved.X = X;
                    c.saved.host = true;
                }
            }
            dl.finish(st);
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_gram_apply_dev(laplex_plan plan, const void* X, size_t rows, void* Y, void* stream) {
    return guarded([&] {
        check_plan(plan);
        if (plan->core->dtype == LAPLEX_F64)
            do_gram_apply<double>(plan, (const double*)X, rows, (double*)Y, as_stream(stream));
        else
            do_gram_apply<float>(plan, (const float*)X, rows, (float*)Y, as_stream(stream));
    });
}

int laplex_gram_apply(laplex_plan plan, const void* X, size_t rows, size_t cols, void* Y) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const int ia = plan->swapped ? 1 : 0;
        const size_t k = c.side[1 - ia].m;
        // the composition's checks: matvec (operator.hpp:162-165,255-257) first
        if (c.phased) fail(LAPLEX_E_PHASE_PRESENT, "matvec: operator has phases");
        if (cols != k) fail(LAPLEX_E_DIMENSION_MISMATCH, "matvec: x length");
        cudaStream_t st = host_stream();
        auto run = [&](auto zero) {
            using R = decltype(zero);
            HostUp<R> dx(X, rows * cols, st);
            DBuf dy(rows * k * sizeof(R), st);
            Flags f(1, st);
            dx.wait(st);
            launch_finite<R>(dx.get(), rows * cols, f.at(0), st);
            f.snapshot(st);
            Downloader dl(sizeof(R));
            dl.check = [&] {
                if (f.wait()[0]) fail(LAPLEX_E_NON_FINITE, "matvec x: non-finite entry");
            };
            dl.add(dy.p, Y, k, (int)rows);
            {
                HookScope hs(&dl.hook);
                do_gram_apply<R>(plan, dx.get(), rows, dy.as<R>(), st);
            }
            dl.finish(st);
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_backward_dev(laplex_plan plan, unsigned flags, const void* X, const void* G, size_t rows, void* x_bar,
                        void* a_bar, void* b_bar, void* phi_bar, void* psi_bar, void* stream) {
    return guarded([&] {
        check_plan(plan);
        if (plan->core->dtype == LAPLEX_F64)
            do_backward<double>(plan, flags, (const double*)X, (const double*)G, rows, (double*)x_bar,
                                (double*)a_bar, (double*)b_bar, (double*)phi_bar, (double*)psi_bar,
                                as_stream(stream));
        else
            do_backward<float>(plan, flags, (const float*)X, (const float*)G, rows, (float*)x_bar, (float*)a_bar,
                               (float*)b_bar, (float*)phi_bar, (float*)psi_bar, as_stream(stream));
    });
}

int laplex_backward(laplex_plan plan, unsigned flags, const void* X, size_t rows, size_t xcols, const void* G,
                    size_t gcols, void* x_bar, void* a_bar, void* b_bar, void* phi_bar, void* psi_bar) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const int ia = plan->swapped ? 1 : 0;
        const size_t n = c.side[ia].m, k = c.side[1 - ia].m;
        const bool ph = flags & LAPLEX_PHASED;
        // gradients.hpp:113-117 / 142-146
        if (ph && !c.phased) fail(LAPLEX_E_PHASE_ABSENT, "phased_matvec_vjp: operator has no phases");
        if (!ph && c.phased) fail(LAPLEX_E_PHASE_PRESENT, "matvec_vjp: use phased_matvec_vjp");
        if (xcols != k) fail(LAPLEX_E_DIMENSION_MISMATCH, "matvec_vjp: x length");
        if (gcols != n) fail(LAPLEX_E_DIMENSION_MISMATCH, "matvec_vjp: g length");
        cudaStream_t st = host_stream();
        const size_t rs = rsize(c.dtype);
        // LAPLEX_REUSE_X after a host-API apply with LAPLEX_SAVE_X of the same
        // X, rows and orientation: x is neither uploaded nor checked again (the
        // caller asserts it is unchanged; the apply checked it)
        bool reuse;
        {
            std::lock_guard<std::mutex> g(c.saved_mu);
            reuse = (flags & LAPLEX_REUSE_X) && c.saved.xs.p && c.saved.host && c.saved.X == X &&
                    c.saved.rows == rows && c.saved.swapped == plan->swapped && c.saved.phased == ph;
        }
        auto run = [&](auto zero) {
            using R = decltype(zero);
            // x first: its gather runs while g is still uploading
            HostUp<R> dx(reuse ? nullptr : X, reuse ? 0 : rows * k, st);
            HostUp<R> dg(G, rows * n, st);
            DBuf xb(rows * k * rs, st), ab(n * rs, st), bb(k * rs, st), pb(ph ? n * rs : 0, st), qb(ph ? k * rs : 0, st);
            Flags f(2, st);
            if (!reuse) {
                dx.wait(st);
                launch_finite<R>(dx.get(), rows * k, f.at(0), st);
            }
            Downloader dl(rs);
            dl.check = [&] {
                const int* h = f.wait();
                if (h[0]) fail(LAPLEX_E_NON_FINITE, "matvec_vjp x: non-finite entry");
                if (h[1]) fail(LAPLEX_E_NON_FINITE, "matvec_vjp g: non-finite entry");
            };
            dl.add(xb.p, x_bar, k, (int)rows);
            dl.add(ab.p, a_bar, n, 1);
            dl.add(bb.p, b_bar, k, 1);
            if (ph) {
                dl.add(pb.p, phi_bar, n, 1);
                dl.add(qb.p, psi_bar, k, 1);
            }
            {
                HookScope hs(&dl.hook);
                do_backward<R>(plan, reuse ? flags : flags & ~LAPLEX_REUSE_X, reuse ? (const R*)X : dx.get(),
                               dg.get(), rows, xb.as<R>(), ab.as<R>(), bb.as<R>(), pb.as<R>(), qb.as<R>(), st,
                               [&] {
                                   dg.wait(st);
                                   launch_finite<R>(dg.get(), rows * n, f.at(1), st);
                                   f.snapshot(st);
                               },
                               reuse);
            }
            dl.finish(st);
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_gram_dev(laplex_plan plan, unsigned flags, const void* D, void* M, void* stream) {
    return guarded([&] {
        check_plan(plan);
        if (plan->core->dtype == LAPLEX_F64)
            do_gram<double>(plan, flags, (const double*)D, (double*)M, as_stream(stream));
        else
            do_gram<float>(plan, flags, (const float*)D, (float*)M, as_stream(stream));
    });
}

int laplex_gram(laplex_plan plan, unsigned flags, const void* D, size_t dlen, void* M) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const int ia = plan->swapped ? 1 : 0;
        const size_t n = c.side[ia].m, k = c.side[1 - ia].m;
        const bool ph = flags & LAPLEX_PHASED;
        // operator.hpp:192,218-220,372-373
        if (ph && !c.phased) fail(LAPLEX_E_PHASE_ABSENT, "phased_gram: operator has no phases");
        if (!ph && c.phased) fail(LAPLEX_E_PHASE_PRESENT, "weighted_gram: operator has phases");
        if (dlen != k) fail(LAPLEX_E_DIMENSION_MISMATCH, "weighted_gram: D length");
        cudaStream_t st = host_stream();
        auto run = [&](auto zero) {
            using R = decltype(zero);
            if (!host_finite((const R*)D, dlen)) fail(LAPLEX_E_NON_FINITE, "weighted_gram D: non-finite entry");
            HostUp<R> dd(D, k, st);
            dd.wait(st);
            DBuf dm(n * n * sizeof(R), st);
            do_gram<R>(plan, flags, dd.get(), dm.as<R>(), st);
            d2h<R>(M, dm, n * n, st);
            ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_gram_vjp_weights(laplex_plan plan, const void* D, size_t dlen, const void* G_bar, size_t grows,
                            size_t gcols, void* D_bar) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const int ia = plan->swapped ? 1 : 0;
        const size_t n = c.side[ia].m, k = c.side[1 - ia].m;
        (void)D;
        // gradients.hpp:193-205
        if (c.phased) fail(LAPLEX_E_PHASE_PRESENT, "gram_vjp_weights: phased operator not supported");
        if (dlen != k) fail(LAPLEX_E_DIMENSION_MISMATCH, "gram_vjp_weights: D length");
        if (grows != n || gcols != n) fail(LAPLEX_E_DIMENSION_MISMATCH, "gram_vjp_weights: G_bar shape");
        cudaStream_t st = host_stream();
        auto run = [&](auto zero) {
            using R = decltype(zero);
            const R* g = (const R*)G_bar;
            if (!host_finite(g, n * n)) fail(LAPLEX_E_NON_FINITE, "gram_vjp_weights G_bar: non-finite entry");
            R max_abs = 0, max_asym = 0;
            for (size_t i = 0; i < n; ++i)
                for (size_t j = 0; j < i; ++j) {
                    max_abs = std::max(max_abs, std::abs(g[i * n + j]));
                    max_asym = std::max(max_asym, std::abs(g[i * n + j] - g[j * n + i]));
                }
            if (max_asym > R(1e-9) * std::max(R(1), max_abs))
                fail(LAPLEX_E_ASYMMETRIC_COTANGENT, "gram_vjp_weights: G_bar is not symmetric");
            HostUp<R> dg(G_bar, n * n, st);
            dg.wait(st);
            DBuf dd(k * sizeof(R), st);
            do_gram_vjp<R>(plan, dg.get(), dd.as<R>(), st);
            d2h<R>(D_bar, dd, k, st);
            ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_sort(int dtype, const void* raw, size_t m, void* values, uint64_t* perm, void* decays) {
    return guarded([&] {
        dtype_check(dtype);
        // scan.hpp:28-29
        if (m == 0) fail(LAPLEX_E_EMPTY_INPUT, "sort_anchors: empty input");
        if (m >= 0x80000000ull) fail(LAPLEX_E_INVALID_SIZE, "m must be < 2^31");
        cudaStream_t st = host_stream();
            auto run = [&](auto zero) {
            using R = decltype(zero);
            if (!host_finite((const R*)raw, m)) fail(LAPLEX_E_NON_FINITE, "sort_anchors: non-finite entry");
            HostUp<R> dr(raw, m, st);
            dr.wait(st);
            DBuf vals(m * sizeof(R), st), pm(m * 4, st), bad(sizeof(int), st), dec(m > 1 ? (m - 1) * sizeof(R) : 0, st);
            ck(cudaMemsetAsync(bad.p, 0, sizeof(int), st), "memset");
            radix_sort<R>(dr.get(), (uint32_t)m, R(1), vals.as<R>(), pm.as<uint32_t>(), bad.as<int>(), st);
            if (m > 1) {
                launch("lx_decays", st, [&] {
                    lx::sort::lx_decays<R><<<(uint32_t)((m + 255) / 256), 256, 0, st>>>(vals.as<R>(), m, dec.as<R>());
                });
            }
            std::vector<uint32_t> hp(m);
            d2h<R>(values, vals, m, st);
            ck(cudaMemcpyAsync(hp.data(), pm.p, m * 4, cudaMemcpyDeviceToHost, st), "D2H");
            if (decays && m > 1) d2h<R>(decays, dec, m - 1, st);
            ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            if (perm)
                for (size_t i = 0; i < m; ++i) perm[i] = hp[i];
        };
        if (dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_scan(int dtype, const void* sorted_values, size_t m, const void* payload, void* prefix, void* suffix) {
    return guarded([&] {
        dtype_check(dtype);
        if (m == 0) return;
        if (m >= 0x80000000ull) fail(LAPLEX_E_INVALID_SIZE, "m must be < 2^31");
        if (dtype == LAPLEX_F64)
            do_scan<double>((const double*)sorted_values, (uint32_t)m, (const double*)payload, (double*)prefix,
                            (double*)suffix, host_stream());
        else
            do_scan<float>((const float*)sorted_values, (uint32_t)m, (const float*)payload, (float*)prefix,
                           (float*)suffix, host_stream());
    });
}

int laplex_sort_dev(int dtype, const void* raw, size_t m, void* values, uint32_t* perm, void* decays,
                    int* nonfinite, void* stream) {
    return guarded([&] {
        dtype_check(dtype);
        if (m == 0) fail(LAPLEX_E_EMPTY_INPUT, "sort_anchors: empty input");
        if (m >= 0x80000000ull) fail(LAPLEX_E_INVALID_SIZE, "m must be < 2^31");
        if (!values || !perm) fail(LAPLEX_E_INVALID_ARGUMENT, "sort_anchors: values and perm are required");
        cudaStream_t st = as_stream(stream);
        auto run = [&](auto zero) {
            using R = decltype(zero);
            DBuf bad(nonfinite ? 0 : sizeof(int), st);
            int* flag = nonfinite ? nonfinite : bad.as<int>();
            ck(cudaMemsetAsync(flag, 0, sizeof(int), st), "memset");
            radix_sort<R>((const R*)raw, (uint32_t)m, R(1), (R*)values, perm, flag, st);
            if (decays && m > 1)
                launch("lx_decays", st, [&] {
                    lx::sort::lx_decays<R><<<(uint32_t)((m + 255) / 256), 256, 0, st>>>((const R*)values, m,
                                                                                       (R*)decays);
                });
            if (!nonfinite) {  // report NonFinite synchronously (scan.hpp:29)
                int h = 0;
                ck(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
                if (h) fail(LAPLEX_E_NON_FINITE, "sort_anchors: non-finite entry");
            }
        };
        if (dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_scan_dev(int dtype, const void* sorted_values, size_t m, const void* payload, void* prefix, void* suffix,
                    void* stream) {
    return guarded([&] {
        dtype_check(dtype);
        if (m == 0) return;
        if (m >= 0x80000000ull) fail(LAPLEX_E_INVALID_SIZE, "m must be < 2^31");
        if (!prefix && !suffix) return;
        if (dtype == LAPLEX_F64)
            do_scan_dev<double>((const double*)sorted_values, (uint32_t)m, (const double*)payload, (double*)prefix,
                                (double*)suffix, as_stream(stream));
        else
            do_scan_dev<float>((const float*)sorted_values, (uint32_t)m, (const float*)payload, (float*)prefix,
                               (float*)suffix, as_stream(stream));
    });
}

int laplex_gram_vjp_weights_dev(laplex_plan plan, const void* G_bar, void* D_bar, void* stream) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        if (c.phased) fail(LAPLEX_E_PHASE_PRESENT, "gram_vjp_weights: phased operator not supported");
        cudaStream_t st = as_stream(stream);
        const int ia = plan->swapped ? 1 : 0;
        const uint32_t n = c.side[ia].m;
        auto run = [&](auto zero) {
            using R = decltype(zero);
            // gradients.hpp:196-205 on the device: finiteness, then symmetry
            // (max |G_ij - G_ji| <= 1e-9 max(1, max |G_ij|)), one synchronisation
            DBuf flags(3 * sizeof(R), st);
            ck(cudaMemsetAsync(flags.p, 0, 3 * sizeof(R), st), "memset");
            launch("lx_gram_sym_check", st, [&] {
                lx::gram::lx_sym_check<R><<<std::max(1u, std::min<uint32_t>((n + 15) / 16, 4096u)), 256, 0, st>>>(
                    (const R*)G_bar, n, flags.as<R>());
            });
            R h[3];
            ck(cudaMemcpyAsync(h, flags.p, sizeof(h), cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "cudaStreamSynchronize");
            if (h[2] != R(0)) fail(LAPLEX_E_NON_FINITE, "gram_vjp_weights G_bar: non-finite entry");
            if (h[1] > R(1e-9) * std::max(R(1), h[0]))
                fail(LAPLEX_E_ASYMMETRIC_COTANGENT, "gram_vjp_weights: G_bar is not symmetric");
            do_gram_vjp<R>(plan, (const R*)G_bar, (R*)D_bar, st);
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

// ---------------------------------------------------------------------------
// range-sharded (multi-GPU) building blocks
// ---------------------------------------------------------------------------
int laplex_shard_plan_create_dev(int dtype, const void* a, size_t n, const void* b, size_t k, double t,
                                 const void* phi, const void* psi, void* stream, laplex_plan* out) {
    return create_dev(dtype, a, n, b, k, t, phi, psi, stream, out, true, true);
}

int laplex_shard_partition_dev(int dtype, const void* raw, size_t m, double t, const void* splitters, int nsplit,
                               uint32_t* perm, uint32_t* counts, void* stream) {
    return guarded([&] {
        dtype_check(dtype);
        if (nsplit < 0 || nsplit >= lx::shard::kMaxShards) fail(LAPLEX_E_INVALID_ARGUMENT, "nsplit");
        cudaStream_t st = as_stream(stream);
            const int nsh = nsplit + 1;
        if (m == 0) {
            ck(cudaMemsetAsync(counts, 0, (size_t)nsh * 4, st), "memset");
            return;
        }
        const uint32_t tiles = (uint32_t)((m + lx::shard::kTile - 1) / lx::shard::kTile);
        DBuf cnt((size_t)tiles * lx::shard::kMaxShards * 4, st);
        auto run = [&](auto zero) {
            using R = decltype(zero);
            const R* rp = (const R*)raw;
            const R* sp = (const R*)splitters;
            const R tr = R(t);
            launch("lx_shard_count", st, [&] {
                lx::shard::lx_shard_count<R><<<tiles, lx::shard::kThreads, 0, st>>>(rp, m, tr, sp, nsplit,
                                                                                    cnt.as<uint32_t>());
            });
            launch("lx_shard_totals", st, [&] {
                lx::shard::lx_shard_totals<<<nsh, lx::shard::kOffThreads, 0, st>>>(cnt.as<uint32_t>(), tiles, counts);
            });
            launch("lx_shard_scan", st, [&] {
                lx::shard::lx_shard_scan<<<nsh, lx::shard::kOffThreads, 0, st>>>(cnt.as<uint32_t>(), tiles, counts);
            });
            launch("lx_shard_scatter", st, [&] {
                lx::shard::lx_shard_scatter<R><<<tiles, lx::shard::kThreads, 0, st>>>(rp, m, tr, sp, nsplit,
                                                                                      cnt.as<uint32_t>(), perm);
            });
        };
        if (dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_gather_dev(int dtype, const void* src, size_t ld_src, const uint32_t* idx, size_t m, size_t rows,
                      void* dst, void* stream) {
    return guarded([&] {
        dtype_check(dtype);
        if (m == 0 || rows == 0) return;
        cudaStream_t st = as_stream(stream);
        auto run = [&](auto zero) {
            using R = decltype(zero);
            using namespace lx::shard;
            const uint32_t chunks = (uint32_t)((m + kRouteChunk - 1) / kRouteChunk);
            for (size_t r0 = 0; r0 < rows; r0 += 65535) {  // grid.y limit
                const uint32_t nr = (uint32_t)std::min<size_t>(65535, rows - r0);
                launch("lx_gather_idx", st, [&] {
                    lx_gather_idx<R><<<dim3(chunks, nr), kRouteThreads, 0, st>>>(
                        (const R*)src + r0 * ld_src, ld_src, idx, m, (R*)dst + r0 * m);
                });
            }
        };
        if (dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_scatter_dev(int dtype, const void* src, const uint32_t* idx, size_t m, size_t rows, void* dst,
                       size_t ld_dst, void* stream) {
    return guarded([&] {
        dtype_check(dtype);
        if (m == 0 || rows == 0) return;
        cudaStream_t st = as_stream(stream);
        auto run = [&](auto zero) {
            using R = decltype(zero);
            using namespace lx::shard;
            const uint32_t chunks = (uint32_t)((m + kRouteChunk - 1) / kRouteChunk);
            for (size_t r0 = 0; r0 < rows; r0 += 65535) {  // grid.y limit
                const uint32_t nr = (uint32_t)std::min<size_t>(65535, rows - r0);
                launch("lx_scatter_idx", st, [&] {
                    lx_scatter_idx<R><<<dim3(chunks, nr), kRouteThreads, 0, st>>>(
                        (const R*)src + r0 * m, idx, m, (R*)dst + r0 * ld_dst, ld_dst);
                });
            }
        };
        if (dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
    });
}

int laplex_shard_totals_count(laplex_plan plan, unsigned flags, int backward, size_t rows, size_t* count) {
    return guarded([&] {
        check_plan(plan);
        const int ch = (flags & LAPLEX_PHASED) ? 2 : 1;
        const int nc = backward ? 2 * ch : ch;
        *count = 3 + 2 * (size_t)(2 * nc) * rows;
    });
}

int laplex_shard_apply_begin(laplex_plan plan, unsigned flags, const void* X, size_t rows, void* totals,
                             laplex_work* work, void* stream) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const bool ph = flags & LAPLEX_PHASED;
        if (ph != c.phased) fail(ph ? LAPLEX_E_PHASE_ABSENT : LAPLEX_E_PHASE_PRESENT, "shard apply: phase mismatch");
        if (flags & LAPLEX_TRANSPOSE) fail(LAPLEX_E_INVALID_ARGUMENT, "shard apply: transpose not supported");
        if (rows == 0 || rows > 0x7fffffff) fail(LAPLEX_E_INVALID_SIZE, "rows");
        cudaStream_t st = as_stream(stream);
        auto w = std::make_unique<laplex_work_s>();
        w->dtype = c.dtype;
        w->phased = ph;
        auto run = [&](auto zero) {
            using R = decltype(zero);
            View<R> v = view<R>(c, plan->swapped, st);
            if (ph) {
                auto f = fwd_begin<R, 2>(v, (const R*)X, (int)rows, st);
                collect_totals<R>(v, f->sc, (int)rows, 4, (R*)totals, st);
                w->impl = std::move(f);
            } else {
                auto f = fwd_begin<R, 1>(v, (const R*)X, (int)rows, st);
                collect_totals<R>(v, f->sc, (int)rows, 2, (R*)totals, st);
                w->impl = std::move(f);
            }
            w->impl->keep = plan->core;
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
        *work = w.release();
    });
}

int laplex_shard_apply_end(laplex_work work, const void* ext, void* Y, void* stream) {
    return guarded([&] {
        if (!work || work->backward) fail(LAPLEX_E_INVALID_ARGUMENT, "invalid work handle");
        cudaStream_t st = as_stream(stream);
        auto run = [&](auto zero) {
            using R = decltype(zero);
            if (work->phased)
                fwd_end<R, 2>(*static_cast<FwdWork<R, 2>*>(work->impl.get()), (const R*)ext, (R*)Y, st);
            else
                fwd_end<R, 1>(*static_cast<FwdWork<R, 1>*>(work->impl.get()), (const R*)ext, (R*)Y, st);
        };
        if (work->dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
        delete work;
    });
}

int laplex_shard_backward_begin(laplex_plan plan, unsigned flags, const void* X, const void* G, size_t rows,
                                void* totals, laplex_work* work, void* stream) {
    return guarded([&] {
        check_plan(plan);
        Core& c = *plan->core;
        const bool ph = flags & LAPLEX_PHASED;
        if (ph != c.phased) fail(ph ? LAPLEX_E_PHASE_ABSENT : LAPLEX_E_PHASE_PRESENT, "shard backward: phases");
        if (rows == 0 || rows > 0x7fffffff) fail(LAPLEX_E_INVALID_SIZE, "rows");
        cudaStream_t st = as_stream(stream);
        auto w = std::make_unique<laplex_work_s>();
        w->dtype = c.dtype;
        w->phased = ph;
        w->backward = true;
        auto run = [&](auto zero) {
            using R = decltype(zero);
            View<R> v = view<R>(c, plan->swapped, st);
            if (ph) {
                auto b = bwd_begin<R, 2>(v, (const R*)X, (const R*)G, (int)rows, st);
                collect_totals<R>(v, b->sc, (int)rows, 8, (R*)totals, st);
                w->impl = std::move(b);
            } else {
                auto b = bwd_begin<R, 1>(v, (const R*)X, (const R*)G, (int)rows, st);
                collect_totals<R>(v, b->sc, (int)rows, 4, (R*)totals, st);
                w->impl = std::move(b);
            }
            w->impl->keep = plan->core;
        };
        if (c.dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
        *work = w.release();
    });
}

int laplex_shard_backward_end(laplex_work work, const void* ext, void* x_bar, void* a_bar, void* b_bar,
                              void* phi_bar, void* psi_bar, void* stream) {
    return guarded([&] {
        if (!work || !work->backward) fail(LAPLEX_E_INVALID_ARGUMENT, "invalid work handle");
        cudaStream_t st = as_stream(stream);
        auto run = [&](auto zero) {
            using R = decltype(zero);
            if (work->phased)
                bwd_end<R, 2>(*static_cast<BwdWork<R, 2>*>(work->impl.get()), (const R*)ext, (R*)x_bar, (R*)a_bar,
                              (R*)b_bar, (R*)phi_bar, (R*)psi_bar, st);
            else
                bwd_end<R, 1>(*static_cast<BwdWork<R, 1>*>(work->impl.get()), (const R*)ext, (R*)x_bar, (R*)a_bar,
                              (R*)b_bar, nullptr, nullptr, st);
        };
        if (work->dtype == LAPLEX_F64)
            run(0.0);
        else
            run(0.0f);
        delete work;
    });
}

int laplex_work_release(laplex_work work) {
    delete work;
    return LAPLEX_OK;
}

}  // extern "C"

// multi-GPU host layer (communicators, range-sharded operator, batch replicas)
#include "lx_dist.inc"
