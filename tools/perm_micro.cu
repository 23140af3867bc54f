// Diagnostic only (not product code): cost of the window-local half of a
// permutation (lx_perm_stage_scatter / lx_perm_stage_gather) on 2^30 fp32
// elements as a function of the window size and of the cache policy, plus the
// shared-memory-window alternative.  dst is a pseudo-random bijection inside
// each window (what a plan's sdst looks like).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/perm_micro tools/perm_micro.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x, int b, uint32_t seed) {
    const uint32_t mask = b == 32 ? 0xffffffffu : ((1u << b) - 1u);
    x = (x ^ seed) & mask;
    for (int r = 0; r < 3; ++r) {
        x = (x * 0x9E3779B1u) & mask;
        x ^= x >> (b / 2 + 1);
        x = (x + 0x7F4A7C15u * (r + 1)) & mask;
    }
    return x;
}

__global__ void make_dst(uint32_t* dst, size_t m, int wbits) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x) {
        const size_t base = q >> wbits << wbits;
        dst[q] = (uint32_t)(base + mix((uint32_t)(q - base), wbits, (uint32_t)(base >> wbits) * 2654435761u));
    }
}

__global__ void fill(float* v, size_t m) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x)
        v[q] = (float)(q & 1023);
}

constexpr int T = 256, I = 8, CH = T * I;

template <int MODE>  // 0 plain, 1 streaming loads, 2 streaming loads + evict_last stores
__global__ void __launch_bounds__(T) scat(const uint32_t* __restrict__ dst, const float* __restrict__ s,
                                          float* __restrict__ o, size_t m) {
    const size_t q0 = (size_t)blockIdx.x * CH + threadIdx.x;
    uint32_t u[I];
    float v[I];
#pragma unroll
    for (int j = 0; j < I; ++j) {
        const size_t q = q0 + (size_t)j * T;
        if (MODE == 0) { u[j] = q < m ? dst[q] : 0u; v[j] = q < m ? s[q] : 0.f; }
        else { u[j] = q < m ? __ldcs(dst + q) : 0u; v[j] = q < m ? __ldcs(s + q) : 0.f; }
    }
    uint64_t pol = 0;
    if (MODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
    for (int j = 0; j < I; ++j) {
        const size_t q = q0 + (size_t)j * T;
        if (q < m) {
            if (MODE == 2)
                asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(o + u[j]), "f"(v[j]), "l"(pol) : "memory");
            else
                o[u[j]] = v[j];
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(T) gath(const uint32_t* __restrict__ dst, const float* __restrict__ x,
                                          float* __restrict__ st, size_t m) {
    const size_t q0 = (size_t)blockIdx.x * CH + threadIdx.x;
    uint32_t u[I];
    float v[I];
#pragma unroll
    for (int j = 0; j < I; ++j) {
        const size_t q = q0 + (size_t)j * T;
        u[j] = q < m ? (MODE ? __ldcs(dst + q) : dst[q]) : 0u;
    }
    uint64_t pol = 0;
    if (MODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
    for (int j = 0; j < I; ++j) {
        const size_t q = q0 + (size_t)j * T;
        if (q < m) {
            if (MODE == 2)
                asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v[j]) : "l"(x + u[j]), "l"(pol));
            else
                v[j] = x[u[j]];
        } else v[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < I; ++j) {
        const size_t q = q0 + (size_t)j * T;
        if (q < m) { if (MODE) __stcs(st + q, v[j]); else st[q] = v[j]; }
    }
}

__global__ void copyk(const float* __restrict__ s, float* __restrict__ o, size_t m) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < m / 4; q += (size_t)gridDim.x * blockDim.x)
        reinterpret_cast<float4*>(o)[q] = reinterpret_cast<const float4*>(s)[q];
}

// shared-memory window: one CTA owns a 2^W-element window of the output and
// receives its entries (value + 16-bit local index) contiguously
template <int W>
__global__ void __launch_bounds__(1024) smem_win(const float* __restrict__ s, const uint16_t* __restrict__ li,
                                                 float* __restrict__ o) {
    extern __shared__ float win[];
    constexpr int N = 1 << W;
    const size_t base = (size_t)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += 1024) win[li[base + i]] = s[base + i];
    __syncthreads();
    for (int i = threadIdx.x; i < N / 4; i += 1024)
        reinterpret_cast<float4*>(o + base)[i] = reinterpret_cast<const float4*>(win)[i];
}

__global__ void make_li(uint16_t* li, size_t m, int wbits) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x) {
        const size_t base = q >> wbits << wbits;
        li[q] = (uint16_t)mix((uint32_t)(q - base), wbits, (uint32_t)(base >> wbits) * 2654435761u);
    }
}

// digit-run writes of a radix pass: tile t (RK keys) writes RK/256 consecutive
// keys (+ values) into each of 256 digit regions, like a uniform-digit pass
template <int RK>
__global__ void __launch_bounds__(256) runs(const uint2* __restrict__ in, uint32_t* __restrict__ ok,
                                            uint32_t* __restrict__ ov, size_t m) {
    constexpr int RUN = RK / 256;
    const size_t tiles = m / RK;
    const size_t t = blockIdx.x;
    const size_t region = m / 256;
    for (int j = 0; j < RK / 256; ++j) {
        const int i = j * 256 + threadIdx.x;  // position in the tile, digit-major
        const uint2 kv = in[t * RK + i];
        const int d = i / RUN, r = i % RUN;
        const size_t o = (size_t)d * region + t * RUN + r;
        ok[o] = kv.x;
        ov[o] = kv.y;
    }
    (void)tiles;
}

template <class F>
float timeit(F f, int reps = 5) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 30;
    const size_t m = size_t(1) << lg;
    uint32_t* dst;
    float *s, *o;
    uint16_t* li;
    CK(cudaMalloc(&dst, m * 4));
    CK(cudaMalloc(&s, m * 4));
    CK(cudaMalloc(&o, m * 4));
    CK(cudaMalloc(&li, m * 2));
    fill<<<2048, 256>>>(s, m);
    const unsigned blocks = (unsigned)((m + CH - 1) / CH);
    printf("copy 8 B/elem: %.3f ms\n", timeit([&] { copyk<<<148 * 16, 256>>>(s, o, m); }));
    for (int wb = 14; wb <= 24; ++wb) {
        make_dst<<<2048, 256>>>(dst, m, wb);
        CK(cudaDeviceSynchronize());
        float t[6];
        t[0] = timeit([&] { scat<0><<<blocks, T>>>(dst, s, o, m); });
        t[1] = timeit([&] { scat<1><<<blocks, T>>>(dst, s, o, m); });
        t[2] = timeit([&] { scat<2><<<blocks, T>>>(dst, s, o, m); });
        t[3] = timeit([&] { gath<0><<<blocks, T>>>(dst, s, o, m); });
        t[4] = timeit([&] { gath<1><<<blocks, T>>>(dst, s, o, m); });
        t[5] = timeit([&] { gath<2><<<blocks, T>>>(dst, s, o, m); });
        printf("window 2^%2d (%6.2f MB): scatter plain %.3f cs %.3f cs+evl %.3f | gather plain %.3f cs %.3f cs+evl %.3f ms\n",
               wb, (4.0 * (1 << wb)) / 1048576.0, t[0], t[1], t[2], t[3], t[4], t[5]);
    }
    {
        uint32_t *k2, *v2;
        CK(cudaMalloc(&k2, m * 4));
        CK(cudaMalloc(&v2, m * 4));
        const uint2* in = reinterpret_cast<const uint2*>(dst);  // m/2 pairs: reuse 2 buffers as 8 B input
        const size_t mm = m / 2;
        printf("digit runs (8 B in, 4+4 B out) of %zu keys: tile 2048 %.3f | 4096 %.3f | 8192 %.3f | 16384 %.3f ms\n", mm,
               timeit([&] { runs<2048><<<(unsigned)(mm / 2048), 256>>>(in, k2, v2, mm); }),
               timeit([&] { runs<4096><<<(unsigned)(mm / 4096), 256>>>(in, k2, v2, mm); }),
               timeit([&] { runs<8192><<<(unsigned)(mm / 8192), 256>>>(in, k2, v2, mm); }),
               timeit([&] { runs<16384><<<(unsigned)(mm / 16384), 256>>>(in, k2, v2, mm); }));
        printf("copy of the same bytes (8 B in, 8 B out): %.3f ms\n",
               timeit([&] { copyk<<<148 * 16, 256>>>(s, o, m); }));
        make_li<<<2048, 256>>>(li, m, 15);
        CK(cudaFuncSetAttribute(smem_win<15>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << 15));
        printf("smem window 2^15 (val 4 B + idx 2 B in, 4 B out): %.3f ms\n",
               timeit([&] { smem_win<15><<<(unsigned)(m >> 15), 1024, 4 << 15>>>(s, li, o); }));
        make_li<<<2048, 256>>>(li, m, 14);
        CK(cudaFuncSetAttribute(smem_win<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 << 14));
        printf("smem window 2^14: %.3f ms\n",
               timeit([&] { smem_win<14><<<(unsigned)(m >> 14), 1024, 4 << 14>>>(s, li, o); }));
    }
    return 0;
}
