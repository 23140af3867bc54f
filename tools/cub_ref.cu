// Reference point only (not product code): CUB onesweep SortPairs on 2^N u32
// key / u32 value pairs on this B200, timed with CUDA events.
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void fill(unsigned* k, unsigned* v, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)(i * 2654435761u) ^ 0x9e3779b9u;
        x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13;
        k[i] = x; v[i] = (unsigned)i;
    }
}

int main(int argc, char** argv) {
    int lg = argc > 1 ? atoi(argv[1]) : 30;
    size_t n = size_t(1) << lg;
    unsigned *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
    fill<<<1184, 256>>>(k0, v0, n);
    void* tmp = nullptr; size_t tmpb = 0;
    cub::DeviceRadixSort::SortPairs(tmp, tmpb, k0, k1, v0, v1, n);
    cudaMalloc(&tmp, tmpb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) cub::DeviceRadixSort::SortPairs(tmp, tmpb, k0, k1, v0, v1, n);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) cub::DeviceRadixSort::SortPairs(tmp, tmpb, k0, k1, v0, v1, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
    printf("cub SortPairs u32/u32 n=2^%d: %.3f ms  (%.1f GB/s at 4 passes x 16 B + 4 B hist)\n", lg, ms,
           n * 68.0 / (ms * 1e6));
    return 0;
}
