// Random-sector read ceiling of this B200: the bound for k_hop's neighbour-rank loads (one 4-byte
// read of cols_rank at a random CSR index per sample, i.e. one 32-byte DRAM sector per load).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/randread tools/randread.cu && /tmp/randread
//
// Tables of 256 MB - 2 GiB (> the 126 MB L2); every thread issues `kBatch` independent loads per iteration at
// hashed indices.  Reports loads/s and sector GB/s (32 B per load) -- the denominator DESIGN.md uses
// for the random-gather kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kBatch = 8;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void k_rand(const int32_t* __restrict__ t, uint32_t mask, int iters, int32_t* out) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    int32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        int32_t v[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) v[j] = __ldg(t + (mix(tid * 131u + it * 7919u + j * 104729u) & mask));
#pragma unroll
        for (int j = 0; j < kBatch; ++j) acc += v[j];
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

int main() {
    const size_t n_max = (size_t)1 << 29;   // up to 2 GiB of int32
    int32_t *t, *out;
    cudaMalloc(&t, n_max * 4);
    cudaMalloc(&out, 4);
    cudaMemset(t, 1, n_max * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t n : {(size_t)1 << 26, (size_t)1 << 27, (size_t)1 << 28, (size_t)1 << 29}) {   // 256 MB .. 2 GiB
        for (int bps : {4, 8}) {
            const int blocks = 148 * bps, threads = 256, iters = 64;
            k_rand<<<blocks, threads>>>(t, (uint32_t)(n - 1), iters, out);
            cudaEventRecord(a);
            const int reps = 5;
            for (int r = 0; r < reps; ++r) k_rand<<<blocks, threads>>>(t, (uint32_t)(n - 1), iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double loads = (double)blocks * threads * iters * kBatch * reps;
            printf("table %4zu MB, blocks/SM %d: %.1f G random loads/s, %.0f GB/s of 32-byte sectors\n", n * 4 >> 20,
                   bps, loads / ms / 1e6, loads * 32 / ms / 1e6);
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
