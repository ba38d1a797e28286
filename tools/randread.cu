// Random-sector read ceiling of this B200: the bound for k_hop's neighbour-rank loads (one 4-byte
// read of cols_rank at a random CSR index per sample, i.e. one 32-byte DRAM sector per load).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/randread tools/randread.cu && /tmp/randread
//
// Tables of 16 MB - 2 GiB (L2-resident up to 64 MB, > the 126 MB L2 from 256 MB); every thread issues
// `kBatch` independent loads per iteration at hashed indices, 4-byte (k_hop's column loads) or 8-byte
// (k_relabel's (bits, position) probes).  Reports loads/s and sector GB/s (32 B per load) -- the
// denominators DESIGN.md uses for the random-access kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kBatch = 8;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

template <class T>
__device__ __forceinline__ int32_t val(T v) { return (int32_t)v; }
template <>
__device__ __forceinline__ int32_t val<int2>(int2 v) { return v.x ^ v.y; }

template <class T>
__global__ void k_rand(const T* __restrict__ t, uint32_t mask, int iters, int32_t* out) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    int32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        T v[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) v[j] = __ldg(t + (mix(tid * 131u + it * 7919u + j * 104729u) & mask));
#pragma unroll
        for (int j = 0; j < kBatch; ++j) acc += val(v[j]);
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

template <class T>
void run(const void* tab, size_t bytes, int32_t* out, cudaEvent_t a, cudaEvent_t b, int sms) {
    const size_t n = bytes / sizeof(T);
    for (int bps : {4, 8}) {
        const int blocks = sms * bps, threads = 256, iters = 64;
        k_rand<T><<<blocks, threads>>>((const T*)tab, (uint32_t)(n - 1), iters, out);
        cudaEventRecord(a);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) k_rand<T><<<blocks, threads>>>((const T*)tab, (uint32_t)(n - 1), iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double loads = (double)blocks * threads * iters * kBatch * reps;
        printf("table %4zu MB, %zu-byte loads, blocks/SM %d: %.1f G random loads/s, %.0f GB/s of 32-byte sectors\n",
               bytes >> 20, sizeof(T), bps, loads / ms / 1e6, loads * 32 / ms / 1e6);
    }
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
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (size_t mb : {16, 32, 64, 256, 512, 1024, 2048}) {   // 16-64 MB fit the 126 MB L2
        run<int32_t>(t, mb << 20, out, a, b, sms);
        run<int2>(t, mb << 20, out, a, b, sms);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}
