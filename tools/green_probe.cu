// Probe: do green contexts (SM partitions) work with runtime-API launches on this driver, and does
// an HBM-streaming kernel on one partition overlap a random-read kernel on the other?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o green_probe tools/green_probe.cu -lcuda
//   ./green_probe [SMs of partition A]
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CU(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* m; cuGetErrorString(r_, &m); \
    printf("%s failed: %s\n", #x, m); exit(1); } } while (0)
#define RT(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s failed: %s\n", #x, \
    cudaGetErrorString(r_)); exit(1); } } while (0)

__global__ void k_smid(int* out) {
    if (threadIdx.x == 0) {
        int s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        out[blockIdx.x] = s;
    }
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

__global__ void k_rand(const int* __restrict__ t, long n, long iters, int* out) {
    unsigned x = blockIdx.x * blockDim.x + threadIdx.x + 1;
    int acc = 0;
    for (long i = 0; i < iters; ++i) {
        int v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x = x * 1664525u + 1013904223u;
            v[j] = __ldg(t + (x % (unsigned)n));
        }
        acc += v[0] ^ v[1] ^ v[2] ^ v[3];
    }
    if (acc == 0x7fffffff) out[0] = acc;
}

static std::set<int> sms_of(cudaStream_t s, int* d, int nb) {
    k_smid<<<nb, 32, 0, s>>>(d);
    RT(cudaGetLastError());
    RT(cudaStreamSynchronize(s));
    std::vector<int> h(nb);
    RT(cudaMemcpy(h.data(), d, nb * 4, cudaMemcpyDeviceToHost));
    return std::set<int>(h.begin(), h.end());
}

int main(int argc, char** argv) {
    const unsigned want = argc > 1 ? atoi(argv[1]) : 100;
    CU(cuInit(0));
    RT(cudaSetDevice(0));
    RT(cudaFree(0));
    CUdevice dev;
    CU(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource ga, rest;
    unsigned nb = 1;
    CU(cuDevSmResourceSplitByCount(&ga, &nb, &all, &rest, 0, want));
    printf("partition A: %u SMs, B (remaining): %u SMs\n", ga.sm.smCount, rest.sm.smCount);
    CUdevResourceDesc da, db;
    CU(cuDevResourceGenerateDesc(&da, &ga, 1));
    CU(cuDevResourceGenerateDesc(&db, &rest, 1));
    CUgreenCtx ca, cb;
    CU(cuGreenCtxCreate(&ca, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CU(cuGreenCtxCreate(&cb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sa, sb;
    CU(cuGreenCtxStreamCreate(&sa, ca, CU_STREAM_NON_BLOCKING, 0));
    CU(cuGreenCtxStreamCreate(&sb, cb, CU_STREAM_NON_BLOCKING, 0));
    int* d;
    RT(cudaMalloc(&d, 4096 * 4));
    auto A = sms_of((cudaStream_t)sa, d, 4096), B = sms_of((cudaStream_t)sb, d, 4096);
    printf("runtime launch on green stream A used %zu SMs, B used %zu SMs\n", A.size(), B.size());
    int overlap = 0;
    for (int s : A) overlap += B.count(s);
    printf("SMs in both: %d\n", overlap);

    const long n4 = (2048L << 20) / 16;                  // 2 GiB copy
    float4 *x, *y;
    RT(cudaMalloc(&x, n4 * 16));
    RT(cudaMalloc(&y, n4 * 16));
    RT(cudaMemset(x, 1, n4 * 16));
    const long nt = (1024L << 20) / 4;                   // 1 GiB random-read table
    int* t;
    RT(cudaMalloc(&t, nt * 4));
    RT(cudaMemset(t, 2, nt * 4));
    cudaStream_t s0;
    RT(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, e2, e3;
    RT(cudaEventCreate(&e0)); RT(cudaEventCreate(&e1)); RT(cudaEventCreate(&e2)); RT(cudaEventCreate(&e3));
    const long iters = 64;
    auto run = [&](cudaStream_t scp, int gcp, cudaStream_t srd, int grd, const char* tag) {
        for (int rep = 0; rep < 2; ++rep) {
            RT(cudaDeviceSynchronize());
            RT(cudaEventRecord(e0, scp));
            RT(cudaStreamWaitEvent(srd, e0, 0));
            k_copy<<<gcp, 512, 0, scp>>>(x, y, n4);
            RT(cudaEventRecord(e1, scp));
            k_rand<<<grd, 256, 0, srd>>>(t, nt, iters, d);
            RT(cudaEventRecord(e2, srd));
            RT(cudaStreamWaitEvent(scp, e2, 0));
            RT(cudaEventRecord(e3, scp));
            RT(cudaEventSynchronize(e3));
            float tc, tr, tt;
            RT(cudaEventElapsedTime(&tc, e0, e1));
            RT(cudaEventElapsedTime(&tr, e0, e2));
            RT(cudaEventElapsedTime(&tt, e0, e3));
            if (rep) printf("%-28s copy %.3f ms (%.0f GB/s)  rand done %.3f ms  total %.3f ms\n", tag, tc,
                            2.0 * n4 * 16 / tc / 1e6, tr, tt);
        }
    };
    const int nsm = all.sm.smCount;
    // alone, whole GPU
    run(s0, nsm * 4, s0, nsm * 8, "serial, whole GPU");
    cudaStream_t s1;
    RT(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    run(s0, nsm * 4, s1, nsm * 8, "two plain streams");
    run((cudaStream_t)sa, ga.sm.smCount * 4, (cudaStream_t)sb, rest.sm.smCount * 8, "green: copy A | rand B");
    run((cudaStream_t)sb, rest.sm.smCount * 4, (cudaStream_t)sa, ga.sm.smCount * 8, "green: copy B | rand A");
    printf("ok\n");
    return 0;
}
