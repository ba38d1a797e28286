// umma_probe.cu -- standalone probe of tcgen05.mma kind::tf32 operand layouts (development tool).
// D[128 x 128] = A^T B with A, B stored "row = K" (MN contiguous), K = 64, SWIZZLE_128B,
// 32-column atoms of 64 rows (8 KB) side by side.  Runs several descriptor variants and prints
// the max error against a CPU reference for each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2410_22697_b200/csrc umma_probe.cu -o probe
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2410_22697_b200/csrc/common.cuh"
#include "../paper_2410_22697_b200/csrc/umma.cuh"

using namespace mgnn;

constexpr int K = 64, MN = 128;

__global__ void probe(const float* A, const float* B, float* D, int variant) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    unsigned char* base = dsm + ((1024u - (su32(dsm) & 1023u)) & 1023u);
    unsigned char* sa = base;
    unsigned char* sb = base + 4 * K * 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // fill: element (k, c) of a [K][MN] row-major matrix -> atom c/32, row k, 16 B unit (c%32)/4 ^ (k%8)
    for (int i = threadIdx.x; i < K * MN; i += blockDim.x) {
        const int k = i / MN, c = i % MN;
        const int atom = c / 32, u = (c % 32) / 4, e = c % 4;
        const size_t off = (size_t)atom * K * 128 + (size_t)k * 128 + ((u ^ (k & 7)) * 16) + e * 4;
        *(float*)(sa + off) = A[i];
        *(float*)(sb + off) = B[i];
    }
    // K-major copies: element (k, c) -> chunk k/32 (M rows x 128 B), row c, unit (k%32)/4 ^ (c%8)
    unsigned char* ka = base + 8 * K * 128;
    unsigned char* kb = ka + 2 * MN * 128;
    for (int i = threadIdx.x; i < K * MN; i += blockDim.x) {
        const int k = i / MN, c = i % MN;
        const int ch = k / 32, u = (k % 32) / 4, e = k % 4;
        const size_t off = (size_t)ch * MN * 128 + (size_t)c * 128 + ((u ^ (c & 7)) * 16) + e * 4;
        *(float*)(ka + off) = A[i];
        *(float*)(kb + off) = B[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (lane == 0) mb_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
        tmem_alloc(&tm, 128);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = tm;
    if (threadIdx.x == 0) {
        uint32_t amaj = 1, bmaj = 1, lbo = K * 128, sbo = 1024;
        if (variant == 1) { lbo = 1024; sbo = K * 128; }          // swapped
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amaj << 15) | (bmaj << 16) | ((MN >> 3) << 17) |
                               ((128u >> 4) << 24);
        for (int kk = 0; kk < K / 8; ++kk) {
            const uint32_t a0 = su32(sa) + kk * 1024, b0 = su32(sb) + kk * 1024;
            uint64_t da = (uint64_t)((a0 >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                          ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
            uint64_t db = (uint64_t)((b0 >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
                          ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
            if (variant >= 3) {   // K-major: chunk kk/4, 32-byte step kk%4 inside the 128-byte row
                const uint32_t ka0 = su32(ka) + (kk / 4) * MN * 128 + (kk % 4) * 32;
                const uint32_t kb0 = su32(kb) + (kk / 4) * MN * 128 + (kk % 4) * 32;
                const uint64_t kd = (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
                db = kd | ((kb0 >> 4) & 0x3FFF);
                if (variant == 3) da = kd | ((ka0 >> 4) & 0x3FFF);
            }
            uint32_t id2 = idesc;
            if (variant == 3) id2 = idesc & ~((1u << 15) | (1u << 16));
            if (variant == 4) id2 = idesc & ~(1u << 16);
            if (variant == 2) {   // per-k advance inside a 1 KB group: 8 rows x 128 B, try 128-byte steps
                da = (da & ~0x3FFFull) | (((su32(sa) + kk * 8 * 128) >> 4) & 0x3FFF);
                db = (db & ~0x3FFFull) | (((su32(sb) + kk * 8 * 128) >> 4) & 0x3FFF);
            }
            mma_tf32(t, da, db, id2, kk > 0 ? 1u : 0u);
        }
        mma_commit(&bar);
    }
    __syncwarp();
    mb_wait(&bar, 0);
    tc_fence_after();
    const int row = warp * 32 + lane;
    for (int c = 0; c < MN; c += 8) {
        float v[8];
        tmem_ld8(t + ((uint32_t)(warp * 32) << 16) + c, v);
        for (int i = 0; i < 8; ++i) D[row * MN + c + i] = v[i];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(t, 128);
}

int main() {
    std::vector<float> A(K * MN), B(K * MN), D(MN * MN), R(MN * MN);
    srand(1);
    for (auto& x : A) x = (float)(rand() % 17 - 8) / 8.0f;
    for (auto& x : B) x = (float)(rand() % 13 - 6) / 4.0f;
    for (int m = 0; m < MN; ++m)
        for (int n = 0; n < MN; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[k * MN + m] * B[k * MN + n];
            R[m * MN + n] = (float)s;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = 1024 + 2 * 4 * K * 128 + 4 * MN * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int v = 0; v < 5; ++v) {
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128, smem>>>(dA, dB, dD, v);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double mx = 0, mr = 0;
        for (int i = 0; i < MN * MN; ++i) {
            mx = fmax(mx, fabs(D[i] - R[i]));
            mr = fmax(mr, fabs(R[i]));
        }
        printf("variant %d: %s max|D-R| = %g (max|R| = %g) D[0..3] = %g %g %g %g R = %g %g %g %g\n", v,
               cudaGetErrorString(e), mx, mr, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
    }
    return 0;
}
