// g4_probe.cu -- standalone probe of the TMA row gather (cp.async.bulk.tensor.2d ... tile::gather4) on
// sm_100a (development tool): 4 arbitrary rows of a [rows][pitch] fp32 table into shared memory in one
// instruction, box = {cols, 1}.  Checks the data and which shared-memory destination offsets work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 g4_probe.cu -lcuda -o g4_probe && ./g4_probe [cols]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int cols, int off, const int* rows, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    unsigned char* dst = sm + off;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(4 * cols * 4)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(s32(dst)),
            "l"(&map), "r"(s32(&bar)), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3])
            : "memory");
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}\n" ::"r"(
                s32(&bar))
            : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * cols; i += blockDim.x) out[i] = reinterpret_cast<const float*>(dst)[i];
}

int main(int argc, char** argv) {
    const int cols = argc > 1 ? atoi(argv[1]) : 100, pitch = (cols + 3) / 4 * 4, n = 1000;
    std::vector<float> h((size_t)n * pitch);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < pitch; ++c) h[(size_t)r * pitch + c] = r * 1000.0f + c;
    float *d, *out;
    int* rows;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&out, 4 * pitch * 4);
    cudaMalloc(&rows, 16);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int want[4] = {7, 3, 999, 500};
    cudaMemcpy(rows, want, 16, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box[2] = {(cuuint32_t)cols, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult rr = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode cols=%d pitch=%d: %d\n", cols, pitch, (int)rr);
    if (rr != CUDA_SUCCESS) return 1;
    const int offs[] = {0, 128, 1664, 1600, 16};
    for (int off : offs) {
        cudaMemset(out, 0, 4 * pitch * 4);
        probe<<<1, 128, 16384>>>(map, cols, off, rows, out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("off %d: %s\n", off, cudaGetErrorString(e));
            return 2;
        }
        std::vector<float> o(4 * cols);
        cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int j = 0; j < 4; ++j)
            for (int c = 0; c < cols; ++c) bad += o[(size_t)j * cols + c] != want[j] * 1000.0f + c;
        printf("off %d: %s (%d bad of %d; rows packed at %d floats)\n", off, bad ? "WRONG" : "ok", bad, 4 * cols, cols);
    }
    return 0;
}
