// load.cu -- partition build on the device (§8(a) A1).
//
// V_p^h = sorted unique non-local neighbours of V_p^l: mark them in a bitmap
// over global ids, then a popcount scan emits them in ascending order.
// deg_in[h] = occurrences of h among the local rows (R#10).  The CSR columns
// are rewritten as LOCAL RANKS: the position of the neighbour in the sorted
// union V_p^h ∪ V_p^l, so that ascending rank == ascending global id, the
// local/halo test is a range check and the halo index is rank arithmetic.
// Feature rows are synthesised with Philox (R#4) into a pitched table.
#include "launch.h"

namespace mgnn {

constexpr int kLThreads = 256;

static inline unsigned lblocks(int64_t n) {
    int64_t b = (n + kLThreads - 1) / kLThreads;
    if (b > (int64_t)num_sms() * 16) b = (int64_t)num_sms() * 16;
    return (unsigned)(b < 1 ? 1 : b);
}

__global__ void k_mark_halo(const int32_t* __restrict__ cols, int64_t nnz, int64_t lo, int64_t hi,
                            uint32_t* __restrict__ bm) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = cols[e];
        if (c < lo || c >= hi) atomicOr(&bm[c >> 5], 1u << (c & 31));
    }
}

void launch_mark_halo(const int32_t* cols, int64_t nnz, int64_t lo, int64_t hi, uint32_t* bm, cudaStream_t s) {
    if (nnz < 1) return;
    k_mark_halo<<<lblocks(nnz), kLThreads, 0, s>>>(cols, nnz, lo, hi, bm);
    count_launches(1, __func__, s);
}

// Bitmap -> ascending ids (decoupled look-back over popcounts, 4 words per thread).
__global__ void __launch_bounds__(kLThreads) k_bitmap_to_ids(const uint32_t* __restrict__ bm, int64_t nwords,
                                                             int32_t* __restrict__ out, long long* out_n, Scratch sc) {
    __shared__ long long sm[8];
    __shared__ int tslot;
    __shared__ long long prefix_sh;
    const int64_t tile_words = kLThreads * 4;
    const int64_t ntiles = (nwords + tile_words - 1) / tile_words;
    const int tile = claim_tile(sc.tilectr, &tslot);
    if (tile >= ntiles) return;
    const int64_t w0 = (int64_t)tile * tile_words + (int64_t)threadIdx.x * 4;
    uint32_t b[4];
    long long cnt = 0;
    for (int i = 0; i < 4; ++i) {
        b[i] = (w0 + i < nwords) ? bm[w0 + i] : 0u;
        cnt += __popc(b[i]);
    }
    long long agg;
    long long excl = block_excl_scan256(cnt, sm, &agg);
    if (threadIdx.x < 32) {
            const unsigned long long pv = lookback_exclusive(sc.status, tile, (unsigned long long)agg);
            if (threadIdx.x == 0) prefix_sh = (long long)pv;
        }
    __syncthreads();
    int64_t pos = prefix_sh + excl;
    for (int i = 0; i < 4; ++i) {
        uint32_t x = b[i];
        while (x) {
            const int bi = __ffs(x) - 1;
            x &= x - 1;
            out[pos++] = (int32_t)((w0 + i) * 32 + bi);
        }
    }
    if (tile == ntiles - 1 && threadIdx.x == 0) *out_n = prefix_sh + agg;
}

void launch_bitmap_to_ids(const uint32_t* bm, int64_t nwords, int32_t* out, long long* out_n, Scratch sc,
                          cudaStream_t s) {
    int64_t tiles = (nwords + kLThreads * 4 - 1) / (kLThreads * 4);
    if (tiles < 1) tiles = 1;
    k_bitmap_to_ids<<<(unsigned)tiles, kLThreads, 0, s>>>(bm, nwords, out, out_n, sc);
    count_launches(1, __func__, s);
}

__global__ void k_lower_bound(const int32_t* __restrict__ arr, int64_t n, int64_t v, long long* out) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (arr[mid] < v) lo = mid + 1; else hi = mid;
    }
    *out = lo;
}

void launch_lower_bound(const int32_t* arr, int64_t n, int64_t v, long long* out, cudaStream_t s) {
    k_lower_bound<<<1, 1, 0, s>>>(arr, n, v, out);
    count_launches(1, __func__, s);
}

__global__ void k_halo_index(const int32_t* __restrict__ halo, int64_t n_h, int32_t* __restrict__ gmap) {
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < n_h; h += (int64_t)gridDim.x * blockDim.x)
        gmap[halo[h]] = (int32_t)h;
}

void launch_halo_index(const int32_t* halo, int64_t n_h, int32_t* gmap, cudaStream_t s) {
    if (n_h < 1) return;
    k_halo_index<<<lblocks(n_h), kLThreads, 0, s>>>(halo, n_h, gmap);
    count_launches(1, __func__, s);
}

// NEXT-1 remote expansion: the global CSR in global ids, assembled from the hosted partitions
// (rows of partition p at [lo_p, hi_p), its edges at base_p = sum of the earlier partitions' nnz).
__global__ void k_gcsr_rows(const int64_t* __restrict__ indptr, int64_t n_local, int64_t lo, int64_t base,
                            int64_t* __restrict__ g_indptr) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n_local; r += (int64_t)gridDim.x * blockDim.x)
        g_indptr[lo + r] = base + indptr[r];
}
__global__ void k_gcsr_cols(const PartDev* __restrict__ pdp, int64_t nnz, int64_t base, int32_t* __restrict__ g_cols) {
    const PartDev& pd = *pdp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
        g_cols[base + e] = rank_to_gid(pd, pd.cols_rank[e]);
}

void launch_global_csr(const PartDev* pd_dev, const int64_t* indptr, int64_t n_local, int64_t lo, int64_t nnz,
                       int64_t base, int64_t* g_indptr, int32_t* g_cols, cudaStream_t s) {
    k_gcsr_rows<<<lblocks(n_local + 1), kLThreads, 0, s>>>(indptr, n_local, lo, base, g_indptr);
    if (nnz > 0) k_gcsr_cols<<<lblocks(nnz), kLThreads, 0, s>>>(pd_dev, nnz, base, g_cols);
    count_launches(2, __func__, s);
}

__global__ void k_deg_rank(const int32_t* __restrict__ cols, int64_t nnz, int64_t lo, int64_t n_local, int64_t h_below,
                           const int32_t* __restrict__ gmap, int32_t* __restrict__ deg_in,
                           int32_t* __restrict__ cols_rank) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = cols[e];
        int64_t r;
        if (c >= lo && c < lo + n_local) {
            r = h_below + (c - lo);
        } else {
            const int32_t h = gmap[c];
            atomicAdd(&deg_in[h], 1);
            r = h < h_below ? h : h + n_local;
        }
        cols_rank[e] = (int32_t)r;
    }
}

void launch_deg_rank(const int32_t* cols, int64_t nnz, int64_t lo, int64_t n_local, int64_t h_below,
                     const int32_t* gmap, int32_t* deg_in, int32_t* cols_rank, cudaStream_t s) {
    if (nnz < 1) return;
    k_deg_rank<<<lblocks(nnz), kLThreads, 0, s>>>(cols, nnz, lo, n_local, h_below, gmap, deg_in, cols_rank);
    count_launches(1, __func__, s);
}

// Feature value (R#4): ((Philox(node, c/4, 0, 3; feat_seed).c%4 >> 8) - 2^23) * 2^-23, exact in fp32.
__global__ void k_features(float* __restrict__ table, int64_t lo, int64_t n_rows, int32_t dim, int32_t pitch,
                           uint32_t k0, uint32_t k1) {
    const int64_t q = pitch / 4;
    const int64_t total = n_rows * q;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / q, c4 = i - row * q;
        const u4 o = philox4x32_10(u4{(uint32_t)(lo + row), (uint32_t)c4, 0u, kStreamFeature}, k0, k1);
        const uint32_t v[4] = {o.x, o.y, o.z, o.w};
        float4 out;
        float* po = &out.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t col = c4 * 4 + j;
            const int32_t iv = (int32_t)(v[j] >> 8) - (1 << 23);
            po[j] = col < dim ? __fmul_rn(__int2float_rn(iv), 1.1920928955078125e-07f) : 0.0f;
        }
        reinterpret_cast<float4*>(table + row * pitch)[c4] = out;
    }
}

void launch_features(float* table, int64_t lo, int64_t n_rows, int32_t dim, int32_t pitch, uint64_t feat_seed,
                     cudaStream_t s) {
    if (n_rows < 1 || pitch < 4) return;
    k_features<<<lblocks(n_rows * (pitch / 4)), kLThreads, 0, s>>>(table, lo, n_rows, dim, pitch, (uint32_t)feat_seed,
                                                                   (uint32_t)(feat_seed >> 32));
    count_launches(1, __func__, s);
}

}  // namespace mgnn
