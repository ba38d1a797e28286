// gather.cu -- classify + feature gather (Alg.2 l.2-5, l.10-11, l.21-22).
//
// One warp per node of F_L, every instance of the window at once:
//   local  (u in V_p^l)           -> row of the partition's own table   (l.10)
//   hit    (u in V_p^h, in BUF)   -> BUF row of its slot                 (l.11)
//   miss   (u in V_p^h, not BUF)  -> row of the OWNER's table, read over
//                                    NVLink peer memory when the owner is
//                                    another GPU (the RPC of l.22, fused into
//                                    the gather: no request/response exchange)
// The class is a range test on the node's local rank plus one slot_of load
// (the compact O(|V_p^h|) S_A of P:228, indexed directly instead of by binary
// search).  Hits set bit w of the slot's hit mask (decay bookkeeping, l.6-9);
// misses add 1 to S_A (l.21).  Every add is +1.0f, so the result does not
// depend on the order of the atomics (bit-exact vs. sequential steps).
// Rows move as 16-byte vectors, coalesced per warp; X stores stream past L2.
#include "launch.h"

namespace mgnn {

constexpr int kGThreads = 256;

__device__ __forceinline__ float4 ld_row(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

__global__ void __launch_bounds__(kGThreads) k_gather(WinDev W, WorldDev G) {
    __shared__ unsigned long long cnt_sh[3];
    const int m = blockIdx.y;
    const int lp = m / W.n_steps, w = m % W.n_steps;
    const PartDev& pd = W.parts[lp];
    if (threadIdx.x < 3) cnt_sh[threadIdx.x] = 0;
    __syncthreads();
    const int64_t U = W.hop_size[(int64_t)m * (kMaxLayers + 1) + W.L];
    const int lane = threadIdx.x & 31;
    const int pitch = W.pitch;
    const int64_t nwarps = (int64_t)gridDim.x * (kGThreads / 32);
    const int32_t* fr = W.fr_rank + (int64_t)m * W.ucap;
    int32_t* fgid = W.fr_gid + (int64_t)m * W.ucap;
    float* X = W.X + (int64_t)m * W.ucap * pitch;
    const int64_t h_below = pd.h_below, n_local = pd.n_local, lo = pd.lo;
    const unsigned long long wbit = 1ull << w;
    unsigned n_loc = 0, n_hit = 0, n_miss = 0;
    for (int64_t f = (int64_t)blockIdx.x * (kGThreads / 32) + (threadIdx.x >> 5); f < U; f += nwarps) {
        const int64_t r = fr[f];
        const float* src;
        int32_t gid;
        if (r >= h_below && r < h_below + n_local) {
            gid = (int32_t)(lo + (r - h_below));
            src = pd.table + (r - h_below) * pitch;
            ++n_loc;
        } else {
            const int64_t h = r < h_below ? r : r - n_local;
            gid = pd.halo_ids[h];
            const int32_t s = pd.slot_of[h];
            if (s >= 0) {
                src = pd.rows + (int64_t)s * pitch;
                if (lane == 0) atomicOr(&pd.hitmask[s], wbit);
                ++n_hit;
            } else {
                const int q = owner_of(G.bounds, G.n_parts, gid);
                src = G.tables[q] + ((int64_t)gid - G.bounds[q]) * pitch;
                if (lane == 0) atomicAdd(&pd.sa[h], 1.0f);
                ++n_miss;
            }
        }
        if (lane == 0) fgid[f] = gid;
        float* dst = X + f * pitch;
        for (int c = lane * 4; c < pitch; c += 128) __stcs(reinterpret_cast<float4*>(dst + c), ld_row(src + c));
    }
    if (lane == 0) {
        if (n_loc) atomicAdd(&cnt_sh[0], n_loc);
        if (n_hit) atomicAdd(&cnt_sh[1], n_hit);
        if (n_miss) atomicAdd(&cnt_sh[2], n_miss);
    }
    __syncthreads();
    long long* cn = W.counts + (int64_t)m * 8;
    if (threadIdx.x == 0) {
        if (cnt_sh[0]) atomicAdd((unsigned long long*)&cn[1], cnt_sh[0]);
        if (cnt_sh[1]) atomicAdd((unsigned long long*)&cn[2], cnt_sh[1]);
        if (cnt_sh[2]) {
            atomicAdd((unsigned long long*)&cn[3], cnt_sh[2]);
            atomicAdd((unsigned long long*)&cn[6], cnt_sh[2]);
        }
        const unsigned long long rows = cnt_sh[0] + cnt_sh[1] + cnt_sh[2];
        if (rows && W.gathered_rows) atomicAdd((unsigned long long*)W.gathered_rows, rows);
        if (blockIdx.x == 0) cn[0] = U;
    }
}

void launch_gather(const WinDev& w, const WorldDev& world, cudaStream_t s) {
    int64_t target = (148 * 8 + w.n_inst - 1) / w.n_inst;   // ~8 resident 256-thread blocks per SM in total
    int64_t need = (w.ucap + 7) / 8;
    unsigned gx = (unsigned)(need < target ? need : target);
    if (gx < 1) gx = 1;
    dim3 grid(gx, w.n_inst);
    k_gather<<<grid, kGThreads, 0, s>>>(w, world);
    count_launches(1, __func__);
}

}  // namespace mgnn
