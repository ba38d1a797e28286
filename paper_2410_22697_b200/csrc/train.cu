// train.cu -- backward of the GraphSAGE-mean consumer: one DDP training step per minibatch
// (Alg.1 l.6-8: every trainer computes the forward
// pass and the backward pass of its minibatch, gradients are all-reduced across trainers,
// and the optimizer updates the replicated model).  The forward is k_sage_layer (sage.cu)
// with the neighbour means kept; here:
//   k_xent      : softmax cross-entropy of the seeds' logits -> dlogits, loss, bias gradient
//   k_relu_mask : dZ = dH * [H > 0] (hidden layers) + bias gradient
//   k_zero_rows : clears a gradient buffer's live rows
//   k_wgrad     : dW[o][c] += sum_rows dZ[r][o] * [H | mean][r][c]  -- tcgen05 kind::tf32, the
//                 row-major operands transposed into K-major shared-memory tiles by the CTA's
//                 threads, split-K over CTAs, partial tiles reduced with red.global.add.v4.f32
//   k_dgrad     : [dZ W_self | dZ W_neigh] per 128-row tile (tcgen05, K-major, transposed
//                 weights); the epilogue stores dZ W_self into dH and dZ W_neigh / deg into dmean
//   k_scatter   : dmean rows added to the sampled neighbours' dH rows (warp per row, atomics)
//   k_sgd_layers, k_transpose : the optimizer step and the dgrad operand layout
// Gradient reductions use fp32 atomics (order-dependent rounding; the parity bound of the
// training step is stated in DESIGN.md §7.2).
#include <algorithm>

#include "launch.h"
#include "umma.cuh"

namespace mgnn {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ int inst_of(int k, int inst0, int inst_step) { return inst0 + k * inst_step; }

// ------------------------------------------------------------------ loss
// warp per seed row: softmax over the C logits, cross-entropy against the seed's label
__global__ void __launch_bounds__(kT) k_xent(XentArgs a) {
    pdl_enter();
    __shared__ float s_db[256];
    __shared__ float s_loss;
    const int k = blockIdx.y;
    const int m = inst_of(k, a.inst0, a.inst_step);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int c = threadIdx.x; c < 256; c += kT) s_db[c] = 0.0f;
    if (threadIdx.x == 0) s_loss = 0.0f;
    __syncthreads();
    const int64_t n0 = a.hop_size[(int64_t)m * (kMaxLayers + 1)];
    const int C = a.n_classes;
    const float inv = a.scale / (float)(n0 > 0 ? n0 : 1);
    for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < a.rows; i += (int64_t)gridDim.x * 8) {
        const float* z = a.logits + ((int64_t)m * a.rows + i) * a.pitch;
        float* dz = a.dlogits + ((int64_t)m * a.rows + i) * a.pitch;
        if (i >= n0) {
            for (int c = lane; c < a.pitch; c += 32) dz[c] = 0.0f;
            continue;
        }
        const int label = a.labels[a.frontier[(int64_t)m * a.ucap + i]];
        float mx = -INFINITY;
        for (int c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
        float se = 0.0f;
        for (int c = lane; c < C; c += 32) se += expf(z[c] - mx);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(kFull, se, o);
        const float lse = logf(se);
        for (int c = lane; c < a.pitch; c += 32) {
            float g = 0.0f;
            if (c < C) {
                const float p = expf(z[c] - mx - lse);
                g = (p - (c == label ? 1.0f : 0.0f)) * inv;
                atomicAdd(&s_db[c], g);
            }
            dz[c] = g;
        }
        if (lane == 0) atomicAdd(&s_loss, (mx + lse - z[label]) * inv);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += kT)
        if (s_db[c] != 0.0f) atomicAdd(&a.db[c], s_db[c]);
    if (threadIdx.x == 0 && s_loss != 0.0f) atomicAdd(a.loss, s_loss);
}

// ------------------------------------------------------------------ ReLU backward + bias gradient
__global__ void __launch_bounds__(kT) k_relu_mask(MaskArgs a) {
    pdl_enter();
    __shared__ float s_db[256];
    const int k = blockIdx.y;
    const int m = inst_of(k, a.inst0, a.inst_step);
    for (int c = threadIdx.x; c < 256; c += kT) s_db[c] = 0.0f;
    __syncthreads();
    const int64_t n = a.hop_size[(int64_t)m * (kMaxLayers + 1) + a.hop];
    const int64_t n64 = (n + 63) / 64 * 64;
    const int q = a.ncols / 4;
    if (kT % q == 0) {
        // fixed column per thread (kT / q rows per block step): no per-element 64-bit division, and the
        // bias gradient accumulates in registers with one shared atomic per thread and column
        const int c4 = threadIdx.x % q;
        const int rpi = kT / q;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t r = (int64_t)blockIdx.x * rpi + threadIdx.x / q; r < n64; r += (int64_t)gridDim.x * rpi) {
            float4* dz = reinterpret_cast<float4*>(a.dz + ((int64_t)m * a.rows + r) * a.pitch) + c4;
            if (r >= n) {
                *dz = make_float4(0.f, 0.f, 0.f, 0.f);
                continue;
            }
            const float4 h = *(reinterpret_cast<const float4*>(a.h + ((int64_t)m * a.h_rows + r) * a.h_pitch) + c4);
            float4 g = *dz;
            g.x = h.x > 0.0f ? g.x : 0.0f;
            g.y = h.y > 0.0f ? g.y : 0.0f;
            g.z = h.z > 0.0f ? g.z : 0.0f;
            g.w = h.w > 0.0f ? g.w : 0.0f;
            *dz = g;
            acc.x += g.x;
            acc.y += g.y;
            acc.z += g.z;
            acc.w += g.w;
        }
        if (acc.x != 0.0f) atomicAdd(&s_db[4 * c4], acc.x);
        if (acc.y != 0.0f) atomicAdd(&s_db[4 * c4 + 1], acc.y);
        if (acc.z != 0.0f) atomicAdd(&s_db[4 * c4 + 2], acc.z);
        if (acc.w != 0.0f) atomicAdd(&s_db[4 * c4 + 3], acc.w);
        __syncthreads();
        for (int c = threadIdx.x; c < a.ncols; c += kT)
            if (s_db[c] != 0.0f) atomicAdd(&a.db[c], s_db[c]);
        return;
    }
    for (int64_t e = (int64_t)blockIdx.x * kT + threadIdx.x; e < n64 * q; e += (int64_t)gridDim.x * kT) {
        const int64_t r = e / q;
        const int c4 = (int)(e - r * q);
        float4* dz = reinterpret_cast<float4*>(a.dz + ((int64_t)m * a.rows + r) * a.pitch) + c4;
        if (r >= n) {
            *dz = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        const float4 h = *(reinterpret_cast<const float4*>(a.h + ((int64_t)m * a.h_rows + r) * a.h_pitch) + c4);
        float4 g = *dz;
        g.x = h.x > 0.0f ? g.x : 0.0f;
        g.y = h.y > 0.0f ? g.y : 0.0f;
        g.z = h.z > 0.0f ? g.z : 0.0f;
        g.w = h.w > 0.0f ? g.w : 0.0f;
        *dz = g;
        if (g.x != 0.0f) atomicAdd(&s_db[4 * c4], g.x);
        if (g.y != 0.0f) atomicAdd(&s_db[4 * c4 + 1], g.y);
        if (g.z != 0.0f) atomicAdd(&s_db[4 * c4 + 2], g.z);
        if (g.w != 0.0f) atomicAdd(&s_db[4 * c4 + 3], g.w);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < a.ncols; c += kT)
        if (s_db[c] != 0.0f) atomicAdd(&a.db[c], s_db[c]);
}

__global__ void __launch_bounds__(kT) k_zero_rows(ZeroRowsArgs a) {
    pdl_enter();
    const int m = inst_of(blockIdx.y, a.inst0, a.inst_step);
    const int64_t n = a.hop_size[(int64_t)m * (kMaxLayers + 1) + a.hop];
    const int64_t n64 = (n + 63) / 64 * 64;
    const int64_t q = a.pitch / 4;
    float4* b = reinterpret_cast<float4*>(a.buf + (int64_t)m * a.rows * a.pitch);
    for (int64_t e = (int64_t)blockIdx.x * kT + threadIdx.x; e < n64 * q; e += (int64_t)gridDim.x * kT)
        b[e] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ------------------------------------------------------------------ weight gradient (tcgen05)
// dW (M = output features o, N = input columns c) = sum over rows r (the K dimension) of
// dZ[r][o] * In[r][c].  Both operands are stored row-major with K = rows, i.e. MN-major, which
// kind::tf32 does not accept (measured: the MMA writes nothing, tools/umma_probe.cu), so the
// CTA's threads load each 64-row chunk and store it TRANSPOSED into the K-major SWIZZLE_128B
// layout (operand row = o or c, 128-byte rows of 32 consecutive K values, 16-byte unit u of
// row x at u ^ (x % 8)); rows past |F_h| and columns past the data read as zero.
// 3xTF32 (SPLIT, DESIGN R#29): the threads split every value into hi (low 13 mantissa bits cleared) and
// lo = v - hi while transposing, so a stage holds A_hi | A_lo | B_hi | B_lo of a 32-row chunk (the same
// 64 KB as the TF32 stage's A | B of 64 rows), and each K step issues a_lo b_hi + a_hi b_lo + a_hi b_hi.
constexpr int kWRegion = 128 * 128;              // 128 operand rows x 32 K values (fp32): 16 KB
constexpr int kWStage = 4 * kWRegion;            // 4 regions: A and B x 2 K-regions, or A/B x hi/lo
constexpr int kWMaxInst = 256;

__device__ __forceinline__ float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

constexpr int kWThreads = 1024;                   // 8 threads per operand row: 8x the loads in flight
template <bool SPLIT>
__global__ void __launch_bounds__(kWThreads, 1) k_wgrad(WgradArgs a) {
    constexpr int kWRows = SPLIT ? 32 : 64;      // K rows per chunk
    constexpr int kNReg = kWRows / 32;           // K-regions per operand part
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) uint64_t bar_empty[2], bar_done;
    __shared__ uint32_t tmem_sh;
    __shared__ int32_t pref[kWMaxInst + 1];
    unsigned char* base = dsm + ((1024u - (su32(dsm) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_nt = (2 * a.kp) / 128, n_mt = (a.npad + 127) / 128;
    const int tile = blockIdx.x % (n_mt * n_nt), ks = blockIdx.x / (n_mt * n_nt);
    const int mt = tile / n_nt, nt = tile % n_nt;
    if (warp == 0) {
        if (lane == 0) {
            mb_init(&bar_empty[0], 1);
            mb_init(&bar_empty[1], 1);
            mb_init(&bar_done, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        tmem_alloc(&tmem_sh, 128);
    }
    pdl_enter();
    if (warp == 1) {     // chunk prefix over the step's instances: ceil(|F_h| / 64) chunks each
        int32_t run = 0;
        if (lane == 0) pref[0] = 0;
        for (int k0 = 0; k0 < a.n_inst; k0 += 32) {
            const int k = k0 + lane;
            int32_t t = 0;
            if (k < a.n_inst)
                t = (int32_t)((a.hop_size[(int64_t)inst_of(k, a.inst0, a.inst_step) * (kMaxLayers + 1) + a.hop] + kWRows -
                               1) / kWRows);
            int32_t x = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= o) x += y;
            }
            if (k < a.n_inst) pref[k + 1] = run + x;
            run += __shfl_sync(kFull, x, 31);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_sh;
    const int total = pref[a.n_inst];
    const int c_lo = (int)(((int64_t)total * ks) / a.ksplit), c_hi = (int)(((int64_t)total * (ks + 1)) / a.ksplit);
    const bool neigh = nt * 128 >= a.kp;               // columns of the mean rows
    const int col0 = neigh ? nt * 128 - a.kp : nt * 128;
    const float* src_b = neigh ? a.mean : a.h_in;
    const int64_t b_rows = neigh ? a.mean_rows : a.in_rows, b_pitch = neigh ? a.mean_pitch : a.in_pitch;
    const int b_cols = neigh ? a.mean_cols : a.in_cols;  // columns carrying data
    // K-major tf32, M = 128, N = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    // thread = (operand row x, rows q*8 .. q*8+7 of the chunk).  Chunk c+1's loads are issued before
    // chunk c's transposed stores (ping-pong registers, no copies), so they are in flight across the
    // barrier and the MMA issue; a full chunk loads without per-row predicates (ncu: the round-1 loop
    // spent ~400 instructions per thread per chunk on 64-bit row addressing and a per-chunk search).
    const int x = threadIdx.x & 127, q = threadIdx.x >> 7;
    constexpr int kQ = kWRows / 4 / (kWThreads / 128);    // K groups of 4 per thread
    constexpr int kR = kQ * 4;                            // rows per thread
    const int o_row = mt * 128 + x, cc = col0 + x;
    const bool oka = o_row < a.npad, okb = cc < b_cols;
    const int sa_p = (int)a.dz_pitch, sb_p = (int)b_pitch;
    int lo = 0;                                           // instance of the chunk (chunks ascend)
    auto load_chunk = [&](int c, float (&va)[kQ][4], float (&vb)[kQ][4]) {
        while (lo + 1 < a.n_inst && pref[lo + 1] <= c) ++lo;
        const int m = inst_of(lo, a.inst0, a.inst_step);
        const int64_t r0 = (int64_t)(c - pref[lo]) * kWRows + q * kR;
        const int nk = (int)min(a.hop_size[(int64_t)m * (kMaxLayers + 1) + a.hop] - r0, (int64_t)kR);
        const float* pa = a.dz + ((int64_t)m * a.dz_rows + r0) * a.dz_pitch + o_row;
        const float* pb = src_b + ((int64_t)m * b_rows + r0) * b_pitch + cc;
        if (nk >= kR) {
#pragma unroll
            for (int j = 0; j < kR; ++j) {
                va[j >> 2][j & 3] = oka ? __ldg(pa + j * sa_p) : 0.0f;
                vb[j >> 2][j & 3] = okb ? __ldg(pb + j * sb_p) : 0.0f;
            }
        } else {                                          // the instance's last chunk: rows past |F_h| are 0
#pragma unroll
            for (int j = 0; j < kR; ++j) {
                va[j >> 2][j & 3] = (oka && j < nk) ? __ldg(pa + j * sa_p) : 0.0f;
                vb[j >> 2][j & 3] = (okb && j < nk) ? __ldg(pb + j * sb_p) : 0.0f;
            }
        }
    };
    auto step = [&](int c, float (&ca)[kQ][4], float (&cb)[kQ][4], float (&na)[kQ][4], float (&nb)[kQ][4]) {
        const int i = c - c_lo, st = i & 1;
        if (i >= 2) mb_wait(&bar_empty[st], ((i >> 1) - 1) & 1);   // MMAs of chunk c-2 read this stage
        if (c + 1 < c_hi) load_chunk(c + 1, na, nb);
        unsigned char* sa = base + st * kWStage;                      // A (hi)
        unsigned char* sb = sa + (SPLIT ? 2 : 1) * kNReg * kWRegion;   // B (hi)
#pragma unroll
        for (int g = 0; g < kQ; ++g) {
            const int k4 = q * kQ + g;
            const int reg = k4 >> 3, u = k4 & 7;            // 32 K values per region, 8 units of 4
            const uint32_t off = (uint32_t)(reg * kWRegion + x * 128 + ((u ^ (x & 7)) << 4));
            if (SPLIT) {
                float4 ah, bh;
                ah.x = tf32_hi(ca[g][0]); ah.y = tf32_hi(ca[g][1]); ah.z = tf32_hi(ca[g][2]); ah.w = tf32_hi(ca[g][3]);
                bh.x = tf32_hi(cb[g][0]); bh.y = tf32_hi(cb[g][1]); bh.z = tf32_hi(cb[g][2]); bh.w = tf32_hi(cb[g][3]);
                *reinterpret_cast<float4*>(sa + off) = ah;
                *reinterpret_cast<float4*>(sb + off) = bh;
                *reinterpret_cast<float4*>(sa + kNReg * kWRegion + off) =
                    make_float4(__fsub_rn(ca[g][0], ah.x), __fsub_rn(ca[g][1], ah.y), __fsub_rn(ca[g][2], ah.z),
                                __fsub_rn(ca[g][3], ah.w));
                *reinterpret_cast<float4*>(sb + kNReg * kWRegion + off) =
                    make_float4(__fsub_rn(cb[g][0], bh.x), __fsub_rn(cb[g][1], bh.y), __fsub_rn(cb[g][2], bh.z),
                                __fsub_rn(cb[g][3], bh.w));
            } else {
                *reinterpret_cast<float4*>(sa + off) = make_float4(ca[g][0], ca[g][1], ca[g][2], ca[g][3]);
                *reinterpret_cast<float4*>(sb + off) = make_float4(cb[g][0], cb[g][1], cb[g][2], cb[g][3]);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        if (threadIdx.x == 0) {
            const uint32_t a0 = su32(sa), b0 = su32(sb);
#pragma unroll
            for (int kk = 0; kk < kWRows / 8; ++kk) {      // UMMA K = 8: region kk/4, 32-byte step kk%4
                const uint32_t ko = (uint32_t)((kk >> 2) * kWRegion + (kk & 3) * 32);
                if (SPLIT) {                                // small terms first
                    const uint32_t lo = (uint32_t)(kNReg * kWRegion);
                    mma_tf32(tmem, sdesc(a0 + lo + ko), sdesc(b0 + ko), idesc, (i > 0 || kk > 0) ? 1u : 0u);
                    mma_tf32(tmem, sdesc(a0 + ko), sdesc(b0 + lo + ko), idesc, 1u);
                    mma_tf32(tmem, sdesc(a0 + ko), sdesc(b0 + ko), idesc, 1u);
                } else {
                    mma_tf32(tmem, sdesc(a0 + ko), sdesc(b0 + ko), idesc, (i > 0 || kk > 0) ? 1u : 0u);
                }
            }
            mma_commit(&bar_empty[st]);
        }
    };
    float ra[2][kQ][4], rb[2][kQ][4];
    if (c_lo < c_hi) load_chunk(c_lo, ra[0], rb[0]);
    for (int c = c_lo; c < c_hi; c += 2) {
        step(c, ra[0], rb[0], ra[1], rb[1]);
        if (c + 1 < c_hi) step(c + 1, ra[1], rb[1], ra[0], rb[0]);
    }
    if (c_lo < c_hi && warp < 4) {                   // TMEM lanes 0-127: warps 0-3 drain the accumulator
        if (threadIdx.x == 0) mma_commit(&bar_done);
        __syncwarp();
        mb_wait(&bar_done, 0);
        tc_fence_after();
        const int o = mt * 128 + warp * 32 + lane;      // TMEM lane = output feature (M)
        float* dst = a.dw + (int64_t)o * (2 * a.kp) + nt * 128;
        for (int c = 0; c < 128; c += 8) {
            float v[8];
            tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
            if (o < a.npad) {
                red_add4(dst + c, v[0], v[1], v[2], v[3]);
                red_add4(dst + c + 4, v[4], v[5], v[6], v[7]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 128);
}

// ------------------------------------------------------------------ input gradient (tcgen05, K-major)
constexpr int kDTile = 128;

// 3xTF32 (SPLIT): warps 1-3 split each landed stage (dZ tile and Wt chunk) into hi in place and lo in a
// second copy of the stage, then arrive on bar_conv; the MMA thread issues a_lo b_hi + a_hi b_lo + a_hi b_hi.
template <bool SPLIT>
__global__ void __launch_bounds__(128, 1)
    k_dgrad(const __grid_constant__ CUtensorMap map_dz, const __grid_constant__ CUtensorMap map_wt, DgradArgs a,
            uint32_t tmem_cols) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) uint64_t bar_full[2], bar_empty[2], bar_done, bar_conv[2];
    __shared__ uint32_t tmem_sh;
    __shared__ int32_t pref[kWMaxInst + 1];
    unsigned char* base = dsm + ((1024u - (su32(dsm) & 1023u)) & 1023u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t a_bytes = kDTile * 128, b_bytes = (uint32_t)(2 * a.kp) * 128;
    const uint32_t plain_bytes = a_bytes + b_bytes;                 // [A | B] (hi in place when SPLIT)
    const uint32_t stage_bytes = SPLIT ? 2 * plain_bytes : plain_bytes;   // + [A_lo | B_lo]
    if (warp == 0) {
        if (lane == 0) {
            mb_init(&bar_full[0], 1);
            mb_init(&bar_full[1], 1);
            mb_init(&bar_conv[0], 3);
            mb_init(&bar_conv[1], 3);
            mb_init(&bar_empty[0], 1);
            mb_init(&bar_empty[1], 1);
            mb_init(&bar_done, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        tmem_alloc(&tmem_sh, tmem_cols);
    }
    pdl_enter();
    if (warp == 1) {
        int32_t run = 0;
        if (lane == 0) pref[0] = 0;
        for (int k0 = 0; k0 < a.n_inst; k0 += 32) {
            const int k = k0 + lane;
            int32_t t = 0;
            if (k < a.n_inst)
                t = (int32_t)((a.hop_size[(int64_t)inst_of(k, a.inst0, a.inst_step) * (kMaxLayers + 1) + a.hop] + kDTile -
                               1) / kDTile);
            int32_t x = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(kFull, x, o);
                if (lane >= o) x += y;
            }
            if (k < a.n_inst) pref[k + 1] = run + x;
            run += __shfl_sync(kFull, x, 31);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_sh;
    const int n_tiles = pref[a.n_inst];
    const int nk = (a.npad_out + 31) / 32;          // K chunks of 32 dZ columns
    // K-major tf32, M = 128, N = kp per half
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(a.kp >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t g = 0;        // chunks issued/consumed by this CTA (both stages alternate)
    uint32_t done_phase = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int lo = 0, hi = a.n_inst;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pref[mid] <= tile) lo = mid; else hi = mid;
        }
        const int m = inst_of(lo, a.inst0, a.inst_step);
        const int64_t row0 = (int64_t)(tile - pref[lo]) * kDTile;
        const int64_t n_dst = a.hop_size[(int64_t)m * (kMaxLayers + 1) + a.hop];
        if (warp == 0 && lane == 0) {
            auto issue = [&](int j, uint32_t gg) {
                const int st = gg & 1;
                if (gg >= 2) mb_wait(&bar_empty[st], ((gg >> 1) - 1) & 1);
                unsigned char* sa = base + st * stage_bytes;
                mb_expect_tx(&bar_full[st], plain_bytes);
                tma_load_2d(sa, &map_dz, j * 32, (int)((int64_t)m * a.dz_rows + row0), &bar_full[st]);
                tma_load_2d(sa + a_bytes, &map_wt, j * 32, 0, &bar_full[st]);
                if (a.kp > 128) tma_load_2d(sa + a_bytes + a.kp * 128, &map_wt, j * 32, a.kp, &bar_full[st]);
            };
            issue(0, g);
            for (int j = 0; j < nk; ++j) {
                const uint32_t gg = g + j;
                if (j + 1 < nk) issue(j + 1, gg + 1);
                const int st = gg & 1;
                mb_wait(SPLIT ? &bar_conv[st] : &bar_full[st], (gg >> 1) & 1);
                tc_fence_after();
                const uint32_t sa = su32(base + st * stage_bytes), sb = sa + a_bytes;
                const uint32_t nb = (uint32_t)a.kp * 128;             // neighbour half of the Wt chunk
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t acc = (j > 0 || k > 0) ? 1u : 0u;
                    if (SPLIT) {
                        const uint32_t al = sa + plain_bytes, bl = sb + plain_bytes;
                        mma_tf32(tmem, sdesc(al + k * 32), sdesc(sb + k * 32), idesc, acc);
                        mma_tf32(tmem, sdesc(sa + k * 32), sdesc(bl + k * 32), idesc, 1u);
                        mma_tf32(tmem, sdesc(sa + k * 32), sdesc(sb + k * 32), idesc, 1u);
                        mma_tf32(tmem + (uint32_t)a.kp, sdesc(al + k * 32), sdesc(sb + nb + k * 32), idesc, acc);
                        mma_tf32(tmem + (uint32_t)a.kp, sdesc(sa + k * 32), sdesc(bl + nb + k * 32), idesc, 1u);
                        mma_tf32(tmem + (uint32_t)a.kp, sdesc(sa + k * 32), sdesc(sb + nb + k * 32), idesc, 1u);
                    } else {
                        mma_tf32(tmem, sdesc(sa + k * 32), sdesc(sb + k * 32), idesc, acc);
                        mma_tf32(tmem + (uint32_t)a.kp, sdesc(sa + k * 32), sdesc(sb + nb + k * 32), idesc, acc);
                    }
                }
                mma_commit(&bar_empty[st]);
            }
            mma_commit(&bar_done);
        }
        if (SPLIT && warp >= 1) {            // converters: hi in place, lo into the stage's second half
            const int t = threadIdx.x - 32;
            const uint32_t n4 = plain_bytes / 16;
            for (int j = 0; j < nk; ++j) {
                const uint32_t gg = g + j;
                const int st = gg & 1;
                mb_wait(&bar_full[st], (gg >> 1) & 1);
                float4* p = reinterpret_cast<float4*>(base + st * stage_bytes);
                float4* pl = reinterpret_cast<float4*>(base + st * stage_bytes + plain_bytes);
                for (uint32_t i = t; i < n4; i += 96) {
                    const float4 v = p[i];
                    float4 h;
                    h.x = tf32_hi(v.x); h.y = tf32_hi(v.y); h.z = tf32_hi(v.z); h.w = tf32_hi(v.w);
                    p[i] = h;
                    pl[i] = make_float4(__fsub_rn(v.x, h.x), __fsub_rn(v.y, h.y), __fsub_rn(v.z, h.z), __fsub_rn(v.w, h.w));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mb_arrive(&bar_conv[st]);
            }
        }
        __syncwarp();
        g += nk;
        mb_wait(&bar_done, done_phase & 1);
        ++done_phase;
        tc_fence_after();
        const int r = warp * 32 + lane;
        const int64_t row = row0 + r;
        const bool live = row < n_dst;
        int64_t e0 = 0, e1 = 0;   // the row's neighbours: only their count (mean divisor) is used here
        if (live) {
            e0 = a.off[(int64_t)m * a.off_stride + row];
            e1 = a.off[(int64_t)m * a.off_stride + row + 1];
        }
        const float inv = e1 > e0 ? 1.0f / (float)(e1 - e0) : 0.0f;
        // dH rows < |F_h| are written here (k_zero_rows cleared them; the scatter adds later);
        // the neighbour part goes to dmean for k_scatter, which spreads it over all SMs
        float* d = a.dh + ((int64_t)m * a.dh_rows + row) * a.dh_pitch;
        float* dm = a.dmean + ((int64_t)m * a.dmean_rows + row) * a.kp;
        for (int c = 0; c < a.k_in; c += 8) {
            float v[8], u[8];
            tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c, v);
            tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a.kp + c), u);
            if (live) {
                reinterpret_cast<float4*>(d + c)[0] = make_float4(v[0], v[1], v[2], v[3]);
                reinterpret_cast<float4*>(d + c)[1] = make_float4(v[4], v[5], v[6], v[7]);
                reinterpret_cast<float4*>(dm + c)[0] = make_float4(u[0] * inv, u[1] * inv, u[2] * inv, u[3] * inv);
                reinterpret_cast<float4*>(dm + c)[1] = make_float4(u[4] * inv, u[5] * inv, u[6] * inv, u[7] * inv);
            }
        }
        tc_fence_before();
        __syncthreads();      // TMEM is rewritten by the next tile's MMAs
        tc_fence_after();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, tmem_cols);
}

// warp per dst row i: dH[j] += dmean[i] over the row's sampled neighbours j, one 16-byte vector
// atomic per lane per neighbour (128 columns per warp instruction)
__global__ void __launch_bounds__(kT) k_scatter(DgradArgs a) {
    pdl_enter();
    const int m = inst_of(blockIdx.y, a.inst0, a.inst_step);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_dst = a.hop_size[(int64_t)m * (kMaxLayers + 1) + a.hop];
    const int64_t* off = a.off + (int64_t)m * a.off_stride;
    const int32_t* nb = a.cols + (int64_t)m * a.col_stride;
    float* dh_m = a.dh + (int64_t)m * a.dh_rows * a.dh_pitch;
    for (int64_t i = (int64_t)blockIdx.x * (kT / 32) + warp; i < n_dst; i += (int64_t)gridDim.x * (kT / 32)) {
        const int64_t e0 = off[i], e1 = off[i + 1];
        if (e0 == e1) continue;
        const float* dm = a.dmean + ((int64_t)m * a.dmean_rows + i) * a.kp;
        for (int c = lane * 4; c < a.k_in; c += 128) {
            const float4 u = *reinterpret_cast<const float4*>(dm + c);
            for (int64_t e = e0; e < e1; ++e) red_add4(dh_m + (int64_t)nb[e] * a.dh_pitch + c, u.x, u.y, u.z, u.w);
        }
    }
}

// ------------------------------------------------------------------ neighbour means (training forward)
// warp per dst row: lanes cover 128 columns as float4, kMeanUnroll neighbour rows in flight
#ifndef MGNN_MEAN_UNROLL
#define MGNN_MEAN_UNROLL 4
#endif
constexpr int kMeanUnroll = MGNN_MEAN_UNROLL;
__global__ void __launch_bounds__(kT) k_mean(SageLayerArgs a) {
    pdl_enter();
    const int m = inst_of(blockIdx.y, a.inst0, a.inst_step);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n_dst = a.hop_size[(int64_t)m * (kMaxLayers + 1) + a.hop];
    const int64_t* off = a.off + (int64_t)m * a.off_stride;
    const int32_t* nb = a.cols + (int64_t)m * a.col_stride;
    const float* h = a.h_in + (int64_t)m * a.in_rows * a.in_pitch;
    for (int64_t i = (int64_t)blockIdx.x * (kT / 32) + warp; i < n_dst; i += (int64_t)gridDim.x * (kT / 32)) {
        const int64_t e0 = off[i], e1 = off[i + 1];
        float* mo = a.mean_out + ((int64_t)m * a.mean_rows + i) * a.mean_pitch;
        const float inv = (float)(e1 - e0);
        for (int c = lane * 4; c < a.mean_pitch; c += 128) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < a.k_in) {
                int64_t e = e0;
                for (; e + kMeanUnroll <= e1; e += kMeanUnroll) {
                    float4 v[kMeanUnroll];
#pragma unroll
                    for (int j = 0; j < kMeanUnroll; ++j)
                        v[j] = __ldg(reinterpret_cast<const float4*>(h + (int64_t)nb[e + j] * a.in_pitch + c));
#pragma unroll
                    for (int j = 0; j < kMeanUnroll; ++j) {
                        acc.x = __fadd_rn(acc.x, v[j].x);
                        acc.y = __fadd_rn(acc.y, v[j].y);
                        acc.z = __fadd_rn(acc.z, v[j].z);
                        acc.w = __fadd_rn(acc.w, v[j].w);
                    }
                }
                for (; e < e1; ++e) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(h + (int64_t)nb[e] * a.in_pitch + c));
                    acc.x = __fadd_rn(acc.x, v.x);
                    acc.y = __fadd_rn(acc.y, v.y);
                    acc.z = __fadd_rn(acc.z, v.z);
                    acc.w = __fadd_rn(acc.w, v.w);
                }
                if (e1 > e0) {
                    acc.x = __fdiv_rn(acc.x, inv);
                    acc.y = __fdiv_rn(acc.y, inv);
                    acc.z = __fdiv_rn(acc.z, inv);
                    acc.w = __fdiv_rn(acc.w, inv);
                }
            }
            *reinterpret_cast<float4*>(mo + c) = acc;
        }
    }
}

// ------------------------------------------------------------------ optimizer
// SGD over every layer's [W_self | W_neigh] block (and bias) in one launch, also refreshing the
// transposed copy the input-gradient GEMM reads
__global__ void __launch_bounds__(kT) k_sgd_layers(SgdLayers d, float lr) {
    pdl_enter();
    for (int l = 0; l < d.n_layers; ++l) {
        const int64_t rows = d.rows[l], cols = d.cols[l];
        float* w = d.w[l];
        float* g = d.g[l];
        float* wt = d.wt[l];
        const int64_t n = rows * cols + rows;          // block then bias (contiguous)
        for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
            const float v = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
            w[i] = v;
            g[i] = 0.0f;
            if (i < rows * cols && d.whi[l]) {          // 3xTF32 operands of the forward GEMM
                const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
                d.whi[l][i] = hi;
                d.wlo[l][i] = __fsub_rn(v, hi);
            }
            if (i < rows * cols && wt) {
                const int64_t o = i / cols, c = i - o * cols;
                wt[c * rows + o] = v;
            }
        }
    }
}

__global__ void __launch_bounds__(kT) k_transpose(const float* __restrict__ w, float* __restrict__ wt, int rows,
                                                  int cols) {
    pdl_enter();
    __shared__ float t[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int j = ty; j < 32; j += kT / 32)
        if (by + j < rows && bx + tx < cols) t[j][tx] = w[(int64_t)(by + j) * cols + bx + tx];
    __syncthreads();
    for (int j = ty; j < 32; j += kT / 32)
        if (bx + j < cols && by + tx < rows) wt[(int64_t)(bx + j) * rows + by + tx] = t[tx][j];
}

}  // namespace

void launch_xent(const XentArgs& a, cudaStream_t s) {
    const unsigned gx = (unsigned)std::max<int64_t>(1, (a.rows + 7) / 8);   // one seed row per warp
    launch_k(k_xent, dim3(gx, a.n_inst), dim3(kT), 0, s, a);
    count_launches(1, __func__, s);
}

// blocks per instance so the whole launch fills every SM (~8 resident 256-thread blocks per SM) even
// when a training step has only its 2-8 instances, capped by the work
static unsigned fill_x(int64_t work_blocks, int n_inst) {
    const int64_t target = ((int64_t)num_sms() * 8 + n_inst - 1) / n_inst;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(work_blocks, std::max<int64_t>(target, 1)));
}

void launch_relu_mask(const MaskArgs& a, cudaStream_t s) {
    const int64_t work = ((a.rows + 63) / 64 * 64) * (a.ncols / 4);
    const unsigned gx = fill_x((work + kT - 1) / kT, a.n_inst);
    launch_k(k_relu_mask, dim3(gx, a.n_inst), dim3(kT), 0, s, a);
    count_launches(1, __func__, s);
}

void launch_zero_rows(const ZeroRowsArgs& a, cudaStream_t s) {
    const int64_t work = a.rows * (a.pitch / 4);
    const unsigned gx = fill_x((work + kT - 1) / kT, a.n_inst);
    launch_k(k_zero_rows, dim3(gx, a.n_inst), dim3(kT), 0, s, a);
    count_launches(1, __func__, s);
}

bool launch_wgrad(const WgradArgs& a_in, cudaStream_t s) {
    const size_t smem = 1024 + 2 * kWStage;
    if (ensure_smem_k(k_wgrad<false>, (int)smem) != cudaSuccess) return false;
    if (ensure_smem_k(k_wgrad<true>, (int)smem) != cudaSuccess) return false;
    WgradArgs a = a_in;
    if (a.n_inst > kWMaxInst || a.kp % 128 || a.npad > 256) return false;
    const int sms = num_sms();
    const int tiles = ((a.npad + 127) / 128) * ((2 * a.kp) / 128);
    // split-K over every SM (measured: fewer CTAs with >= 8 chunks each was slower, 16 -> 26 us; the
    // chunk loads are latency-bound, the partial-tile atomics are not)
    a.ksplit = std::max(1, sms / tiles);
    if (a.split3)
        launch_k(k_wgrad<true>, dim3(tiles * a.ksplit), dim3(kWThreads), smem, s, a);
    else
        launch_k(k_wgrad<false>, dim3(tiles * a.ksplit), dim3(kWThreads), smem, s, a);
    count_launches(1, __func__, s);
    return true;
}

bool launch_dgrad(const void* map_dz, const void* map_wt, const DgradArgs& a, cudaStream_t s) {
    if (a.n_inst > kWMaxInst || a.kp % 32 || a.kp > 256 || a.npad_out > 256) return false;
    const size_t plain = (size_t)kDTile * 128 + (size_t)2 * a.kp * 128;
    const bool split = a.split3 && 1024 + 4 * plain <= 227 * 1024;     // kp <= 128 (hidden layers)
    const size_t smem = 1024 + 2 * (split ? 2 : 1) * plain;
    if (ensure_smem_k(k_dgrad<false>, 1024 + 2 * (int)plain) != cudaSuccess) return false;
    if (split && ensure_smem_k(k_dgrad<true>, (int)smem) != cudaSuccess) return false;
    uint32_t cols = 32;
    while ((int)cols < 2 * a.kp) cols <<= 1;
    const int sms = num_sms();
    if (split)
        launch_k(k_dgrad<true>, dim3(sms), dim3(128), smem, s, *(const CUtensorMap*)map_dz,
                 *(const CUtensorMap*)map_wt, a, cols);
    else
        launch_k(k_dgrad<false>, dim3(sms), dim3(128), smem, s, *(const CUtensorMap*)map_dz,
                 *(const CUtensorMap*)map_wt, a, cols);
    count_launches(1, __func__, s);
    return true;
}

void launch_scatter(const DgradArgs& a, cudaStream_t s) {
    launch_k(k_scatter, dim3(fill_x((a.dz_rows + 7) / 8, a.n_inst), a.n_inst), dim3(kT), 0, s, a);
    count_launches(1, __func__, s);
}

void launch_mean(const SageLayerArgs& a, cudaStream_t s) {
    // warp per dst row: enough blocks that every SM keeps ~8 of them (the training step's forward has
    // only 2-8 instances; 128 blocks per instance left ~14 warps per SM and 1.7 TB/s on products)
    launch_k(k_mean, dim3(std::max(128u, fill_x((a.out_rows + 7) / 8, a.n_inst)), a.n_inst), dim3(kT), 0, s, a);
    count_launches(1, __func__, s);
}

void launch_sgd_layers(const SgdLayers& d, float lr, cudaStream_t s) {
    launch_k(k_sgd_layers, dim3(num_sms()), dim3(kT), 0, s, d, lr);
    count_launches(1, __func__, s);
}

void launch_transpose(const float* w, float* wt, int32_t rows, int32_t cols, cudaStream_t s) {
    launch_k(k_transpose, dim3((cols + 31) / 32, (rows + 31) / 32), dim3(kT), 0, s, w, wt, rows, cols);
    count_launches(1, __func__, s);
}

}  // namespace mgnn
