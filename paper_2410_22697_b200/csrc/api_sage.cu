// api_sage.cu -- the consumer (A14: GraphSAGE-mean forward) and training (NEXT-3: DDP step) calls
// of include/mgnn.h.  Host code only: marshals sizes/pointers and launches sage.cu / train.cu.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/mgnn.h"
#include "ctx.h"
#include "launch.h"

using namespace mgnn;
using namespace mgnn::host;

namespace mgnn {
namespace host {

void free_sage(mgnn_ctx_s* ctx) {
    auto& S = ctx->sage;
    dfree(S.params);
    dfree(S.w3);
    for (int l = 0; l < kMaxLayers; ++l) {
        S.w[l] = S.b[l] = S.whi[l] = S.wlo[l] = nullptr;
        dfree(S.h[l]);
        dfree(S.wt[l]);
        dfree(S.mean[l]);
        dfree(S.dh[l]);
    }
    dfree(S.labels);
    dfree(S.dmean);
    dfree(S.grads);
    dfree(S.logits);
    dfree(S.dlogits);
    dfree(S.loss);
    if (S.side) {
        cudaStreamDestroy(S.side);
        for (auto& e : S.ev_fork) cudaEventDestroy(e);
        cudaEventDestroy(S.ev_join);
        cudaEventDestroy(S.ev_start);
        cudaEventDestroy(S.ev_zero);
        S.side = nullptr;
    }
    S.ready = S.train = false;
}

}  // namespace host
}  // namespace mgnn

namespace mgnn {
namespace host {
mgnn_status rebind_sage_input(mgnn_ctx ctx, int slot) {
    auto& S = ctx->sage;
    if (!S.ready) return MGNN_OK;
    const int64_t M = (int64_t)ctx->parts.size() * ctx->max_window;
    if (!sage_encode_map(S.map_in[slot][0], ctx->win[slot].X, M * ctx->ucap, ctx->pitch, ctx->pitch, 128))
        return fail(ctx, MGNN_ECUDA, "bind_x: cuTensorMapEncodeTiled (layer 0 input) failed");
    return MGNN_OK;
}
}  // namespace host
}  // namespace mgnn

extern "C" {

// ------------------------------------------------------------------ A14: GraphSAGE-mean consumer
mgnn_status mgnn_sage_config(mgnn_ctx ctx, const mgnn_sage_desc* d) {
    GUARD();
    if (!ctx->configured) return fail(ctx, MGNN_ESTATE, "sage_config before sampler_config");
    if (!d || d->n_layers != ctx->L || !d->dims || !d->w_self || !d->w_neigh || !d->bias)
        return fail(ctx, MGNN_EINVAL, "sage: n_layers must equal the sampler's and all arrays given");
    if (d->dims[0] != ctx->D) return fail(ctx, MGNN_EINVAL, "sage: dims[0] must equal feat_dim");
    for (int l = 1; l <= d->n_layers; ++l)
        if (d->dims[l] < 1 || d->dims[l] > 256) return fail(ctx, MGNN_EINVAL, "sage: dims[l] must be 1..256");
    for (int l = 0; l < d->n_layers; ++l)
        if (!d->w_self[l] || !d->w_neigh[l] || !d->bias[l]) return fail(ctx, MGNN_EINVAL, "sage: null weight");
    CK(cudaDeviceSynchronize());
    free_sage(ctx);
    auto& S = ctx->sage;
    const int L = d->n_layers;
    S.L = L;
    for (int l = 0; l <= L; ++l) S.dims[l] = d->dims[l];
    const int64_t M = (int64_t)ctx->parts.size() * ctx->max_window;
    // padded parameter layout (one buffer: the optimizer and the gradient all-reduce see one array)
    int64_t off = 0;
    for (int l = 0; l < L; ++l) {
        S.npad[l] = (S.dims[l + 1] + 15) / 16 * 16;
        S.kp[l] = (S.dims[l] + 127) / 128 * 128;
        S.w_off[l] = off;
        off += (int64_t)S.npad[l] * 2 * S.kp[l];
        S.b_off[l] = off;
        off += S.npad[l];
    }
    S.n_params = off;
    std::vector<float> hp((size_t)off, 0.0f);
    for (int l = 0; l < L; ++l) {
        const int kin = S.dims[l], n = S.dims[l + 1];
        const int64_t wc = 2 * (int64_t)S.kp[l];
        float* w = hp.data() + S.w_off[l];
        for (int o = 0; o < n; ++o) {
            for (int k = 0; k < kin; ++k) {
                w[(size_t)o * wc + k] = d->w_self[l][(size_t)o * kin + k];
                w[(size_t)o * wc + S.kp[l] + k] = d->w_neigh[l][(size_t)o * kin + k];
            }
            hp[(size_t)S.b_off[l] + o] = d->bias[l][o];
        }
    }
    CK(dalloc(&S.params, off));
    CK(cudaMemcpy(S.params, hp.data(), off * sizeof(float), cudaMemcpyHostToDevice));
    {
        const char* e = getenv("MGNN_SAGE_TF32");
        S.split3 = !(e && e[0] == '1');
    }
    if (S.split3) {
        int64_t wn = 0;
        for (int l = 0; l < L; ++l) wn += (int64_t)S.npad[l] * 2 * S.kp[l];
        CK(dalloc(&S.w3, 2 * wn));
        int64_t o = 0;
        for (int l = 0; l < L; ++l) {
            S.whi[l] = S.w3 + o;
            S.wlo[l] = S.w3 + wn + o;
            o += (int64_t)S.npad[l] * 2 * S.kp[l];
        }
    }
    for (int l = 0; l < L; ++l) {
        S.w[l] = S.params + S.w_off[l];
        S.b[l] = S.params + S.b_off[l];
        const int64_t wc = 2 * (int64_t)S.kp[l];
        if (!sage_encode_map(S.map_w[l], S.w[l], S.npad[l], wc, wc, S.npad[l]))
            return fail(ctx, MGNN_ECUDA, "sage: cuTensorMapEncodeTiled (weights) failed");
        if (S.split3) {
            launch_split_tf32(S.w[l], S.whi[l], S.wlo[l], (int64_t)S.npad[l] * wc, 0);
            if (!sage_encode_map(S.map_whi[l], S.whi[l], S.npad[l], wc, wc, S.npad[l]) ||
                !sage_encode_map(S.map_wlo[l], S.wlo[l], S.npad[l], wc, wc, S.npad[l]))
                return fail(ctx, MGNN_ECUDA, "sage: cuTensorMapEncodeTiled (split weights) failed");
        }
        S.out_rows[l] = ctx->fcap[L - 1 - l];
        if (l < L - 1) {
            const int64_t n = M * S.out_rows[l] * S.npad[l];
            CK(dalloc(&S.h[l], n));
            CK(cudaMemset(S.h[l], 0, n * sizeof(float)));   // rows never written stay finite (tensor-core operands)
        }
    }
    for (int slot = 0; slot < 2; ++slot)
        for (int l = 0; l < L; ++l) {
            const int hop = L - 1 - l;
            const float* base;
            int64_t rows, cols, pitch;
            if (l == 0) {
                base = ctx->win[slot].X;
                rows = M * ctx->ucap;
                cols = pitch = ctx->pitch;
            } else {
                base = S.h[l - 1];
                rows = M * ctx->fcap[hop + 1];
                cols = pitch = S.npad[l - 1];
            }
            if (!sage_encode_map(S.map_in[slot][l], base, rows, cols, pitch, 128))
                return fail(ctx, MGNN_ECUDA, "sage: cuTensorMapEncodeTiled (activations) failed");
        }
    CK(cudaDeviceSynchronize());                 // the weight split (legacy stream) precedes every forward
    S.ready = true;
    return MGNN_OK;
}

namespace {
// one forward layer over `n_inst` instances inst0, inst0 + inst_step, ... of a window slot
mgnn_status sage_layer(mgnn_ctx ctx, Win& w, int slot, int l, int n_inst, int inst0, int inst_step, float* out,
                       int64_t out_rows, int64_t out_pitch, int n_out, float* mean_out, cudaStream_t s,
                       bool mean_first = false) {
    auto& S = ctx->sage;
    const int L = S.L, hop = L - 1 - l;
    SageLayerArgs a;
    memset(&a, 0, sizeof(a));
    a.n_inst = n_inst;
    a.inst0 = inst0;
    a.inst_step = inst_step;
    a.hop = hop;
    a.k_in = S.dims[l];
    a.kp = S.kp[l];
    a.npad = S.npad[l];
    a.relu = l < L - 1;
    a.k_hop = ctx->k_hop[hop];
    a.hop_size = w.hop_size;
    a.off = w.off[hop];
    a.off_stride = ctx->fcap[hop] + 1;
    a.cols = w.cols[hop];
    a.col_stride = ctx->ecap[hop];
    if (l == 0) {
        a.h_in = w.X;
        a.in_rows = ctx->ucap;
        a.in_pitch = ctx->pitch;
    } else {
        a.h_in = S.h[l - 1];
        a.in_rows = ctx->fcap[hop + 1];
        a.in_pitch = S.npad[l - 1];
    }
    a.h_out = out;
    a.out_rows = out_rows;
    a.out_pitch = out_pitch;
    a.n_out = n_out;
    a.bias = S.b[l];
    a.mean_out = mean_out;
    a.mean_rows = S.out_rows[l];
    a.mean_pitch = S.kp[l];
    if (mean_first) {          // means by k_mean over all SMs, then the warp-specialised TMA-fed GEMM
        launch_mean(a, s);
        a.split3 = S.split3 ? 1 : 0;
        if (!launch_sage_gemm(S.map_in[slot][l], S.split3 ? S.map_whi[l] : S.map_w[l], S.map_wlo[l],
                              S.map_mean128[l], a, s))
            return fail(ctx, MGNN_ECUDA, "sage: gemm launch configuration failed");
        return MGNN_OK;
    }
    if (!launch_sage_layer(S.map_in[slot][l], S.map_w[l], a, s))
        return fail(ctx, MGNN_ECUDA, "sage: layer launch configuration failed");
    return MGNN_OK;
}
}  // namespace

namespace {
// neighbour-mean buffers [M][out_rows][kp] per layer and their TMA maps (training; split forward)
mgnn_status ensure_mean_buffers(mgnn_ctx ctx) {
    auto& S = ctx->sage;
    const int64_t M = (int64_t)ctx->parts.size() * ctx->max_window;
    for (int l = 0; l < S.L; ++l) {
        if (S.mean[l]) continue;
        const int64_t nm = M * S.out_rows[l] * S.kp[l];
        CK(dalloc(&S.mean[l], nm));
        CK(cudaMemset(S.mean[l], 0, nm * sizeof(float)));
        if (!sage_encode_map(S.map_mean128[l], S.mean[l], M * S.out_rows[l], S.kp[l], S.kp[l], 128))
            return fail(ctx, MGNN_ECUDA, "cuTensorMapEncodeTiled (means) failed");
    }
    return MGNN_OK;
}
// Window forward as k_mean (neighbour means, warp per row over all SMs, stored in HBM) + the
// TMA-fed GEMM (default; measured faster than aggregating inside the GEMM kernel on every config:
// arxiv 0.64 -> 0.44 ms, reddit 7.2 -> 4.6 ms, products 6.6 -> 5.6 ms per window).
// MGNN_SAGE_SPLIT=0 selects the fused in-kernel aggregation (A/B, tested).
bool split_forward() {
    const char* e = getenv("MGNN_SAGE_SPLIT");
    return !(e && e[0] == '0');
}
}  // namespace

mgnn_status mgnn_sage_forward(mgnn_ctx ctx, int32_t slot, float* logits, int64_t logits_pitch, mgnn_stream stream) {
    GUARD();
    if (slot < 0 || slot > 1 || !logits) return fail(ctx, MGNN_EINVAL, "bad slot / logits");
    auto& S = ctx->sage;
    if (!S.ready) return fail(ctx, MGNN_ESTATE, "sage_forward before sage_config");
    if (logits_pitch < S.dims[S.L]) return fail(ctx, MGNN_EINVAL, "logits_pitch < dims[L]");
    Win& w = ctx->win[slot];
    if (!w.gathered) return fail(ctx, MGNN_ESTATE, "sage_forward needs a gathered window");
    if (w.relabel_pending) return fail(ctx, MGNN_ESTATE, "sage_forward: the window's columns are not relabelled (mgnn_relabel)");
    cudaStream_t s = (cudaStream_t)stream;
    const int L = S.L;
    const int n_inst = (int)ctx->parts.size() * w.n_steps;
    const bool split = split_forward();
    if (split) {
        mgnn_status st = ensure_mean_buffers(ctx);
        if (st) return st;
    }
    for (int l = 0; l < L; ++l) {
        float* mo = split ? S.mean[l] : nullptr;
        mgnn_status st = l < L - 1 ? sage_layer(ctx, w, slot, l, n_inst, 0, 1, S.h[l], S.out_rows[l], S.npad[l],
                                                S.npad[l], mo, s, split)
                                   : sage_layer(ctx, w, slot, l, n_inst, 0, 1, logits, ctx->batch, logits_pitch,
                                                S.dims[L], mo, s, split);
        if (st) return st;
    }
    CKL();
    return MGNN_OK;
}

// ------------------------------------------------------------------ NEXT-3: DDP training step
mgnn_status mgnn_sage_train_config(mgnn_ctx ctx, const int32_t* labels) {
    GUARD();
    auto& S = ctx->sage;
    if (!S.ready) return fail(ctx, MGNN_ESTATE, "train_config before sage_config");
    if (!labels) return fail(ctx, MGNN_EINVAL, "labels");
    for (int64_t v = 0; v < ctx->n_global; ++v)
        if (labels[v] < 0 || labels[v] >= S.dims[S.L]) return fail(ctx, MGNN_EINVAL, "label out of range");
    CK(cudaDeviceSynchronize());
    const int L = S.L;
    const int64_t M = (int64_t)ctx->parts.size() * ctx->max_window;
    dfree(S.labels);
    CK(dalloc(&S.labels, ctx->n_global));
    CK(cudaMemcpy(S.labels, labels, ctx->n_global * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (!S.grads) {
        CK(dalloc(&S.grads, S.n_params));
        CK(cudaMemset(S.grads, 0, S.n_params * sizeof(float)));
        CK(dalloc(&S.loss, 1));
        CK(cudaMemset(S.loss, 0, sizeof(float)));
        CK(cudaStreamCreateWithFlags(&S.side, cudaStreamNonBlocking));
        for (auto& e : S.ev_fork) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&S.ev_join, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&S.ev_start, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&S.ev_zero, cudaEventDisableTiming));
        S.rows64 = (ctx->batch + 63) / 64 * 64;
        const int64_t nl = M * S.rows64 * S.npad[L - 1];
        CK(dalloc(&S.logits, nl));
        CK(dalloc(&S.dlogits, nl));
        CK(cudaMemset(S.logits, 0, nl * sizeof(float)));
        CK(cudaMemset(S.dlogits, 0, nl * sizeof(float)));
        int64_t ndm = 1;
        for (int l = 1; l < L; ++l) ndm = std::max(ndm, M * S.out_rows[l] * S.kp[l]);
        CK(dalloc(&S.dmean, ndm));
        {
            mgnn_status st = ensure_mean_buffers(ctx);
            if (st) return st;
        }
        for (int l = 0; l < L; ++l) {
            CK(dalloc(&S.wt[l], (int64_t)2 * S.kp[l] * S.npad[l]));
            if (l < L - 1) {
                S.dh_rows[l] = (S.out_rows[l] + 63) / 64 * 64;
                const int64_t nd = M * S.dh_rows[l] * S.npad[l];
                CK(dalloc(&S.dh[l], nd));
                CK(cudaMemset(S.dh[l], 0, nd * sizeof(float)));
            }
        }
        for (int l = 0; l < L; ++l) {
            float* dz = l == L - 1 ? S.dlogits : S.dh[l];
            const int64_t dzr = l == L - 1 ? S.rows64 : S.dh_rows[l];
            const int64_t wtr = 2 * (int64_t)S.kp[l];
            // the input gradient (and its transposed-weight operand) exists for layers >= 1 only
            if (!sage_encode_map(S.map_dz128[l], dz, M * dzr, S.npad[l], S.npad[l], 128) ||
                (l > 0 && !sage_encode_map(S.map_wt[l], S.wt[l], wtr, S.npad[l], S.npad[l],
                                           (int)(wtr <= 256 ? wtr : S.kp[l]))))
                return fail(ctx, MGNN_ECUDA, "train: cuTensorMapEncodeTiled failed");
            launch_transpose(S.w[l], S.wt[l], S.npad[l], (int32_t)wtr, 0);
        }
        CKL();
        CK(cudaDeviceSynchronize());
    }
    S.train = true;
    return MGNN_OK;
}

mgnn_status mgnn_sage_train_step(mgnn_ctx ctx, int32_t slot, int32_t step_in_window, int32_t n_trainers,
                                 mgnn_stream stream) {
    GUARD();
    auto& S = ctx->sage;
    if (!S.train) return fail(ctx, MGNN_ESTATE, "train_step before train_config");
    if (slot < 0 || slot > 1 || n_trainers < 1) return fail(ctx, MGNN_EINVAL, "bad slot / n_trainers");
    Win& w = ctx->win[slot];
    if (!w.gathered) return fail(ctx, MGNN_ESTATE, "train_step needs a gathered window");
    if (w.relabel_pending) return fail(ctx, MGNN_ESTATE, "train_step: the window's columns are not relabelled (mgnn_relabel)");
    if (step_in_window < 0 || step_in_window >= w.n_steps) return fail(ctx, MGNN_EINVAL, "step_in_window");
    cudaStream_t s = (cudaStream_t)stream;
    const int L = S.L;
    const int n_lp = (int)ctx->parts.size();
    const int i0 = step_in_window, is = w.n_steps;   // instances lp * n_steps + step_in_window
    // every early return after the side stream forked joins it back into `s` first, so a CUDA-graph
    // capture of the caller's stream never ends with an un-joined fork
    bool forked = false;
    auto joined = [&](mgnn_status st) -> mgnn_status {
        if (forked && cudaEventRecord(S.ev_join, S.side) == cudaSuccess) cudaStreamWaitEvent(s, S.ev_join, 0);
        return st;
    };
    // The input-gradient buffers dH[l-1] (l >= 1) are cleared on the side stream beside the forward:
    // nothing of this step touches them before the first dgrad, and every write of the previous
    // step (dgrad, scatter, ReLU mask on `s`) precedes the fork of that step's last weight gradient,
    // which the side stream already follows.
    if (L > 1) {
        CK(cudaEventRecord(S.ev_start, s));
        CK(cudaStreamWaitEvent(S.side, S.ev_start, 0));
        forked = true;
        for (int l = 1; l < L; ++l) {
            ZeroRowsArgs za;
            memset(&za, 0, sizeof(za));
            za.n_inst = n_lp;
            za.inst0 = i0;
            za.inst_step = is;
            za.hop = L - l;
            za.hop_size = w.hop_size;
            za.buf = S.dh[l - 1];
            za.rows = S.dh_rows[l - 1];
            za.pitch = S.npad[l - 1];
            launch_zero_rows(za, S.side);
        }
        CK(cudaEventRecord(S.ev_zero, S.side));
    }
    // forward, keeping every layer's output and neighbour means
    for (int l = 0; l < L; ++l) {
        mgnn_status st = l < L - 1 ? sage_layer(ctx, w, slot, l, n_lp, i0, is, S.h[l], S.out_rows[l], S.npad[l],
                                                S.npad[l], S.mean[l], s, true)
                                   : sage_layer(ctx, w, slot, l, n_lp, i0, is, S.logits, S.rows64, S.npad[l],
                                                S.npad[l], S.mean[l], s, true);
        if (st) return joined(st);
    }
    // loss: mean cross-entropy per trainer, averaged over the n_trainers of the DDP step
    XentArgs xa;
    memset(&xa, 0, sizeof(xa));
    xa.n_inst = n_lp;
    xa.inst0 = i0;
    xa.inst_step = is;
    xa.n_classes = S.dims[L];
    xa.hop_size = w.hop_size;
    xa.frontier = w.fr_gid;
    xa.ucap = ctx->ucap;
    xa.labels = S.labels;
    xa.logits = S.logits;
    xa.dlogits = S.dlogits;
    xa.rows = S.rows64;
    xa.pitch = S.npad[L - 1];
    xa.scale = 1.0f / (float)n_trainers;
    xa.db = S.grads + S.b_off[L - 1];
    xa.loss = S.loss;
    launch_xent(xa, s);
    for (int l = L - 1; l >= 0; --l) {
        const int hop = L - 1 - l;
        float* dz = l == L - 1 ? S.dlogits : S.dh[l];
        const int64_t dzr = l == L - 1 ? S.rows64 : S.dh_rows[l];
        if (l < L - 1) {
            MaskArgs ma;
            memset(&ma, 0, sizeof(ma));
            ma.n_inst = n_lp;
            ma.inst0 = i0;
            ma.inst_step = is;
            ma.hop = hop;
            ma.hop_size = w.hop_size;
            ma.dz = dz;
            ma.rows = dzr;
            ma.pitch = S.npad[l];
            ma.h = S.h[l];
            ma.h_rows = S.out_rows[l];
            ma.h_pitch = S.npad[l];
            ma.ncols = S.npad[l];
            ma.db = S.grads + S.b_off[l];
            launch_relu_mask(ma, s);
        }
        WgradArgs wa;
        memset(&wa, 0, sizeof(wa));
        wa.n_inst = n_lp;
        wa.inst0 = i0;
        wa.inst_step = is;
        wa.hop = hop;
        wa.hop_size = w.hop_size;
        wa.dz = dz;
        wa.dz_rows = dzr;
        wa.dz_pitch = S.npad[l];
        if (l == 0) {
            wa.h_in = w.X;
            wa.in_rows = ctx->ucap;
            wa.in_pitch = ctx->pitch;
        } else {
            wa.h_in = S.h[l - 1];
            wa.in_rows = ctx->fcap[hop + 1];
            wa.in_pitch = S.npad[l - 1];
        }
        wa.in_cols = S.dims[l];
        wa.mean = S.mean[l];
        wa.mean_rows = S.out_rows[l];
        wa.mean_pitch = S.kp[l];
        wa.mean_cols = S.dims[l];
        wa.kp = S.kp[l];
        wa.npad = S.npad[l];
        wa.dw = S.grads + S.w_off[l];
        wa.max_chunks = (int64_t)n_lp * ((S.out_rows[l] + 63) / 64);
        wa.split3 = S.split3 ? 1 : 0;
        // the weight gradient only reads dZ, H and the means: it runs on the side stream while the
        // input gradient and the next layer's mask proceed on `s` (joined before returning)
        CK(cudaEventRecord(S.ev_fork[l], s));
        CK(cudaStreamWaitEvent(S.side, S.ev_fork[l], 0));
        forked = true;
        if (!launch_wgrad(wa, S.side))
            return joined(fail(ctx, MGNN_ECUDA, "train: wgrad launch configuration failed"));
        if (l > 0) {
            if (l == L - 1) CK(cudaStreamWaitEvent(s, S.ev_zero, 0));
            DgradArgs da;
            memset(&da, 0, sizeof(da));
            da.n_inst = n_lp;
            da.inst0 = i0;
            da.inst_step = is;
            da.hop = hop;
            da.hop_size = w.hop_size;
            da.off = w.off[hop];
            da.off_stride = ctx->fcap[hop] + 1;
            da.cols = w.cols[hop];
            da.col_stride = ctx->ecap[hop];
            da.dz_rows = dzr;
            da.npad_out = S.npad[l];
            da.kp = S.kp[l];
            da.k_in = S.dims[l];
            da.dh = S.dh[l - 1];
            da.dh_rows = S.dh_rows[l - 1];
            da.dh_pitch = S.npad[l - 1];
            da.dmean = S.dmean;
            da.dmean_rows = S.out_rows[l];
            da.split3 = S.split3 ? 1 : 0;
            if (!launch_dgrad(S.map_dz128[l], S.map_wt[l], da, s))
                return joined(fail(ctx, MGNN_ECUDA, "train: dgrad launch configuration failed"));
            launch_scatter(da, s);
        }
    }
    CK(cudaEventRecord(S.ev_join, S.side));
    CK(cudaStreamWaitEvent(s, S.ev_join, 0));
    CKL();
    return MGNN_OK;
}

mgnn_status mgnn_sage_grads(mgnn_ctx ctx, float** grads, int64_t* n_floats) {
    GUARD();
    if (!grads || !n_floats) return fail(ctx, MGNN_EINVAL, "null output");
    if (!ctx->sage.train) return fail(ctx, MGNN_ESTATE, "grads before train_config");
    *grads = ctx->sage.grads;
    *n_floats = ctx->sage.n_params;
    return MGNN_OK;
}

mgnn_status mgnn_sage_sgd(mgnn_ctx ctx, float lr, mgnn_stream stream) {
    GUARD();
    auto& S = ctx->sage;
    if (!S.train) return fail(ctx, MGNN_ESTATE, "sgd before train_config");
    cudaStream_t s = (cudaStream_t)stream;
    SgdLayers d;
    memset(&d, 0, sizeof(d));
    d.n_layers = S.L;
    for (int l = 0; l < S.L; ++l) {     // the bias follows its layer's block (b_off = w_off + npad * 2 kp)
        d.w[l] = S.w[l];
        d.g[l] = S.grads + S.w_off[l];
        d.wt[l] = S.wt[l];
        d.whi[l] = S.whi[l];
        d.wlo[l] = S.wlo[l];
        d.rows[l] = S.npad[l];
        d.cols[l] = 2 * (int64_t)S.kp[l];
    }
    launch_sgd_layers(d, lr, s);
    CKL();
    return MGNN_OK;
}

mgnn_status mgnn_sage_loss(mgnn_ctx ctx, float* host_loss, mgnn_stream stream) {
    GUARD();
    auto& S = ctx->sage;
    if (!S.train || !host_loss) return fail(ctx, MGNN_ESTATE, "loss before train_config");
    cudaStream_t s = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(host_loss, S.loss, sizeof(float), cudaMemcpyDeviceToHost, s));
    CK(cudaMemsetAsync(S.loss, 0, sizeof(float), s));
    CK(cudaStreamSynchronize(s));
    return MGNN_OK;
}

mgnn_status mgnn_sage_params(mgnn_ctx ctx, int32_t l, float* w_self, float* w_neigh, float* bias) {
    GUARD();
    auto& S = ctx->sage;
    if (!S.ready || l < 0 || l >= S.L) return fail(ctx, MGNN_EINVAL, "layer");
    CK(cudaDeviceSynchronize());
    const int kin = S.dims[l], n = S.dims[l + 1];
    const int64_t wc = 2 * (int64_t)S.kp[l];
    std::vector<float> w((size_t)S.npad[l] * wc), b((size_t)S.npad[l]);
    CK(cudaMemcpy(w.data(), S.w[l], w.size() * sizeof(float), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), S.b[l], b.size() * sizeof(float), cudaMemcpyDeviceToHost));
    for (int o = 0; o < n; ++o) {
        for (int k = 0; k < kin; ++k) {
            if (w_self) w_self[(size_t)o * kin + k] = w[(size_t)o * wc + k];
            if (w_neigh) w_neigh[(size_t)o * kin + k] = w[(size_t)o * wc + S.kp[l] + k];
        }
        if (bias) bias[o] = b[o];
    }
    return MGNN_OK;
}

}  // extern "C"
