"""GPU consumer (mgnn_sage_forward, tcgen05 TF32) vs the fp64 oracle (oracle/sage.py).

Tolerance ("consumer"): the tensor cores read fp32 operands as TF32
(10 explicit mantissa bits; unit roundoff u = 2^-10 covers truncation as well as
rounding) and accumulate in fp32.  For one output z = sum_k a_k w_k + b of a layer
with K = 2*d_in terms the error is bounded by
    (2u + u^2 + (K+2) 2^-24) * sum_k |a_k||w_k|  +  sum_k |w_k| e(a_k)  +  2^-24 |z|,
where e(a) is the propagated bound of the layer's input (0 for X, exact in fp32;
the mean adds (deg+1) 2^-24 |h| of fp32 summation and division).  ReLU is
1-Lipschitz.  The test bound is that running bound times 2 (slack for the order of
the fp32 accumulation inside the tensor core), evaluated in fp64 from the oracle's
own quantities -- nothing from the CUDA path enters it.
"""
from __future__ import annotations

import numpy as np

from inputs import synth
from oracle import oracle as O
from oracle import sage as S

U_TF32 = 2.0 ** -10
U32 = 2.0 ** -24


def gpu_precision() -> str:
    """The forward GEMM's operand precision in this process: "3xtf32" (k_sage_gemm default), or "tf32"
    (MGNN_SAGE_TF32=1, or the fused in-kernel aggregation MGNN_SAGE_SPLIT=0)."""
    import os
    if os.environ.get("MGNN_SAGE_TF32") == "1" or os.environ.get("MGNN_SAGE_SPLIT") == "0":
        return "tf32"
    return "3xtf32"


def error_bound(X, blocks, weights, precision: str = "tf32"):
    """Running elementwise bound on |GPU - exact| of every layer's output (see module doc).
    precision "3xtf32": a = a_hi + a_lo, w = w_hi + w_lo exactly (TF32 hi parts), three TF32 products
    a_hi w_hi + a_hi w_lo + a_lo w_hi, each within 3 u^2 |a||w| of a w (dropped a_lo w_lo, the TF32
    conversion of the lo parts), accumulated in fp32 over 3K terms."""
    h = np.asarray(X, np.float64)
    e = np.zeros_like(h)
    L = len(weights)
    for l in range(L):
        off, nbr = blocks[L - 1 - l]
        n = len(off) - 1
        ws, wn, b = (np.abs(np.asarray(a, np.float64)) for a in weights[l])
        K = 2 * h.shape[1]
        if precision == "3xtf32":
            u_op = 3 * U_TF32 ** 2
            c = u_op + (3 * K + 2) * U32
        else:
            u_op = 2 * U_TF32
            c = 2 * U_TF32 + U_TF32 ** 2 + (K + 2) * U32
        mean_abs = np.zeros((n, h.shape[1]))
        mean_err = np.zeros((n, h.shape[1]))
        for i in range(n):
            nb = nbr[off[i]:off[i + 1]]
            if len(nb):
                mean_abs[i] = np.abs(h[nb]).mean(axis=0)
                mean_err[i] = e[nb].mean(axis=0) + (len(nb) + 1) * U32 * mean_abs[i]
        mag = np.abs(h[:n]) @ ws.T + mean_abs @ wn.T
        ws_, wn_, b_ = (np.asarray(a, np.float64) for a in weights[l])
        z = S.sage_layer(h, n, np.asarray(off), np.asarray(nbr), ws_, wn_, b_, relu=False)
        e = 2.0 * (c * mag + (e[:n] @ ws.T + mean_err @ wn.T) * (1 + u_op) + U32 * np.abs(z))
        h = np.maximum(z, 0.0) if l < L - 1 else z
    return e


def oracle_instance(op, step, fanouts, batch, run_seed=synth.RUN_SEED):
    """Run oracle partition `op` at global step `step`; return (F_L, blocks with positions, X)."""
    op.step(run_seed, step, fanouts, batch)
    F = op.frontier()
    blocks = []
    for h in range(len(fanouts)):
        off, cols = op.hop_block(h)
        blocks.append((off, S.positions(F, cols)))
    return F, blocks, op.features()


def run_sage_parity(g, P, D, fanouts, batch, dims, windows, f_bp=2500, gamma=0.95, delta=0,
                    inst_every=1, weight_seed=synth.SAGE_SEED, device=0, bind_x=False, precision=None):
    """Sample/gather windows on the GPU, run the consumer, compare every checked instance's
    logits with the fp64 oracle within error_bound.  Returns max |err| / bound."""
    import torch
    from paper_2410_22697_b200 import pipeline as PL

    parts = synth.partition(g, P)
    alpha = float(O.alpha_default(gamma, delta)) if delta > 0 else 0.0
    W = O.World(parts, D, synth.FEAT_SEED)
    for p in W.parts:
        p.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    ctx = PL.build_context(device, parts, D, synth.FEAT_SEED)
    ctx.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    ctx.sampler_config(fanouts, batch, synth.RUN_SEED, max(windows))
    wts = synth.sage_weights(dims, seed=weight_seed)
    ctx.sage_config(dims, [w[0] for w in wts], [w[1] for w in wts], [w[2] for w in wts])
    if bind_x:                        # caller-owned X (mgnn_window_bind_x) after the consumer exists
        rs, pitch, mi = ctx.window_shape()
        for sl in (0, 1):
            ctx.bind_x(sl, torch.full((mi * rs * pitch,), float("nan"), device="cuda", dtype=torch.float32))
    C = dims[-1]
    worst = 0.0
    t, slot = 1, 0
    checked = 0
    for wlen in windows:
        n_inst = len(ctx.parts) * wlen
        logits = torch.full((n_inst, batch, C), float("nan"), device="cuda", dtype=torch.float32)
        ctx.sample(slot, t, wlen)
        ctx.lookup_gather(slot)
        ctx.sage_forward(slot, logits)
        ctx.score(slot)
        torch.cuda.synchronize()
        got_all = logits.cpu().numpy()
        for w in range(wlen):
            for lp, pid in enumerate(ctx.parts):
                m = lp * wlen + w
                op = W.parts[pid]
                F, blocks, X = oracle_instance(op, t + w, fanouts, batch)
                if (checked := checked + 1) % inst_every:
                    continue
                ref = S.sage_forward(X, blocks, wts)[-1]
                bound = error_bound(X, blocks, wts, precision or gpu_precision())
                n0 = ref.shape[0]
                got = got_all[m, :n0, :]
                assert np.all(np.isfinite(got)), (pid, t + w)
                err = np.abs(got.astype(np.float64) - ref)
                ratio = float(np.max(err / (bound + 1e-30)))
                assert np.all(err <= bound), (pid, t + w, ratio, np.unravel_index(np.argmax(err / bound), err.shape))
                worst = max(worst, ratio)
                # rows past |F_0| are never written
                assert np.all(np.isnan(got_all[m, n0:, :])), (pid, t + w)
        t += wlen
        slot ^= 1
    ctx.close()
    W.close()
    print(f"[sage parity] worst |err|/bound = {worst:.3e}")
    return worst
