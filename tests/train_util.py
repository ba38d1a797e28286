"""GPU training step (mgnn_sage_train_step / mgnn_sage_sgd, NEXT-3) vs the fp64 oracle
(oracle/sage.py sage_loss_grads / sgd), step by step.

Tolerance: the GPU multiplies in TF32 (u = 2^-10) and reduces gradients
with fp32 atomics in a data-dependent order, and its ReLU masks follow its own TF32
pre-activations, so a unit whose pre-activation is within the forward error bound of 0 may
be masked differently from the oracle's.  Gradients therefore match in norm, not elementwise:
per tensor ||g - g_ref|| <= REL_l ||g_ref||, and for the last layer (whose dZ = dlogits has no
mask) also per output row o ||g_o - g_ref_o|| <= REL_l (||g_ref_o|| + ||g_ref|| / sqrt(rows)),
REL = 16 u = 1/64 (two TF32
products per layer on the forward path and two on the backward path, times the depth, with
2x slack).  Weights after SGD: ||W - W_ref|| <= 2 REL lr sum_steps ||g_ref||.
"""
from __future__ import annotations

import numpy as np

from inputs import synth
from oracle import oracle as O
from oracle import sage as S
from tests.sage_util import oracle_instance

REL = 1.0 / 64


def unpack(flat: np.ndarray, dims):
    """Padded parameter/gradient layout of the library -> [(W_self, W_neigh, b)] per layer."""
    out, off = [], 0
    for l in range(len(dims) - 1):
        d_in, d_out = dims[l], dims[l + 1]
        npad, kp = (d_out + 15) // 16 * 16, (d_in + 127) // 128 * 128
        w = flat[off:off + npad * 2 * kp].reshape(npad, 2 * kp)
        off += npad * 2 * kp
        b = flat[off:off + npad]
        off += npad
        out.append((w[:d_out, :d_in].copy(), w[:d_out, kp:kp + d_in].copy(), b[:d_out].copy()))
    return out


def close(got, ref, what, rows=True, rel=REL):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    nerr = np.linalg.norm(got - ref)
    nref = np.linalg.norm(ref)
    assert nerr <= rel * nref + 1e-9, (what, nerr, nref)
    if rows and ref.ndim == 2:
        rows_err = np.linalg.norm(got - ref, axis=1)
        rows_ref = np.linalg.norm(ref, axis=1)
        lim = rel * (rows_ref + nref / np.sqrt(ref.shape[0])) + 1e-9
        bad = np.nonzero(rows_err > lim)[0]
        assert len(bad) == 0, (what, "rows", bad[:5], rows_err[bad[:5]], lim[bad[:5]])
    return nerr / max(nref, 1e-30)


def run_train_parity(g, P, D, fanouts, batch, dims, n_steps, lr=0.05, window=None, device=0, hosted=None,
                     exchange=False):
    """P trainers (partitions) on one GPU, `n_steps` DDP steps of one window: per step compare the
    loss and every gradient with the oracle's average over the P minibatches, then SGD on both
    sides and compare the weights.  Returns the worst (relative gradient error / tolerance)."""
    import torch
    from paper_2410_22697_b200 import pipeline as PL

    parts = synth.partition(g, P)
    W = O.World(parts, D, synth.FEAT_SEED)
    for p in W.parts:
        p.buffer_init(0.95, 0.0, 1.0, 0, 2500)
    ctx = PL.build_context(device, parts, D, synth.FEAT_SEED, hosted)
    if exchange:                      # multi-process: map the other ranks' tables (CUDA IPC, NVLink)
        PL.exchange_tables(ctx)
    multi = exchange
    ctx.buffer_init(0.95, 0.0, 1.0, 0, 2500)
    window = window or n_steps
    ctx.sampler_config(fanouts, batch, synth.RUN_SEED, window)
    wts = synth.sage_weights(dims, seed=7)
    ctx.sage_config(dims, [w[0] for w in wts], [w[1] for w in wts], [w[2] for w in wts])
    labels = synth.node_labels(g.n_nodes, dims[-1])
    ctx.train_config(labels)
    ref_w = [tuple(np.asarray(a, np.float64) for a in w) for w in wts]
    worst = 0.0
    gsum = {}
    t = 1
    slot = 0
    done = 0
    while done < n_steps:
        wl = min(window, n_steps - done)
        ctx.sample(slot, t, wl)
        ctx.lookup_gather(slot)
        for w in range(wl):
            ctx.train_step(slot, w, P)
            if multi:                 # DDP: sum the ranks' gradient buffers (NCCL) and losses
                import torch.distributed as dist
                dist.all_reduce(ctx.grads())
            torch.cuda.synchronize()
            gpu_g = unpack(ctx.grads().cpu().numpy(), dims)
            gpu_loss = ctx.loss()
            if multi:
                lt = torch.tensor([gpu_loss], dtype=torch.float64, device="cuda")
                dist.all_reduce(lt)
                gpu_loss = float(lt.item())
            ref_g = None
            ref_loss = 0.0
            for pid in range(P):
                _, blocks, X = oracle_instance(W.parts[pid], t + w, fanouts, batch)
                F0 = W.parts[pid].frontier()[:W.parts[pid].hop_sizes()[0]]
                loss, gr = S.sage_loss_grads(X, blocks, ref_w, labels[F0])
                ref_loss += loss / P
                gr = [tuple(x / P for x in layer) for layer in gr]
                ref_g = gr if ref_g is None else [tuple(a + b for a, b in zip(x, y)) for x, y in zip(ref_g, gr)]
            assert abs(gpu_loss - ref_loss) <= REL * abs(ref_loss) + 1e-6, (t + w, gpu_loss, ref_loss)
            L = len(dims) - 1
            for l in range(L):
                for k, name in enumerate(("W_self", "W_neigh", "b")):
                    rel = REL * 2.0 ** (L - 1 - l)
                    worst = max(worst, close(gpu_g[l][k], ref_g[l][k], f"step {t + w} layer {l} d{name}",
                                             rows=l == L - 1, rel=rel) / rel)
            ctx.sgd(lr)
            ref_w = S.sgd(ref_w, ref_g, lr)
            for l in range(len(dims) - 1):
                got = ctx.params(l)
                for k, name in enumerate(("W_self", "W_neigh", "b")):
                    gsum[(l, k)] = gsum.get((l, k), 0.0) + np.linalg.norm(ref_g[l][k])
                    err = np.linalg.norm(np.asarray(got[k], np.float64) - ref_w[l][k])
                    assert err <= 2 * REL * 2.0 ** (L - 1 - l) * lr * gsum[(l, k)] + 1e-6, (t + w, l, name, err)
            done += 1
        ctx.score(slot)
        t += wl
        slot ^= 1
    if multi:                         # peers may still read our tables until every rank is done
        import torch.distributed as dist
        torch.cuda.synchronize()
        dist.barrier()
    ctx.close()
    W.close()
    print(f"[train parity] worst gradient error / tolerance {worst:.3f}")
    return worst
