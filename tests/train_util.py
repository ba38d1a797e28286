"""GPU training step (mgnn_sage_train_step / mgnn_sage_sgd, NEXT-3) vs the fp64 oracle
(oracle/sage.py sage_loss_grads / sgd), step by step.

Tolerance.  The forward GEMMs and the backward GEMMs (k_wgrad, k_dgrad) multiply in
3xTF32 by default (fp32-grade products, per-product error 3 u_tf32^2 ~ 2.9e-6), MGNN_SAGE_TF32=1 in one
TF32 pass (u_tf32 = 2^-10); gradients are reduced with fp32 atomics in a data-dependent order.
  * Every DDP step (one process or several ranks, the all-reduce's fp32 sum added): ELEMENTWISE, |g - g_ref| <= the running bound of grad_bounds()
    (rigorous worst case: operand errors propagated from the forward's running bound, product errors,
    fp32 accumulation over the step's rows in any order, ReLU units whose pre-activation lies within its
    forward bound of 0 counted as masked either way, and the weights' drift from earlier SGD steps,
    e_W <- (e_W + lr B_g)(1 + 2 u32) + 2 u32 (|W| + lr |g|)); the weights after SGD within e_W.
  * Every step, NORMWISE per tensor: ||g - g_ref|| <= REL_l ||g_ref||, and for the last layer per output
    row o ||g_o - g_ref_o|| <= REL_l (||g_ref_o|| + ||g_ref|| / sqrt(rows)), REL_l = REL 2^(L-1-l):
    REL = 16 u_tf32 = 1/64 for one TF32 pass (two TF32 products per layer forward and backward, times the
    depth, 2x slack); REL = 2^-10 for 3xTF32 (per-product 3 u_tf32^2 plus sqrt(n) u32 accumulation over
    n <= 1e5 rows ~ 2e-5 per GEMM, four GEMMs per layer on the path, 8x slack -- a probabilistic, not a
    worst-case, bound; the first step's elementwise check is the rigorous one).
  * Weights after SGD: ||W - W_ref|| <= 2 REL_l lr sum_steps ||g_ref||.
"""
from __future__ import annotations

import numpy as np

from inputs import synth
from oracle import oracle as O
from oracle import sage as S
from tests.sage_util import oracle_instance

REL_TF32 = 1.0 / 64
REL_3XTF32 = 2.0 ** -10
U32 = 2.0 ** -24
U_TF32 = 2.0 ** -10


def forward_bounds(X, blocks, weights, precision, e_w=None):
    """Per layer (h, e_h, mean, e_mean, z, e_z): the oracle's fp64 quantities and the running elementwise
    bounds on |GPU - exact| of the layer's input, neighbour means and pre-activation -- the recurrence of
    tests/sage_util.error_bound (module doc there), kept layer by layer.  e_w: per layer elementwise
    bounds (e_Ws, e_Wn, e_b) on |W_gpu - W_ref| after earlier SGD steps (None: identical weights); their
    products with |input| + e_input join e_z."""
    h = np.asarray(X, np.float64)
    e = np.zeros_like(h)
    L = len(weights)
    out = []
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
        mean = np.zeros((n, h.shape[1]))
        mean_abs = np.zeros((n, h.shape[1]))
        mean_err = np.zeros((n, h.shape[1]))
        for i in range(n):
            nb = nbr[off[i]:off[i + 1]]
            if len(nb):
                mean[i] = h[nb].mean(axis=0)
                mean_abs[i] = np.abs(h[nb]).mean(axis=0)
                mean_err[i] = e[nb].mean(axis=0) + (len(nb) + 1) * U32 * mean_abs[i]
        mag = np.abs(h[:n]) @ ws.T + mean_abs @ wn.T
        ws_, wn_, b_ = (np.asarray(a, np.float64) for a in weights[l])
        z = S.sage_layer(h, n, np.asarray(off), np.asarray(nbr), ws_, wn_, b_, relu=False)
        ez = 2.0 * (c * mag + (e[:n] @ ws.T + mean_err @ wn.T) * (1 + u_op) + U32 * np.abs(z))
        if e_w is not None:                      # the GPU's weights differ from the oracle's by e_w
            ews, ewn, eb = e_w[l]
            ez += 2.0 * (((np.abs(h[:n]) + e[:n]) @ ews.T + (mean_abs + mean_err) @ ewn.T) * (1 + u_op) + eb)
        out.append((h, e, mean, mean_err, z, ez))
        h = np.maximum(z, 0.0) if l < L - 1 else z
        e = ez
    return out


def grad_bounds(X, blocks, weights, labels, scale, n_acc, precision, e_w=None):
    """Elementwise bounds on |GPU - exact| of one trainer's gradient contribution (scaled by `scale` =
    1 / n_trainers, as the GPU scales dlogits) per layer: [(dW_self, dW_neigh, db)].  A running bound
    through the backward, evaluated in fp64 from the oracle's own quantities (nothing from the CUDA path):
      * dlogits = (softmax(z) - y) / n:  |d p_j| <= 2 p_j max_k |dz_k| (softmax Jacobian) plus the fp32
        evaluation of expf(z - max - lse) (argument rounding, the C-term sum, a few ulp);
      * ReLU: dZ = dH [z > 0]; a unit whose pre-activation is within its forward bound of 0 (|z| <= e_z)
        may be masked either way on the GPU, so its dZ error is |dH| + e_dH -- mask flips are covered;
      * every product sum (dW = dZ^T In, dH = dZ W, over K terms) carries the operand errors
        (e_a |b| + (|a| + e_a) e_b)(1 + u_op) plus (u_op + (K + 2) u32) sum |a||b| -- u_op = 3 u_tf32^2
        for 3xTF32 products, 2 u_tf32 + u_tf32^2 for one TF32 pass, K the rows the step accumulates
        (n_acc[l], every trainer of the step: split-K partial sums and atomics in any order);
      * the neighbour scatter dH[j] += dZ_i W_neigh / deg(i) by fp32 atomics adds (count_j + 1) u32 sum |.|."""
    fw = forward_bounds(X, blocks, weights, precision, e_w)
    u_op = 3 * U_TF32 ** 2 if precision == "3xtf32" else 2 * U_TF32 + U_TF32 ** 2
    L = len(weights)
    zL, ezL = fw[-1][4], fw[-1][5]
    n0 = zL.shape[0]
    zm = zL - zL.max(axis=1, keepdims=True)
    p = np.exp(zm)
    p /= p.sum(axis=1, keepdims=True)
    y = np.zeros_like(p)
    y[np.arange(n0), labels] = 1.0
    lse = np.log(np.exp(zm).sum(axis=1, keepdims=True))
    C = zL.shape[1]
    dh = (p - y) * (scale / n0)
    # fp32 p = expf(z - max - lse): the argument's rounding (|z - max| + lse) u32, the sum over C classes,
    # expf / logf within a few ulp; then p - y and the 1/n scaling
    rel_p = 2.0 * (np.abs(zm) + lse + C + 8) * U32
    edh = (2.0 * p * ezL.max(axis=1, keepdims=True) + rel_p * p + 4 * U32 * np.abs(p - y)) * (scale / n0)
    out = [None] * L
    for l in range(L - 1, -1, -1):
        off, nbr = blocks[L - 1 - l]
        h, eh, mean, emean, z, ez = fw[l]
        n = len(off) - 1
        if l < L - 1:
            live = z > 0.0
            amb = np.abs(z) <= ez
            dz = dh * live
            edz = np.where(amb, np.abs(dh) + edh, edh * live)
        else:
            dz, edz = dh, edh
        adz = np.abs(dz)
        c = u_op + (n_acc[l] + 2) * U32
        bounds = []
        for inp, ein in ((h[:n], eh[:n]), (mean, emean)):
            ain = np.abs(inp)
            bounds.append((edz.T @ ain + (adz + edz).T @ ein) * (1 + u_op) + c * (adz.T @ ain))
        bounds.append(edz.sum(axis=0) + (n_acc[l] + 2) * U32 * adz.sum(axis=0))
        out[l] = tuple(bounds)
        if l > 0:
            ws, wn, _ = (np.asarray(a, np.float64) for a in weights[l])
            aws, awn = np.abs(ws), np.abs(wn)
            cK = u_op + (dz.shape[1] + 2) * U32
            deg = np.diff(np.asarray(off)).astype(np.float64)
            inv = np.where(deg > 0, 1.0 / np.maximum(deg, 1.0), 0.0)[:, None]
            dh_in = np.zeros_like(h)
            e_in = np.zeros_like(h)
            acc = np.zeros_like(h)
            cnt = np.zeros((h.shape[0], 1))
            mag_s = adz @ aws
            dh_in[:n] += dz @ ws
            e_in[:n] += edz @ aws * (1 + u_op) + cK * mag_s
            if e_w is not None:                  # dZ W with the GPU's weights
                e_in[:n] += (adz + edz) @ e_w[l][0] * (1 + u_op)
            acc[:n] += mag_s
            cnt[:n] += 1
            dm = (dz @ wn) * inv
            mag_n = (adz @ awn) * inv
            e_n = (edz @ awn * (1 + u_op) + cK * (adz @ awn)) * inv + U32 * mag_n
            if e_w is not None:
                e_n += ((adz + edz) @ e_w[l][1] * (1 + u_op)) * inv
            for i in range(n):
                nb = nbr[off[i]:off[i + 1]]
                if len(nb):
                    np.add.at(dh_in, nb, dm[i])
                    np.add.at(e_in, nb, e_n[i])
                    np.add.at(acc, nb, mag_n[i])
                    np.add.at(cnt, nb, 1.0)
            e_in += (cnt + 1) * U32 * acc
            dh, edh = dh_in, e_in
    return out


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


def close(got, ref, what, rows=True, rel=REL_TF32):
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
    elem_worst = 0.0
    from tests.sage_util import gpu_precision
    precision = gpu_precision()
    REL = REL_3XTF32 if precision == "3xtf32" else REL_TF32
    e_w = [tuple(np.zeros_like(np.asarray(a, np.float64)) for a in layer) for layer in ref_w]
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
            first = True                          # elementwise bounds at every step (weight drift in e_w)
            inst = []
            gabs = None                           # sum over trainers of |g_p| (the all-reduce's rounding)
            for pid in range(P):
                _, blocks, X = oracle_instance(W.parts[pid], t + w, fanouts, batch)
                F0 = W.parts[pid].frontier()[:W.parts[pid].hop_sizes()[0]]
                loss, gr = S.sage_loss_grads(X, blocks, ref_w, labels[F0])
                ref_loss += loss / P
                gr = [tuple(x / P for x in layer) for layer in gr]
                ref_g = gr if ref_g is None else [tuple(a + b for a, b in zip(x, y)) for x, y in zip(ref_g, gr)]
                if first:
                    inst.append((X, blocks, labels[F0]))
                    ga = [tuple(np.abs(x) for x in layer) for layer in gr]
                    gabs = ga if gabs is None else [tuple(a + b for a, b in zip(x, y)) for x, y in zip(gabs, ga)]
            if first:
                Ld = len(dims) - 1
                n_acc = [sum(len(b[Ld - 1 - l][0]) - 1 for _, b, _ in inst) for l in range(Ld)]
                bsum = None
                for X_, b_, y_ in inst:
                    bd = grad_bounds(X_, b_, ref_w, y_, 1.0 / P, n_acc, precision, e_w)
                    bsum = bd if bsum is None else [tuple(a + c for a, c in zip(x, y)) for x, y in zip(bsum, bd)]
                if multi:                         # NCCL sum over the ranks' gradient buffers in fp32
                    import torch.distributed as dist
                    nr = dist.get_world_size()
                    bsum = [tuple(b + (nr + 1) * U32 * (a + b) for a, b in zip(ga_, bs_))
                            for ga_, bs_ in zip(gabs, bsum)]
                for l in range(Ld):
                    for k, name in enumerate(("W_self", "W_neigh", "b")):
                        err = np.abs(np.asarray(gpu_g[l][k], np.float64) - ref_g[l][k])
                        ratio = float(np.max(err / (bsum[l][k] + 1e-30)))
                        elem_worst = max(elem_worst, ratio)
                        assert np.all(err <= bsum[l][k]), (f"step {t + w} layer {l} d{name} elementwise", ratio,
                                                           np.unravel_index(np.argmax(err / (bsum[l][k] + 1e-30)),
                                                                            err.shape))
            assert abs(gpu_loss - ref_loss) <= REL * abs(ref_loss) + 1e-6, (t + w, gpu_loss, ref_loss)
            L = len(dims) - 1
            for l in range(L):
                for k, name in enumerate(("W_self", "W_neigh", "b")):
                    rel = REL * 2.0 ** (L - 1 - l)
                    worst = max(worst, close(gpu_g[l][k], ref_g[l][k], f"step {t + w} layer {l} d{name}",
                                             rows=l == L - 1, rel=rel) / rel)
            ctx.sgd(lr)
            ref_w = S.sgd(ref_w, ref_g, lr)
            if first:                             # W_gpu = fl(W - lr g_gpu): drift bound of the next step
                Ld = len(dims) - 1
                e_w = [tuple((ew + lr * bsum[l][k]) * (1 + 2 * U32)
                             + 2 * U32 * (np.abs(ref_w[l][k]) + lr * np.abs(ref_g[l][k]))
                             for k, ew in enumerate(e_w[l])) for l in range(Ld)]
            for l in range(len(dims) - 1):
                got = ctx.params(l)
                if first:                         # weights elementwise within the drift bound
                    for k in range(3):
                        errw = np.abs(np.asarray(got[k], np.float64) - ref_w[l][k])
                        assert np.all(errw <= e_w[l][k] + 1e-30), ("weights elementwise", t + w, l, k,
                                                                  float(np.max(errw / (e_w[l][k] + 1e-30))))
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
    print(f"[train parity] worst gradient error / tolerance {worst:.3f} (normwise, every step); "
          f"elementwise (every step) worst |err| / bound {elem_worst:.3e} ({precision})")
    return worst
