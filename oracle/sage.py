"""CPU oracle of the GraphSAGE-mean consumer.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg, never by the product package.  Shares no code
with the CUDA path (paper_2410_22697_b200/csrc/sage.cu).

What it computes (Alg.1 l.6-7: each trainer "computes the
forward pass" of GraphSAGE over the minibatch's sampled blocks; P:343 names
GraphSAGE with DGL's mean aggregator; P:133-137 the DDP step we stop short of).
DGL's SAGEConv('mean') on block b_l with input features H^l:

    H^{l+1}[i] = act( W_self^l H^l[i] + W_neigh^l * mean_{j in N_l(i)} H^l[j] + b^l )

with i over the destination nodes of the block (the first |dst| source nodes,
DGL block convention), act = ReLU between layers and identity after the last,
and mean over an empty neighbourhood = 0.  Layer l uses the block of sampling
hop h = L-1-l (the hop nearest the seeds feeds the last layer).  Everything is
float64, one destination node at a time (no blocking, no fusion).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def sage_layer(h_in: np.ndarray, n_dst: int, off: np.ndarray, nbr: np.ndarray,
               w_self: np.ndarray, w_neigh: np.ndarray, bias: np.ndarray, relu: bool) -> np.ndarray:
    """One SAGEConv('mean') layer over one block.

    h_in [n_src][d_in] (float64), destination i = source row i for i < n_dst;
    off [n_dst+1], nbr [off[-1]] = source rows of each destination's sampled
    neighbours; w_* [d_out][d_in] (nn.Linear layout), bias [d_out]."""
    d_out = w_self.shape[0]
    out = np.zeros((n_dst, d_out), np.float64)
    for i in range(n_dst):
        nb = nbr[off[i]:off[i + 1]]
        if len(nb):
            mean = h_in[nb].sum(axis=0) / len(nb)
        else:
            mean = np.zeros(h_in.shape[1], np.float64)
        z = w_self @ h_in[i] + w_neigh @ mean + bias
        out[i] = np.maximum(z, 0.0) if relu else z
    return out


def sage_forward(X: np.ndarray, blocks: Sequence[Tuple[np.ndarray, np.ndarray]],
                 weights: Sequence[Tuple[np.ndarray, np.ndarray, np.ndarray]]) -> List[np.ndarray]:
    """Forward pass over the sampled blocks of one minibatch.

    X [|F_L|][D]: input features of F_L (row i = node F_L[i]).
    blocks[h] = (off_h [|F_h|+1], nbr_h) for sampling hop h = 0..L-1, nbr_h
    holding POSITIONS in F_{h+1} (so |F_h| = len(off_h) - 1).
    weights[l] = (W_self, W_neigh, b) of layer l = 0..L-1 (input layer first).
    Returns [H^1, ..., H^L]; H^L [|F_0|][C] are the logits of the seeds."""
    L = len(weights)
    assert len(blocks) == L
    h = np.asarray(X, np.float64)
    outs = []
    for l in range(L):
        hop = L - 1 - l
        off, nbr = blocks[hop]
        ws, wn, b = (np.asarray(a, np.float64) for a in weights[l])
        h = sage_layer(h, len(off) - 1, np.asarray(off), np.asarray(nbr), ws, wn, b, relu=l < L - 1)
        outs.append(h)
    return outs


def positions(frontier: np.ndarray, cols_global: np.ndarray) -> np.ndarray:
    """Map global ids of sampled neighbours to their positions in F_L (the oracle's blocks
    hold global ids; F_{h+1} is a prefix of F_L, so a position in F_L is a position in F_{h+1})."""
    pos = {int(v): i for i, v in enumerate(frontier)}
    return np.array([pos[int(v)] for v in cols_global], np.int64)


# ---------------------------------------------------------------------------------------------
# Training step ("GraphSAGE forward/backward with ncclAllReduce gradients",
# Alg.1 l.6-8: forward, loss, backward, gradient all-reduce across trainers (DDP),
# optimizer step).  Loss = mean softmax cross-entropy over the seeds (F_0) of the minibatch; the
# gradient of a DDP step over P trainers is the average of the trainers' gradients.
# Written out by hand (chain rule, layer by layer, one destination row at a time), float64.

def sage_forward_cache(X, blocks, weights):
    """Forward pass keeping what the backward needs: per layer (h_in, mean rows, z)."""
    L = len(weights)
    h = np.asarray(X, np.float64)
    cache = []
    for l in range(L):
        off, nbr = blocks[L - 1 - l]
        n = len(off) - 1
        ws, wn, b = (np.asarray(a, np.float64) for a in weights[l])
        mean = np.zeros((n, h.shape[1]))
        for i in range(n):
            nb = nbr[off[i]:off[i + 1]]
            if len(nb):
                mean[i] = h[nb].sum(axis=0) / len(nb)
        z = h[:n] @ ws.T + mean @ wn.T + b
        cache.append((h, mean, z))
        h = np.maximum(z, 0.0) if l < L - 1 else z
    return h, cache


def softmax_xent(logits, labels):
    """Mean cross-entropy of rows of logits against integer labels; returns (loss, dlogits)."""
    z = np.asarray(logits, np.float64)
    zm = z - z.max(axis=1, keepdims=True)
    e = np.exp(zm)
    p = e / e.sum(axis=1, keepdims=True)
    n = z.shape[0]
    loss = float(-np.mean(np.log(p[np.arange(n), labels])))
    d = p.copy()
    d[np.arange(n), labels] -= 1.0
    return loss, d / n


def sage_backward(blocks, weights, cache, dlogits):
    """Gradients (dW_self, dW_neigh, db) per layer of the loss whose gradient w.r.t. the
    logits is dlogits.  Backward of H' = act(H[:n] Ws^T + mean(H[N(i)]) Wn^T + b):
    dZ = dH' * [Z > 0] (hidden layers), dWs = dZ^T H[:n], dWn = dZ^T mean, db = sum_i dZ_i,
    dH[i] += dZ_i Ws (i < n), dH[j] += (dZ_i Wn) / |N(i)| for every sampled neighbour j of i."""
    L = len(weights)
    grads = [None] * L
    dh = np.asarray(dlogits, np.float64)
    for l in range(L - 1, -1, -1):
        off, nbr = blocks[L - 1 - l]
        h, mean, z = cache[l]
        n = len(off) - 1
        ws, wn, _ = (np.asarray(a, np.float64) for a in weights[l])
        dz = dh if l == L - 1 else dh * (z > 0.0)
        grads[l] = (dz.T @ h[:n], dz.T @ mean, dz.sum(axis=0))
        if l > 0:
            dh_in = np.zeros_like(h)
            dh_in[:n] += dz @ ws
            dmean = dz @ wn
            for i in range(n):
                nb = nbr[off[i]:off[i + 1]]
                for j in nb:
                    dh_in[j] += dmean[i] / len(nb)
            dh = dh_in
    return grads


def sage_loss_grads(X, blocks, weights, labels):
    """(loss, grads) of one minibatch (labels of the seeds F_0, in F_0 order)."""
    logits, cache = sage_forward_cache(X, blocks, weights)
    loss, dlog = softmax_xent(logits, labels)
    return loss, sage_backward(blocks, weights, cache, dlog)


def sgd(weights, grads, lr):
    """W <- W - lr * g for every tensor (plain SGD, the optimizer of the training step)."""
    return [tuple(np.asarray(w, np.float64) - lr * np.asarray(g, np.float64) for w, g in zip(wl, gl))
            for wl, gl in zip(weights, grads)]
