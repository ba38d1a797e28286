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
