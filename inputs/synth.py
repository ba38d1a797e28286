"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module is INPUT GENERATION ONLY.  It holds none of the method's
arithmetic (no sampler, no Philox, no scores, no feature values): it builds
the graph G(V, E), the contiguous-range partition bounds that
define V_p^l and the per-partition training-seed sets.  Node features
are NOT produced here: the oracle (oracle/orc.c) and the CUDA library
(paper_2410_22697_b200/csrc) each synthesise them with their own Philox from
`feat_seed`.

Graph recipe ("planted-block R-MAT", DESIGN.md §Input recipe):
  * V = [0, N) is cut into 8 contiguous blocks b (block boundaries b*N//8).
  * Each raw edge picks a source block uniformly, a source inside that block by
    R-MAT(a=.57, b=.19, c=.19, d=.05) over the block (skewed degrees), and with
    probability 1-mu a destination inside the same block (R-MAT), otherwise in
    a uniformly chosen block (R-MAT inside it).  mu is the per-config
    "cross-block" knob that sets the halo/local ratio.
  * Ids are randomly relabelled inside each block, the edge set is
    symmetrised, self-loops are dropped and duplicates removed; batches are
    added until nnz (directed entries) is within 2% of the target.
  * Partitions are P contiguous ranges bounds[q] = q*N//P (aligned to the
    blocks whenever P divides 8).
  * Training nodes: each node independently with probability `train_frac`.
All randomness is numpy PCG64 seeded from `graph_seed`.
"""
from __future__ import annotations

import dataclasses
import hashlib
import os
from typing import List, Optional

import numpy as np

GRAPH_SEED = 24102269
FEAT_SEED = GRAPH_SEED + 1
RUN_SEED = GRAPH_SEED + 2

_A, _B, _C = 0.57, 0.19, 0.19   # R-MAT quadrant probabilities (d = 0.05)


@dataclasses.dataclass
class GraphConfig:
    name: str
    n_nodes: int
    nnz_target: int
    feat_dim: int
    mu: float
    train_frac: float
    fanouts: List[int]            # GNN-layer order, input layer first (DGL), e.g. [10, 25]
    batch: int
    graph_seed: int = GRAPH_SEED


# BASELINE.json "configs"; nnz targets follow SURVEY §8(c) reading #27.
CONFIGS = {
    "cfg1": GraphConfig("cfg1", 10_000, 100_000, 64, 0.2, 1.0, [10, 25], 256),
    "arxiv": GraphConfig("arxiv", 169_343, 2 * 1_166_243, 128, 0.6, 0.537, [10, 25], 1000),
    "reddit": GraphConfig("reddit", 232_965, 114_615_892, 602, 0.05, 0.659, [10, 25], 1000),
    "products": GraphConfig("products", 2_449_029, 2 * 61_859_140, 100, 0.2, 0.080, [5, 10, 15], 2000),
    "papers": GraphConfig("papers", 111_059_956, 2 * 1_615_685_872, 128, 0.15, 0.0109, [5, 10, 15], 2000),
    # 1/32-scale papers100M shape (same degree, dims, train fraction, fanout) for routine parity runs
    "papers_s32": GraphConfig("papers_s32", 111_059_956 // 32, 2 * 1_615_685_872 // 32, 128, 0.15, 0.0109,
                              [5, 10, 15], 2000),
}


@dataclasses.dataclass
class Graph:
    n_nodes: int
    indptr: np.ndarray            # int64 [N+1]
    cols: np.ndarray              # int32 [nnz], each row ascending, no dups / self loops
    train_mask: np.ndarray        # bool [N]

    @property
    def nnz(self) -> int:
        return int(self.cols.shape[0])


@dataclasses.dataclass
class PartitionInput:
    """Host arrays for one partition p (what mgnn_partition_desc / orc_part_new take)."""
    part_id: int
    n_parts: int
    n_global: int
    bounds: np.ndarray            # int64 [P+1]
    indptr: np.ndarray            # int64 [hi-lo+1], local rows, starting at 0
    cols: np.ndarray              # int32 view of the global cols for rows lo..hi-1
    train_ids: np.ndarray         # int32 sorted local train ids


def _rmat_in(rng: np.random.Generator, m: int, size: np.ndarray) -> np.ndarray:
    """m R-MAT row draws mapped into [0, size) (size may be per-edge)."""
    levels = max(1, int(np.ceil(np.log2(max(2, int(np.max(size)))))))
    x = np.zeros(m, dtype=np.int64)
    for _ in range(levels):
        r = rng.random(m, dtype=np.float32)
        # row bit is 1 for quadrants c, d  (P(c or d) = 0.24)
        x = (x << 1) | (r >= (_A + _B)).astype(np.int64)
    # scale [0, 2^levels) -> [0, size), preserving the skew toward low ids
    return (x * size.astype(np.int64)) >> levels


def _raw_edges(rng: np.random.Generator, m: int, n: int, mu: float):
    nb = 8
    blo = (np.arange(nb + 1, dtype=np.int64) * n) // nb
    bsz = np.diff(blo)
    sb = rng.integers(0, nb, size=m)
    u = blo[sb] + _rmat_in(rng, m, bsz[sb])
    cross = rng.random(m, dtype=np.float32) < mu
    db = np.where(cross, rng.integers(0, nb, size=m), sb)
    v = blo[db] + _rmat_in(rng, m, bsz[db])
    return u, v


def _unique_sorted(x: np.ndarray) -> np.ndarray:
    """Sorted unique int64 keys (torch's multithreaded CPU sort; identical result to np.unique)."""
    import torch
    return torch.unique(torch.from_numpy(x), sorted=True).numpy()


def generate(cfg: GraphConfig, cache_dir: Optional[str] = "/tmp/mgnn_inputs") -> Graph:
    """Deterministic planted-block R-MAT graph for `cfg` (see module doc)."""
    key = hashlib.sha1(repr(dataclasses.astuple(cfg)).encode() + b"v2").hexdigest()[:12]
    path = None
    if cache_dir:
        os.makedirs(cache_dir, exist_ok=True)
        path = os.path.join(cache_dir, f"{cfg.name}_{key}.npz")
        if os.path.exists(path):
            z = np.load(path)
            return Graph(cfg.n_nodes, z["indptr"], z["cols"], z["train_mask"])
    n = cfg.n_nodes
    rng = np.random.default_rng(cfg.graph_seed)
    nb = 8
    blo = (np.arange(nb + 1, dtype=np.int64) * n) // nb
    relabel = np.empty(n, dtype=np.int64)
    for b in range(nb):
        relabel[blo[b]:blo[b + 1]] = blo[b] + rng.permutation(blo[b + 1] - blo[b])
    keys = np.zeros(0, dtype=np.int64)
    target = cfg.nnz_target
    m = max(1024, target // 2)
    chunk = 1 << 24
    while True:
        parts = [keys]
        left = m
        while left > 0:
            c = min(chunk, left)
            u, v = _raw_edges(rng, c, n, cfg.mu)
            u = relabel[u]
            v = relabel[v]
            keep = u != v
            u, v = u[keep], v[keep]
            parts.append(u * n + v)
            parts.append(v * n + u)
            left -= c
        new_keys = _unique_sorted(np.concatenate(parts))
        gained = new_keys.shape[0] - keys.shape[0]
        keys = new_keys
        if keys.shape[0] >= 0.98 * target or gained <= 0:
            break
        # next batch sized from the observed yield of this one
        m = int((target - keys.shape[0]) * m / max(gained, 1) * 1.02) + 1024
    src = keys // n
    cols = (keys % n).astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    train_mask = rng.random(n) < cfg.train_frac
    g = Graph(n, indptr, cols, train_mask)
    if path:
        tmp = f"{path}.{os.getpid()}.tmp.npz"
        np.savez(tmp, indptr=indptr, cols=cols, train_mask=train_mask)
        os.replace(tmp, path)
    return g


def from_edges(n: int, edges, train_mask=None) -> Graph:
    """Symmetric simple CSR from an undirected edge list (tests / worked examples)."""
    s = set()
    for a, b in edges:
        if a != b:
            s.add((a, b))
            s.add((b, a))
    keys = np.array(sorted(a * n + b for a, b in s), dtype=np.int64)
    src = keys // n if keys.size else np.zeros(0, np.int64)
    cols = (keys % n).astype(np.int32) if keys.size else np.zeros(0, np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    if train_mask is None:
        train_mask = np.ones(n, dtype=bool)
    return Graph(n, indptr, cols, np.asarray(train_mask, dtype=bool))


def random_graph(n: int, p_edge: float, seed: int, train_frac: float = 1.0) -> Graph:
    """Small Erdos-Renyi graph for brute-force tests."""
    rng = np.random.default_rng(seed)
    edges = [(a, b) for a in range(n) for b in range(a + 1, n) if rng.random() < p_edge]
    return from_edges(n, edges, rng.random(n) < train_frac)


def range_bounds(n: int, n_parts: int) -> np.ndarray:
    return (np.arange(n_parts + 1, dtype=np.int64) * n) // n_parts


def partition(g: Graph, n_parts: int, bounds: Optional[np.ndarray] = None) -> List[PartitionInput]:
    """Split `g` into P contiguous-range partitions (first level of P:63)."""
    if bounds is None:
        bounds = range_bounds(g.n_nodes, n_parts)
    bounds = np.asarray(bounds, dtype=np.int64)
    out = []
    for p in range(n_parts):
        lo, hi = int(bounds[p]), int(bounds[p + 1])
        ip = g.indptr[lo:hi + 1]
        indptr = (ip - ip[0]).astype(np.int64)
        cols = np.ascontiguousarray(g.cols[ip[0]:ip[-1]])
        train_ids = (np.nonzero(g.train_mask[lo:hi])[0] + lo).astype(np.int32)
        out.append(PartitionInput(p, n_parts, g.n_nodes, bounds, np.ascontiguousarray(indptr), cols, train_ids))
    return out


def hash_relabel(g: Graph, seed: int = GRAPH_SEED + 5) -> Graph:
    """The same graph under a uniformly random relabelling of its ids: contiguous-range partitions of
    the result are a hash partition of the original (SURVEY §8(f) NEXT-4's worst-case halo stress)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = g.n_nodes
    new_of = rng.permutation(n).astype(np.int64)           # old id -> new id
    old_of = np.empty(n, np.int64)
    old_of[new_of] = np.arange(n, dtype=np.int64)
    deg = np.diff(g.indptr)[old_of]
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=indptr[1:])
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    starts = g.indptr[old_of]
    idx = np.arange(indptr[-1], dtype=np.int64) - np.repeat(indptr[:-1], deg) + np.repeat(starts, deg)
    cols = new_of[g.cols[idx]]
    key = src * n + cols                                    # rows ascending after relabelling
    order = np.argsort(key, kind="stable")
    cols = cols[order].astype(np.int32)
    return Graph(n, indptr, cols, g.train_mask[old_of])


def describe(g: Graph, parts: List[PartitionInput]) -> dict:
    """Achieved shape statistics reported beside every result."""
    deg = np.diff(g.indptr)
    halo = []
    seen = np.zeros(g.n_nodes, dtype=bool)
    for pi in parts:
        lo, hi = int(pi.bounds[pi.part_id]), int(pi.bounds[pi.part_id + 1])
        c = pi.cols
        seen[:] = False
        seen[c] = True                      # distinct neighbours without a sort (papers: 400M per part)
        n_h = int(seen[:lo].sum()) + int(seen[hi:].sum())
        halo.append(n_h / max(1, hi - lo))
    # degree histogram in power-of-two buckets: bucket b counts nodes with 2^(b-1) <= deg < 2^b (b = 0: deg 0)
    b = np.zeros(deg.shape, np.int64)
    nz = deg > 0
    b[nz] = np.floor(np.log2(deg[nz])).astype(np.int64) + 1
    hist = np.bincount(b, minlength=1).tolist() if deg.size else []
    return {
        "n_nodes": g.n_nodes, "nnz": g.nnz, "avg_deg": g.nnz / max(1, g.n_nodes),
        "max_deg": int(deg.max()) if deg.size else 0, "median_deg": float(np.median(deg)) if deg.size else 0.0,
        "n_train": int(g.train_mask.sum()), "halo_over_local": [round(h, 4) for h in halo],
        "deg_hist_log2": hist, "deg_hist_note": "bucket 0: degree 0; bucket b >= 1: 2^(b-1) <= degree < 2^b",
    }


# ------------------------------------------------------------------ consumer weights (A14)
HIDDEN = 128                    # GraphSAGE hidden size (unstated in the paper -> 128)
N_CLASSES = {"cfg1": 16, "arxiv": 40, "reddit": 41, "products": 47, "papers": 172, "papers_s32": 172}
SAGE_SEED = GRAPH_SEED + 3


def sage_dims(feat_dim: int, n_layers: int, n_classes: int, hidden: int = HIDDEN) -> List[int]:
    """[D, hidden, ..., hidden, C]: layer widths of an n_layers-deep GraphSAGE."""
    return [feat_dim] + [hidden] * (n_layers - 1) + [n_classes]


def sage_weights(dims: List[int], seed: int = SAGE_SEED):
    """Random-init fp32 weights, one (W_self, W_neigh, bias) triple per layer in nn.Linear
    layout [d_out][d_in]: Glorot-uniform matrices, small uniform biases.  Input generation
    only (the stand-in for a trained model; there are no trained weights to load)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for l in range(len(dims) - 1):
        d_in, d_out = dims[l], dims[l + 1]
        lim = float(np.sqrt(6.0 / (d_in + d_out)))
        ws = rng.uniform(-lim, lim, (d_out, d_in)).astype(np.float32)
        wn = rng.uniform(-lim, lim, (d_out, d_in)).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, d_out).astype(np.float32)
        out.append((ws, wn, b))
    return out


def node_labels(n_nodes: int, n_classes: int, seed: int = SAGE_SEED + 1) -> np.ndarray:
    """Synthetic class labels (int32 [n_nodes], uniform in [0, n_classes)): the stand-in for the
    dataset's labels the training step's loss needs (input generation only)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, n_classes, size=n_nodes, dtype=np.int64).astype(np.int32)
