"""Shared driver for GPU-vs-oracle parity (tests/ only).

Runs the CUDA path (window-batched) and the CPU oracle (step by step, the
paper's Alg.2 order) on the same seeded inputs and compares, per step and
per partition, element by element:
  * F_L (global ids) and |F_i| per hop,
  * per-hop CSR offsets and sampled columns (GPU: positions in F_{i+1},
    mapped back through F_L; oracle: global ids),
  * X (first D columns), bit-exact,
  * counts (nodes, local, hits, misses, evicted, rows fetched),
  * after each window: BUF membership per slot, S_E bits per slot, S_A bits
    per halo node (0 ULP, BASELINE.json north_star).
"""
from __future__ import annotations

import hashlib

import numpy as np

from inputs import synth
from oracle import oracle as O


def assert_bits_equal(a, b, what):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if a.dtype == np.float32:
        ok = np.array_equal(a.view(np.uint32), b.view(np.uint32))
    else:
        ok = np.array_equal(a, b)
    if not ok:
        bad = np.nonzero((a.view(np.uint32) != b.view(np.uint32)) if a.dtype == np.float32 else (a != b))
        idx = tuple(x[:5] for x in bad)
        raise AssertionError(f"{what}: {len(bad[0])} mismatches, first at {idx}: gpu={a[idx]} oracle={b[idx]}")


def run_parity(g: synth.Graph, P: int, D: int, fanouts, batch: int, f_bp: int, gamma: float, delta: int,
               theta_r: float, windows, run_seed: int = synth.RUN_SEED, feat_seed: int = synth.FEAT_SEED,
               alpha=None, hosted=None, sample_every: int = 1, check_x_rows: int = 0, ext_seeds=None,
               device: int = 0, exchange: bool = False, remote: bool = False, dense: bool = False,
               rows_bound: int = 0, bind_x: bool = False):
    """windows: list of window lengths run back to back from step 1."""
    from paper_2410_22697_b200 import pipeline as PL

    parts = synth.partition(g, P)
    if alpha is None:
        alpha = float(O.alpha_default(gamma, delta))
    W = O.World(parts, D, feat_seed, dense=dense)
    for p in W.parts:
        p.buffer_init(gamma, alpha, theta_r, delta, f_bp)
        p.set_expand_remote(remote)
    ctx = PL.build_context(device, parts, D, feat_seed, hosted, dense=dense)
    if remote:                        # NEXT-1: non-local frontier nodes sampled from their owners
        if hosted is not None:        # other partitions live elsewhere: replicate the global CSR
            ctx.load_global_csr(g.indptr, g.cols)
        ctx.expand_remote(True)
    if exchange:                      # multi-process: map the other ranks' tables (CUDA IPC, NVLink)
        PL.exchange_tables(ctx)
    ctx.buffer_init(gamma, alpha, theta_r, delta, f_bp)
    if rows_bound < 0:                # realistic arenas from a pilot (pipeline.estimate_rows_bound)
        rows_bound = PL.estimate_rows_bound(ctx, fanouts, batch, run_seed)
    ctx.sampler_config(fanouts, batch, run_seed, max(windows), rows_bound=rows_bound)
    x_user = {}
    if bind_x:                        # caller-owned X (mgnn_window_bind_x): torch tensors, NaN-filled
        import torch
        rs, pitch, mi = ctx.window_shape()
        for sl in (0, 1):
            x_user[sl] = torch.full((mi, rs, pitch), float("nan"), device="cuda", dtype=torch.float32)
            ctx.bind_x(sl, x_user[sl])
    lps = {pid: lp for lp, pid in enumerate(ctx.parts)}
    # static partition facts
    for pid, lp in lps.items():
        gi, gd = ctx.halo(lp)
        oi, od = W.parts[pid].halo()
        assert_bits_equal(gi, oi, f"halo ids p{pid}")
        assert_bits_equal(gd, od, f"deg_in p{pid}")
        assert ctx.part_info(lp)["cap"] == W.parts[pid].cap
    L = len(fanouts)
    t = 1
    slot = 0
    stats = {"steps": 0, "hits": 0, "misses": 0, "evicted": 0}
    digests = {pid: hashlib.sha256() for pid in lps}     # per-partition digest of everything compared
    for wlen in windows:
        seeds_arr = cnt_arr = None
        if ext_seeds is not None:
            n_lp = len(ctx.parts)
            seeds_arr = np.zeros((n_lp, wlen, batch), np.int32)
            cnt_arr = np.zeros((n_lp, wlen), np.int32)
            for pid, lp in lps.items():
                for w in range(wlen):
                    sd = ext_seeds(pid, t + w)
                    seeds_arr[lp, w, :len(sd)] = sd
                    cnt_arr[lp, w] = len(sd)
        ctx.sample(slot, t, wlen, seeds=seeds_arr, seed_counts=cnt_arr)
        ctx.lookup_gather(slot)
        ctx.score(slot)
        counts = ctx.counts(slot)
        for w in range(wlen):
            step = t + w
            for pid, lp in lps.items():
                op = W.parts[pid]
                op.step(run_seed, step, fanouts, batch,
                        seeds=None if ext_seeds is None else np.asarray(ext_seeds(pid, step), np.int32))
                m = lp * wlen + w
                oc = op.counts()
                gc = counts[m]
                got = [gc[0], gc[1], gc[2], gc[3], gc[4], gc[6]]
                want = [oc["n_nodes"], oc["n_local"], oc["n_hit"], oc["n_miss"], oc["n_evicted"], oc["rows_fetched"]]
                assert got == want, (pid, step, got, want)      # counts: every step
                digests[pid].update(np.asarray(got, np.int64).tobytes())
                # NVLink rows (counts[7]): misses + refills owned by a partition on another GPU
                refill = gc[5] if w == wlen - 1 else 0
                assert 0 <= gc[7] <= gc[3] + refill, (pid, step, gc[7])
                if not exchange:
                    assert gc[7] == 0, (pid, step, gc[7])
                stats["peer_rows"] = stats.get("peer_rows", 0) + int(gc[7])
                stats["steps"] += 1
                stats["hits"] += oc["n_hit"]
                stats["misses"] += oc["n_miss"]
                stats["evicted"] += oc["n_evicted"]
                if (step - 1) % sample_every:
                    continue
                inst = ctx.instance(slot, m, with_x=True)
                hs = op.hop_sizes()
                assert_bits_equal(inst["hop_size"], np.array(hs, np.int64), f"hop sizes p{pid} t{step}")
                F = op.frontier()
                assert_bits_equal(inst["frontier"], F, f"F_L p{pid} t{step}")
                for i in range(L):
                    off, cols = op.hop_block(i)
                    assert_bits_equal(inst[f"off{i}"], off, f"offsets hop{i} p{pid} t{step}")
                    gcols = inst["frontier"][inst[f"cols{i}"]] if len(cols) else inst[f"cols{i}"]
                    assert_bits_equal(gcols.astype(np.int32), cols, f"cols hop{i} p{pid} t{step}")
                    assert np.all(inst[f"cols{i}"] < hs[i + 1])
                X = op.features()
                if bind_x:                    # the rows landed in the caller's tensor
                    assert_bits_equal(x_user[slot][m, :X.shape[0], :D].cpu().numpy(), X, f"user X p{pid} t{step}")
                if check_x_rows and X.shape[0] > check_x_rows:
                    sel = np.linspace(0, X.shape[0] - 1, check_x_rows).astype(np.int64)
                    assert_bits_equal(inst["X"][sel], X[sel], f"X p{pid} t{step}")
                else:
                    assert_bits_equal(inst["X"], X, f"X p{pid} t{step}")
        for pid, lp in lps.items():
            gs = ctx.snapshot(lp, rows=True)
            os_ = W.parts[pid].buffer_state(rows=True)
            assert_bits_equal(gs["node_of_slot"], os_["node_of_slot"], f"BUF p{pid} after t{t + wlen - 1}")
            assert_bits_equal(gs["se"], os_["se"], f"S_E p{pid} after t{t + wlen - 1}")
            assert_bits_equal(gs["sa"], os_["sa"], f"S_A p{pid} after t{t + wlen - 1}")
            assert_bits_equal(gs["slot_of"], os_["slot_of"], f"slot_of p{pid} after t{t + wlen - 1}")
            assert_bits_equal(gs["rows"], os_["rows"], f"BUF rows p{pid} after t{t + wlen - 1}")
            for k in ("node_of_slot", "se", "sa", "slot_of"):
                digests[pid].update(np.ascontiguousarray(gs[k]).tobytes())
        t += wlen
        slot ^= 1
    stats["digest"] = {int(pid): h.hexdigest() for pid, h in digests.items()}
    if exchange:                      # peers may still read our tables until every rank is done
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        dist.barrier()
    ctx.close()
    W.close()
    return stats
