"""Parity of the TIMED schedule (tests/ only): bench.py's loop, checked against the oracle.

paper_2410_22697_b200.schedule.PrepareAhead is the loop bench.py times: two streams (sampling of
window w+1 on stream A beside classify/gather/score of window w on stream B), programmatic
dependent launches (the library default), the 256 MB L2 flush before every iteration, CUDA events
around every iteration.  This driver runs exactly that loop with no host synchronisation between
iterations; after each consumed window it only ENQUEUES device-side copies on stream B (counters
of every instance, and for two instances per window their hop sizes, F_L, every hop's offsets and
columns, and sampled X rows), then compares everything with the oracle (Alg.2 step by
step, oracle/orc.c) once the run is over:
  * counts (|F_L|, local, hits, misses, evicted, rows fetched) of every instance of every window,
  * hop sizes, F_L, offsets and columns of the captured instances, element by element,
  * X rows of the captured instances: every row (x_rows = 0) or `x_rows` evenly spaced positions,
  * BUF membership, S_E, S_A, slot_of and BUF rows after the last window (0 ULP).
"""
from __future__ import annotations

import numpy as np

from inputs import synth
from oracle import oracle as O
from tests.parity_util import assert_bits_equal


class _Perturbed:
    """Race probe: forwards to the context but first enqueues a random-length spin kernel on the stream
    of every sample / lookup_gather / score call, so the two streams interleave differently on every
    run (compute-sanitizer is closed on this pool; an ordering bug between the streams shows up here as
    a mismatch with the oracle)."""

    def __init__(self, ctx, seed: int, max_cycles: int = 400_000):
        self._c = ctx
        self._rng = np.random.default_rng(seed)
        self._max = max_cycles

    def __getattr__(self, k):
        return getattr(self._c, k)

    def _spin(self, stream):
        import torch
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(self._rng.integers(0, self._max)))

    def sample(self, sl, tt, n, stream=None, **kw):
        self._spin(stream)
        return self._c.sample(sl, tt, n, stream=stream, **kw)

    def sample_ptr(self, sl, tt, n, sp, cp, on_host, stream=None):
        self._spin(stream)
        return self._c.sample_ptr(sl, tt, n, sp, cp, on_host, stream)

    def lookup_gather(self, sl, stream=None):
        self._spin(stream)
        return self._c.lookup_gather(sl, stream)

    def relabel(self, sl, stream=None):
        self._spin(stream)
        return self._c.relabel(sl, stream)

    def score(self, sl, stream=None):
        self._spin(stream)
        return self._c.score(sl, stream)


def run_schedule_parity(g: synth.Graph, P: int, D: int, fanouts, batch: int, f_bp: int, gamma: float, delta: int,
                        window: int, n_windows: int, x_rows: int = 2048, warm: int = 0, flush_bytes: int = 256 << 20,
                        run_seed: int = synth.RUN_SEED, feat_seed: int = synth.FEAT_SEED, rows_bound: int = -1,
                        perturb=None, relabel_stream: bool = False, sm_split: int = 0, sampling_priority: int = 0):
    import torch
    from paper_2410_22697_b200 import pipeline as PL
    from paper_2410_22697_b200.schedule import PrepareAhead

    parts = synth.partition(g, P)
    alpha = float(O.alpha_default(gamma, delta))
    ctx = PL.build_context(0, parts, D, feat_seed)
    ctx.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    if rows_bound < 0:                 # realistic arenas, as bench.py sizes them
        rows_bound = PL.estimate_rows_bound(ctx, fanouts, batch, run_seed)
    ctx.sampler_config(fanouts, batch, run_seed, window, rows_bound=rows_bound)
    if sm_split:                       # mgnn_sm_partition: the calls run on green-context SM subsets
        g_sms, p_sms = ctx.sm_partition(sm_split)
        assert g_sms >= 1 and p_sms >= 1 and g_sms + p_sms <= torch.cuda.get_device_properties(0).multi_processor_count
    L = len(fanouts)
    n_inst = P * window
    pipe = PrepareAhead(ctx if perturb is None else _Perturbed(ctx, perturb), window, t0=1, flush_bytes=flush_bytes,
                        relabel_stream=relabel_stream, sampling_priority=sampling_priority)
    grabbed = []
    xpos_n = x_rows

    def grab(slot, t0, sB):
        wv = ctx.window(slot)
        wi = len(grabbed)
        picks = sorted({(3 * wi) % n_inst, (5 * wi + n_inst // 2 + 1) % n_inst})
        rec = {"t0": t0, "picks": picks}
        with torch.cuda.stream(sB):
            rec["counts"] = PL.device_view(wv.counts, (n_inst, 8), "i8").clone()
            hs_all = PL.device_view(wv.hop_size, (n_inst, 9), "i8")
            rec["hs"] = hs_all.clone()
            fr = PL.device_view(wv.frontier, (n_inst, wv.rows_stride), "i4")
            X = PL.device_view(wv.X, (n_inst, wv.rows_stride, wv.pitch), "f4")
            for m in picks:
                U = hs_all[m, L]
                rec[f"fr{m}"] = fr[m].clone()
                if xpos_n > 0:               # x_rows evenly spaced rows
                    k = torch.arange(xpos_n, device="cuda", dtype=torch.int64)
                    pos = torch.minimum((k * (U - 1)) // max(1, xpos_n - 1), U - 1)
                    rec[f"xpos{m}"] = pos
                    rec[f"x{m}"] = X[m].index_select(0, pos)[:, :D].clone()
                else:                        # x_rows = 0: every row of the arena (compared up to |F_L|)
                    rec[f"xpos{m}"] = None
                    rec[f"x{m}"] = X[m][:, :D].clone()
                for i in range(L):
                    rec[f"off{m}_{i}"] = PL.device_view(wv.offsets[i], (n_inst, wv.off_stride[i]), "i8")[m].clone()
                    rec[f"cols{m}_{i}"] = PL.device_view(wv.cols[i], (n_inst, wv.col_stride[i]), "i4")[m].clone()
        grabbed.append(rec)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_windows)]
    for i in range(n_windows):                   # the bench loop, no host sync inside
        pipe.iteration(events=ev[i], after_consume=grab, prepare_next=i + 1 < n_windows)
    torch.cuda.synchronize()
    ctx.counts(pipe.slot ^ 1)                    # raises MGNN_EOVERFLOW if any window overflowed its arena
    ms = [a.elapsed_time(b) for a, b in ev]
    snaps = {pid: ctx.snapshot(lp, rows=True) for lp, pid in enumerate(ctx.parts)}
    lps = {pid: lp for lp, pid in enumerate(ctx.parts)}

    # ---------------- the oracle, step by step (Alg.2 order), same inputs
    W = O.World(parts, D, feat_seed)
    for p in W.parts:
        p.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    stats = {"steps": 0, "hits": 0, "misses": 0, "evicted": 0, "checked_instances": 0, "x_rows": 0}
    for rec in grabbed:
        counts = rec["counts"].cpu().numpy()
        hs = rec["hs"].cpu().numpy()
        for w in range(window):
            step = rec["t0"] + w
            for pid, lp in lps.items():
                op = W.parts[pid]
                op.step(run_seed, step, fanouts, batch)
                m = lp * window + w
                oc = op.counts()
                gc = counts[m]
                got = [gc[0], gc[1], gc[2], gc[3], gc[4], gc[6]]
                want = [oc["n_nodes"], oc["n_local"], oc["n_hit"], oc["n_miss"], oc["n_evicted"], oc["rows_fetched"]]
                assert got == want, ("counts", pid, step, got, want)
                stats["steps"] += 1
                stats["hits"] += oc["n_hit"]
                stats["misses"] += oc["n_miss"]
                stats["evicted"] += oc["n_evicted"]
                if m not in rec["picks"]:
                    continue
                stats["checked_instances"] += 1
                ohs = np.array(op.hop_sizes(), np.int64)
                assert_bits_equal(hs[m, :L + 1], ohs, f"hop sizes p{pid} t{step}")
                U = int(ohs[L])
                F = op.frontier()
                gF = rec[f"fr{m}"].cpu().numpy()[:U]
                assert_bits_equal(gF, F, f"F_L p{pid} t{step}")
                for i in range(L):
                    off, cols = op.hop_block(i)
                    goff = rec[f"off{m}_{i}"].cpu().numpy()[:ohs[i] + 1]
                    assert_bits_equal(goff, off, f"offsets hop{i} p{pid} t{step}")
                    gc_ = rec[f"cols{m}_{i}"].cpu().numpy()[:int(off[-1])]
                    assert np.all(gc_ < ohs[i + 1])
                    assert_bits_equal(gF[gc_].astype(np.int32) if len(gc_) else gc_, cols,
                                      f"cols hop{i} p{pid} t{step}")
                X = op.features()
                if rec[f"xpos{m}"] is None:
                    assert_bits_equal(rec[f"x{m}"][:U].cpu().numpy(), X, f"X p{pid} t{step}")
                    stats["x_rows"] += U
                else:
                    pos = rec[f"xpos{m}"].cpu().numpy()
                    assert_bits_equal(rec[f"x{m}"].cpu().numpy(), X[pos], f"X p{pid} t{step}")
                    stats["x_rows"] += len(pos)
    for pid, lp in lps.items():
        gs = snaps[pid]
        os_ = W.parts[pid].buffer_state(rows=True)
        for k in ("node_of_slot", "se", "sa", "slot_of", "rows"):
            assert_bits_equal(gs[k], os_[k], f"{k} p{pid} after the last window")
    ctx.close()
    W.close()
    stats["ms_per_window"] = ms
    return stats
