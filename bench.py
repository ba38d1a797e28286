"""Benchmark: sampled+feature-ready minibatches/s of the halo feature pipeline
(arXiv 2410.22697 prefetch + eviction) on B200, per BASELINE.json.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {mgnn,reference}]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, one rank per GPU)

Workload (BASELINE.json configs[1], fits one GPU): ogbn-arxiv-shaped synthetic
graph (169,343 nodes, ~2.33M directed edges, 128-dim fp32 features), fanout
[10, 25], batch 1000, P = 2 partitions per GPU (trainers), policy for P from
the paper's GPU optima: P=2 (f=.25, gamma=.995, Delta=32), P=4
(.50, .995, 32), P>=8 (.35, .995, 128); theta_R = 1.
One bench "step" = one WINDOW of 32 consecutive minibatch steps for every
partition on the GPU (sample, classify, gather, tally, decay, and the eviction
round that ends the window when 32 | Delta): 32 x 2 minibatches per GPU.
Software pipeline (the paper's prepare-ahead, Alg.1 l.9): in timed iteration i
the sampling of window i+1 runs on a second stream concurrently with the
classify/gather/score of window i; both streams join at the end of the
iteration.  Timing: per-iteration CUDA events, L2 flushed (256 MB write)
between timed iterations, max over ranks.  `e2e` drives the same pipeline
through the C ABI with the seeds in pinned HOST memory (H2D inside mgnn_sample)
and every window's per-minibatch counters read back to the host (D2H).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from inputs import synth  # noqa: E402

METRIC = "sampled+feature-ready minibatches/sec"
UNIT = "minibatches/s"
WINDOW = 32
PARTS_PER_GPU = 2
CFG = synth.CONFIGS["arxiv"]
REMOTE = False                     # NEXT-1 remote expansion (--remote)
DENSE = False                      # NEXT-1 dense S_A (--dense)

# Measurement policy (f_p in basis points, gamma, Delta) by config and total partitions P: the
# paper's GPU optima; theta_R = 1.
POLICY = {
    "cfg1": {2: (2500, 0.995, 64)},
    "arxiv": {2: (2500, 0.995, 32), 4: (5000, 0.995, 32), 8: (3500, 0.995, 128)},
    "reddit": {2: (3500, 0.995, 32), 4: (5000, 0.995, 256), 8: (5000, 0.95, 32)},
    "products": {2: (5000, 0.995, 32), 4: (5000, 0.995, 32), 8: (5000, 0.9995, 16)},
    "papers_s32": {8: (5000, 0.9995, 512)},
}
# partitions per GPU and window length per config (papers: all 8 partitions on one GPU at N=1,
# short windows so the statically bounded window arenas fit in HBM)
LAYOUT = {"cfg1": (2, 32), "arxiv": (2, 32), "reddit": (2, 32), "products": (2, 32), "papers_s32": (8, 8)}
WORKLOAD_TEXT = {
    "cfg1": "synthetic 10k-node graph, avg degree 10, 64-d fp32, fanout [10,25], batch 256 (BASELINE.json configs[0])",
    "arxiv": "ogbn-arxiv-shaped synthetic (169,343 nodes, ~2.33M directed edges, 128-d fp32), "
             "fanout [10,25], batch 1000 (BASELINE.json configs[1])",
    "reddit": "Reddit-shaped synthetic (232,965 nodes, ~114.6M directed edges, 602-d fp32), fanout [10,25], "
              "batch 1000 (BASELINE.json configs[2])",
    "products": "ogbn-products-shaped synthetic (2,449,029 nodes, ~123.7M directed edges, 100-d fp32), "
                "fanout [5,10,15], batch 2000 (BASELINE.json configs[3])",
    "papers_s32": "ogbn-papers100M-shaped synthetic at 1/32 scale (3.47M nodes, ~101M directed edges, 128-d fp32), "
                  "8 partitions, fanout [5,10,15], batch 2000 (BASELINE.json configs[4], scaled)",
}


def select_config(name: str) -> None:
    global CFG, WINDOW, PARTS_PER_GPU
    CFG = synth.CONFIGS[name]
    PARTS_PER_GPU, WINDOW = LAYOUT[name]


def policy_for(P: int):
    table = POLICY[CFG.name]
    k = min((q for q in table if q >= P), default=max(table))
    f_bp, gamma, delta = table[k]
    return f_bp, gamma, delta


def window_for(delta: int) -> int:
    """Steps per window: a window may end on an eviction step but not contain one earlier."""
    return min(WINDOW, delta) if delta > 0 else WINDOW


def workload(P: int) -> dict:
    f_bp, gamma, delta = policy_for(P)
    return {
        "workload": WORKLOAD_TEXT[CFG.name],
        "partitions": P, "partitions_per_gpu": PARTS_PER_GPU, "f_p": f_bp / 10000, "gamma": gamma, "delta": delta,
        "theta_r": 1.0, "window_steps": WINDOW, "minibatches_per_step_per_gpu": WINDOW * PARTS_PER_GPU,
        "l2": "flushed (256 MB write) between timed windows",
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every ~1 ms on a
    background thread while the timed region runs (the nvidia-smi clocks line of the
    profiling recipe, at a rate that resolves a few-millisecond region)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, cuda_index: int):
        self.idx = cuda_index
        self.rows = []
        self.stop = threading.Event()
        self.h = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(self.idx)
            want = (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
            for i in range(pynvml.nvmlDeviceGetCount()):        # match the CUDA device by PCI location
                h = pynvml.nvmlDeviceGetHandleByIndex(i)
                pci = pynvml.nvmlDeviceGetPciInfo(h)
                if (int(pci.domain), int(pci.bus), int(pci.device)) == want:
                    self.h = h
                    break
            if self.h is None:
                raise RuntimeError("no NVML device matches the CUDA device")
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # NVML unavailable: report it, do not fail the bench
            self.err = repr(e)
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.001)

    def __exit__(self, *a):
        self.stop.set()
        if self.h is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0,
                    "source": "nvml"}
        mask = 0
        for _, r in self.rows:
            mask |= r
        return {"sm_mhz": statistics.median(c for c, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": [n for n, bit in self.REASONS if mask & bit], "samples": len(self.rows), "source": "nvml"}


def peer_copy_gbs(src: int, dst: int):
    """Achievable NVLink bandwidth: 256 MB copy from GPU src to GPU dst (CUDA events, best of 5)."""
    import torch
    if src == dst:
        return None
    try:
        a = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{src}")
        b = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dst}")
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a, non_blocking=True)
            e1.record()
            torch.cuda.synchronize(src)
            torch.cuda.synchronize(dst)
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        return (256 << 20) / (best / 1e3) / 1e9
    except Exception:
        return None


# ---------------------------------------------------------------- oracle timings (test infrastructure)
def oracle_rate(parts, P, f_bp, gamma, delta, budget_s: float, min_steps: int = 8):
    """Oracle (oracle/orc.c, single thread) on the same workload: minibatches/s over a bounded sample."""
    from oracle import oracle as O
    W = O.World(parts, CFG.feat_dim, synth.FEAT_SEED, dense=DENSE)
    alpha = O.alpha_default(gamma, delta)
    for p in W.parts:
        p.buffer_init(gamma, alpha, 1.0, delta, f_bp)
        p.set_expand_remote(REMOTE)
    t0 = time.perf_counter()
    n_mb, step = 0, 1
    while True:
        for p in W.parts:
            p.step(synth.RUN_SEED, step, CFG.fanouts, CFG.batch)
            n_mb += 1
        step += 1
        el = time.perf_counter() - t0
        if step > min_steps and el >= budget_s:
            break
    W.close()
    return n_mb / el, n_mb, el


def oracle_rate_threads(parts, P, f_bp, gamma, delta, budget_s: float):
    """The same oracle with one host thread per partition (the C steps release the GIL; partitions
    are independent between eviction rounds of their own buffers): SURVEY §8(d)'s P-thread rate."""
    import threading as th
    from oracle import oracle as O
    W = O.World(parts, CFG.feat_dim, synth.FEAT_SEED, dense=DENSE)
    alpha = O.alpha_default(gamma, delta)
    for p in W.parts:
        p.buffer_init(gamma, alpha, 1.0, delta, f_bp)
        p.set_expand_remote(REMOTE)
    counts = [0] * len(W.parts)
    t0 = time.perf_counter()

    def run(i):
        step = 1
        while time.perf_counter() - t0 < budget_s or step <= 8:
            W.parts[i].step(synth.RUN_SEED, step, CFG.fanouts, CFG.batch)
            counts[i] += 1
            step += 1

    ts = [th.Thread(target=run, args=(i,)) for i in range(len(W.parts))]
    for t_ in ts:
        t_.start()
    for t_ in ts:
        t_.join()
    el = time.perf_counter() - t0
    n_thr = len(ts)
    W.close()
    return sum(counts) / el, n_thr


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    global WINDOW
    P = PARTS_PER_GPU * args.gpus
    f_bp, gamma, delta = policy_for(P)
    WINDOW = window_for(delta)
    g = synth.generate(CFG)
    parts = synth.partition(g, P)
    # each reference "step" = the same 32 x (partitions on one GPU) minibatches, bounded by time
    per_step = WINDOW * PARTS_PER_GPU
    from oracle import oracle as O
    W = O.World(parts, CFG.feat_dim, synth.FEAT_SEED)
    alpha = O.alpha_default(gamma, delta)
    for p in W.parts:
        p.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    mine = W.parts[:PARTS_PER_GPU]
    t = 1
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for w in range(WINDOW):
            for p in mine:
                p.step(synth.RUN_SEED, t + w, CFG.fanouts, CFG.batch)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
        t += WINDOW
    W.close()
    total = sum(times)
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload(P),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} windows x {per_step} minibatches of partitions 0-1 (P={P}), "
                                   "single-threaded C oracle"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mgnn", choices=["mgnn", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-train-graph", action="store_true", help="training steps as eager launches")
    ap.add_argument("--remote", action="store_true",
                    help="NEXT-1: sample non-local frontier nodes from their owner's CSR")
    ap.add_argument("--dense", action="store_true", help="NEXT-1: dense S_A (every non-local node scorable)")
    ap.add_argument("--hash-partition", action="store_true",
                    help="NEXT-4 stress: partitions of a randomly relabelled graph (hash partitioner)")
    ap.add_argument("--config", default="arxiv", choices=sorted(LAYOUT),
                    help="workload (default: arxiv-shaped, BASELINE.json configs[1])")
    args = ap.parse_args()
    global WINDOW, REMOTE, DENSE
    select_config(args.config)
    REMOTE = args.remote
    DENSE = args.dense
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2410_22697_b200 import pipeline as PL

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        saved = os.dup(1)                 # keep stdout to the one JSON line: NCCL's banner goes to stderr
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    P = PARTS_PER_GPU * world
    f_bp, gamma, delta = policy_for(P)
    WINDOW = window_for(delta)
    g = synth.generate(CFG)
    if args.hash_partition:
        g = synth.hash_relabel(g)
    parts = synth.partition(g, P)
    hosted = list(range(PARTS_PER_GPU * rank, PARTS_PER_GPU * (rank + 1)))
    ctx = PL.build_context(local, parts, CFG.feat_dim, synth.FEAT_SEED, hosted, dense=args.dense)
    if world > 1:
        PL.exchange_tables(ctx)
    alpha = PL.alpha_default(gamma, delta)
    # INITIALIZE_PREFETCHER cost ("<1% of overall training"), CUDA events on the init stream
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    i0.record()
    ctx.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    i1.record()
    torch.cuda.synchronize()
    init_ms = i0.elapsed_time(i1)
    if args.remote:
        if world > 1:
            ctx.load_global_csr(g.indptr, g.cols)       # replicated global CSR on every GPU
        ctx.expand_remote(True)
    ctx.sampler_config(CFG.fanouts, CFG.batch, synth.RUN_SEED, WINDOW)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # Two streams = the paper's prepare-ahead overlap (Alg.1 l.9): NeighborSampler of window w+1
    # (needs no buffer state) runs on sA while window w is classified/gathered/scored on sB.
    sA = torch.cuda.Stream()
    sB = stream
    ev_sampled = [torch.cuda.Event(), torch.cuda.Event()]
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]

    def sample_async(sl, tt):
        sA.wait_event(ev_done[sl])            # slot free once its previous window was gathered + scored
        ctx.sample(sl, tt, WINDOW, stream=sA)
        ev_sampled[sl].record(sA)

    def consume(sl):
        sB.wait_event(ev_sampled[sl])
        ctx.lookup_gather(sl, sB)
        ctx.score(sl, sB)
        ev_done[sl].record(sB)

    t = 1
    slot = 0
    sample_async(0, t)
    for _ in range(args.warmup):
        sample_async(slot ^ 1, t + WINDOW)
        consume(slot)
        t += WINDOW
        slot ^= 1
    # ---------------- timed region (device path: inputs resident in HBM)
    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    launches0 = ctx.launch_count()
    ctx.profile(True)
    ctx.profile_read()
    hits = misses = 0
    barrier()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for i in range(K):
            flush.zero_()                      # L2 flush between timed iterations (not timed)
            ev[i][0].record(sB)
            sA.wait_event(ev[i][0])
            sample_async(slot ^ 1, t + WINDOW)  # window i+1: sampling stream
            consume(slot)                       # window i: buffer stream
            sB.wait_stream(sA)
            ev[i][1].record(sB)
            t += WINDOW
            slot ^= 1
        barrier()
        wall = time.perf_counter() - wall0
    launches = ctx.launch_count() - launches0
    gms, glaunch, gbytes = ctx.profile_read()
    ctx.profile(False)
    c = ctx.counts(slot ^ 1, stream)            # the last consumed window
    hits += int(c[:, 2].sum())
    misses += int(c[:, 3].sum())
    peer_rows = int(c[:, 7].sum())              # rows read from another GPU's table over NVLink
    ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(ms)
    mine_ms = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(mine_ms, op=dist.ReduceOp.MAX)
    max_ms = float(mine_ms.item())
    mb_total = WINDOW * PARTS_PER_GPU * world * K
    value = mb_total / (max_ms / 1e3)

    # ---------------- e2e: host seeds (pinned) -> C ABI -> counts back to host, every window
    # The seeds a user passes are this window's F_0; take them from the library's epoch order by
    # sampling the same steps first (sampling reads no buffer state), outside the timed region.
    n_inst = PARTS_PER_GPU * WINDOW
    E2E = max(3, K)
    t_e2e = t
    seeds_h, counts_h = [], []
    for i in range(E2E):
        ctx.sample(slot, t_e2e + i * WINDOW, WINDOW, stream=stream)
        wv = ctx.window(slot)
        n0 = PL.device_view(wv.hop_size, (wv.n_inst, 9), "i8")[:, 0].to(torch.int32)
        f0 = PL.device_view(wv.frontier, (wv.n_inst, wv.rows_stride), "i4")[:, :CFG.batch]
        seeds_h.append(f0.cpu().pin_memory())
        counts_h.append(n0.cpu().pin_memory())
    h2d = n_inst * CFG.batch * 4 + n_inst * 4
    d2h = n_inst * 8 * 8
    cbuf = [torch.zeros((n_inst, 8), dtype=torch.int64).pin_memory() for _ in range(2)]
    ev_cnt = [torch.cuda.Event(), torch.cuda.Event()]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_hits = 0

    def sample_host(sl, i):                    # H2D of window i's seeds inside mgnn_sample (stream A)
        sA.wait_event(ev_done[sl])
        ctx.sample_ptr(sl, t_e2e + i * WINDOW, WINDOW, seeds_h[i].data_ptr(), counts_h[i].data_ptr(), True, sA)
        ev_sampled[sl].record(sA)

    barrier()
    ev0.record(sB)
    sA.wait_event(ev0)
    sample_host(slot, 0)
    for i in range(E2E):                       # same two-stream pipeline, host buffers at both ends
        if i + 1 < E2E:
            sample_host(slot ^ 1, i + 1)
        sB.wait_event(ev_sampled[slot])
        ctx.lookup_gather(slot, sB)
        ctx.score(slot, sB)
        ctx.counts_async(slot, cbuf[i % 2].data_ptr(), sB)      # D2H of the window's counters
        ev_cnt[i % 2].record(sB)
        ev_done[slot].record(sB)
        if i >= 1:                             # read the previous window's counters on the host
            ev_cnt[(i - 1) % 2].synchronize()
            e2e_hits += int(cbuf[(i - 1) % 2][:, 2].sum())
        slot ^= 1
    ev1.record(sB)
    ev_cnt[(E2E - 1) % 2].synchronize()
    e2e_hits += int(cbuf[(E2E - 1) % 2][:, 2].sum())
    barrier()
    e2e_ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = WINDOW * PARTS_PER_GPU * world * E2E / (float(e2e_ms.item()) / 1e3)

    # ---------------- with consumer (A14): the same pipeline plus the GraphSAGE-mean forward of every
    # minibatch (mgnn_sage_forward, tcgen05 TF32) between gather and score on the buffer stream, with
    # the sampling of the next window still overlapped on stream A (Alg.1 l.6-9).
    dims = synth.sage_dims(CFG.feat_dim, len(CFG.fanouts), synth.N_CLASSES[CFG.name])
    wts = synth.sage_weights(dims)
    ctx.sage_config(dims, [w_[0] for w_ in wts], [w_[1] for w_ in wts], [w_[2] for w_ in wts])
    logits = torch.empty((PARTS_PER_GPU * WINDOW, CFG.batch, dims[-1]), dtype=torch.float32, device="cuda")
    fwd_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]

    # Alg.1 overlap: the consumer of window w runs on its own stream C while stream B gathers and
    # scores window w+1 and stream A samples window w+2; a slot is resampled only after both its
    # score (B) and its forward pass (C) are done.
    sC = torch.cuda.Stream()
    ev_gathered = [torch.cuda.Event(), torch.cuda.Event()]
    ev_fwd = [torch.cuda.Event(), torch.cuda.Event()]
    logits2 = [logits, torch.empty_like(logits)]

    def sample_async_c(sl, tt):
        sA.wait_event(ev_done[sl])
        sA.wait_event(ev_fwd[sl])
        ctx.sample(sl, tt, WINDOW, stream=sA)
        ev_sampled[sl].record(sA)

    def consume_fwd(sl, i=None):
        sB.wait_event(ev_sampled[sl])
        ctx.lookup_gather(sl, sB)
        ev_gathered[sl].record(sB)
        ctx.score(sl, sB)
        ev_done[sl].record(sB)
        sC.wait_event(ev_gathered[sl])
        if i is not None:
            fwd_ev[i][0].record(sC)
        ctx.sage_forward(sl, logits2[sl], sC)
        if i is not None:
            fwd_ev[i][1].record(sC)
        ev_fwd[sl].record(sC)

    t_c = t_e2e + E2E * WINDOW
    barrier()
    sample_async_c(slot, t_c)
    for _ in range(args.warmup):
        sample_async_c(slot ^ 1, t_c + WINDOW)
        consume_fwd(slot)
        t_c += WINDOW
        slot ^= 1
    barrier()
    # timed as one span (no per-window flush / join: the three streams run windows back to back)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    c0.record(sB)
    sA.wait_event(c0)
    sC.wait_event(c0)
    for i in range(K):
        sample_async_c(slot ^ 1, t_c + WINDOW)
        consume_fwd(slot, i)
        t_c += WINDOW
        slot ^= 1
    sB.wait_stream(sA)
    sB.wait_stream(sC)
    c1.record(sB)
    barrier()
    c_ms = torch.tensor([c0.elapsed_time(c1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(c_ms, op=dist.ReduceOp.MAX)
    c_value = mb_total / (float(c_ms.item()) / 1e3)
    fwd_ms = sum(a.elapsed_time(b) for a, b in fwd_ev) / K
    # algorithmic work of the last forward (window slot ^ 1): per layer 2 * n_dst * (2 d_in) * d_out
    # flops (dense part) and the neighbour rows it averages (4 * d_in bytes per sampled edge)
    wv = ctx.window(slot ^ 1)
    hs = PL.device_view(wv.hop_size, (wv.n_inst, 9), "i8").cpu().numpy()
    L_ = len(CFG.fanouts)
    flops = 0.0
    agg_bytes = 0.0
    for l in range(L_):
        hop = L_ - 1 - l
        n_dst = hs[:, hop].astype(np.float64)
        flops += float((2.0 * n_dst * 2 * dims[l] * dims[l + 1]).sum())
        offs = PL.device_view(wv.offsets[hop], (wv.n_inst, wv.off_stride[hop]), "i8")
        n_edges = np.array([int(offs[m, int(hs[m, hop])]) for m in range(wv.n_inst)], np.float64)
        agg_bytes += float((n_edges * dims[l] * 4).sum())

    # ---------------- with training (NEXT-3): every minibatch trains the model -- forward, loss,
    # backward, NCCL all-reduce of the gradients across ranks (N > 1), SGD -- on stream C, one
    # DDP step per window step (the steps of a window are sequential through the weights), while
    # streams A/B prepare the next windows (Alg.1: prepare(t+1) || train(t)).
    labels = synth.node_labels(CFG.n_nodes, dims[-1])
    ctx.train_config(labels)
    n_trainers = PARTS_PER_GPU * world
    lr = 0.01
    ev_trained = [torch.cuda.Event(), torch.cuda.Event()]

    def sample_async_t(sl, tt):
        sA.wait_event(ev_done[sl])
        sA.wait_event(ev_trained[sl])
        ctx.sample(sl, tt, WINDOW, stream=sA)
        ev_sampled[sl].record(sA)

    # The WINDOW DDP steps of a slot are one CUDA graph (captured once per slot, replayed every
    # window): ~12 launches per step, all device-resident sizes, so the graph is static.
    graphs = {}
    # one rank: graph capture; N > 1 keeps eager launches (the step is GPU-bound either way, and a
    # graph holding captured NCCL work hung the process teardown)
    use_graph = [not args.no_train_graph and world == 1]

    def train_window(sl):
        if use_graph[0]:
            if sl not in graphs:
                try:
                    g_ = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g_, stream=sC):
                        for w_ in range(WINDOW):
                            PL.ddp_step(ctx, sl, w_, n_trainers, lr, stream=torch.cuda.current_stream())
                    graphs[sl] = g_
                except Exception as e:  # capture unsupported here: stay eager
                    print(f"[bench] training graph capture failed ({e!r}); eager launches", file=sys.stderr)
                    use_graph[0] = False
            if use_graph[0]:
                with torch.cuda.stream(sC):
                    graphs[sl].replay()
                return
        for w_ in range(WINDOW):
            PL.ddp_step(ctx, sl, w_, n_trainers, lr, stream=sC)

    def consume_train(sl):
        sB.wait_event(ev_sampled[sl])
        ctx.lookup_gather(sl, sB)
        ev_gathered[sl].record(sB)
        ctx.score(sl, sB)
        ev_done[sl].record(sB)
        sC.wait_event(ev_gathered[sl])
        train_window(sl)
        ev_trained[sl].record(sC)

    KT = max(3, min(K, 6))
    t_t = t_c                   # the window pending in `slot` (sampled, not yet gathered)
    barrier()
    sample_async_t(slot, t_t)
    for _ in range(args.warmup):
        sample_async_t(slot ^ 1, t_t + WINDOW)
        consume_train(slot)
        t_t += WINDOW
        slot ^= 1
    barrier()
    ctx.loss(sC)
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    t0e.record(sB)
    sA.wait_event(t0e)
    sC.wait_event(t0e)
    for i in range(KT):
        sample_async_t(slot ^ 1, t_t + WINDOW)
        consume_train(slot)
        t_t += WINDOW
        slot ^= 1
    sB.wait_stream(sA)
    sB.wait_stream(sC)
    t1e.record(sB)
    barrier()
    tr_ms = torch.tensor([t0e.elapsed_time(t1e)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tr_ms, op=dist.ReduceOp.MAX)
    tr_value = WINDOW * PARTS_PER_GPU * world * KT / (float(tr_ms.item()) / 1e3)
    tr_loss_t = torch.tensor([ctx.loss(sC) / (KT * WINDOW)], dtype=torch.float64, device="cuda")
    if world > 1:                       # each rank holds its trainers' share of the mean loss
        dist.all_reduce(tr_loss_t)
    tr_loss = float(tr_loss_t.item())

    clocks = clk.summary()
    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
        g_avg_ms = gms / max(glaunch, 1)
        g_bytes = gbytes / max(glaunch, 1)
        achieved = g_bytes / (g_avg_ms / 1e3) / 1e9 if g_avg_ms > 0 else None
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "gather_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get("bytes_per_launch")
            except (OSError, ValueError):
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": dict(workload(P), **({"sampling": "remote expansion (NEXT-1)"} if args.remote else {}),
                           **({"scores": "dense S_A (NEXT-1)"} if args.dense else {}),
                           **({"partitioner": "hash (random relabel)"} if args.hash_partition else {})),
            "buffer_init_ms": init_ms,
            "hit_rate": hits / max(1, hits + misses),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": E2E, "path": "two-stream pipeline: mgnn_sample(host pinned seeds, H2D) | "
                                          "lookup_gather + score_evict_refill + counts_read_async (D2H), "
                                          "host reads each window's counters"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": "k_gather (classify + feature-row gather)",
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": (achieved / hbm_peak) if achieved else None, "traffic": traffic,
                         "peak_source": peak_src, "launch_ms": g_avg_ms, "share_of_step": gms / max(tot_ms, 1e-9),
                         "algorithmic_bytes_per_launch": g_bytes},
            "clocks": clocks,
            "wall_s_timed_region": wall,
            "with_consumer": {
                "value": c_value, "unit": UNIT, "ms_per_step": float(c_ms.item()) / K,
                "model": f"GraphSAGE-mean {dims} (random init), forward of every minibatch",
                "consumer_ms_per_step": fwd_ms, "consumer_launches_per_step": L_,
                "pipeline": "3 streams: sample(w+2) | gather+score(w+1) | forward(w), timed as one span",
                "kernel": "k_mean (neighbour means, all SMs) + k_sage_gemm (warp-specialised: TMA ring of self "
                          "rows / means / weights -> tcgen05.mma kind::tf32 into 2 TMEM accumulators -> "
                          "bias/ReLU epilogue warps)",
                "tflops": flops / (fwd_ms / 1e3) / 1e12 if fwd_ms > 0 else None,
                "agg_gbs": agg_bytes / (fwd_ms / 1e3) / 1e9 if fwd_ms > 0 else None,
                "dtype": "tf32 x tf32 -> f32"},
            "with_training": {
                "value": tr_value, "unit": UNIT, "ms_per_step": float(tr_ms.item()) / KT, "steps": KT,
                "model": f"GraphSAGE-mean {dims}, softmax cross-entropy, SGD lr {lr}",
                "ddp": f"{n_trainers} trainers; gradient all-reduce " + ("NCCL (torch.distributed)" if world > 1
                                                                          else "none (one rank)"),
                "mean_loss_in_timed_steps": tr_loss,
                "pipeline": "3 streams: sample(w+2) | gather+score(w+1) | DDP steps of window w",
                "cuda_graph": bool(use_graph[0]),
                "dtype": "tf32 x tf32 -> f32"},
        }
        if world > 1:
            nv_bytes = peer_rows * CFG.feat_dim * 4
            gbs = nv_bytes / (g_avg_ms / 1e3) / 1e9 if g_avg_ms > 0 else None
            peer = peer_copy_gbs(local, (local + 1) % torch.cuda.device_count())
            line["nvlink"] = {"peer_rows_per_window": peer_rows, "bytes_per_window": nv_bytes,
                              "gbs_during_gather": gbs,
                              "peak_gbs": 900.0, "peak_source": "NVLink 5 nominal per direction per GPU",
                              "frac": gbs / 900.0 if gbs else None,
                              "achievable_peer_copy_gbs": peer,
                              "frac_of_achievable": gbs / peer if (gbs and peer) else None,
                              "note": "miss + refill rows whose owner is on another GPU, read by peer loads "
                                      "inside k_gather / k_swap_refill (last timed window); achievable = "
                                      "256 MB device-to-device copy to the next GPU, best of 5"}
        if world == 1 and not args.no_cpu_baseline:
            rate, n_mb, el = oracle_rate(parts, P, f_bp, gamma, delta, args.cpu_budget)
            rate_p, n_thr = oracle_rate_threads(parts, P, f_bp, gamma, delta, min(args.cpu_budget, 6.0))
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                                    "sample": f"{n_mb} minibatches (steps 1..{n_mb // P} of all {P} partitions), "
                                              f"{el:.1f} s, single-threaded C oracle",
                                    "value_one_thread_per_partition": rate_p, "threads": n_thr,
                                    "host_cpu": host_cpu(), "host_nproc": os.cpu_count()}
        print(json.dumps(line), flush=True)
    graphs.clear()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()                 # peers read our feature tables until everyone is done
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
