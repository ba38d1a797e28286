"""Per-call GPU time of one window (serial, no overlap): sample / lookup_gather / score_evict_refill.

    python tools/breakdown.py [--windows 10]
Uses the bench workload (arxiv-shaped, 2 partitions, 32-step windows) and CUDA events on one stream.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from inputs import synth  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--windows", type=int, default=12)
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--parts", type=int, default=2)
    a = ap.parse_args()
    S = bench.Setup(a.config, 1, parts=a.parts)
    cfg = S.cfg
    P = S.P
    f_bp, gamma, delta = S.f_bp, S.gamma, S.delta
    g = synth.generate(cfg)
    parts = synth.partition(g, P)
    ctx = PL.build_context(0, parts, cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(gamma, PL.alpha_default(gamma, delta), 1.0, delta, f_bp)
    W = S.window
    ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, W)
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t, slot = 1, 0
    acc = {"sample": [], "gather": [], "score": []}
    import ctypes
    from paper_2410_22697_b200 import _lib
    L = _lib.load()
    prof_from = a.windows + 3                  # per-launcher events only in a second pass (they add overhead)
    for i in range(2 * a.windows + 3):
        if i == prof_from:
            L.mgnn_profile_kernels(1, None, 0)
        flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(s)
        ctx.sample(slot, t, W, stream=s)
        e[1].record(s)
        ctx.lookup_gather(slot, s)
        e[2].record(s)
        ctx.score(slot, s)
        e[3].record(s)
        torch.cuda.synchronize()
        if 3 <= i < prof_from:
            acc["sample"].append(e[0].elapsed_time(e[1]))
            acc["gather"].append(e[1].elapsed_time(e[2]))
            acc["score"].append(e[2].elapsed_time(e[3]))
        t += W
        slot ^= 1
    buf = ctypes.create_string_buffer(1 << 16)
    L.mgnn_profile_kernels(0, buf, len(buf))
    for k, v in acc.items():
        print(f"{k:8s} mean {1e3 * sum(v) / len(v):8.1f} us   min {1e3 * min(v):8.1f} us")
    print(f"per launcher over {a.windows} windows (time since the previous launcher on the stream):")
    print(buf.value.decode())


if __name__ == "__main__" and "--timeline" not in sys.argv:
    main()


def timeline(windows=6):
    """Pipelined (two-stream) iterations: event timestamps after each call, relative to iteration start."""
    S = bench.Setup("arxiv", 1)
    cfg, P = S.cfg, S.P
    f_bp, gamma, delta = S.f_bp, S.gamma, S.delta
    g = synth.generate(cfg)
    parts = synth.partition(g, P)
    ctx = PL.build_context(0, parts, cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(gamma, PL.alpha_default(gamma, delta), 1.0, delta, f_bp)
    W = 32
    ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, W)
    sA, sB = torch.cuda.Stream(), torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t, slot = 1, 0
    ctx.sample(0, t, W, stream=sA)
    torch.cuda.synchronize()
    for i in range(windows + 4):
        flush.zero_()
        torch.cuda.synchronize()
        ev = {k: torch.cuda.Event(enable_timing=True) for k in ("start", "sampleA", "gatherB", "scoreB", "end")}
        h0 = time.perf_counter()
        ev["start"].record(sB)
        sA.wait_event(ev["start"])
        ctx.sample(slot ^ 1, t + W, W, stream=sA)
        ev["sampleA"].record(sA)
        ctx.lookup_gather(slot, sB)
        ev["gatherB"].record(sB)
        ctx.score(slot, sB)
        ev["scoreB"].record(sB)
        sB.wait_stream(sA)
        ev["end"].record(sB)
        host_us = 1e6 * (time.perf_counter() - h0)
        torch.cuda.synchronize()
        if i >= 4:
            print("  ".join(f"{k} {1e3 * ev['start'].elapsed_time(e):7.1f}" for k, e in ev.items() if k != "start")
                  + f"  host_issue {host_us:7.1f}")
        t += W
        slot ^= 1


if __name__ == "__main__" and "--timeline" in sys.argv:
    timeline()
