"""NEXT-4 policy study on the GPU pipeline: buffer hit rate, remote feature rows and throughput
over a grid of prefetch fraction f, decay gamma and eviction interval Delta (§4-5 trade-offs,
P:276-288), including f = 0 (no prefetch: every halo access is a remote fetch, the DistDGL
baseline) and Delta = 0 (prefetch without eviction).

    python tools/policy_sweep.py [--config arxiv] [--parts 2] [--steps 512]

Per policy: a fresh context, `steps` minibatch steps of every partition in windows of
min(32, Delta) steps (sample -> gather -> score on one stream), counters read per window.
Remote rows = misses + refills + initial buffer fill (the rows that cross partitions).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from inputs import synth  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402


def run(parts, cfg, f_bp, gamma, delta, steps, window=32):
    ctx = PL.build_context(0, parts, cfg.feat_dim, synth.FEAT_SEED)
    alpha = PL.alpha_default(gamma, delta) if delta > 0 else 0.0
    ctx.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    W = min(window, delta) if delta > 0 else window
    ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, W)
    init_rows = sum(ctx.part_info(lp)["cap"] for lp in range(len(ctx.parts)))
    hits = misses = refills = 0
    t, slot = 1, 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    done = 0
    while done < steps:
        e0.record()
        ctx.sample(slot, t, W)
        ctx.lookup_gather(slot)
        ctx.score(slot)
        e1.record()
        c = ctx.counts(slot)
        ms += e0.elapsed_time(e1)
        hits += int(c[:, 2].sum())
        misses += int(c[:, 3].sum())
        refills += int(c[:, 5].sum())
        t += W
        done += W
        slot ^= 1
    ctx.close()
    mb = done * len(parts)
    return {"hit_rate": hits / max(1, hits + misses), "remote_rows_per_mb": (misses + refills + init_rows) / mb,
            "misses_per_mb": misses / mb, "refills_per_mb": refills / mb, "mb_per_s": mb / (ms / 1e3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--parts", type=int, default=2)
    ap.add_argument("--steps", type=int, default=512)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    g = synth.generate(cfg)
    parts = synth.partition(g, a.parts)
    grid = [(0, 0.995, 0)]                                            # no prefetch (all halo misses)
    grid += [(f, 0.995, 0) for f in (1000, 2500, 5000, 10000)]        # prefetch, no eviction
    grid += [(f, gm, d) for f in (2500, 5000) for gm in (0.95, 0.995) for d in (16, 32, 64, 128, 256)]
    print(f"config {a.config}, P = {a.parts}, {a.steps} steps per partition, theta_R = 1")
    print(f"{'f':>5s} {'gamma':>6s} {'Delta':>5s} {'hit rate':>8s} {'misses/mb':>10s} {'refills/mb':>10s} "
          f"{'remote rows/mb':>14s} {'mb/s':>9s}")
    for f_bp, gm, d in grid:
        r = run(parts, cfg, f_bp, gm, d, a.steps)
        print(f"{f_bp / 1e4:5.2f} {gm:6.3f} {d:5d} {r['hit_rate']:8.3f} {r['misses_per_mb']:10.1f} "
              f"{r['refills_per_mb']:10.1f} {r['remote_rows_per_mb']:14.1f} {r['mb_per_s']:9.0f}", flush=True)


if __name__ == "__main__":
    main()
