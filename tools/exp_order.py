"""Diagnostic: one stream, a fixed call order per window, CUDA events around each call.
    python tools/exp_order.py --config products --order gather,sample,score
Orders: gather / score of window w, sample of window w+1, relabel of window w (deferred)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from inputs import synth  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--windows", type=int, default=10)
    ap.add_argument("--order", default="gather,score,sample")
    a = ap.parse_args()
    S = bench.Setup(a.config, 1)
    g = synth.generate(S.cfg)
    parts = synth.partition(g, S.P)
    ctx = PL.build_context(0, parts, S.cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(S.gamma, PL.alpha_default(S.gamma, S.delta), 1.0, S.delta, S.f_bp)
    ctx.sampler_config(S.cfg.fanouts, S.cfg.batch, synth.RUN_SEED, S.window)
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    order = a.order.split(",")
    t, slot = 1, 0
    ctx.sample(slot, t, S.window, stream=s)
    acc = {k: [] for k in order}
    tot = []
    for it in range(a.windows + 3):
        flush.zero_()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(order) + 1)]
        evs[0].record(s)
        for i, op in enumerate(order):
            if op == "gather":
                ctx.lookup_gather(slot, s)
            elif op == "score":
                ctx.score(slot, s)
            elif op == "sample":
                ctx.sample(slot ^ 1, t + S.window, S.window, stream=s)
            evs[i + 1].record(s)
        torch.cuda.synchronize()
        if it >= 3:
            for i, op in enumerate(order):
                acc[op].append(evs[i].elapsed_time(evs[i + 1]))
            tot.append(evs[0].elapsed_time(evs[-1]))
        t += S.window
        slot ^= 1
    med = lambda x: sorted(x)[len(x) // 2]
    print(json.dumps({"config": a.config, "order": a.order, "window_ms": med(tot),
                      **{k + "_ms": med(v) for k, v in acc.items()}}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
