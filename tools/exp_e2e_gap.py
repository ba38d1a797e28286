"""Diagnostic: the bench schedule with device seeds (the epoch order built on the GPU) against host seeds
(pinned, copied by mgnn_sample) on consecutive windows of one run: where does e2e's margin come from?
    python tools/exp_e2e_gap.py --config products --windows 20"""
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
from paper_2410_22697_b200.schedule import PrepareAhead  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--windows", type=int, default=20)
    a = ap.parse_args()
    tune = bench.TUNING.get(a.config, {})
    for k_, v_ in tune.get("env", {}).items():
        os.environ.setdefault(k_, v_)
    S = bench.Setup(a.config, 1)
    g = synth.generate(S.cfg)
    parts = synth.partition(g, S.P)
    ctx = PL.build_context(0, parts, S.cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(S.gamma, PL.alpha_default(S.gamma, S.delta), 1.0, S.delta, S.f_bp)
    rb = PL.estimate_rows_bound(ctx, S.cfg.fanouts, S.cfg.batch, synth.RUN_SEED)
    ctx.sampler_config(S.cfg.fanouts, S.cfg.batch, synth.RUN_SEED, S.window, rows_bound=rb)
    ctx.defer_relabel(True)
    W = S.window
    prio = tune.get("sampling_priority", 0)

    def timed(pipe, n):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i in range(n):
            pipe.iteration(events=ev[i])
        torch.cuda.synchronize()
        ms = [x.elapsed_time(y) for x, y in ev]
        return sum(ms) / n, sorted(ms)[n // 2]

    out = {"config": a.config}
    pipe = PrepareAhead(ctx, W, t0=1, relabel_stream=True, sampling_priority=prio)
    for _ in range(4):
        pipe.iteration()
    out["device_1"] = timed(pipe, a.windows)
    pipe.iteration(prepare_next=False)
    t0, slot = pipe.t, pipe.slot
    seeds, counts = {}, {}
    for i in range(a.windows + 1):
        tt = t0 + i * W
        ctx.sample(slot, tt, W)
        wv = ctx.window(slot)
        counts[tt] = PL.device_view(wv.hop_size, (wv.n_inst, 9), "i8")[:, 0].to(torch.int32).cpu().pin_memory()
        seeds[tt] = PL.device_view(wv.frontier, (wv.n_inst, wv.rows_stride), "i4")[:, :S.cfg.batch].cpu().pin_memory()
    torch.cuda.synchronize()
    hp = PrepareAhead(ctx, W, t0=t0, relabel_stream=True, sampling_priority=prio,
                      host_seeds=lambda sl, tt: (seeds[tt].data_ptr(), counts[tt].data_ptr()))
    out["host"] = timed(hp, a.windows)
    hp.iteration(prepare_next=False)
    # the same seeds from DEVICE memory (mgnn_sample copies them device -> device)
    t1 = hp.t
    dseeds, dcounts = {}, {}
    for i in range(a.windows + 1):
        tt = t1 + i * W
        ctx.sample(hp.slot, tt, W)
        wv = ctx.window(hp.slot)
        dcounts[tt] = PL.device_view(wv.hop_size, (wv.n_inst, 9), "i8")[:, 0].to(torch.int32).clone()
        dseeds[tt] = PL.device_view(wv.frontier, (wv.n_inst, wv.rows_stride), "i4")[:, :S.cfg.batch].clone()
    torch.cuda.synchronize()

    class Dev(PrepareAhead):
        def _sample(self, sl, tt):
            self.sA.wait_event(self.ev_done[sl])
            if self.relabel_stream:
                self.sA.wait_event(self.ev_relabeled[sl])
            self.ctx.sample_ptr(sl, tt, self.W, dseeds[tt].data_ptr(), dcounts[tt].data_ptr(), False, self.sA)
            self.ev_sampled[sl].record(self.sA)

    xp = Dev(ctx, W, t0=t1, relabel_stream=True, sampling_priority=prio)
    out["device_seeds_d2d"] = timed(xp, a.windows)
    xp.iteration(prepare_next=False)
    hp = xp
    dp = PrepareAhead(ctx, W, t0=hp.t, relabel_stream=True, sampling_priority=prio)
    out["device_2"] = timed(dp, a.windows)
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
