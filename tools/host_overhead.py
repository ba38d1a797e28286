"""Host (CPU) time per window of the bench schedule against its device time: is a config launch-bound?

    python tools/host_overhead.py --config cfg1 [--windows 200] [--profile]
Prints the wall time per PrepareAhead.iteration() measured WITHOUT synchronising (the host runs ahead
as far as the GPU lets it), the device time per iteration (CUDA events), and the host time of each
library call (perf_counter around the ctypes call, GPU busy so nothing blocks).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from inputs import synth  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402
from paper_2410_22697_b200.schedule import PrepareAhead  # noqa: E402


class Timed:
    """Proxy that accumulates host seconds per method of the wrapped context."""

    def __init__(self, ctx):
        self._c = ctx
        self.t = {}
        self.n = {}

    def __getattr__(self, name):
        f = getattr(self._c, name)
        if not callable(f):
            return f

        def g(*a, **k):
            t0 = time.perf_counter()
            r = f(*a, **k)
            self.t[name] = self.t.get(name, 0.0) + time.perf_counter() - t0
            self.n[name] = self.n.get(name, 0) + 1
            return r
        return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--windows", type=int, default=200)
    ap.add_argument("--profile", action="store_true", help="per-call stage events on (as in bench's timed runs)")
    a = ap.parse_args()
    S = bench.Setup(a.config, 1)
    g = synth.generate(S.cfg)
    parts = synth.partition(g, S.P)
    ctx = PL.build_context(0, parts, S.cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(S.gamma, PL.alpha_default(S.gamma, S.delta), 1.0, S.delta, S.f_bp)
    ctx.sampler_config(S.cfg.fanouts, S.cfg.batch, synth.RUN_SEED, S.window)
    tc = Timed(ctx)
    pipe = PrepareAhead(tc, S.window, relabel_stream=True)
    for _ in range(5):
        pipe.iteration()
    torch.cuda.synchronize()
    ctx.profile(a.profile)
    tc.t.clear()
    tc.n.clear()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.windows)]
    t0 = time.perf_counter()
    for i in range(a.windows):
        pipe.iteration(events=ev[i])
    host = time.perf_counter() - t0
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    dev = sorted(x.elapsed_time(y) for x, y in ev)
    out = {"config": a.config, "profile": a.profile, "windows": a.windows,
           "host_us_per_iteration": 1e6 * host / a.windows, "wall_us_per_iteration": 1e6 * total / a.windows,
           "device_us_per_iteration_median": 1e3 * dev[len(dev) // 2],
           "per_call_host_us": {k: round(1e6 * v / tc.n[k], 1) for k, v in tc.t.items()}}
    print(json.dumps(out), flush=True)
    ctx.profile(False)
    ctx.close()


if __name__ == "__main__":
    main()
