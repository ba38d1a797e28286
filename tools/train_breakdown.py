"""Per-launcher GPU time of DDP training steps (arxiv bench workload, one GPU, eager launches,
per-launcher CUDA events; diagnostics only).   python tools/train_breakdown.py [--steps 32]"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from inputs import synth  # noqa: E402
from paper_2410_22697_b200 import _lib  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--steps", type=int, default=32)
    a = ap.parse_args()
    S = bench.Setup(a.config, 1)
    cfg, P = S.cfg, S.P
    f_bp, gamma, delta = S.f_bp, S.gamma, S.delta
    g = synth.generate(cfg)
    parts = synth.partition(g, P)
    ctx = PL.build_context(0, parts, cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(gamma, PL.alpha_default(gamma, delta), 1.0, delta, f_bp)
    W = S.window
    ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, W)
    dims = synth.sage_dims(cfg.feat_dim, len(cfg.fanouts), synth.N_CLASSES[cfg.name])
    wts = synth.sage_weights(dims)
    ctx.sage_config(dims, [w[0] for w in wts], [w[1] for w in wts], [w[2] for w in wts])
    ctx.train_config(synth.node_labels(cfg.n_nodes, dims[-1]))
    ctx.sample(0, 1, W)
    ctx.lookup_gather(0)
    for w in range(min(4, W)):                     # warm-up
        PL.ddp_step(ctx, 0, w, P, 0.01)
    torch.cuda.synchronize()
    L = _lib.load()
    L.mgnn_profile_kernels(1, None, 0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.steps):
        PL.ddp_step(ctx, 0, i % W, P, 0.01)
    e1.record()
    torch.cuda.synchronize()
    buf = ctypes.create_string_buffer(1 << 16)
    L.mgnn_profile_kernels(0, buf, len(buf))
    print(f"{a.steps} DDP steps of {P} trainers: {e0.elapsed_time(e1) / a.steps * 1e3:.1f} us per step "
          "(with per-launcher events)")
    print(buf.value.decode())


if __name__ == "__main__":
    main()
