"""End-to-end use of the library: MassiveGNN-style prefetching feeding DDP GraphSAGE training.

    python examples/train_ddp.py [--config arxiv] [--windows 40]                      # one GPU
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 examples/train_ddp.py        # one rank per GPU

Each rank hosts 2 partitions (trainers).  Per window of W steps: stream A samples the next window
(no buffer state needed), stream B classifies / gathers / scores the current one (prefetch buffer
hits, misses over NVLink from the owner GPU, decay, eviction + refill every Delta steps), stream C
trains on it: one DDP step per window step for every local trainer -- forward, cross-entropy,
backward on the tensor cores, NCCL all-reduce of the gradients across ranks, SGD.
Labels are the planted block of each node (8 classes, a structural task the aggregation can learn).
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from inputs import synth  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="arxiv")
    ap.add_argument("--windows", type=int, default=40)
    ap.add_argument("--lr", type=float, default=0.5)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[a.config]
    P = 2 * world
    g = synth.generate(cfg)
    parts = synth.partition(g, P)
    ctx = PL.build_context(local, parts, cfg.feat_dim, synth.FEAT_SEED, hosted=[2 * rank, 2 * rank + 1])
    if world > 1:
        PL.exchange_tables(ctx)                       # remote feature tables mapped over NVLink
    gamma, delta, W = 0.995, 32, 32
    ctx.buffer_init(gamma, PL.alpha_default(gamma, delta), 1.0, delta, 2500)
    ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, W)
    dims = synth.sage_dims(cfg.feat_dim, len(cfg.fanouts), 8)
    wts = synth.sage_weights(dims)
    ctx.sage_config(dims, [w[0] for w in wts], [w[1] for w in wts], [w[2] for w in wts])
    labels = (np.arange(g.n_nodes, dtype=np.int64) * 8 // g.n_nodes).astype(np.int32)   # planted block
    ctx.train_config(labels)

    sA, sB, sC = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev_s = [torch.cuda.Event(), torch.cuda.Event()]
    ev_g = [torch.cuda.Event(), torch.cuda.Event()]
    ev_d = [torch.cuda.Event(), torch.cuda.Event()]
    ev_t = [torch.cuda.Event(), torch.cuda.Event()]
    t, slot = 1, 0

    def sample(sl, tt):
        sA.wait_event(ev_d[sl])
        sA.wait_event(ev_t[sl])
        ctx.sample(sl, tt, W, stream=sA)
        ev_s[sl].record(sA)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sample(slot, t)
    for i in range(a.windows):
        sample(slot ^ 1, t + W)
        sB.wait_event(ev_s[slot])
        ctx.lookup_gather(slot, sB)
        ev_g[slot].record(sB)
        ctx.score(slot, sB)
        ev_d[slot].record(sB)
        sC.wait_event(ev_g[slot])
        for w in range(W):
            PL.ddp_step(ctx, slot, w, P, a.lr, stream=sC)
        ev_t[slot].record(sC)
        if i % 10 == 9 or i == a.windows - 1:
            loss = torch.tensor([ctx.loss(sC) / (10 * W)], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(loss)
            c = ctx.counts(slot ^ 0, sB)
            if rank == 0:
                print(f"window {i + 1:4d}  steps {t + W - 1:6d}  mean loss {loss.item():.4f}  "
                      f"hit rate {c[:, 2].sum() / max(1, c[:, 2].sum() + c[:, 3].sum()):.3f}", flush=True)
        t += W
        slot ^= 1
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if rank == 0:
        print(f"{a.windows * W * P} minibatches trained in {el:.2f} s "
              f"({a.windows * W * P / el:.0f} minibatches/s incl. host, {world} GPU(s))")
    if world > 1:
        dist.barrier()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
