"""Multi-GPU parity (one process per GPU): run with
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/multi_gpu_parity.py [--config cfg1|arxiv]
Each rank hosts 2 partitions of P = 2N; miss and refill rows of partitions owned by
other ranks are read over NVLink through CUDA-IPC-mapped feature tables.  Every
rank compares its windows with the oracle (which runs all P partitions on the CPU).
Exit code 0 iff every rank matched bit for bit.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from inputs import synth  # noqa: E402
from tests.parity_util import run_parity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--delta", type=int, default=4)
    ap.add_argument("--windows", type=int, default=4)
    ap.add_argument("--train", action="store_true", help="DDP training-step parity (NEXT-3) instead")
    ap.add_argument("--remote", action="store_true", help="NEXT-1 remote expansion (replicated global CSR)")
    ap.add_argument("--parts", type=int, default=0, help="total partitions P (default 2 per GPU)")
    ap.add_argument("--digest-out", default="", help="write this rank's per-partition result digests (JSON)")
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = synth.CONFIGS[a.config]
    g = synth.generate(cfg)
    P = a.parts or 2 * world
    assert P % world == 0
    per = P // world
    hosted = list(range(per * rank, per * (rank + 1)))
    ok = torch.ones(1, device="cuda")
    try:
        if a.train:
            from tests.train_util import run_train_parity
            r = run_train_parity(g, P, cfg.feat_dim, cfg.fanouts, cfg.batch, synth.sage_dims(cfg.feat_dim, 2, 16), 3,
                                 hosted=hosted, device=local, exchange=True)
            print(f"[rank {rank}] train parity ok: worst error / tolerance {r:.3f}", flush=True)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            dist.destroy_process_group()
            sys.exit(0 if ok.item() == 1 else 1)
        st = run_parity(g, P, cfg.feat_dim, cfg.fanouts, cfg.batch, 2500, 0.9, a.delta, 1.0,
                        [a.delta] * a.windows, hosted=hosted, device=local, exchange=True, remote=a.remote,
                        sample_every=1 if a.config == "cfg1" else 9, check_x_rows=0 if a.config == "cfg1" else 2048)
        print(f"[rank {rank}] parity ok: {st}", flush=True)
        if a.digest_out:
            import json
            with open(f"{a.digest_out}.rank{rank}", "w") as f:
                json.dump(st["digest"], f)
        assert st["misses"] > 0 and st["evicted"] > 0 and st["peer_rows"] > 0
    except Exception as e:  # report, then fail the collective result
        print(f"[rank {rank}] FAILED: {e!r}", flush=True)
        ok.zero_()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if ok.item() == 1 else 1)


if __name__ == "__main__":
    main()
