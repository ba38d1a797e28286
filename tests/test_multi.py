"""Multi-process paths.

* gloo (CPU, world_size 2, -m "not gpu"): the host logic of the multi-GPU setup --
  partition ownership per rank, all-gather of the feature-table handles and the
  import of every remote table, and the max-over-ranks timing reduction of bench.py.
* NCCL (>= 2 GPUs, -m gpu): tests/multi_gpu_parity.py under torchrun -- every rank's
  windows bit-exact vs the oracle while miss/refill rows are NVLink peer loads.
"""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class FakeCtx:
    """Stands in for pipeline.Context: records exports/imports (no CUDA)."""

    def __init__(self, rank, parts_per_rank, P):
        self.parts = list(range(parts_per_rank * rank, parts_per_rank * (rank + 1)))
        self.P = P
        self.imported = {}

    def export_table(self, pid):
        return bytes([pid]) * 64

    def import_table(self, pid, handle):
        assert pid not in self.parts and pid not in self.imported
        assert handle == bytes([pid]) * 64
        self.imported[pid] = handle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2410_22697_b200.pipeline import exchange_tables
    ctx = FakeCtx(rank, 2, 2 * world)
    exchange_tables(ctx)
    # bench.py reduces the timed region as the MAX over ranks
    t = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    q.put((rank, sorted(ctx.imported), float(t.item())))
    dist.destroy_process_group()


class FakeTrainCtx:
    """Stands in for pipeline.Context in ddp_step: CPU gradient buffer, records the call order."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []
        self.g = torch.full((6,), float(rank + 1))

    def train_step(self, slot, w, n, stream=None):
        self.calls.append(("train_step", slot, w, n))

    def grads(self):
        return self.g

    def sgd(self, lr, stream=None):
        self.calls.append(("sgd", lr, self.g.tolist()))


def _train_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    from paper_2410_22697_b200.pipeline import ddp_step
    ctx = FakeTrainCtx(rank)
    ddp_step(ctx, 1, 3, 4, 0.5)
    q.put((rank, ctx.calls))
    dist.destroy_process_group()


def test_gloo_two_ranks_ddp_step():
    """NEXT-3 host logic: train_step, then the SUM all-reduce of the gradient buffer across ranks,
    then SGD on the reduced gradients, on every rank."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, calls in res:
        assert calls == [("train_step", 1, 3, 4), ("sgd", 0.5, [3.0] * 6)], (rank, calls)


@pytest.mark.gpu
def test_nccl_two_gpus_train_parity():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "multi_gpu_parity.py"), "--train"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


def test_gloo_two_ranks_table_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == (0, [2, 3], 11.0)
    assert res[1] == (1, [0, 1], 11.0)


@pytest.mark.gpu
def test_nccl_two_gpus_parity():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "multi_gpu_parity.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.gpu
def test_nccl_two_gpus_remote_expansion_parity():
    """NEXT-1 across GPUs: replicated global CSR, far rows over NVLink, bit-exact per rank."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    port = _free_port()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "multi_gpu_parity.py"), "--remote"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


def _digests(prefix, world):
    import json
    out = {}
    for r in range(world):
        with open(f"{prefix}.rank{r}") as f:
            out.update({int(k): v for k, v in json.load(f).items()})
    return out


@pytest.mark.gpu
def test_placement_invariance_p8(tmp_path):
    """SURVEY §4 layer 4 / north_star's layout: P = 8 partitions give the SAME per-partition results
    (counts of every step, final BUF / S_E / S_A / slot_of -- each run also checked against the oracle)
    whether one GPU hosts all 8, two GPUs host 4 each or four GPUs host 2 each (miss and refill rows of
    partitions on other GPUs then cross NVLink)."""
    sys.path.insert(0, ROOT)
    from inputs import synth
    from tests.parity_util import run_parity
    g = synth.generate(synth.CONFIGS["cfg1"])
    one = run_parity(g, 8, 64, [10, 25], 256, 2500, 0.9, 4, 1.0, [4] * 4)["digest"]
    assert sorted(one) == list(range(8))
    n = torch.cuda.device_count()
    for world in (2, 4):
        if n < world:
            continue
        prefix = str(tmp_path / f"dig{world}")
        port = _free_port()
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                            "--master-addr", "127.0.0.1", "--master-port", str(port),
                            os.path.join(ROOT, "tests", "multi_gpu_parity.py"), "--parts", "8",
                            "--digest-out", prefix],
                           capture_output=True, text=True, timeout=900, cwd=ROOT)
        print(r.stdout[-3000:], r.stderr[-3000:])
        assert r.returncode == 0
        assert _digests(prefix, world) == one, world
