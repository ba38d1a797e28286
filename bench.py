"""Benchmark: sampled+feature-ready minibatches/s of the halo feature pipeline
(arXiv 2410.22697 prefetch + eviction) on B200, per BASELINE.json.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {mgnn,reference}] [--config C]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, one rank per GPU)

Default workload (BASELINE.json configs[3], the largest config that fits one GPU with its own
partitioning): ogbn-products-shaped synthetic graph (2,449,029 nodes, ~123.7M directed edges,
100-dim fp32 features), fanout [5, 10, 15], batch 2000, 2 partitions (trainers) per GPU, policy
for the total partition count P from the paper's GPU optima: P=2 (f=.50, gamma=.995,
Delta=32), P=4 (.50, .995, 32), P=8 (.50, .9995, 16); theta_R = 1.  `--config arxiv` etc. select
the other configs (arxiv's tables are L2-resident, so its line is not an HBM roofline).
One bench "step" = one WINDOW of consecutive minibatch steps for every partition on the GPU
(sample, classify, gather, tally, decay, and the eviction round that ends the window when the
window length divides Delta): e.g. 32 x 2 minibatches per GPU for products at P = 2.
Schedule (paper_2410_22697_b200/schedule.py, the paper's prepare-ahead, Alg.1 l.9): in timed
iteration i the sampling of window i+1 runs on a second stream concurrently with the
classify/gather/score of window i, and window i's column relabel on a third stream beside its
gather; the streams join at the end of the iteration.  Timing: per-
iteration CUDA events, L2 flushed (256 MB write) between timed iterations, the K-iteration run
repeated 3 times and the median reported, max over ranks.  `e2e` drives the same schedule through
the C ABI with the seeds in pinned HOST memory (H2D inside mgnn_sample) and every window's
per-minibatch counters read back to the host (D2H), same flush and per-iteration events.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from inputs import synth  # noqa: E402

METRIC = "sampled+feature-ready minibatches/sec"
UNIT = "minibatches/s"
DEFAULT_CONFIG = "products"
# the columns' relabel on a third stream beside the gather (schedule.PrepareAhead relabel_stream):
# products window 2.207 -> 2.162 ms, arxiv 0.214 -> 0.206 ms
RELABEL_STREAM = True
# Launch tuning by config (libmgnn reads these once per process, before its first launch; every variant
# is parity-tested in tests/test_gpu_variants.py): on products the next window's sampling stream runs at
# high priority with the persistent k_hop / k_compact grids capped at 5 blocks per SM, so its kernels
# are dispatched beside the gather instead of queueing behind the gather's blocks (products window
# 1.90 -> 1.80 ms, profiles/r02/gather_flat/exp_s29*); neutral on arxiv / cfg1, 1-4 % slower on reddit /
# papers_s32, which keep the defaults.
TUNING = {
    "products": {"env": {"MGNN_HOP_GRID_BPS": "5", "MGNN_COMPACT_BPS": "5"}, "sampling_priority": -1},
    # cfg1's ~2 MB tables: the TMA row gather (k_gather_g4) beats the flat gather by 4 % in the bench loop
    # (profiles/r02/tuning/exp_s37: 832-835k vs 796-799k minibatches/s); arxiv is equal or better flat
    "cfg1": {"env": {"MGNN_GATHER": "tma"}},
}

# Measurement policy (f_p in basis points, gamma, Delta) by config and total partitions P: the
# paper's GPU optima; theta_R = 1.  Looked up for the P actually used.
POLICY = {
    "cfg1": {2: (2500, 0.995, 64)},
    "arxiv": {2: (2500, 0.995, 32), 4: (5000, 0.995, 32), 8: (3500, 0.995, 128)},
    "reddit": {2: (3500, 0.995, 32), 4: (5000, 0.995, 256), 8: (5000, 0.95, 32)},
    "products": {2: (5000, 0.995, 32), 4: (5000, 0.995, 32), 8: (5000, 0.9995, 16)},
    "papers_s32": {8: (5000, 0.9995, 512)},
    "papers": {8: (5000, 0.9995, 512)},
}
# default partitions per GPU (configs 1-4: 2 trainers per GPU, P = 2N; papers: P = 8 at every N,
# 8/N per GPU) and the window length (steps per window; papers shorter: 8 trainers per GPU)
LAYOUT = {"cfg1": (2, 32), "arxiv": (2, 32), "reddit": (2, 32), "products": (2, 32), "papers_s32": (8, 16),
          "papers": (8, 16)}
FIXED_P = {"papers_s32": 8, "papers": 8}
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
    "papers": "ogbn-papers100M-shaped synthetic (111,059,956 nodes, ~3.23B directed edges, 128-d fp32), "
              "8 partitions, fanout [5,10,15], batch 2000 (BASELINE.json configs[4])",
}


class Setup:
    """Workload + layout chosen by the command line."""

    def __init__(self, name: str, world: int, parts_per_gpu=None, parts=None, window=None):
        self.name = name
        self.cfg = synth.CONFIGS[name]
        ppg, win = LAYOUT[name]
        if parts is None and name in FIXED_P:
            parts = FIXED_P[name]
        if parts is not None:
            if parts % world:
                raise SystemExit(f"--parts {parts} is not a multiple of the {world} GPUs")
            ppg = parts // world
        elif parts_per_gpu is not None:
            ppg = parts_per_gpu
        self.ppg = ppg
        self.P = ppg * world
        table = POLICY[name]
        k = min((q for q in table if q >= self.P), default=max(table))
        self.policy_P = k
        self.f_bp, self.gamma, self.delta = table[k]
        w = window or win
        self.window = min(w, self.delta) if self.delta > 0 else w
        self.sampling_priority = 0

    def workload(self) -> dict:
        return {
            "workload": WORKLOAD_TEXT[self.name], "config_name": self.name,
            "partitions": self.P, "partitions_per_gpu": self.ppg,
            "layout": ("P = 2 trainers per GPU (P = 2N)" if self.ppg == 2 and self.name not in FIXED_P else
                       f"P = {self.P} partitions, {self.ppg} per GPU"),
            "policy_for_P": self.policy_P, "f_p": self.f_bp / 10000, "gamma": self.gamma, "delta": self.delta,
            "theta_r": 1.0, "window_steps": self.window, "minibatches_per_step_per_gpu": self.window * self.ppg,
            "l2": "flushed (256 MB write) between timed windows",
            "launch": {"gather": os.environ.get("MGNN_GATHER", "flat"),
                       **{k: v for k, v in os.environ.items() if k.startswith("MGNN_")},
                       "sampling_stream_priority": self.sampling_priority},
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
        self.period = float(os.environ.get("BENCH_CLOCK_PERIOD_MS", "1")) / 1e3

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
            time.sleep(self.period)

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


def nvlink_counters(index: int):
    """NVLink throughput counters of one GPU (NVML field values, KiB since driver load; None if the
    driver does not expose them): read before and after the timed region, so the difference is the
    bytes that crossed this GPU's links while it ran."""
    try:
        import pynvml as nv
        import torch
        nv.nvmlInit()
        pr = torch.cuda.get_device_properties(index)
        want = (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
        h = None
        for i in range(nv.nvmlDeviceGetCount()):              # the NVML device of this CUDA ordinal
            hh = nv.nvmlDeviceGetHandleByIndex(i)
            pci = nv.nvmlDeviceGetPciInfo(hh)
            if (int(pci.domain), int(pci.bus), int(pci.device)) == want:
                h = hh
        if h is None:
            return None
        ids = [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX]
        vals = nv.nvmlDeviceGetFieldValues(h, ids)
        if all(v.nvmlReturn == 0 for v in vals):
            return [int(v.value.ullVal) * 1024 for v in vals] + ["NVLINK_THROUGHPUT_DATA_TX/RX (KiB)"]
        # per-link byte counters, summed over the links (scopeId = link index)
        tx = rx = 0
        ok = False
        for link in range(18):
            vv = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, link),
                                                 (nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, link)])
            if vv[0].nvmlReturn == 0 and vv[1].nvmlReturn == 0:
                tx += int(vv[0].value.ullVal)
                rx += int(vv[1].value.ullVal)
                ok = True
        if ok:
            return [tx, rx, "NVLINK_COUNT_XMIT/RCV_BYTES summed over links"]
        return nvidia_smi_nvlink(nv.nvmlDeviceGetIndex(h))
    except Exception:
        return None


def nvidia_smi_nvlink(nvml_index: int):
    """`nvidia-smi nvlink -gt d -i N`: per-link data Tx / Rx counters (KiB), summed; None if unavailable."""
    import re
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(nvml_index)], capture_output=True,
                             text=True, timeout=20).stdout
    except Exception:
        return None
    tx = rx = 0
    found = False
    for line in out.splitlines():
        m = re.search(r"(Tx|Rx)\s*:?\s*([0-9]+)\s*KiB", line)
        if m:
            found = True
            if m.group(1) == "Tx":
                tx += int(m.group(2)) * 1024
            else:
                rx += int(m.group(2)) * 1024
    return [tx, rx, "nvidia-smi nvlink -gt d (KiB per link, summed)"] if found else None


def traffic_table(name: str):
    """Per-config ncu DRAM bytes per launch (profiles/r02/traffic_<config>.json, written by
    tools/ncu_traffic.py from a committed `ncu --set full` capture of this config); None if absent."""
    p = os.path.join(ROOT, "profiles", "r02", f"traffic_{name}.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d if d.get("config") == name else None
    except (OSError, ValueError):
        return None


def gather_kernel_name(g4_eligible: bool = False) -> str:
    """The gather kernel the library launches (MGNN_GATHER, read once per process by libmgnn): flat
    (default) -> k_gather_flat; tma -> k_gather_g4 (TMA row gather) when the hosted tables fit in 3/4 of
    L2 and the rows are unpadded and at most 256 floats (the library's rule, api.cu / gather.cu; also
    MGNN_GATHER_G4), else k_gather_tma; reg -> k_gather."""
    e = os.environ.get("MGNN_GATHER", "flat")
    if e.startswith("t"):
        g4 = os.environ.get("MGNN_GATHER_G4", "2")
        return "k_gather_g4" if (g4 == "1" or (g4 == "2" and g4_eligible)) else "k_gather_tma"
    return "k_gather" if e.startswith("r") else "k_gather_flat"


def sampler_ncu_dram(tt, layers: int, peak: float):
    """The sampler kernels' DRAM rate from the committed ncu table alone (one source for bytes and time):
    (k_hop x L + k_compact x L + k_relabel) DRAM bytes per window / their ncu time per window, against the
    HBM peak -- next to the SURVEY §8(d) algorithmic-bytes fraction, which counts 8 B per sampled edge
    although every edge is one random DRAM burst."""
    ks = (tt or {}).get("kernels", {})
    if not all(k in ks for k in ("k_hop", "k_compact", "k_relabel")):
        return None
    n = {"k_hop": layers, "k_compact": layers, "k_relabel": 1}
    b = sum(ks[k]["dram_bytes_per_launch"] * n[k] for k in n)
    us = sum(ks[k]["us_per_launch"] * n[k] for k in n)
    gbs = b / (us * 1e-6) / 1e9 if us > 0 else None
    return {"bytes_per_window": b, "us_per_window_serialised": us, "gbs": gbs,
            "frac": (gbs / peak) if gbs else None, "source": (tt or {}).get("source")}


def random_load_peak(table_bytes=None):
    """Measured random-load ceiling (profiles/r02/randread.json, tools/randread.cu): of an L2-resident
    table, or (table_bytes given) of the smallest measured table at least that large (DRAM-resident)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "randread.json")) as f:
            d = json.load(f)
        if table_bytes is None:
            return float(d["l2_resident_random_loads_g_per_s"]), "L2-resident table"
        rows = sorted((r for r in d["rows"] if (r["table_mb"] << 20) >= table_bytes), key=lambda r: r["table_mb"])
        rows = rows or sorted(d["rows"], key=lambda r: -r["table_mb"])
        best = max(r["g_loads_per_s"] for r in rows if r["table_mb"] == rows[0]["table_mb"])
        return float(best), f"{rows[0]['table_mb']} MB table"
    except (OSError, ValueError, KeyError, IndexError):
        return None, None


def git_head():
    if os.environ.get("MGNN_GIT_HEAD"):          # the GPU box's copy has no .git: the caller passes it
        return os.environ["MGNN_GIT_HEAD"]
    try:
        return subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], cwd=ROOT, capture_output=True,
                              text=True, timeout=10).stdout.strip() or None
    except Exception:
        return None


# ---------------------------------------------------------------- oracle timings (test infrastructure)
def oracle_rate(S: Setup, parts, budget_s: float, remote=False, dense=False, min_steps: int = 8):
    """Oracle (oracle/orc.c, single thread) on the same workload: minibatches/s over a bounded sample."""
    from oracle import oracle as O
    W = O.World(parts, S.cfg.feat_dim, synth.FEAT_SEED, dense=dense)
    alpha = O.alpha_default(S.gamma, S.delta)
    for p in W.parts:
        p.buffer_init(S.gamma, alpha, 1.0, S.delta, S.f_bp)
        p.set_expand_remote(remote)
    t0 = time.perf_counter()
    n_mb, step = 0, 1
    while True:
        for p in W.parts:
            p.step(synth.RUN_SEED, step, S.cfg.fanouts, S.cfg.batch)
            n_mb += 1
        step += 1
        el = time.perf_counter() - t0
        if step > min_steps and el >= budget_s:
            break
    W.close()
    return n_mb / el, n_mb, el


def oracle_rate_threads(S: Setup, parts, budget_s: float, remote=False, dense=False):
    """The same oracle with one host thread per partition (the C steps release the GIL; partitions
    are independent between eviction rounds of their own buffers): SURVEY §8(d)'s P-thread rate."""
    import threading as th
    from oracle import oracle as O
    W = O.World(parts, S.cfg.feat_dim, synth.FEAT_SEED, dense=dense)
    alpha = O.alpha_default(S.gamma, S.delta)
    for p in W.parts:
        p.buffer_init(S.gamma, alpha, 1.0, S.delta, S.f_bp)
        p.set_expand_remote(remote)
    counts = [0] * len(W.parts)
    t0 = time.perf_counter()

    def run(i):
        step = 1
        while time.perf_counter() - t0 < budget_s or step <= 8:
            W.parts[i].step(synth.RUN_SEED, step, S.cfg.fanouts, S.cfg.batch)
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


def run_reference(args, S: Setup):
    """The reference arm: the oracle (no reference code exists; /root/reference holds only the paper)
    on the same workload, the GPU's hosted partitions, steps in order from t = 1.  Each bench step is
    a bounded sample of a window (`ref_steps` consecutive steps of every hosted partition) so the
    whole --steps K --warmup W run stays within a few minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    g = synth.generate(S.cfg)
    parts = synth.partition(g, S.P)
    from oracle import oracle as O
    mine_ids = list(range(S.ppg))
    W = O.World([parts[i] for i in range(S.P)], S.cfg.feat_dim, synth.FEAT_SEED)
    alpha = O.alpha_default(S.gamma, S.delta)
    for p in W.parts:
        p.buffer_init(S.gamma, alpha, 1.0, S.delta, S.f_bp)
    mine = [W.parts[i] for i in mine_ids]
    # steps per reference bench step: ~1 s of single-thread work at the oracle's rate on this config
    per_mb_s = {"cfg1": 0.001, "arxiv": 0.006, "reddit": 0.035, "products": 0.075, "papers_s32": 0.04,
                "papers": 0.1}.get(S.name, 0.05)
    ref_steps = int(max(1, min(S.window, round(1.0 / (per_mb_s * S.ppg)))))
    t = 1
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for w in range(ref_steps):
            for p in mine:
                p.step(synth.RUN_SEED, t + w, S.cfg.fanouts, S.cfg.batch)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
        t += ref_steps
    W.close()
    total = sum(times)
    per_step = ref_steps * S.ppg
    value = per_step * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": S.workload(),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} bench steps x {ref_steps} consecutive steps x {S.ppg} hosted "
                                   f"partitions (P={S.P}), steps 1..{t - 1} in order, single-threaded C oracle"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--runs", type=int, default=3, help="timed runs of --steps iterations; the median is reported")
    ap.add_argument("--impl", default="mgnn", choices=["mgnn", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(LAYOUT),
                    help=f"workload (default: {DEFAULT_CONFIG}-shaped, BASELINE.json configs[3])")
    ap.add_argument("--parts-per-gpu", type=int, default=None, help="partitions (trainers) per GPU")
    ap.add_argument("--parts", type=int, default=None, help="total partitions P (a multiple of the GPU count)")
    ap.add_argument("--window", type=int, default=None, help="steps per window (default per config)")
    ap.add_argument("--static-arenas", action="store_true",
                    help="size window arenas for the static worst case instead of a pilot-measured bound")
    ap.add_argument("--sm-split", type=int, default=0,
                    help="mgnn_sm_partition: gather + scoring on this many SMs, sampling on the rest (0 = whole GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-extras", action="store_true", help="skip the with_consumer / with_training lines")
    ap.add_argument("--no-tuning", action="store_true", help="library launch defaults (ignore TUNING)")
    ap.add_argument("--no-gather-events", action="store_true",
                    help="experiment: no events around the gather in the timed runs (roofline then unavailable)")
    ap.add_argument("--no-train-graph", action="store_true", help="training steps as eager launches")
    ap.add_argument("--remote", action="store_true",
                    help="NEXT-1: sample non-local frontier nodes from their owner's CSR")
    ap.add_argument("--dense", action="store_true", help="NEXT-1: dense S_A (every non-local node scorable)")
    ap.add_argument("--hash-partition", action="store_true",
                    help="NEXT-4 stress: partitions of a randomly relabelled graph (hash partitioner)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    S = Setup(args.config, world if args.impl == "mgnn" else args.gpus, args.parts_per_gpu, args.parts, args.window)
    if args.impl == "reference":
        return run_reference(args, S)

    tune = {} if args.no_tuning else TUNING.get(S.name, {})
    for k_, v_ in tune.get("env", {}).items():
        os.environ.setdefault(k_, v_)
    S.sampling_priority = tune.get("sampling_priority", 0)
    import torch
    import torch.distributed as dist
    from paper_2410_22697_b200 import pipeline as PL
    from paper_2410_22697_b200.schedule import PrepareAhead

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
    cfg = S.cfg
    WINDOW = S.window
    g = synth.generate(cfg)
    if args.hash_partition:
        g = synth.hash_relabel(g)
    parts = synth.partition(g, S.P)
    hosted = list(range(S.ppg * rank, S.ppg * (rank + 1)))
    ctx = PL.build_context(local, parts, cfg.feat_dim, synth.FEAT_SEED, hosted, dense=args.dense)
    if world > 1:
        PL.exchange_tables(ctx)
    alpha = PL.alpha_default(S.gamma, S.delta)
    # INITIALIZE_PREFETCHER cost ("<1% of overall training"), CUDA events on the init stream
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    i0.record()
    ctx.buffer_init(S.gamma, alpha, 1.0, S.delta, S.f_bp)
    i1.record()
    torch.cuda.synchronize()
    init_ms = i0.elapsed_time(i1)
    if args.remote:
        if world > 1:
            ctx.load_global_csr(g.indptr, g.cols)       # replicated global CSR on every GPU
        ctx.expand_remote(True)
    # realistic window arenas (mgnn_sampler_config_bounded): the largest |F_L| of a one-step pilot x 1.25;
    # a window that still overflows is skipped on the device and reported, and the run is redone with a
    # doubled bound (resuming at the overflowed step)
    rows_bound = 0 if args.static_arenas else PL.estimate_rows_bound(ctx, cfg.fanouts, cfg.batch, synth.RUN_SEED)
    if world > 1:                                # one bound for every rank (the largest)
        rb = torch.tensor([rows_bound], dtype=torch.int64, device="cuda")
        dist.all_reduce(rb, op=dist.ReduceOp.MAX)
        rows_bound = int(rb.item())
    ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, WINDOW, rows_bound=rows_bound)
    sm_split = ctx.sm_partition(args.sm_split) if args.sm_split else None
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        t_ = torch.tensor([x], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        return float(t_.item())

    # Two streams = the paper's prepare-ahead overlap (Alg.1 l.9): NeighborSampler of window w+1
    # (needs no buffer state) runs on stream A while window w is classified/gathered/scored on B.
    from paper_2410_22697_b200._lib import MgnnError
    K = args.steps
    R = max(1, args.runs)
    mb_total = WINDOW * S.ppg * world * K
    t_first = 1
    for attempt in range(4):
        pipe = PrepareAhead(ctx, WINDOW, t0=t_first, stream_b=stream, relabel_stream=RELABEL_STREAM,
                            sampling_priority=tune.get("sampling_priority", 0))
        for _ in range(args.warmup):
            pipe.iteration()
        # ---------------- timed region (device path: inputs resident in HBM); R runs, median reported
        nv0 = nvlink_counters(local) if world > 1 else None
        launches0 = ctx.launch_count()
        # events around the gather launch only (its roofline); events between the other launches
        # would end their programmatic overlap (PDL) and lengthen the step (cfg1: 72 -> 85 us)
        ctx.profile(not args.no_gather_events, gather_only=True)
        ctx.profile_stages()                     # reset
        runs = []
        prof = {}
        wall = 0.0
        with ClockSampler(local) as clk:
            for r in range(R):
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
                barrier()
                wall0 = time.perf_counter()
                for i in range(K):
                    pipe.iteration(events=ev[i])
                barrier()
                wall += time.perf_counter() - wall0
                tot_ms = sum(a.elapsed_time(b) for a, b in ev)
                max_ms = max_over_ranks(tot_ms)
                runs.append({"value": mb_total / (max_ms / 1e3), "ms_per_step": max_ms / K, "my_ms": tot_ms})
                ps = ctx.profile_stages()
                for k_, v_ in ps.items():
                    prof[k_] = prof.get(k_, 0.0) + v_
        # one more run with every stage bracketed by events: the per-stage times and the sampler's
        # roofline (not part of `value`)
        ctx.profile(True)
        ev_s = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        barrier()
        for i in range(K):
            pipe.iteration(events=ev_s[i])
        barrier()
        stage_prof = ctx.profile_stages()
        stage_prof["window_ms"] = sum(a.elapsed_time(b) for a, b in ev_s) / K
        ctx.profile(False)
        ovf = 0
        try:
            ctx.counts(pipe.slot ^ 1, stream)    # EOVERFLOW if any window of the run overflowed its arena
        except MgnnError as e:
            if e.status != 6:
                raise
            ovf = 1
        if world > 1:
            ot = torch.tensor([ovf], dtype=torch.int64, device="cuda")
            dist.all_reduce(ot, op=dist.ReduceOp.MAX)
            ovf = int(ot.item())
        if not ovf:
            break
        print(f"[bench] arena bound {rows_bound} rows overflowed; retrying with {2 * rows_bound}", file=sys.stderr)
        barrier()
        rows_bound *= 2
        ctx.sampler_config(cfg.fanouts, cfg.batch, synth.RUN_SEED, WINDOW, rows_bound=rows_bound)
        t_first = ctx.next_step()                # resume at the overflowed window
    launches = ctx.launch_count() - launches0
    nv1 = nvlink_counters(local) if world > 1 else None
    clocks = clk.summary()
    order = sorted(range(R), key=lambda j: runs[j]["value"])
    med = runs[order[R // 2]]
    value = med["value"]
    c = ctx.counts(pipe.slot ^ 1, stream)       # the last consumed window
    hits = int(c[:, 2].sum())
    misses = int(c[:, 3].sum())
    peer_rows = int(c[:, 7].sum())              # rows read from another GPU's table over NVLink

    # ---------------- e2e: host seeds (pinned) -> C ABI -> counts back to host, every window, through the
    # same schedule (flush between iterations, per-iteration events).  The seeds a user passes are the
    # window's F_0; take them from the library's epoch order by sampling the same steps first (sampling
    # reads no buffer state), outside the timed region.
    n_inst = S.ppg * WINDOW
    E2E = max(3, K)
    pipe.iteration(prepare_next=False)          # consume the window the device run left prepared
    t_e2e = pipe.t
    seeds_h, counts_h = {}, {}
    slot = pipe.slot
    for i in range(E2E):
        tt = t_e2e + i * WINDOW
        ctx.sample(slot, tt, WINDOW, stream=stream)
        wv = ctx.window(slot)
        n0 = PL.device_view(wv.hop_size, (wv.n_inst, 9), "i8")[:, 0].to(torch.int32)
        f0 = PL.device_view(wv.frontier, (wv.n_inst, wv.rows_stride), "i4")[:, :cfg.batch]
        seeds_h[tt] = f0.cpu().pin_memory()
        counts_h[tt] = n0.cpu().pin_memory()
    h2d = n_inst * cfg.batch * 4 + n_inst * 4
    d2h = n_inst * 8 * 8
    cbuf = [torch.zeros((n_inst, 8), dtype=torch.int64).pin_memory() for _ in range(2)]
    ev_cnt = [torch.cuda.Event(), torch.cuda.Event()]
    state = {"i": 0, "hits": 0}
    epipe = PrepareAhead(ctx, WINDOW, t0=t_e2e, stream_b=stream, relabel_stream=RELABEL_STREAM,
                         host_seeds=lambda sl, tt: (seeds_h[tt].data_ptr(), counts_h[tt].data_ptr()))
    epipe.sA = pipe.sA
    epipe.flush = pipe.flush

    def read_counts(sl, t0_, sB):
        i = state["i"]
        ctx.counts_async(sl, cbuf[i % 2].data_ptr(), sB)      # D2H of the window's counters
        ev_cnt[i % 2].record(sB)

    ev_e = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(E2E)]
    barrier()
    for i in range(E2E):
        state["i"] = i
        epipe.iteration(events=ev_e[i], after_consume=read_counts, prepare_next=i + 1 < E2E)
        if i >= 1:                             # read the previous window's counters on the host
            ev_cnt[(i - 1) % 2].synchronize()
            state["hits"] += int(cbuf[(i - 1) % 2][:, 2].sum())
    ev_cnt[(E2E - 1) % 2].synchronize()
    state["hits"] += int(cbuf[(E2E - 1) % 2][:, 2].sum())
    barrier()
    e2e_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev_e))
    e2e_value = WINDOW * S.ppg * world * E2E / (e2e_ms / 1e3)
    t_next = epipe.t
    slot = epipe.slot
    ctx.defer_relabel(False)                     # the consumer / training loops below relabel in mgnn_sample

    line_extra = {}
    if not args.no_extras:
        try:
            line_extra = extras(args, S, ctx, pipe, t_next, slot, world, barrier, max_over_ranks, mb_total, K,
                                med["ms_per_step"], prof, R)
        except MgnnError as e:              # e.g. the training buffers of a 128-instance window do not fit
            torch.cuda.synchronize()
            line_extra = {"with_consumer_or_training": {"skipped": str(e)}}

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        peak_src = ("MEASURED_PEAKS.json hbm_gbs (measured copy, burst: each kernel is timed alone per launch)"
                    if "hbm_gbs" in peaks else "fallback 6.65 TB/s (B200_PROFILING.md)")
        n_win = R * K
        g_ms = prof["gather_ms"] / max(prof["gather_calls"], 1)
        g_bytes = 2.0 * prof["gather_rows"] * cfg.feat_dim * 4 / max(prof["gather_calls"], 1)
        achieved = g_bytes / (g_ms / 1e3) / 1e9 if g_ms > 0 else None
        sp_ = stage_prof
        s_ms = sp_["sample_ms"] / max(sp_["sample_calls"], 1)
        s_bytes = (8.0 * sp_["edges"] + 24.0 * sp_["frontier"] + 8.0 * sp_["unique"]) / max(sp_["sample_calls"], 1)
        s_ach = s_bytes / (s_ms / 1e3) / 1e9 if s_ms > 0 else None
        tt_ = traffic_table(S.name)
        cfg_layers = len(cfg.fanouts)
        pitch_ = (cfg.feat_dim + 3) // 4 * 4
        l2_res = (sum(len(parts[q].indptr) - 1 for q in hosted) * pitch_ * 4
                  <= torch.cuda.get_device_properties(local).L2_cache_size * 3 // 4)
        g_kernel = gather_kernel_name(l2_res and pitch_ == cfg.feat_dim and pitch_ <= 256 and S.ppg <= 8)
        # k_relabel is bound by dependent random probes of L2-resident (bits, position) pairs, not bytes:
        # probes per window (counted by the kernel) / its event time vs the measured L2 random-load ceiling
        rl_ms = sp_["relabel_ms"] / max(sp_["relabel_calls"], 1)
        rl_probes = sp_["relabel_probes"] / max(sp_["relabel_calls"], 1)
        rl_peak, _ = random_load_peak()
        rl_rate = rl_probes / (rl_ms / 1e3) / 1e9 if rl_ms > 0 and rl_probes > 0 else None
        # k_hop: one random 4-byte column load per sampled edge from the hosted partitions' cols_rank
        # (ncu per-launch time at HEAD from the committed traffic table) vs the random-load ceiling of a
        # DRAM table of that size
        cols_bytes = sum(int(parts[q].cols.nbytes) for q in hosted)
        hop_peak, hop_tab = random_load_peak(cols_bytes)
        hop_us = ((tt_ or {}).get("kernels", {}).get("k_hop", {}) or {}).get("us_per_launch")
        e_win = sp_["edges"] / max(sp_["sample_calls"], 1)
        hop_rate = e_win / (cfg_layers * hop_us * 1e-6) / 1e9 if hop_us else None
        hop_roof = {"bound": "dram_random_loads", "edges_per_window": e_win, "launches_per_window": cfg_layers,
                    "us_per_launch_ncu": hop_us, "achieved": hop_rate, "unit": "G loads/s", "peak": hop_peak,
                    "frac": (hop_rate / hop_peak) if hop_rate and hop_peak else None,
                    "peak_source": f"profiles/r02/randread.json ({hop_tab}: hosted cols_rank = {cols_bytes >> 20} MB)",
                    "note": "k > 1 samples of a node share its CSR row, so the loads beat fully random ones"}
        relabel_roof = {"bound": "l2_random_loads", "probes_per_window": rl_probes,
                        "probes_per_edge": rl_probes / max(sp_["edges"] / max(sp_["sample_calls"], 1), 1.0),
                        "ms_per_window": rl_ms, "achieved": rl_rate, "unit": "G loads/s", "peak": rl_peak,
                        "frac": (rl_rate / rl_peak) if rl_rate and rl_peak else None,
                        "peak_source": "profiles/r02/randread.json (tools/randread.cu, L2-resident random loads)",
                        "note": "deferred k_relabel on its own stream beside the gather (time includes the sharing)"}
        step_ms_sum = sum(r_["my_ms"] for r_ in runs)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": med["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded planted-block R-MAT graph, Philox features)",
            "config": dict(S.workload(), **({"sampling": "remote expansion (NEXT-1)"} if args.remote else {}),
                           **({"scores": "dense S_A (NEXT-1)"} if args.dense else {}),
                           **({"partitioner": "hash (random relabel)"} if args.hash_partition else {}),
                           **({"sm_partition": {"gather_sms": sm_split[0], "prepare_sms": sm_split[1]}}
                              if sm_split else {}),
                           graph_stats=synth.describe(g, parts)),
            "runs": [r_["value"] for r_ in runs], "median_of": R,
            "buffer_init_ms": init_ms,
            "arenas": {"rows_bound_per_instance": rows_bound or "static worst case",
                       "static_bound": static_ucap(S),
                       "x_bytes_per_slot": (rows_bound or static_ucap(S)) * (((cfg.feat_dim + 3) // 4) * 4) * 4
                       * S.ppg * WINDOW,
                       "note": "mgnn_sampler_config_bounded: pilot max |F_L| x 1.25; overflow -> skipped + retried"},
            "hit_rate": prof["hits"] / max(1.0, prof["hits"] + prof["misses"]),
            "hit_rate_note": "buffer hits / halo accesses over every timed window (R#23 unique nodes per minibatch)",
            "hit_rate_last_window": hits / max(1, hits + misses),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": E2E, "path": "schedule.PrepareAhead with host seeds: mgnn_sample(pinned host seeds, "
                                          "H2D) | lookup_gather + score_evict_refill + counts_read_async (D2H); "
                                          "host reads each window's counters; L2 flushed between windows"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": f"{g_kernel} (classify + feature-row gather)",
                         "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": (achieved / hbm_peak) if achieved else None,
                         "traffic": (tt_ or {}).get(g_kernel),
                         "traffic_source": (tt_ or {}).get("source"),
                         "peak_source": peak_src, "launch_ms": g_ms, "share_of_step": prof["gather_ms"] / max(step_ms_sum, 1e-9),
                         "algorithmic_bytes_per_launch": g_bytes,
                         "algorithmic": "2 * rows * D * 4 (row read + X write, SURVEY §8(d))"},
            "sampler_roofline": {
                "bound": "hbm", "kernels": "k_hop x L + k_compact x L + k_relabel (stream A, beside the gather)",
                "achieved": s_ach, "peak": hbm_peak, "unit": "GB/s", "frac": (s_ach / hbm_peak) if s_ach else None,
                "ms_per_window": s_ms, "share_of_step": s_ms / max(sp_["window_ms"], 1e-9),
                "measured": "stage-profiled run after the timed runs (every call bracketed by events)",
                "algorithmic_bytes_per_window": s_bytes,
                "algorithmic": "8 E + 24 F + 8 U (SURVEY §8(d)): E sampled edges, F expanded frontier nodes, U = |F_L|",
                "per_window": {"E": sp_["edges"] / max(sp_["sample_calls"], 1),
                               "F": sp_["frontier"] / max(sp_["sample_calls"], 1),
                               "U": sp_["unique"] / max(sp_["sample_calls"], 1)},
                "traffic": {k_: v_ for k_, v_ in (tt_ or {}).items() if k_ in ("k_hop", "k_compact", "k_relabel")}
                or None,
                "ncu_dram": sampler_ncu_dram(tt_, cfg_layers, hbm_peak),
                "relabel": relabel_roof, "hop": hop_roof},
            "stages_ms_per_window": {"sample": s_ms,
                                     "gather": sp_["gather_ms"] / max(sp_["gather_calls"], 1),
                                     "score": sp_["score_ms"] / max(sp_["score_calls"], 1),
                                     "relabel": sp_["relabel_ms"] / max(sp_["relabel_calls"], 1),
                                     "window_pipelined": sp_["window_ms"],
                                     "note": "CUDA events per call on the stream it runs on, in one extra run of "
                                             "K windows after the timed runs (stage events end the launches' "
                                             "programmatic overlap, so they are kept out of `value`)"},
            "clocks": clocks,
            "wall_s_timed_region": wall,
            "git_head": git_head(),
        }
        line.update(line_extra)
        if world > 1:
            nv_bytes = peer_rows * cfg.feat_dim * 4
            gbs = nv_bytes / (g_ms / 1e3) / 1e9 if g_ms > 0 else None
            peer = peer_copy_gbs(local, (local + 1) % torch.cuda.device_count())
            cnt = None
            if nv0 and nv1:
                txw, rxw = (nv1[0] - nv0[0]) / n_win, (nv1[1] - nv0[1]) / n_win
                cnt = {"tx_bytes_per_window": txw, "rx_bytes_per_window": rxw,
                       "rx_gbs_over_window": rxw / (med["ms_per_step"] / 1e3) / 1e9,
                       "source": f"NVML {nv0[2]} of this GPU around the timed runs"}
            else:
                cnt = {"unavailable": "NVML NVLink throughput / byte counters not exposed on this driver"}
            line["nvlink"] = {"peer_rows_per_window": peer_rows, "bytes_per_window": nv_bytes,
                              "gbs_during_gather": gbs,
                              "peak_gbs": 900.0, "peak_source": "NVLink 5 nominal per direction per GPU",
                              "frac": gbs / 900.0 if gbs else None,
                              "achievable_peer_copy_gbs": peer,
                              "frac_of_achievable": gbs / peer if (gbs and peer) else None,
                              "counters": cnt,
                              "note": "miss + refill rows whose owner is on another GPU, read by peer loads "
                                      "inside k_gather / k_swap_refill (last timed window); achievable = "
                                      "256 MB device-to-device copy to the next GPU, best of 5"}
        if world == 1 and not args.no_cpu_baseline:
            rate, n_mb, el = oracle_rate(S, parts, args.cpu_budget, args.remote, args.dense)
            rate_p, n_thr = oracle_rate_threads(S, parts, min(args.cpu_budget, 6.0), args.remote, args.dense)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                                    "sample": f"{n_mb} minibatches (steps 1..{n_mb // S.P} of all {S.P} partitions), "
                                              f"{el:.1f} s, single-threaded C oracle",
                                    "value_one_thread_per_partition": rate_p, "threads": n_thr,
                                    "host_cpu": host_cpu(), "host_nproc": os.cpu_count()}
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()                 # peers read our feature tables until everyone is done
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def static_ucap(S) -> int:
    """min(B * prod(1 + k_i), |V|): the worst-case |F_L| the static arenas are sized for."""
    u = S.cfg.batch
    for k in S.cfg.fanouts:
        u *= 1 + k
    return int(min(u, S.cfg.n_nodes))


def extras(args, S, ctx, pipe, t_start, slot, world, barrier, max_over_ranks, mb_total, K, prep_ms, prof, R):
    """with_consumer (A14) and with_training (NEXT-3) lines, plus the Eq.4-5 stage report."""
    import torch
    from paper_2410_22697_b200._lib import MgnnError
    from paper_2410_22697_b200 import pipeline as PL
    cfg = S.cfg
    WINDOW = S.window
    sA, sB = pipe.sA, pipe.sB
    ev_sampled = [torch.cuda.Event(), torch.cuda.Event()]
    ev_done = [torch.cuda.Event(), torch.cuda.Event()]
    flush = pipe.flush
    # ---------------- with consumer (A14): the same pipeline plus the GraphSAGE-mean forward of every
    # minibatch (mgnn_sage_forward, tcgen05 TF32) on stream C, while stream B gathers and scores window
    # w+1 and stream A samples window w+2; a slot is resampled only after its score (B) and forward (C).
    dims = synth.sage_dims(cfg.feat_dim, len(cfg.fanouts), synth.N_CLASSES[cfg.name])
    wts = synth.sage_weights(dims)
    ctx.sage_config(dims, [w_[0] for w_ in wts], [w_[1] for w_ in wts], [w_[2] for w_ in wts])
    logits = torch.empty((S.ppg * WINDOW, cfg.batch, dims[-1]), dtype=torch.float32, device="cuda")
    fwd_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
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

    t_c = t_start
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
    c_ms = max_over_ranks(c0.elapsed_time(c1))
    c_value = mb_total / (c_ms / 1e3)
    fwd_ms = sum(a.elapsed_time(b) for a, b in fwd_ev) / K
    # algorithmic work of the last forward (window slot ^ 1): per layer 2 * n_dst * (2 d_in) * d_out
    # flops (dense part) and the neighbour rows it averages (4 * d_in bytes per sampled edge)
    wv = ctx.window(slot ^ 1)
    hs = PL.device_view(wv.hop_size, (wv.n_inst, 9), "i8").cpu().numpy()
    L_ = len(cfg.fanouts)
    flops = 0.0
    agg_bytes = 0.0
    for l in range(L_):
        hop = L_ - 1 - l
        n_dst = hs[:, hop].astype(np.float64)
        flops += float((2.0 * n_dst * 2 * dims[l] * dims[l + 1]).sum())
        offs = PL.device_view(wv.offsets[hop], (wv.n_inst, wv.off_stride[hop]), "i8")
        n_edges = np.array([int(offs[m, int(hs[m, hop])]) for m in range(wv.n_inst)], np.float64)
        agg_bytes += float((n_edges * dims[l] * 4).sum())

    out = {"with_consumer": {
            "value": c_value, "unit": UNIT, "ms_per_step": c_ms / K,
            "model": f"GraphSAGE-mean {dims} (random init), forward of every minibatch",
            "consumer_ms_per_step": fwd_ms, "consumer_launches_per_step": 2 * L_,
            "pipeline": "3 streams: sample(w+2) | gather+score(w+1) | forward(w), timed as one span",
            "kernel": "k_mean (neighbour means, all SMs) + k_sage_gemm (warp-specialised: TMA ring of self "
                      "rows / means / weights -> tcgen05.mma kind::tf32, 3 products per term (3xTF32), into 2 TMEM accumulators -> "
                      "bias/ReLU epilogue warps)",
            "tflops": flops / (fwd_ms / 1e3) / 1e12 if fwd_ms > 0 else None,
            "agg_gbs": agg_bytes / (fwd_ms / 1e3) / 1e9 if fwd_ms > 0 else None,
            "dtype": ("tf32 x tf32 -> f32" if os.environ.get("MGNN_SAGE_TF32") == "1"
                      else "3xtf32 (hi/lo split, fp32-grade products) -> f32")}}
    try:
        out.update(_train_extras(args, S, ctx, WINDOW, world, barrier, max_over_ranks, K, prep_ms, sA, sB, sC,
                                 ev_sampled, ev_done, ev_gathered, flush, slot, t_c, dims, lr_=0.01))
    except MgnnError as e:             # e.g. the training buffers of a 128-instance window do not fit
        torch.cuda.synchronize()
        out["with_training"] = {"skipped": str(e)}
    return out


def _train_extras(args, S, ctx, WINDOW, world, barrier, max_over_ranks, K, prep_ms, sA, sB, sC, ev_sampled, ev_done,
                  ev_gathered, flush, slot, t_c, dims, lr_):
    import torch
    from paper_2410_22697_b200 import pipeline as PL
    cfg = S.cfg
    # ---------------- with training (NEXT-3): every minibatch trains the model -- forward, loss,
    # backward, NCCL all-reduce of the gradients across ranks (N > 1), SGD -- on stream C, one
    # DDP step per window step (the steps of a window are sequential through the weights), while
    # streams A/B prepare the next windows (Alg.1: prepare(t+1) || train(t)).
    labels = synth.node_labels(cfg.n_nodes, dims[-1])
    ctx.train_config(labels)
    n_trainers = S.ppg * world
    lr = lr_
    ev_trained = [torch.cuda.Event(), torch.cuda.Event()]

    def sample_async_t(sl, tt):
        sA.wait_event(ev_done[sl])
        sA.wait_event(ev_trained[sl])
        ctx.sample(sl, tt, WINDOW, stream=sA)
        ev_sampled[sl].record(sA)

    graphs = {}
    # one rank: graph capture; N > 1 keeps eager launches (the step is GPU-bound either way, and a
    # graph holding captured NCCL work hung the process teardown)
    use_graph = [not args.no_train_graph and world == 1]

    def train_window(sl, stream_):
        if use_graph[0]:
            if sl not in graphs:
                try:
                    g_ = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g_, stream=stream_):
                        for w_ in range(WINDOW):
                            PL.ddp_step(ctx, sl, w_, n_trainers, lr, stream=torch.cuda.current_stream())
                    graphs[sl] = g_
                except Exception as e:  # capture unsupported here: stay eager
                    print(f"[bench] training graph capture failed ({e!r}); eager launches", file=sys.stderr)
                    use_graph[0] = False
            if use_graph[0]:
                with torch.cuda.stream(stream_):
                    graphs[sl].replay()
                return
        for w_ in range(WINDOW):
            PL.ddp_step(ctx, sl, w_, n_trainers, lr, stream=stream_)

    tw_ev = []

    def consume_train(sl, timed=False):
        sB.wait_event(ev_sampled[sl])
        ctx.lookup_gather(sl, sB)
        ev_gathered[sl].record(sB)
        ctx.score(sl, sB)
        ev_done[sl].record(sB)
        sC.wait_event(ev_gathered[sl])
        if timed:
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e[0].record(sC)
        train_window(sl, sC)
        if timed:
            e[1].record(sC)
            tw_ev.append(e)
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
        consume_train(slot, timed=True)
        t_t += WINDOW
        slot ^= 1
    sB.wait_stream(sA)
    sB.wait_stream(sC)
    t1e.record(sB)
    barrier()
    tr_ms = max_over_ranks(t0e.elapsed_time(t1e))
    tr_value = WINDOW * S.ppg * world * KT / (tr_ms / 1e3)
    tr_loss_t = torch.tensor([ctx.loss(sC) / (KT * WINDOW)], dtype=torch.float64, device="cuda")
    if world > 1:                       # each rank holds its trainers' share of the mean loss
        import torch.distributed as dist
        dist.all_reduce(tr_loss_t)
    tr_loss = float(tr_loss_t.item())
    t_ddp_overlapped = sum(a.elapsed_time(b) for a, b in tw_ev) / len(tw_ev)
    # t_DDP alone: the training of one already-prepared window with nothing else running (the slot
    # consumed last still holds its gathered window; training it again only moves the weights)
    last = slot ^ 1
    alone = []
    for _ in range(3):
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sC)
        train_window(last, sC)
        b.record(sC)
        barrier()
        alone.append(a.elapsed_time(b))
    t_ddp = max_over_ranks(statistics.median(alone))
    T_win = tr_ms / KT
    t_prep = prep_ms
    graphs.clear()
    return {
        "with_training": {
            "value": tr_value, "unit": UNIT, "ms_per_step": T_win, "steps": KT,
            "model": f"GraphSAGE-mean {dims}, softmax cross-entropy, SGD lr {lr}",
            "ddp": f"{n_trainers} trainers; gradient all-reduce " + ("NCCL (torch.distributed)" if world > 1
                                                                      else "none (one rank)"),
            "mean_loss_in_timed_steps": tr_loss,
            "pipeline": "3 streams: sample(w+2) | gather+score(w+1) | DDP steps of window w",
            "cuda_graph": bool(use_graph[0]),
            "dtype": ("tf32 x tf32 -> f32" if os.environ.get("MGNN_SAGE_TF32") == "1"
                      else "3xtf32 (forward and backward GEMMs) -> f32"),
            # Eq.4-5 per window; overlap efficiency read as the trainer's busy
            # fraction t_DDP / T (1 = the preparation is fully hidden; DESIGN R#31)
            "stage_model": {
                "t_prepare_ms": t_prep, "t_ddp_ms": t_ddp, "t_ddp_under_overlap_ms": t_ddp_overlapped,
                "T_window_ms": T_win, "eq5_max_ms": max(t_prep, t_ddp),
                "T_over_eq5": T_win / max(t_prep, t_ddp),
                "overlap_efficiency": t_ddp / T_win,
                "stall_ms_per_window": max(0.0, T_win - t_ddp),
                "hidden_fraction_of_shorter_stage": max(0.0, min(1.0, (t_prep + t_ddp - T_win) /
                                                                 max(1e-9, min(t_prep, t_ddp)))),
                "t_prepare_source": "pipeline-only window time of the timed runs (sample || gather + score)",
                "t_ddp_source": "training of one prepared window with nothing else running (median of 3)"}}}



if __name__ == "__main__":
    main()
