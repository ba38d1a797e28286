"""Window time of one config under the bench schedule, pipelined (two streams) or serial, with the
per-stage CUDA-event times (mgnn_profile_stages).  Experiments only (env knobs of the library).

    python tools/exp_window.py --config products [--serial] [--windows 12]
"""
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
    ap.add_argument("--windows", type=int, default=12)
    ap.add_argument("--serial", action="store_true")
    ap.add_argument("--relabel-stream", action="store_true")
    ap.add_argument("--relabel-after-gather", action="store_true")
    ap.add_argument("--prio-b", action="store_true", help="buffer stream (gather + score) at high priority")
    ap.add_argument("--score-after-sample", action="store_true")
    ap.add_argument("--prio-a", action="store_true", help="sampling stream at high priority")
    ap.add_argument("--gather-events", action="store_true", help="events around the gather launch in the timed run")
    ap.add_argument("--score-prio", type=int, default=None, help="eviction round on its own stream at this priority")
    ap.add_argument("--kprof", action="store_true", help="per-launch event times on each stream (stderr)")
    ap.add_argument("--parts", type=int, default=None)
    ap.add_argument("--tag", default="")
    ap.add_argument("--sm-split", type=int, default=0, help="gather-side SMs of mgnn_sm_partition (0 = off)")
    ap.add_argument("--tuned", action="store_true", help="bench.py's launch tuning for the config (TUNING)")
    a = ap.parse_args()
    if a.tuned:                                  # before the library's first launch reads them
        for k_, v_ in bench.TUNING.get(a.config, {}).get("env", {}).items():
            os.environ.setdefault(k_, v_)
        a.prio_a = a.prio_a or bench.TUNING.get(a.config, {}).get("sampling_priority", 0) < 0
    S = bench.Setup(a.config, 1, parts=a.parts)
    g = synth.generate(S.cfg)
    parts = synth.partition(g, S.P)
    ctx = PL.build_context(0, parts, S.cfg.feat_dim, synth.FEAT_SEED)
    ctx.buffer_init(S.gamma, PL.alpha_default(S.gamma, S.delta), 1.0, S.delta, S.f_bp)
    ctx.sampler_config(S.cfg.fanouts, S.cfg.batch, synth.RUN_SEED, S.window)
    sms = ctx.sm_partition(a.sm_split) if a.sm_split else (0, 0)
    sb = torch.cuda.Stream(priority=-1) if a.prio_b else None
    pipe = PrepareAhead(ctx, S.window, serial=a.serial, stream_b=sb, relabel_stream=a.relabel_stream,
                        relabel_after_gather=a.relabel_after_gather, score_after_sample=a.score_after_sample,
                        sampling_priority=-1 if a.prio_a else 0, score_priority=a.score_prio)
    for _ in range(4):
        pipe.iteration()
    torch.cuda.synchronize()
    # window times without per-stage events (those end the launches' programmatic overlap) ...
    if a.gather_events:
        ctx.profile(True, gather_only=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.windows)]
    for i in range(a.windows):
        pipe.iteration(events=ev[i])
    torch.cuda.synchronize()
    ms = sorted(x.elapsed_time(y) for x, y in ev)
    # ... then the stages of as many windows with them
    ctx.profile(True)
    ctx.profile_stages()
    evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.windows)]
    for i in range(a.windows):
        pipe.iteration(events=evp[i])
    torch.cuda.synchronize()
    msp = sorted(x.elapsed_time(y) for x, y in evp)
    pr = ctx.profile_stages()
    n = max(pr["sample_calls"], 1)
    out = {"tag": a.tag, "config": a.config, "serial": a.serial, "env": {k: v for k, v in os.environ.items() if k.startswith("MGNN_")},
           "ms_median": ms[len(ms) // 2], "ms_mean": sum(ms) / len(ms), "ms_min": ms[0], "ms_median_staged": msp[len(msp) // 2], "mb_per_s": S.window * S.ppg / (ms[len(ms) // 2] / 1e3),
           "sample_ms": pr["sample_ms"] / n, "gather_ms": pr["gather_ms"] / max(pr["gather_calls"], 1),
           "score_ms": pr["score_ms"] / max(pr["score_calls"], 1),
           "relabel_ms": pr["relabel_ms"] / max(pr["relabel_calls"], 1), "relabel_stream": a.relabel_stream,
           "relabel_probes": pr["relabel_probes"] / max(pr["relabel_calls"], 1),
           "edges": pr["edges"] / n, "frontier": pr["frontier"] / n, "unique": pr["unique"] / n,
           "sm_split": sms, "prio_b": a.prio_b, "score_after_sample": a.score_after_sample, "prio_a": a.prio_a, "score_prio": a.score_prio}
    if a.kprof:
        import ctypes as C
        from paper_2410_22697_b200 import _lib
        L = _lib.load()
        torch.cuda.synchronize()
        L.mgnn_profile_kernels(1, None, 0)
        for i in range(a.windows):
            pipe.iteration()
        torch.cuda.synchronize()
        buf = C.create_string_buffer(1 << 22)
        L.mgnn_profile_kernels(0, buf, len(buf))
        print(f"[kprof {a.config} {a.tag}] per launcher, {a.windows} windows:\n" + buf.value.decode(), file=sys.stderr)
    cn = ctx.counts(pipe.slot ^ 1)                  # the last consumed window: evictions per instance (col 4)
    out["evicted_last_window"] = int(cn[:, 4].sum())
    out["parts"] = [ctx.part_info(lp) for lp in range(S.ppg)]
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
