"""Markdown table of the round's final bench lines (profiles/r02/final/bench_<config>.json) for DESIGN §8."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def k(x):
    return f"{x / 1000:.1f}k" if x >= 1000 else f"{x:.0f}"


def main(d=os.path.join(ROOT, "profiles", "r02", "final")):
    print("| config | P | window | minibatches/s (runs) | e2e | hit rate | gather kernel | gather frac | gather share |"
          " with consumer | with DDP training | overlap eff. (R#31) | oracle 1 thread / 1 per partition |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for c in ["cfg1", "arxiv", "reddit", "products", "papers_s32", "papers"]:
        p = os.path.join(d, f"bench_{c}.json")
        if not os.path.exists(p):
            continue
        x = json.loads(open(p).read().strip().splitlines()[-1])
        cf, r = x["config"], x["roofline"]
        cons, tr = x.get("with_consumer", {}), x.get("with_training", {})
        cv = k(cons["value"]) if isinstance(cons.get("value"), (int, float)) else "skipped"
        tv = k(tr["value"]) if isinstance(tr.get("value"), (int, float)) else "skipped"
        oe = tr.get("stage_model", {}).get("overlap_efficiency") if isinstance(tr, dict) else None
        cb = x.get("cpu_baseline") or {}
        cpu = (f"{cb['value']:.1f} / {cb.get('value_one_thread_per_partition', 0):.1f}"
               if cb.get("value") else "—")
        runs = ", ".join(k(v) for v in x.get("runs", []))
        name = f"**{c}** (headline)" if c == "products" else c
        print(f"| {name} | {cf['partitions']} | {cf['window_steps']} | {k(x['value'])} ({runs}) | {k(x['e2e']['value'])} |"
              f" {x['hit_rate']:.2f} | {r['kernel'].split(' ')[0]} | {r['frac']:.2f} | {r.get('share_of_step', 0):.2f} |"
              f" {cv} | {tv} | {oe:.2f} |" if oe is not None else
              f"| {name} | {cf['partitions']} | {cf['window_steps']} | {k(x['value'])} ({runs}) | {k(x['e2e']['value'])} |"
              f" {x['hit_rate']:.2f} | {r['kernel'].split(' ')[0]} | {r['frac']:.2f} | {r.get('share_of_step', 0):.2f} |"
              f" {cv} | {tv} | — |", end="")
        print(f" {cpu} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
