"""The timed two-stream schedule (bench.py's loop) against the oracle -- bit-exact (-m gpu).

Closes SURVEY §8(a) A13 (Alg.1 l.5-9; queue depth P:403) for the schedule the bench
actually times: paper_2410_22697_b200.schedule.PrepareAhead with two streams, PDL (library
default), the per-iteration L2 flush and events, at the bench's window length and partition
layout (tests/schedule_util.py says what is compared).
"""
import pytest

from inputs import synth
from tests.schedule_util import run_schedule_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_schedule_cfg1_windows_with_eviction_rounds():
    """configs[0], 4-step windows ending in eviction rounds (Delta = 4), 8 windows back to back."""
    g = synth.generate(synth.CONFIGS["cfg1"])
    st = run_schedule_parity(g, 2, 64, [10, 25], 256, 2500, 0.9, 4, 4, 8, x_rows=0)
    assert st["evicted"] > 0 and st["hits"] > 0 and st["misses"] > 0


def test_schedule_cfg1_bench_window():
    """configs[0] at the bench's 32-step window and the paper's Delta = 64 for it."""
    g = synth.generate(synth.CONFIGS["cfg1"])
    st = run_schedule_parity(g, 2, 64, [10, 25], 256, 2500, 0.995, 64, 32, 6, x_rows=4096)
    assert st["evicted"] > 0


@pytest.mark.slow
def test_schedule_arxiv_full_size_bench_config():
    """configs[1] at full size in the bench's configuration: P = 2 on one GPU, 32-step windows,
    f = 0.25, gamma = 0.995, Delta = 32 (every window ends in an eviction round)."""
    g = synth.generate(synth.CONFIGS["arxiv"])
    st = run_schedule_parity(g, 2, 128, [10, 25], 1000, 2500, 0.995, 32, 32, 6, x_rows=0,    # every X row
                             relabel_stream=True)                                       # as bench.py
    assert st["evicted"] > 0


PRODUCTS_SCRIPT = """
import sys
sys.path.insert(0, {root!r})
from inputs import synth
from tests.schedule_util import run_schedule_parity
g = synth.generate(synth.CONFIGS["products"])
st = run_schedule_parity(g, 2, 100, [5, 10, 15], 2000, 5000, 0.995, 32, 32, 4, x_rows=0,   # every X row
                         relabel_stream=True, sampling_priority={prio})                   # as bench.py
assert st["evicted"] > 0 and st["misses"] > 0, st
print("products schedule parity ok", st)
"""


@pytest.mark.slow
def test_schedule_products_full_size_bench_config():
    """configs[3] (the bench default) at full size in the bench's configuration: P = 2 on one GPU,
    32-step windows, f = 0.5, gamma = 0.995, Delta = 32, 3 hops [5, 10, 15], batch 2000, with
    bench.py's launch tuning for products (sampling stream priority, sampler grid caps: environment read
    once per process, so a fresh interpreter)."""
    import os
    import subprocess
    import sys
    import bench
    tune = bench.TUNING.get("products", {})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, **tune.get("env", {}))
    r = subprocess.run([sys.executable, "-c", PRODUCTS_SCRIPT.format(root=root, prio=tune.get("sampling_priority", 0))],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0 and "products schedule parity ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


@pytest.mark.parametrize("seed,relabel_stream", [(1, False), (2, False), (3, False), (4, True), (5, True)])
def test_schedule_perturbed_interleavings(seed, relabel_stream):
    """Race probe of the schedule: random spin kernels before every call shift how the sampling
    stream, the buffer stream (and the relabel stream) interleave; every run must equal the oracle."""
    g = synth.generate(synth.CONFIGS["cfg1"])
    st = run_schedule_parity(g, 2, 64, [10, 25], 256, 2500, 0.9, 4, 4, 6, x_rows=1024, perturb=seed,
                             relabel_stream=relabel_stream)
    assert st["evicted"] > 0


def test_schedule_relabel_stream_bench_window():
    """The deferred relabel on a third stream (mgnn_relabel beside the gather) at the bench window."""
    g = synth.generate(synth.CONFIGS["cfg1"])
    st = run_schedule_parity(g, 2, 64, [10, 25], 256, 2500, 0.995, 64, 32, 4, x_rows=0, relabel_stream=True)
    assert st["evicted"] > 0


@pytest.mark.parametrize("sm_split,relabel_stream", [(40, False), (72, True)])
def test_schedule_sm_partition(sm_split, relabel_stream):
    """mgnn_sm_partition: gather + scoring and sampling (+ relabel) on disjoint green-context SM
    subsets, ordered with the caller's streams by event hand-offs -- every window equals the oracle."""
    g = synth.generate(synth.CONFIGS["cfg1"])
    st = run_schedule_parity(g, 2, 64, [10, 25], 256, 2500, 0.9, 4, 4, 6, x_rows=0, relabel_stream=relabel_stream,
                             sm_split=sm_split)
    assert st["evicted"] > 0


def test_sm_partition_api_contract():
    """EINVAL for negative / too-large SM counts; 0 removes the partition; sizes reported."""
    from paper_2410_22697_b200 import pipeline as PL
    from paper_2410_22697_b200._lib import MgnnError
    g = synth.generate(synth.CONFIGS["cfg1"])
    ctx = PL.build_context(0, synth.partition(g, 2), 64, synth.FEAT_SEED)
    n = torch.cuda.get_device_properties(0).multi_processor_count
    for bad in (-1, n, n + 10):
        with pytest.raises(MgnnError):
            ctx.sm_partition(bad)
    a, b = ctx.sm_partition(48)
    assert a >= 48 and b >= 1 and a + b <= n
    assert ctx.sm_partition(0) == (0, 0)
    ctx.close()


def test_checked_library_schedule_and_parity():
    """The device bounds checks (-DMGNN_CHECKS: every MGNN_CHECK traps) on the timed schedule, the
    window-batching parity tests and the API tests, in a fresh interpreter that loads
    libmgnn_checked.so (MGNN_LIB) with MGNN_DEBUG_SYNC=1 (every launch synchronised and checked)."""
    import os
    import subprocess
    import sys
    from paper_2410_22697_b200 import build
    lib = build.build(checked=True)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MGNN_LIB=lib, MGNN_DEBUG_SYNC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_schedule.py::test_schedule_cfg1_windows_with_eviction_rounds",
                        "tests/test_gpu_parity.py::test_cfg1_windows", "tests/test_gpu_parity.py::test_cfg1_policy_grid",
                        "tests/test_gpu_api.py::test_arena_overflow_skips_windows_and_resumes"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "libmgnn_checked" in lib
