"""bench.py contract on CPU: the --impl reference arm prints exactly one JSON line with the
keys the driver reads (the GPU arm is exercised on the B200 box)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3",
                        "--config", "arxiv"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["config"]["workload"].startswith("ogbn-arxiv-shaped")


def test_gpu_arm_rejects_short_warmup():
    r = subprocess.run([sys.executable, "bench.py", "--warmup", "2"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode != 0 and "warmup" in r.stderr


def test_layouts_and_policy_lookup():
    """bench.Setup: configs 1-4 default to 2 trainers per GPU (P = 2N), papers keeps P = 8 at every N
    (8/N per GPU), --parts / --parts-per-gpu override, and the policy is the paper's GPU optimum for
    the P actually used, windows never straddle an eviction step."""
    import importlib
    sys.path.insert(0, ROOT)
    bench = importlib.import_module("bench")
    s = bench.Setup("products", 1)
    assert (s.P, s.ppg, s.f_bp, s.gamma, s.delta, s.window) == (2, 2, 5000, 0.995, 32, 32)
    s = bench.Setup("products", 4)
    assert (s.P, s.ppg, s.gamma, s.delta, s.window) == (8, 2, 0.9995, 16, 16)
    s = bench.Setup("products", 2, parts_per_gpu=1)
    assert (s.P, s.ppg, s.delta) == (2, 1, 32)
    for world, ppg in ((1, 8), (2, 4), (4, 2), (8, 1)):
        s = bench.Setup("papers", world)
        assert (s.P, s.ppg, s.delta, s.window) == (8, ppg, 512, 16)
    s = bench.Setup("arxiv", 4, parts=8)
    assert (s.P, s.ppg, s.f_bp, s.delta, s.window) == (8, 2, 3500, 128, 32)
    s = bench.Setup("cfg1", 1)
    assert s.window == 32 and s.delta == 64
    try:
        bench.Setup("papers", 3)
        raise AssertionError("8 partitions cannot be split over 3 GPUs")
    except SystemExit:
        pass
    assert bench.static_ucap(bench.Setup("products", 1)) == 2000 * 6 * 11 * 16


def test_gather_kernel_name_follows_the_library_rule(monkeypatch):
    """The roofline names the gather the library launches: flat by default, the TMA row gather only
    under MGNN_GATHER=tma for L2-resident, unpadded rows (or MGNN_GATHER_G4=1), reg -> k_gather."""
    import bench
    monkeypatch.delenv("MGNN_GATHER", raising=False)
    monkeypatch.delenv("MGNN_GATHER_G4", raising=False)
    assert bench.gather_kernel_name(True) == "k_gather_flat"
    monkeypatch.setenv("MGNN_GATHER", "tma")
    assert bench.gather_kernel_name(True) == "k_gather_g4"
    assert bench.gather_kernel_name(False) == "k_gather_tma"
    monkeypatch.setenv("MGNN_GATHER_G4", "0")
    assert bench.gather_kernel_name(True) == "k_gather_tma"
    monkeypatch.setenv("MGNN_GATHER_G4", "1")
    assert bench.gather_kernel_name(False) == "k_gather_g4"
    monkeypatch.setenv("MGNN_GATHER", "reg")
    assert bench.gather_kernel_name(True) == "k_gather"


def test_launch_tuning_is_per_config_and_known():
    """bench.TUNING only names configs bench.py knows and library variables the parity suite covers
    (tests/test_gpu_variants.py runs each of these settings against the oracle)."""
    import bench
    known_env = {"MGNN_HOP_GRID_BPS", "MGNN_COMPACT_BPS", "MGNN_GATHER"}
    for name, t in bench.TUNING.items():
        assert name in bench.POLICY
        assert set(t.get("env", {})) <= known_env
        assert t.get("sampling_priority", 0) in (0, -1)
    src = open(bench.__file__.replace("bench.py", "tests/test_gpu_variants.py")).read()
    assert '"MGNN_HOP_GRID_BPS": "5", "MGNN_COMPACT_BPS": "5"' in src and '"MGNN_GATHER": "tma"' in src
