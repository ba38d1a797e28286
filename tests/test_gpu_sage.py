"""GPU consumer (A14: mgnn_sage_forward, tcgen05 kind::tf32 + TMA + TMEM) vs the fp64
oracle (oracle/sage.py), elementwise within the TF32 error bound derived in
tests/sage_util.py (-m gpu)."""
import numpy as np
import pytest

from inputs import synth
from tests.sage_util import run_sage_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg1():
    return synth.generate(synth.CONFIGS["cfg1"])


def test_cfg1_two_layers(cfg1):
    """configs[0]: D = 64 (one partial panel), hidden 128, 16 classes, two windows of 4 steps."""
    r = run_sage_parity(cfg1, 2, 64, [10, 25], 256, synth.sage_dims(64, 2, 16), [4, 4])
    assert r <= 1.0


def test_cfg1_three_layers(cfg1):
    """3 hops / 3 layers ([5,10,15]), 3 partitions on one GPU."""
    run_sage_parity(cfg1, 3, 64, [5, 10, 15], 128, synth.sage_dims(64, 3, 47), [3, 3])


def test_wide_ragged_dims():
    """D = 150 (two panels, the second a single 32-column chunk with padding), hidden 40
    (N padded to 48), 7 classes (logits pitch not a multiple of 4), isolated nodes
    (empty neighbourhoods)."""
    g = synth.random_graph(900, 0.006, seed=21)
    run_sage_parity(g, 2, 150, [4, 6], 64, [150, 40, 7], [2, 3])


def test_single_layer_many_tiles():
    """one layer (fanout [25]): dst = seeds; batch 700 spans 6 tiles with a ragged tail."""
    g = synth.random_graph(3000, 0.004, seed=5)
    run_sage_parity(g, 2, 128, [25], 700, [128, 256], [2])


def test_arxiv_window_sampled_instances():
    """configs[1] (arxiv-shaped, the bench workload) at full size, the bench's launch
    configuration (32-step window x 2 partitions); every 8th instance checked."""
    g = synth.generate(synth.CONFIGS["arxiv"])
    run_sage_parity(g, 2, 128, [10, 25], 1000, synth.sage_dims(128, 2, 40), [32], f_bp=2500, gamma=0.995,
                    delta=32, inst_every=8)


@pytest.mark.parametrize("split", ["0", "1"])
def test_fused_and_split_aggregation(cfg1, split, monkeypatch):
    """Both forward variants: neighbour means inside the GEMM kernel (MGNN_SAGE_SPLIT=0) and
    k_mean + TMA-fed GEMM (default)."""
    monkeypatch.setenv("MGNN_SAGE_SPLIT", split)
    run_sage_parity(cfg1, 2, 64, [10, 25], 256, synth.sage_dims(64, 2, 16), [3])
    g = synth.random_graph(900, 0.006, seed=21)
    run_sage_parity(g, 2, 150, [4, 6], 64, [150, 40, 7], [2])


def test_reddit_width_features():
    """D = 602 (Reddit's width: pitch 604, ten 64-column panels / nineteen 32-column chunks, a ragged
    last chunk), 41 classes, on a small graph."""
    g = synth.random_graph(700, 0.01, seed=41)
    run_sage_parity(g, 2, 602, [4, 8], 48, [602, 128, 41], [2])


@pytest.mark.parametrize("tf32", ["0", "1"])
def test_gemm_3xtf32_and_tf32(cfg1, tf32, monkeypatch):
    """k_sage_gemm's operand precision: 3xTF32 (default: hi/lo split of A in shared memory and of W
    in HBM, three TF32 products per term -- checked against the fp32-grade bound) and one TF32 pass
    (MGNN_SAGE_TF32=1, the TF32 bound); wide layers (npad 256, streamed weights) included."""
    monkeypatch.setenv("MGNN_SAGE_TF32", tf32)
    run_sage_parity(cfg1, 2, 64, [10, 25], 256, synth.sage_dims(64, 2, 16), [3])
    g = synth.random_graph(1200, 0.006, seed=77)
    run_sage_parity(g, 2, 100, [5, 10, 15], 64, [100, 256, 256, 47], [2])
