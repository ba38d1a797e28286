"""GPU DDP training step (NEXT-3: forward, cross-entropy, backward with tcgen05 weight/input
gradients, SGD) vs the fp64 oracle, step by step (-m gpu)."""
import pytest

from inputs import synth
from tests.train_util import run_train_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_two_layers_small():
    g = synth.random_graph(1500, 0.006, seed=31)
    run_train_parity(g, 2, 64, [4, 6], 64, [64, 32, 7], 3)


def test_cfg1_two_layers_hidden128():
    g = synth.generate(synth.CONFIGS["cfg1"])
    run_train_parity(g, 2, 64, [10, 25], 256, synth.sage_dims(64, 2, 16), 3)


def test_three_layers_wide_input():
    """D = 150 (two 128-column K panels in the weight gradient), 3 layers, 3 trainers."""
    g = synth.random_graph(2000, 0.005, seed=9)
    run_train_parity(g, 3, 150, [3, 4, 5], 48, [150, 48, 40, 10], 2)


def test_reddit_width_training():
    """Training with D = 602: the weight gradient's self/neighbour halves span five 128-column
    N-tiles each (kp = 640), pitch 604 inputs, 41 classes."""
    g = synth.random_graph(700, 0.01, seed=43)
    run_train_parity(g, 2, 602, [4, 8], 48, [602, 128, 41], 2)
