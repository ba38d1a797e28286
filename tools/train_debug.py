"""Debug: per-tensor gradient norms, GPU vs oracle, for one DDP step (not a test)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from inputs import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402
from oracle import sage as S  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402
from tests.sage_util import oracle_instance  # noqa: E402
from tests.train_util import unpack  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "3":
    g = synth.random_graph(2000, 0.005, seed=9)
    P, D, fan, B, dims = 3, 150, [3, 4, 5], 48, [150, 48, 40, 10]
else:
    g = synth.random_graph(1500, 0.006, seed=31)
    P, D, fan, B, dims = 2, 64, [4, 6], 64, [64, 32, 7]
parts = synth.partition(g, P)
W = O.World(parts, D, synth.FEAT_SEED)
for p in W.parts:
    p.buffer_init(0.95, 0.0, 1.0, 0, 2500)
ctx = PL.build_context(0, parts, D, synth.FEAT_SEED)
ctx.buffer_init(0.95, 0.0, 1.0, 0, 2500)
ctx.sampler_config(fan, B, synth.RUN_SEED, 1)
wts = synth.sage_weights(dims, seed=7)
ctx.sage_config(dims, [w[0] for w in wts], [w[1] for w in wts], [w[2] for w in wts])
labels = synth.node_labels(g.n_nodes, dims[-1])
ctx.train_config(labels)
ctx.sample(0, 1, 1)
ctx.lookup_gather(0)
ctx.train_step(0, 0, P)
torch.cuda.synchronize()
gg = unpack(ctx.grads().cpu().numpy(), dims)
ref = None
zmin = []
ref_w = [tuple(np.asarray(a, np.float64) for a in w) for w in wts]
for pid in range(P):
    _, blocks, X = oracle_instance(W.parts[pid], 1, fan, B)
    F0 = W.parts[pid].frontier()[:W.parts[pid].hop_sizes()[0]]
    loss, gr = S.sage_loss_grads(X, blocks, ref_w, labels[F0])
    _, cache = S.sage_forward_cache(X, blocks, ref_w)
    for l in range(len(dims) - 2):
        z = cache[l][2]
        print("layer", l, "pre-activations |z| < 1e-3 * max:", int(np.sum(np.abs(z) < 1e-3 * np.abs(z).max())), "of", z.size)
    gr = [tuple(x / P for x in layer) for layer in gr]
    ref = gr if ref is None else [tuple(a + b for a, b in zip(x, y)) for x, y in zip(ref, gr)]
for l in range(len(dims) - 1):
    for k, nm in enumerate(("Ws", "Wn", "b")):
        a, b = np.asarray(gg[l][k], np.float64), ref[l][k]
        print(l, nm, "ref", round(np.linalg.norm(b), 5), "rel err", np.linalg.norm(a - b) / np.linalg.norm(b))
print("loss", ctx.loss())
