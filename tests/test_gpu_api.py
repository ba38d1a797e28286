"""C-ABI contract on the GPU (include/mgnn.h): status codes, call order, sticky errors,
zero-copy views and the per-launcher profile (-m gpu)."""
import ctypes

import numpy as np
import pytest

from inputs import synth
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2410_22697_b200 import _lib  # noqa: E402
from paper_2410_22697_b200 import pipeline as PL  # noqa: E402
from paper_2410_22697_b200._lib import MgnnError  # noqa: E402

EINVAL, ESTATE = 1, 5


@pytest.fixture(scope="module")
def graph():
    return synth.generate(synth.CONFIGS["cfg1"])


def _ctx(graph, hosted=None, init=True, window=4, delta=4):
    parts = synth.partition(graph, 2)
    ctx = PL.build_context(0, parts, 64, synth.FEAT_SEED, hosted)
    if init:
        ctx.buffer_init(0.9, PL.alpha_default(0.9, delta), 1.0, delta, 2500)
        ctx.sampler_config([10, 25], 256, synth.RUN_SEED, window)
    return ctx


def _status(excinfo):
    return excinfo.value.status


def test_call_order(graph):
    ctx = _ctx(graph, init=False)
    with pytest.raises(MgnnError) as e:
        ctx.sample(0, 1, 1)                          # before buffer_init / sampler_config
    assert _status(e) == ESTATE
    ctx.buffer_init(0.9, 0.5, 1.0, 4, 2500)
    ctx.sampler_config([10, 25], 256, synth.RUN_SEED, 4)
    with pytest.raises(MgnnError) as e:
        ctx.lookup_gather(0)                         # gather before sample
    assert _status(e) == ESTATE
    ctx.sample(0, 1, 4)
    with pytest.raises(MgnnError) as e:
        ctx.score(0)                                 # score before gather
    assert _status(e) == ESTATE
    ctx.lookup_gather(0)
    ctx.sample(1, 9, 4)                              # skips steps 5..8
    with pytest.raises(MgnnError) as e:
        ctx.lookup_gather(1)                         # previous window not scored
    assert _status(e) == ESTATE
    ctx.score(0)
    with pytest.raises(MgnnError) as e:
        ctx.lookup_gather(1)                         # windows must be gathered in step order
    assert _status(e) == ESTATE
    ctx.close()


def test_invalid_arguments_leave_state(graph):
    ctx = _ctx(graph)
    for bad in (dict(slot=2, t0=1, n=4), dict(slot=0, t0=0, n=4), dict(slot=0, t0=1, n=5),
                dict(slot=0, t0=3, n=3)):            # t=4 (eviction) inside [3, 5]
        with pytest.raises(MgnnError) as e:
            ctx.sample(bad["slot"], bad["t0"], bad["n"])
        assert _status(e) == EINVAL
    for pol in ((0.0, 0.5, 1.0, 4, 2500), (1.5, 0.5, 1.0, 4, 2500), (0.9, -1.0, 1.0, 4, 2500),
                (0.9, 0.5, 1.0, -1, 2500), (0.9, 0.5, 1.0, 4, 10001), (0.9, float("nan"), 1.0, 4, 2500)):
        with pytest.raises(MgnnError) as e:
            ctx.buffer_init(*pol)
        assert _status(e) == EINVAL
    with pytest.raises(MgnnError) as e:
        ctx.sampler_config([10, 33], 256, 1, 4)      # fanout > 32
    assert _status(e) == EINVAL
    # the context is still usable
    ctx.sample(0, 1, 4)
    ctx.lookup_gather(0)
    ctx.score(0)
    assert ctx.counts(0).shape == (8, 8)
    ctx.close()


def test_partition_validation(graph):
    parts = synth.partition(graph, 2)
    ctx = PL.Context(0, parts[0].bounds, 64, synth.FEAT_SEED)
    p = parts[0]
    bad_cols = p.cols.copy()
    r = int(np.argmax(np.diff(p.indptr) >= 2))
    a, b = int(p.indptr[r]), int(p.indptr[r] + 1)
    bad_cols[a], bad_cols[b] = bad_cols[b], bad_cols[a]      # row not ascending
    with pytest.raises(MgnnError) as e:
        ctx.load_partition(0, p.indptr, bad_cols, p.train_ids)
    assert _status(e) == EINVAL
    with pytest.raises(MgnnError) as e:
        ctx.load_partition(0, p.indptr, p.cols, p.train_ids[::-1].copy())   # unsorted train ids
    assert _status(e) == EINVAL
    ctx.load_partition(0, p.indptr, p.cols, p.train_ids)
    with pytest.raises(MgnnError) as e:
        ctx.load_partition(0, p.indptr, p.cols, p.train_ids)                # loaded twice
    assert _status(e) == EINVAL
    with pytest.raises(MgnnError) as e:
        ctx.buffer_init(0.9, 0.5, 1.0, 4, 2500)       # partition 1's table neither hosted nor imported
    assert _status(e) == ESTATE
    ctx.close()


def test_bad_external_seeds_are_reported(graph):
    ctx = _ctx(graph)
    seeds = np.zeros((2, 4, 256), np.int32)
    counts = np.full((2, 4), 2, np.int32)
    seeds[:, :, 0] = 7
    seeds[:, :, 1] = 7                                # duplicate seed
    seeds[1, :, :2] += 5000                           # partition 1 owns [5000, 10000)
    ctx.sample(0, 1, 4, seeds=seeds, seed_counts=counts)
    with pytest.raises(MgnnError) as e:
        ctx.counts(0)
    assert _status(e) == EINVAL
    with pytest.raises(MgnnError):                    # sticky
        ctx.sample(1, 5, 4)
    ctx.close()


def test_zero_copy_views_match_instance(graph):
    ctx = _ctx(graph)
    ctx.sample(0, 1, 4)
    ctx.lookup_gather(0)
    ctx.score(0)
    torch.cuda.synchronize()
    w = ctx.window(0)
    assert w.n_inst == 8 and w.n_steps == 4 and w.pitch == 64
    X = PL.device_view(w.X, (w.n_inst, w.rows_stride, w.pitch), "f4")
    inst = ctx.instance(0, 3)
    U = int(inst["hop_size"][-1])
    assert torch.equal(X[3, :U, :64].cpu(), torch.from_numpy(inst["X"]))
    F = inst["frontier"]
    for i in range(0, U, 97):
        assert np.array_equal(inst["X"][i], O.feature_row(int(F[i]), 64, synth.FEAT_SEED))
    ctx.close()


def test_kernel_profile_and_launch_count(graph):
    L = _lib.load()
    ctx = _ctx(graph)
    n0 = ctx.launch_count()
    L.mgnn_profile_kernels(1, None, 0)
    ctx.prepare(0, 1, 4)
    buf = ctypes.create_string_buffer(1 << 14)
    L.mgnn_profile_kernels(0, buf, len(buf))
    report = buf.value.decode()
    assert "launch_gather" in report and "launch_hop" in report
    assert ctx.launch_count() - n0 >= 8
    ctx.close()


def test_consumer_training_remote_call_order_and_arguments(graph):
    """Status codes of the consumer (A14), training (NEXT-3) and remote-expansion (NEXT-1) calls."""
    ctx = _ctx(graph)
    dims = synth.sage_dims(64, 2, 16)
    wts = synth.sage_weights(dims)
    logits = torch.zeros((8, 256, 16), device="cuda")
    with pytest.raises(MgnnError) as e:                       # forward before sage_config
        ctx.sage_forward(0, logits)
    assert _status(e) == ESTATE
    with pytest.raises(MgnnError) as e:                       # remote expansion after sampler_config
        ctx.expand_remote(True)
    assert _status(e) == ESTATE
    with pytest.raises(MgnnError) as e:                       # a hidden width above 256
        ctx.sage_config([64, 300, 16], *[[w[i] for w in synth.sage_weights([64, 300, 16])] for i in range(3)])
    assert _status(e) == EINVAL
    with pytest.raises(MgnnError) as e:                       # dims[0] != feat_dim
        ctx.sage_config([32, 128, 16], *[[w[i] for w in synth.sage_weights([32, 128, 16])] for i in range(3)])
    assert _status(e) == EINVAL
    ctx.sage_config(dims, [w[0] for w in wts], [w[1] for w in wts], [w[2] for w in wts])
    ctx.sample(0, 1, 4)
    with pytest.raises(MgnnError) as e:                       # forward before the window is gathered
        ctx.sage_forward(0, logits)
    assert _status(e) == ESTATE
    ctx.lookup_gather(0)
    with pytest.raises(MgnnError) as e:                       # logits pitch below the class count
        ctx.sage_forward(0, torch.zeros((8, 256, 8), device="cuda"))
    assert _status(e) == EINVAL
    ctx.sage_forward(0, logits)
    with pytest.raises(MgnnError) as e:                       # training step before train_config
        ctx.train_step(0, 0, 2)
    assert _status(e) == ESTATE
    with pytest.raises(MgnnError) as e:                       # a label outside [0, C)
        ctx.train_config(np.full(graph.n_nodes, 16, np.int32))
    assert _status(e) == EINVAL
    ctx.train_config(synth.node_labels(graph.n_nodes, 16))
    with pytest.raises(MgnnError) as e:                       # step beyond the window
        ctx.train_step(0, 4, 2)
    assert _status(e) == EINVAL
    ctx.train_step(0, 0, 2)
    ctx.sgd(0.01)
    assert np.isfinite(ctx.loss())
    ctx.score(0)
    ctx.close()
    # dense scores must precede partition loading; remote expansion needs the global CSR when
    # other partitions live in other contexts
    parts = synth.partition(graph, 2)
    c2 = PL.build_context(0, parts, 64, synth.FEAT_SEED, hosted=[0])
    with pytest.raises(MgnnError) as e:
        c2._chk("mgnn_ctx_set_dense_scores", c2.L.mgnn_ctx_set_dense_scores(c2._h, 1))
    assert _status(e) == ESTATE
    with pytest.raises(MgnnError) as e:
        c2.expand_remote(True)
    assert _status(e) == ESTATE
    c2.close()


def test_arena_overflow_skips_windows_and_resumes(graph):
    """mgnn_sampler_config_bounded: a window whose frontier exceeds the arena bound is detected on the
    device, it and every later window are skipped by the buffer-state kernels, counts_read reports
    MGNN_EOVERFLOW (not sticky), and reconfiguring with a larger bound resumes at the overflowed
    step -- the run then matches the oracle's uninterrupted run bit for bit."""
    EOVERFLOW = 6
    P, fan, B, f_bp, gamma, delta = 2, [10, 25], 256, 2500, 0.9, 4
    parts = synth.partition(graph, P)
    alpha = float(O.alpha_default(gamma, delta))
    ctx = PL.build_context(0, parts, 64, synth.FEAT_SEED)
    ctx.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    bound = PL.estimate_rows_bound(ctx, fan, B, synth.RUN_SEED)
    assert B <= bound
    ctx.sampler_config(fan, B, synth.RUN_SEED, 4, rows_bound=bound)
    counts = []
    t, slot = 1, 0
    for _ in range(2):                                  # steps 1-8 fit
        ctx.sample(slot, t, 4)
        ctx.lookup_gather(slot)
        ctx.score(slot)
        counts.append(ctx.counts(slot))
        t += 4
        slot ^= 1
    snap_before = [ctx.snapshot(lp, rows=True) for lp in range(P)]
    ctx.sampler_config(fan, B, synth.RUN_SEED, 4, rows_bound=B + 1)   # far too small: overflows at step 9
    for _ in range(2):                                  # steps 9-16: both windows skipped on the device
        ctx.sample(slot, t, 4)
        ctx.lookup_gather(slot)
        ctx.score(slot)
        with pytest.raises(MgnnError) as e:
            ctx.counts(slot)
        assert _status(e) == EOVERFLOW and "step 9" in str(e.value)
        t += 4
        slot ^= 1
    for lp in range(P):                                 # buffer state untouched by the skipped windows
        snap = ctx.snapshot(lp, rows=True)
        for k in ("node_of_slot", "se", "sa", "slot_of", "rows"):
            assert np.array_equal(np.asarray(snap[k]).view(np.uint8), np.asarray(snap_before[lp][k]).view(np.uint8))
    ctx.sampler_config(fan, B, synth.RUN_SEED, 4, rows_bound=0)       # resume at step 9
    t = 9
    with pytest.raises(MgnnError) as e:                 # the step order now restarts at 9, not 17
        ctx.sample(slot, 17, 4)
        ctx.lookup_gather(slot)
    assert _status(e) == ESTATE
    for _ in range(2):
        ctx.sample(slot, t, 4)
        ctx.lookup_gather(slot)
        ctx.score(slot)
        counts.append(ctx.counts(slot))
        t += 4
        slot ^= 1
    W = O.World(parts, 64, synth.FEAT_SEED)
    for p in W.parts:
        p.buffer_init(gamma, alpha, 1.0, delta, f_bp)
    for wi in range(4):
        for w in range(4):
            step = 1 + 4 * wi + w
            for pid in range(P):
                op = W.parts[pid]
                op.step(synth.RUN_SEED, step, fan, B)
                oc = op.counts()
                gc = counts[wi][pid * 4 + w]
                assert [gc[0], gc[2], gc[3], gc[4]] == [oc["n_nodes"], oc["n_hit"], oc["n_miss"], oc["n_evicted"]]
    for pid in range(P):
        gs = ctx.snapshot(pid, rows=True)
        os_ = W.parts[pid].buffer_state(rows=True)
        for k in ("node_of_slot", "se", "sa", "slot_of", "rows"):
            assert np.array_equal(np.asarray(gs[k]).view(np.uint8), np.asarray(os_[k]).view(np.uint8)), k
    ctx.close()
    W.close()


def test_bounded_arenas_parity(graph):
    """Realistic arenas from the pilot bound (the bench's sizing) give the oracle's results."""
    from tests.parity_util import run_parity
    st = run_parity(graph, 2, 64, [10, 25], 256, 2500, 0.9, 4, 1.0, [4, 4, 4], rows_bound=-1)
    assert st["evicted"] > 0


def test_caller_owned_x(graph):
    """SURVEY §8(b)'s caller-owned X: torch tensors bound with mgnn_window_bind_x receive every
    gathered row (bit-exact against the oracle), also as the consumer's input."""
    from tests.parity_util import run_parity
    from tests.sage_util import run_sage_parity
    run_parity(graph, 2, 64, [10, 25], 256, 2500, 0.9, 4, 1.0, [4, 4], bind_x=True)
    assert run_sage_parity(graph, 2, 64, [10, 25], 256, synth.sage_dims(64, 2, 16), [4], bind_x=True) <= 1.0
    ctx = _ctx(graph)
    rs, pitch, mi = ctx.window_shape()
    small = torch.zeros(mi * rs * pitch - 4, device="cuda")
    with pytest.raises(MgnnError) as e:
        ctx.bind_x(0, small)
    assert _status(e) == EINVAL
    ctx.close()
