"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins (PAPER.md P:n, SPEC.md S:n, DESIGN.md
reading R#n).  None of them compares the oracle with itself.
"""
import itertools
import json
import math
import os
from collections import Counter

import numpy as np
import pytest

from inputs import synth
from oracle import oracle as O
from tests.policy_ref import PolicyRef

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RUN_SEED = synth.RUN_SEED
FEAT_SEED = synth.FEAT_SEED


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def h32(s):
    return int(s, 16)


def world_from(g, P, D=4, bounds=None):
    parts = synth.partition(g, P, bounds)
    return O.World(parts, D, FEAT_SEED), parts


# ------------------------------------------------------------------ Philox / counter layout (R#4-#6)
def test_philox_random123_kat():
    for v in gold("philox_kat.json")["vectors"]:
        out = O.philox([h32(x) for x in v["ctr"]], [h32(x) for x in v["key"]])
        assert out == [h32(x) for x in v["out"]]


def test_counter_layout_golden():
    g = gold("counter_layout.json")
    s = g["sample"]
    key = [s["run_seed"] & 0xFFFFFFFF, s["run_seed"] >> 32]
    u = [O.philox([s["node"], (s["hop"] << 16) | j, s["step"], (s["part"] << 8) | 1], key)[0] for j in range(3)]
    assert u == [h32(x) for x in s["u"]]
    d, k = s["d"], s["k"]
    r = [O.urange(u[j], d - k + j + 1) for j in range(k)]
    assert r == s["r"]
    assert O.floyd(d, k, r) == s["pos"]
    c = g["floyd_collision"]
    assert O.floyd(c["d"], c["k"], c["r"]) == c["pos"]
    sh = g["shuffle"]
    for node, hexkey in sh["keys"].items():
        o = O.philox([int(node), sh["epoch"], 0, (sh["part"] << 8) | 2], key)
        assert ((o[0] << 32) | o[1]) == h32(hexkey)
    f = g["features"]
    row = O.feature_row(f["node"], 4, f["feat_seed"])
    assert [int(x) for x in row.view(np.uint32)] == [h32(x) for x in f["bits"]]


def test_feature_values_on_grid():
    row = O.feature_row(12345, 600, FEAT_SEED)
    assert np.all(row >= -1.0) and np.all(row < 1.0)
    q = row.astype(np.float64) * 2 ** 23          # exact multiples of 2^-23 (R#4)
    assert np.all(q == np.round(q))
    assert not np.array_equal(row, O.feature_row(12346, 600, FEAT_SEED))


@pytest.mark.parametrize("d,k,expect", [(5, 2, 2), (6, 3, 6), (7, 4, 24), (8, 3, 6), (9, 5, 120)])
def test_floyd_bruteforce_uniform(d, k, expect):
    """Every k-subset of {0..d-1} arises from exactly k! of the prod(t_j+1) draw vectors (R#6)."""
    ranges = [range(d - k + j + 1) for j in range(k)]
    cnt = Counter()
    for r in itertools.product(*ranges):
        pos = O.floyd(d, k, list(r))
        assert len(set(pos)) == k and all(0 <= x < d for x in pos)
        cnt[frozenset(pos)] += 1
    assert len(cnt) == math.comb(d, k)
    assert set(cnt.values()) == {expect}


def test_range_reduction_bounds():
    for t1 in (1, 2, 7, 1000, 2 ** 31):
        assert O.urange(0, t1) == 0
        assert O.urange(2 ** 32 - 1, t1) == t1 - 1
        assert O.urange(2 ** 31, t1) == t1 // 2


# ------------------------------------------------------------------ threshold, Eq.1 (R#13)
def test_alpha_grid_bits():
    for gamma, delta, bits in gold("alpha_grid.json")["cells"]:
        a = O.alpha_default(gamma, delta)
        assert int(np.float32(a).view(np.uint32)) == h32(bits), (gamma, delta)
        g32 = float(np.float32(gamma))
        exact = g32 ** delta                                   # error bound of Delta RN products
        assert abs(float(a) - exact) <= ((1 + 2.0 ** -24) ** delta - 1) * exact * 1.0000001


def test_alpha_closed_forms():
    for d in (0, 1, 16, 100, 149):
        assert float(O.alpha_default(0.5, d)) == 2.0 ** -d          # exact powers of two, denormals kept
    assert float(O.alpha_default(0.5, 150)) == 0.0                  # 2^-150 rounds to zero (RN)
    assert float(O.alpha_default(1.0, 1024)) == 1.0
    assert float(O.alpha_default(0.9, 0)) == 1.0


# ------------------------------------------------------------------ halo sets
def test_halo_path_graph():
    g = synth.from_edges(4, [(0, 1), (1, 2), (2, 3)])
    W, _ = world_from(g, 2)
    assert list(W.parts[0].halo()[0]) == [2]
    assert list(W.parts[1].halo()[0]) == [1]


def test_halo_ring_alternating():
    # ring a0 b0 a1 b1 ... with a_i = i in p0 = {0..3}, b_i = 4+i in p1
    ring = [0, 4, 1, 5, 2, 6, 3, 7]
    g = synth.from_edges(8, [(ring[i], ring[(i + 1) % 8]) for i in range(8)])
    W, _ = world_from(g, 2)
    assert W.parts[0].n_halo == 4 and W.parts[1].n_halo == 4


def test_halo_single_partition_empty():
    g = synth.random_graph(20, 0.3, 1)
    W, _ = world_from(g, 1)
    assert W.parts[0].n_halo == 0


@pytest.mark.parametrize("seed", range(8))
def test_halo_and_deg_in_bruteforce(seed):
    g = synth.random_graph(20, 0.25, seed)
    P = 3
    W, parts = world_from(g, P)
    edges = {(u, int(v)) for u in range(20) for v in g.cols[g.indptr[u]:g.indptr[u + 1]]}
    for p, pi in enumerate(parts):
        lo, hi = int(pi.bounds[p]), int(pi.bounds[p + 1])
        local = set(range(lo, hi))
        halo = sorted({v for (u, v) in edges if u in local and v not in local})
        ids, deg = W.parts[p].halo()
        assert list(ids) == halo
        assert list(deg) == [sum(1 for u in local if (u, h) in edges) for h in halo]


# ------------------------------------------------------------------ init
def _init_example():
    # locals L0..L5 = 0..5 (p0), halo a,b,c,d = 6,7,8,9 (p1): deg_in a=5, b=3, c=2, d=1
    a, b, c, d = 6, 7, 8, 9
    edges = [(a, i) for i in range(5)] + [(b, 0), (b, 1), (b, 5), (c, 5), (c, 1), (d, 2)]
    g = synth.from_edges(10, edges)
    return g, (a, b, c, d)


def test_init_top_by_degree():
    g, (a, b, c, d) = _init_example()
    W, _ = world_from(g, 2, bounds=np.array([0, 6, 10]))
    p = W.parts[0]
    assert list(p.halo()[1]) == [5, 3, 2, 1]
    p.buffer_init(0.9, 0.5, 1.0, 0, 5000)                    # f = 0.5
    st = p.buffer_state()
    assert sorted(st["node_of_slot"]) == [a, b]
    assert list(st["se"]) == [1.0, 1.0]
    assert list(st["sa"]) == [-1.0, -1.0, 0.0, 0.0]
    p.buffer_init(0.9, 0.5, 1.0, 0, 0)                       # f = 0: empty buffer is valid
    assert p.cap == 0 and list(p.buffer_state()["sa"]) == [0.0] * 4
    p.buffer_init(0.9, 0.5, 1.0, 0, 10000)
    assert p.cap == 4
    p.buffer_init(0.9, 0.5, 1.0, 0, 1)                       # ceil(0.0001 * 4) = 1 (R#11)
    assert p.cap == 1 and list(p.buffer_state()["node_of_slot"]) == [a]


def test_classify_example():
    """buffer {a,b}, sampled halo {b,c} -> hit {b}, miss {c} (Alg.2 l.4-5)."""
    g, (a, b, c, d) = _init_example()
    W, _ = world_from(g, 2, bounds=np.array([0, 6, 10]))
    p = W.parts[0]
    p.buffer_init(0.9, 0.5, 1.0, 0, 5000)
    p.step(RUN_SEED, 1, [25], 1, seeds=np.array([5], np.int32))     # N(5) = {b, c}
    F = p.frontier()
    assert sorted(F.tolist()) == [5, b, c]
    cls = dict(zip(F.tolist(), p.classes().tolist()))
    assert cls[b] == 1 and cls[c] == 2 and cls[5] == 0
    cnt = p.counts()
    assert (cnt["n_hit"], cnt["n_miss"], cnt["n_local"]) == (1, 1, 1)
    st = p.buffer_state()
    se = dict(zip(st["node_of_slot"].tolist(), st["se"].tolist()))
    assert se[b] == 1.0 and se[a] == np.float32(0.9)          # decay only the unused
    assert st["sa"][2] == 1.0                                  # c tallied


# ------------------------------------------------------------------ decay / threshold boundary
def _decay_graph():
    # p0 = {0,1,2}; halo 3 (deg_in 1, sampled every step from seed 0), halo 4 (deg_in 2, never sampled)
    g = synth.from_edges(6, [(0, 1), (0, 3), (2, 4), (1, 4)], train_mask=[1, 0, 0, 0, 0, 0])
    W, _ = world_from(g, 2, bounds=np.array([0, 3, 6]))
    return W.parts[0]


def test_decay_closed_form_gamma_half():
    """gamma = 0.5: S_E = 2^-t exactly for t <= 149 and 0 at t = 150 (denormals kept, R#12)."""
    p = _decay_graph()
    p.buffer_init(0.5, 0.0, 1.0, 0, 5000)                    # cap 1 -> node 4 (higher deg_in)
    assert list(p.buffer_state()["node_of_slot"]) == [4]
    for t in range(1, 151):
        p.step(RUN_SEED, t, [2], 1)
        se = float(p.buffer_state()["se"][0])
        assert se == (2.0 ** -t if t <= 149 else 0.0), t


def test_gamma_one_constant_and_alpha_zero_never_evicts():
    p = _decay_graph()
    p.buffer_init(1.0, 1.0, 1.0, 4, 5000)
    for t in range(1, 41):
        p.step(RUN_SEED, t, [2], 1)
    st = p.buffer_state()
    assert list(st["node_of_slot"]) == [4] and float(st["se"][0]) == 1.0 and p.totals()["refills"] == 0
    p.buffer_init(0.5, 0.0, 1.0, 1, 5000)                    # alpha = 0: S_E >= 0 is never < 0
    for t in range(1, 200):
        p.step(RUN_SEED, t, [2], 1)
    assert list(p.buffer_state()["node_of_slot"]) == [4] and p.totals()["refills"] == 0


@pytest.mark.parametrize("gamma", [0.95, 0.995, 0.9995])
@pytest.mark.parametrize("delta", [16, 32, 64])
def test_threshold_boundary_and_swap(gamma, delta):
    """Fresh never-hit entry: kept at round Delta (S_E == alpha), evicted at 2*Delta (R#13, R#16),
    then the swap of P:224: S_A[e] <- last S_E, S_E[r] <- last S_A, S_A[r] <- -1."""
    p = _decay_graph()
    alpha = O.alpha_default(gamma, delta)
    p.buffer_init(gamma, alpha, 1.0, delta, 5000)
    for t in range(1, delta + 1):
        p.step(RUN_SEED, t, [2], 1)
    st = p.buffer_state()
    assert list(st["node_of_slot"]) == [4] and st["se"][0] == alpha
    for t in range(delta + 1, 2 * delta + 1):
        p.step(RUN_SEED, t, [2], 1)
    st = p.buffer_state()
    se_last = alpha
    for _ in range(delta):
        se_last = np.float32(se_last * np.float32(gamma))
    assert list(st["node_of_slot"]) == [3]
    assert st["se"][0] == np.float32(2 * delta)             # node 3 missed 2*Delta times
    assert st["sa"][0] == -1.0 and st["sa"][1] == se_last
    assert p.counts()["n_evicted"] == 1 and p.totals()["refills"] == 1


# ------------------------------------------------------------------ EVICT_AND_REPLACE
def test_evict_hand_trace():
    """buffer {a: S_E .3, b: .9}, alpha .5, outside {c: S_A 4, d: 2} -> evict a, admit c."""
    a, b, c, d = 10, 11, 12, 13
    halo = np.array([a, b, c, d], np.int32)
    node = np.array([a, b], np.int32)
    se = np.array([0.3, 0.9], np.float32)
    sa = np.array([-1, -1, 4, 2], np.float32)
    slot = np.array([0, 1, -1, -1], np.int32)
    ev, rp, sl = O.evict_and_replace(node, se, sa, slot, halo, np.ones(4, np.int32), 0.5, 1.0)
    assert list(ev) == [a] and list(rp) == [c] and list(sl) == [0]
    assert list(node) == [c, b]
    assert sa[0] == np.float32(0.3) and se[0] == 4.0 and sa[2] == -1.0 and list(slot) == [-1, 1, 0, -1]


def test_evict_candidates_exceed_replacements():
    """3 candidates, 1 eligible replacement -> exactly 1 pair, lowest S_E evicted (R#19)."""
    halo = np.arange(6, dtype=np.int32)
    node = np.array([0, 1, 2], np.int32)
    se = np.array([0.2, 0.1, 0.3], np.float32)
    sa = np.array([-1, -1, -1, 3, 0, 0], np.float32)
    slot = np.array([0, 1, 2, -1, -1, -1], np.int32)
    ev, rp, _ = O.evict_and_replace(node, se, sa, slot, halo, np.ones(6, np.int32), 0.5, 1.0)
    assert list(ev) == [1] and list(rp) == [3]
    ev, rp, _ = O.evict_and_replace(node, se, sa, slot, halo, np.ones(6, np.int32), 0.05, 1.0)
    assert len(ev) == 0                                     # no S_E below alpha -> no-op round


def _random_state(rng):
    n_h = int(rng.integers(1, 65))
    cap = int(rng.integers(0, min(32, n_h) + 1))
    halo = np.sort(rng.choice(10 ** 6, n_h, replace=False)).astype(np.int32)
    deg = rng.integers(1, 4, n_h).astype(np.int32)            # many degree ties
    buffered = rng.choice(n_h, cap, replace=False)
    node = halo[buffered].astype(np.int32)
    se = rng.choice(np.array([0.0, 0.125, 0.25, 0.5, 0.7, 1.0, 3.0], np.float32), cap)   # many ties
    sa = rng.choice(np.array([0.0, 1.0, 2.0, 0.25, 5.0], np.float32), n_h)
    slot = np.full(n_h, -1, np.int32)
    slot[buffered] = np.arange(cap, dtype=np.int32)
    sa[buffered] = -1.0
    return halo, deg, node, se.astype(np.float32), sa.astype(np.float32), slot


def test_evict_vs_straight_line_reference_1000():
    rng = np.random.default_rng(2410)
    for inst in range(1000):
        halo, deg, node, se, sa, slot = _random_state(rng)
        alpha = float(rng.choice([0.0, 0.2, 0.5, 1.0, 2.0]))
        theta = float(rng.choice([0.0, 1.0]))
        ref = PolicyRef(halo, deg, 0, 1.0, alpha, theta, 1)
        ref.slot = {int(n): s for s, n in enumerate(node)}
        ref.cap = len(node)
        ref.se = {int(n): np.float32(se[s]) for s, n in enumerate(node)}
        ref.sa = {int(h): np.float32(sa[i]) for i, h in enumerate(halo)}
        ref.gamma = np.float32(1.0)
        ref.step(1, [])                                       # gamma=1: decay is identity, no misses
        O.evict_and_replace(node, se, sa, slot, halo, deg, alpha, theta)
        rn, rse, rsa = ref.arrays()
        assert np.array_equal(rn, node) and np.array_equal(rse.view(np.uint32), se.view(np.uint32)), inst
        assert np.array_equal(rsa.view(np.uint32), sa.view(np.uint32)), inst


# ------------------------------------------------------------------ sampler (Alg.2 l.1)
def _check_sampler_invariants(p, g, lo, hi, fanouts):
    L = len(fanouts)
    sizes = p.hop_sizes()
    F = p.frontier()
    assert len(set(F.tolist())) == len(F)                       # F_L has no duplicates
    for i in range(L):
        k = fanouts[L - 1 - i]
        off, cols = p.hop_block(i)
        Fi = F[:sizes[i]]
        for f, x in enumerate(Fi.tolist()):
            s = cols[off[f]:off[f + 1]].tolist()
            nbr = g.cols[g.indptr[x]:g.indptr[x + 1]].tolist()
            if lo <= x < hi:
                assert len(s) == min(len(nbr), k)              # |sample| = min(deg, k)
                assert len(set(s)) == len(s)                   # without replacement
                assert set(s) <= set(nbr)                      # true neighbours
                if len(nbr) <= k:
                    assert s == nbr
            else:
                assert s == []                                 # halo nodes are leaves (R#1)
        new = F[sizes[i]:sizes[i + 1]].tolist()
        assert new == sorted(set(cols.tolist()) - set(Fi.tolist()))   # R#7


@pytest.mark.parametrize("seed", range(6))
def test_sampler_invariants_random_graphs(seed):
    g = synth.random_graph(20, 0.3, seed)
    W, parts = world_from(g, 2)
    for p in W.parts:
        p.buffer_init(0.9, 0.5, 1.0, 3, 5000)
    lo, hi = 0, 10
    for t in range(1, 12):
        W.parts[0].step(RUN_SEED, t, [2, 3], 4)
        _check_sampler_invariants(W.parts[0], g, lo, hi, [2, 3])


def test_sampler_fanouts_above_the_gpu_cap():
    """The oracle follows the paper for any fanout (the CUDA library caps k at 32, MGNN_MAX_FANOUT):
    k = 40 and 64 on a dense graph (degrees ~50-90) keep every sampler invariant."""
    g = synth.random_graph(120, 0.7, 11)
    W, parts = world_from(g, 2)
    for p in W.parts:
        p.buffer_init(0.9, 0.5, 1.0, 3, 5000)
    for t in range(1, 4):
        W.parts[0].step(RUN_SEED, t, [40, 64], 4)
        _check_sampler_invariants(W.parts[0], g, 0, 60, [40, 64])


@pytest.mark.parametrize("seed", range(6))
def test_sampler_full_fanout_is_local_bfs(seed):
    """fanout >= max degree -> F_L is exactly the L-hop neighbourhood expanded through local nodes."""
    g = synth.random_graph(20, 0.2, seed)
    W, _ = world_from(g, 2)
    p = W.parts[0]
    p.buffer_init(0.9, 0.5, 1.0, 0, 0)
    seeds = np.array([1, 3, 7], np.int32)
    p.step(RUN_SEED, 1, [32, 32, 32], 3, seeds=seeds)
    reach = set(seeds.tolist())
    front = set(reach)
    for _ in range(3):
        nxt = set()
        for x in front:
            if x < 10:
                nxt |= set(g.cols[g.indptr[x]:g.indptr[x + 1]].tolist())
        front = nxt - reach
        reach |= nxt
    assert set(p.frontier().tolist()) == reach


def test_star_graph_two_leaves():
    g = synth.from_edges(12, [(0, i) for i in range(1, 12)])
    W, _ = world_from(g, 1)
    p = W.parts[0]
    p.buffer_init(0.9, 0.5, 1.0, 0, 0)
    for t in range(1, 20):
        p.step(RUN_SEED, t, [2], 1, seeds=np.array([0], np.int32))
        F = p.frontier().tolist()
        assert F[0] == 0 and len(F) == 3 and all(1 <= x < 12 for x in F[1:])


def test_sampler_uniform_chi2():
    """Uniform k-of-d sampling: chi^2 over the C(7,3) = 35 subsets across steps."""
    g = synth.from_edges(8, [(0, i) for i in range(1, 8)])
    W, _ = world_from(g, 1)
    p = W.parts[0]
    p.buffer_init(0.9, 0.5, 1.0, 0, 0)
    n = 7000
    cnt = Counter()
    for t in range(1, n + 1):
        p.step(RUN_SEED, t, [3], 1, seeds=np.array([0], np.int32))
        cnt[frozenset(p.frontier().tolist()[1:])] += 1
    assert len(cnt) == 35
    exp = n / 35
    chi2 = sum((c - exp) ** 2 / exp for c in cnt.values())
    assert chi2 < 75.0        # 34 dof: P(chi2 > 75) ~ 6e-5


# ------------------------------------------------------------------ seed order (R#8; Table 3)
def test_table3_minibatches_per_epoch():
    t3 = gold("table3_minibatches.json")
    B = t3["batch"]
    for ds, T, mb in t3["cells"]:
        nt = -(-t3["train_sizes"][ds] // T)
        n = nt + 1
        g = synth.Graph(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.array([1] * nt + [0], bool))
        W, _ = world_from(g, 1, D=0)
        p = W.parts[0]
        p.buffer_init(0.9, 0.5, 1.0, 0, 0)
        seen, t = [], 1
        while True:                      # walk epoch 0; the step after its last batch starts epoch 1
            p.step(RUN_SEED, t, [1], B)
            seen.extend(p.frontier()[:p.hop_sizes()[0]].tolist())
            if len(seen) >= nt:
                break
            t += 1
        assert sorted(seen) == list(range(nt))                 # each train node once per epoch
        assert t * t3["epochs"] == mb, (ds, T)


def test_epoch_permutations():
    g = synth.Graph(40, np.zeros(41, np.int64), np.zeros(0, np.int32), np.ones(40, bool))
    W, _ = world_from(g, 1, D=0)
    p = W.parts[0]
    e0 = p.epoch_perm(RUN_SEED, 0, 40)
    e1 = p.epoch_perm(RUN_SEED, 1, 40)
    assert sorted(e0.tolist()) == list(range(40)) and sorted(e1.tolist()) == list(range(40))
    assert not np.array_equal(e0, e1) and np.array_equal(e0, p.epoch_perm(RUN_SEED, 0, 40))


def test_epoch_permutation_order_is_ascending_philox_key():
    """R#8 pins the ORDER, not just the permutation: epoch e of partition p lists the train ids by
    ascending 64-bit key (out[0] << 32 | out[1]) of Philox(ctr = (id, e, 0, (p << 8) | 2), run_seed),
    ties by ascending id.  The keys are recomputed through the KAT-pinned Philox (test above), so a
    descending sort, a swapped key word, a wrong counter word or a dropped partition id all fail."""
    n = 120
    train = np.zeros(n, bool)
    train[np.random.default_rng(3).choice(n, 70, replace=False)] = True
    g = synth.Graph(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), train)
    W, parts = world_from(g, 2, D=0)
    key = [RUN_SEED & 0xFFFFFFFF, RUN_SEED >> 32]
    for pid in (0, 1):
        ids = parts[pid].train_ids
        for e in (0, 1, 7):
            perm = W.parts[pid].epoch_perm(RUN_SEED, e, len(ids))
            k = []
            for v in perm.tolist():
                o = O.philox([v, e, 0, (pid << 8) | 2], key)
                k.append(((o[0] << 32) | o[1], v))
            assert k == sorted(k), (pid, e)
            assert sorted(perm.tolist()) == sorted(ids.tolist())
        # seeds of step 1 = the first B ids of epoch 0 (R#8, O5)
        p = W.parts[pid]
        p.buffer_init(0.9, 0.5, 1.0, 0, 0)
        p.step(RUN_SEED, 1, [1], 16)
        assert p.frontier()[:p.hop_sizes()[0]].tolist() == p.epoch_perm(RUN_SEED, 0, len(ids))[:16].tolist()


# ------------------------------------------------------------------ whole-step pins
def _run_world(g, P, fanouts, B, f_bp, gamma, delta, theta, steps, D=4, bounds=None, check=None):
    W, parts = world_from(g, P, D=D, bounds=bounds)
    alpha = O.alpha_default(gamma, delta)
    refs = []
    for p in W.parts:
        p.buffer_init(gamma, alpha, theta, delta, f_bp)
        ids, deg = p.halo()
        refs.append(PolicyRef(ids, deg, f_bp, gamma, alpha, theta, delta))
    for t in range(1, steps + 1):
        for p, ref in zip(W.parts, refs):
            p.step(RUN_SEED, t, fanouts, B)
            if check:
                check(p, ref, t)
    return W, refs


def test_policy_vs_straight_line_reference_20_node_graphs():
    """Oracle buffer state == straight-line Alg.2 reference at every step, on 300 random
    20-node instances (north_star 'brute-force enumeration on 20-node graphs')."""
    rng = np.random.default_rng(7)
    n_inst = 0
    for inst in range(300):
        g = synth.random_graph(20, float(rng.uniform(0.1, 0.4)), 1000 + inst, train_frac=0.6)
        if g.train_mask[:10].sum() == 0 or g.train_mask[10:].sum() == 0:
            continue
        P = int(rng.integers(2, 4))
        f_bp = int(rng.choice([0, 2500, 5000, 10000]))
        gamma = float(rng.choice([0.5, 0.9, 1.0]))
        delta = int(rng.choice([0, 1, 2, 3]))
        theta = float(rng.choice([0.0, 1.0]))
        fan = [int(x) for x in rng.integers(1, 4, int(rng.integers(1, 3)))]
        if any(g.train_mask[int(lo):int(hi)].sum() == 0 for lo, hi in
               zip(synth.range_bounds(20, P)[:-1], synth.range_bounds(20, P)[1:])):
            continue

        def check(p, ref, t):
            h, m, k = ref.step(t, p.frontier().tolist())
            c = p.counts()
            assert (c["n_hit"], c["n_miss"], c["n_evicted"]) == (h, m, k)
            st = p.buffer_state()
            rn, rse, rsa = ref.arrays()
            assert np.array_equal(rn, st["node_of_slot"])
            assert np.array_equal(rse.view(np.uint32), st["se"].view(np.uint32))
            assert np.array_equal(rsa.view(np.uint32), st["sa"].view(np.uint32))

        _run_world(g, P, fan, 3, f_bp, gamma, delta, theta, 12, check=check)
        n_inst += 1
    assert n_inst >= 150


def test_content_equivalence_and_accounting():
    """X[i] == features(F_L[i]) (R#24); hits+misses == sampled halo nodes and
    remote fetches == misses + refills + init."""
    g = synth.generate(synth.CONFIGS["cfg1"])
    D = 64
    state = {"halo_acc": 0}

    def check(p, ref, t):
        F = p.frontier()
        X = p.features()
        lo, hi = p.world.bounds[p.pid], p.world.bounds[p.pid + 1]
        assert X.shape == (len(F), D)
        for i in range(0, len(F), 37):
            assert np.array_equal(X[i], O.feature_row(int(F[i]), D, FEAT_SEED))
        c = p.counts()
        n_halo_s = int(((F < lo) | (F >= hi)).sum())
        assert c["n_hit"] + c["n_miss"] == n_halo_s and c["n_local"] + n_halo_s == len(F)
        state["halo_acc"] += n_halo_s
        # buffer invariants: S_A == -1 <=> buffered; |BUF| constant; maps consistent
        st = p.buffer_state(rows=True)
        ids, _ = p.halo()
        buffered = set(st["node_of_slot"].tolist())
        assert len(buffered) == p.cap
        assert set(ids[st["sa"] == -1.0].tolist()) == buffered
        for s, n in enumerate(st["node_of_slot"].tolist()):
            assert st["slot_of"][np.searchsorted(ids, n)] == s
        for s in range(0, p.cap, 29):
            assert np.array_equal(st["rows"][s], O.feature_row(int(st["node_of_slot"][s]), D, FEAT_SEED))

    W, _ = _run_world(g, 2, [10, 25], 256, 2500, 0.9, 4, 1.0, 16, D=D, check=check)
    tot = [p.totals() for p in W.parts]
    assert sum(t["hits"] + t["misses"] for t in tot) == state["halo_acc"]
    assert all(t["refills"] > 0 for t in tot)


@pytest.mark.parametrize("delta", [0, 3])
def test_f0_all_misses_f1_all_hits(delta):
    g = synth.generate(synth.CONFIGS["cfg1"])
    for f_bp, want in ((0, "n_miss"), (10000, "n_hit")):
        def check(p, ref, t):
            c = p.counts()
            assert c[want] == c["n_nodes"] - c["n_local"]
            assert c["n_evicted"] == 0
        _run_world(g, 2, [10, 25], 256, f_bp, 0.5, delta, 1.0, 2 * max(delta, 1), check=check)


# ------------------------------------------------------------------ NEXT-1: remote expansion
def test_remote_expansion_path_hand_trace():
    """Path 0-1-2-3-4, partitions {0,1,2} | {3,4}, seed 2, full fanout, 2 hops.  Local reading
    (R#1): the halo node 3 is a leaf -> F_2 = [2, 1, 3, 0].  Remote expansion: 3 is sampled from
    partition 1's row {2, 4} -> F_2 = [2, 1, 3, 0, 4]; 4 is outside V_0^l and V_0^h = {3}: a
    class-3 miss."""
    g = synth.from_edges(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    for remote, want_F, want_cls in ((False, [2, 1, 3, 0], [0, 0, 2, 0]), (True, [2, 1, 3, 0, 4], [0, 0, 2, 0, 3])):
        W, _ = world_from(g, 2, bounds=np.array([0, 3, 5]))
        p = W.parts[0]
        p.buffer_init(0.9, 0.5, 1.0, 0, 0)
        p.set_expand_remote(remote)
        p.step(RUN_SEED, 1, [32, 32], 1, seeds=np.array([2], np.int32))
        assert p.frontier().tolist() == want_F
        assert p.classes().tolist() == want_cls
        off, cols = p.hop_block(1)
        assert cols[off[2]:off[3]].tolist() == ([2, 4] if remote else [])
        c = p.counts()
        assert c["n_local"] == 3 and c["n_hit"] == 0 and c["n_miss"] == (2 if remote else 1)
        X = p.features()
        for i, v in enumerate(want_F):
            assert np.array_equal(X[i], O.feature_row(v, 4, FEAT_SEED))   # far rows fetched too
        W.close()


@pytest.mark.parametrize("seed", range(4))
def test_remote_expansion_invariants(seed):
    """Every frontier node (local, halo or far) draws min(deg, k) distinct true neighbours from the
    GLOBAL graph; hits + misses = non-local nodes; only halo nodes are tallied."""
    g = synth.random_graph(24, 0.2, seed)
    W, _ = world_from(g, 3)
    for p in W.parts:
        p.buffer_init(0.9, 0.5, 1.0, 3, 5000)
        p.set_expand_remote(True)
    p = W.parts[0]
    lo, hi = 0, 8
    halo = set(p.halo()[0].tolist())
    fan = [2, 3]
    for t in range(1, 10):
        p.step(RUN_SEED, t, fan, 3)
        sizes = p.hop_sizes()
        F = p.frontier()
        for i in range(2):
            k = fan[1 - i]
            off, cols = p.hop_block(i)
            for f, x in enumerate(F[:sizes[i]].tolist()):
                s = cols[off[f]:off[f + 1]].tolist()
                nbr = g.cols[g.indptr[x]:g.indptr[x + 1]].tolist()
                assert len(s) == min(len(nbr), k) and len(set(s)) == len(s) and set(s) <= set(nbr)
        cls = p.classes().tolist()
        for x, c in zip(F.tolist(), cls):
            assert c == (0 if lo <= x < hi else (3 if x not in halo else c)) and c in (0, 1, 2, 3)
        cn = p.counts()
        assert cn["n_local"] + cn["n_hit"] + cn["n_miss"] == cn["n_nodes"]
    W.close()


def test_remote_expansion_single_partition_is_identity():
    """P = 1: no remote nodes, so remote expansion changes nothing."""
    g = synth.random_graph(30, 0.15, 5)
    outs = []
    for remote in (False, True):
        W, _ = world_from(g, 1)
        p = W.parts[0]
        p.buffer_init(0.9, 0.5, 1.0, 0, 0)
        p.set_expand_remote(remote)
        p.step(RUN_SEED, 3, [3, 4], 5)
        outs.append((p.frontier().tolist(), [p.hop_block(i)[1].tolist() for i in range(2)]))
        W.close()
    assert outs[0] == outs[1]


def _path6_world(dense):
    g = synth.from_edges(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)])
    W, _ = world_from(g, 2, bounds=np.array([0, 3, 6]))
    return W


def test_dense_scores_far_node_enters_buffer():
    """Path 0-..-5, partitions {0,1,2} | {3,4,5}, seed 2, full fanout, 2 hops, remote expansion:
    F = [2, 1, 3, 0, 4].  True halo of p0 = {3} (cap = 1 at f = 1); 4 is remote but scorable with
    the dense S_A.  alpha = 2 (an explicit override) makes the buffered 3 evictable at the round
    of step 2, when S_A[4] = 2 >= theta_R: 4 replaces 3 (S_A[3] <- S_E = 1, S_E[slot] <- 2).
    Step 3 then hits 4 and misses 3.  Without the dense S_A, 4 is an unscored miss forever."""
    g = synth.from_edges(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)])
    for dense in (False, True):
        parts = synth.partition(g, 2, np.array([0, 3, 6]))
        W = O.World(parts, 4, FEAT_SEED, dense=dense)
        p = W.parts[0]
        p.buffer_init(0.9, 2.0, 1.0, 2, 10000)
        p.set_expand_remote(True)
        assert p.cap == 1
        seeds = np.array([2], np.int32)
        for t in (1, 2):
            p.step(RUN_SEED, t, [32, 32], 1, seeds=seeds)
            assert p.frontier().tolist() == [2, 1, 3, 0, 4]
        st = p.buffer_state()
        halo = p.halo()[0].tolist()
        if dense:
            assert halo == [3, 4, 5]
            assert st["node_of_slot"].tolist() == [4]
            assert st["se"].tolist() == [2.0]
            assert st["sa"].tolist() == [1.0, -1.0, 0.0]
        else:
            assert halo == [3] and st["node_of_slot"].tolist() == [3]
        p.step(RUN_SEED, 3, [32, 32], 1, seeds=seeds)
        c = p.counts()
        assert (c["n_hit"], c["n_miss"]) == ((1, 1) if dense else (1, 1))
        cls = p.classes().tolist()
        assert cls == ([0, 0, 2, 0, 1] if dense else [0, 0, 1, 0, 3])
        if dense:
            assert p.buffer_state()["sa"].tolist() == [2.0, -1.0, 0.0]
        W.close()


@pytest.mark.parametrize("seed", range(3))
def test_dense_scores_without_remote_expansion_is_identity(seed):
    """Local sampling never reaches nodes outside V_p^h; with theta_R = 1 their S_A (0) never
    qualifies them, so the dense scoreboard changes nothing on the true halo."""
    g = synth.random_graph(30, 0.15, seed)
    res = []
    for dense in (False, True):
        W, parts = world_from(g, 3)
        W.close()
        W = O.World(parts, 4, FEAT_SEED, dense=dense)
        p = W.parts[1]
        p.buffer_init(0.8, float(O.alpha_default(0.8, 2)), 1.0, 2, 5000)
        out = []
        for t in range(1, 9):
            p.step(RUN_SEED, t, [2, 3], 3)
            out.append((p.frontier().tolist(), p.counts()))
        st = p.buffer_state()
        halo = p.halo()[0]
        true = [i for i, d in enumerate(p.halo()[1].tolist()) if d > 0]
        res.append((out, st["node_of_slot"].tolist(), st["se"].tolist(), halo[true].tolist(),
                    st["sa"][true].tolist()))
        W.close()
    assert res[0] == res[1]


def test_hash_relabel_is_an_isomorphism():
    """NEXT-4 stress input: the relabelled graph has exactly the relabelled edge set, ascending rows."""
    g = synth.random_graph(60, 0.08, 4)
    h = synth.hash_relabel(g, 11)
    rng = np.random.Generator(np.random.PCG64(11))
    new_of = rng.permutation(60)
    e_g = {(int(new_of[u]), int(new_of[v])) for u in range(60) for v in g.cols[g.indptr[u]:g.indptr[u + 1]]}
    e_h = {(u, int(v)) for u in range(60) for v in h.cols[h.indptr[u]:h.indptr[u + 1]]}
    assert e_g == e_h
    assert all(np.all(np.diff(h.cols[h.indptr[u]:h.indptr[u + 1]]) > 0) for u in range(60))
    assert sorted(np.nonzero(h.train_mask)[0].tolist()) == sorted(int(new_of[v]) for v in np.nonzero(g.train_mask)[0])
