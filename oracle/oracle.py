"""ctypes wrapper of the CPU oracle (oracle/orc.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package (paper_2410_22697_b200).  The oracle shares no code with the CUDA
path; see orc.h for the citations of every function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")
_SRC = [os.path.join(HERE, "orc.c")]
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-Wall"]

_lib = None


def build(force: bool = False) -> str:
    """Compile liborc.so with gcc (plain C, no fast-math)."""
    newest = max(os.path.getmtime(s) for s in _SRC + [os.path.join(HERE, "orc.h")])
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, *_SRC, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P, I32, I64, U32, U64, F32 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
        sig = {
            "orc_philox4x32_10": (None, [P, P, P]),
            "orc_feature_row": (None, [I64, I32, U64, P]),
            "orc_floyd": (None, [I64, I32, P, P]),
            "orc_range": (U32, [U32, U32]),
            "orc_alpha_default": (F32, [F32, I32]),
            "orc_world_new": (P, [I32, I64, P, I32, U64]),
            "orc_world_free": (None, [P]),
            "orc_part_new": (P, [P, I32, P, P, P, I64]),
            "orc_part_free": (None, [P]),
            "orc_n_local": (I64, [P]),
            "orc_n_halo": (I64, [P]),
            "orc_halo": (None, [P, P, P]),
            "orc_buffer_init": (C.c_int, [P, F32, F32, F32, I32, U32]),
            "orc_capacity": (I64, [P]),
            "orc_epoch_perm": (None, [P, U64, U64, P]),
            "orc_step": (C.c_int, [P, U64, U64, P, I32, I32, P, I32]),
            "orc_counts": (None, [P, P]),
            "orc_hop_size": (I64, [P, I32]),
            "orc_hop_edges": (I64, [P, I32]),
            "orc_frontier": (None, [P, P]),
            "orc_hop_block": (None, [P, I32, P, P]),
            "orc_features_out": (None, [P, P]),
            "orc_classes": (None, [P, P]),
            "orc_buffer_state": (None, [P, P, P, P, P, P]),
            "orc_totals": (None, [P, P]),
            "orc_evict_and_replace": (I64, [I64, I64, P, P, P, P, P, P, F32, F32, P, P, P]),
            "orc_set_expand_remote": (None, [P, I32]),
            "orc_world_set_dense": (None, [P, I32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------------- primitives
def philox(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    c = np.array(ctr, dtype=np.uint32)
    k = np.array(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(o))
    return [int(x) for x in o]


def feature_row(node: int, dim: int, feat_seed: int) -> np.ndarray:
    out = np.zeros(dim, dtype=np.float32)
    lib().orc_feature_row(node, dim, feat_seed, _p(out))
    return out


def floyd(d: int, k: int, r: Sequence[int]) -> List[int]:
    rr = np.array(r, dtype=np.uint32)
    pos = np.zeros(k, dtype=np.int64)
    lib().orc_floyd(d, k, _p(rr), _p(pos))
    return [int(x) for x in pos]


def urange(u: int, t_plus_1: int) -> int:
    return int(lib().orc_range(u, t_plus_1))


def alpha_default(gamma: float, delta: int) -> np.float32:
    return np.float32(lib().orc_alpha_default(float(np.float32(gamma)), delta))


def evict_and_replace(node_of_slot, se, sa, slot_of, halo, deg_in, alpha, theta_r):
    """EVICT_AND_REPLACE on explicit arrays (modified in place). Returns (evicted, replaced, slots)."""
    for a, t in ((node_of_slot, np.int32), (se, np.float32), (sa, np.float32), (slot_of, np.int32)):
        assert a.dtype == t and a.flags.c_contiguous
    halo = np.ascontiguousarray(halo, np.int32)
    deg_in = np.ascontiguousarray(deg_in, np.int32)
    m = max(1, min(len(se), len(sa)))
    ev, rp, sl = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m, np.int32)
    k = lib().orc_evict_and_replace(len(se), len(sa), _p(node_of_slot), _p(se), _p(sa), _p(slot_of),
                                    _p(halo), _p(deg_in), float(np.float32(alpha)),
                                    float(np.float32(theta_r)), _p(ev), _p(rp), _p(sl))
    return ev[:k].copy(), rp[:k].copy(), sl[:k].copy()


# --------------------------------------------------------------------- partitions
class World:
    """All P partitions of one graph, each a trainer with its own prefetcher."""

    def __init__(self, parts_in, feat_dim: int, feat_seed: int, dense: bool = False):
        L = lib()
        p0 = parts_in[0]
        self.P = p0.n_parts
        self.D = feat_dim
        self.bounds = np.ascontiguousarray(p0.bounds, dtype=np.int64)
        self._w = L.orc_world_new(self.P, p0.n_global, _p(self.bounds), feat_dim, feat_seed)
        if not self._w:
            raise ValueError("orc_world_new: invalid input")
        L.orc_world_set_dense(self._w, 1 if dense else 0)   # NEXT-1 dense S_A (orc.h)
        self._keep = []
        self.parts = []
        for pi in parts_in:
            indptr = np.ascontiguousarray(pi.indptr, dtype=np.int64)
            cols = np.ascontiguousarray(pi.cols, dtype=np.int32)
            tr = np.ascontiguousarray(pi.train_ids, dtype=np.int32)
            h = L.orc_part_new(self._w, pi.part_id, _p(indptr), _p(cols), _p(tr), tr.shape[0])
            if not h:
                raise ValueError(f"orc_part_new({pi.part_id}): invalid input")
            self.parts.append(Part(self, h, pi.part_id))

    def close(self):
        L = lib()
        for p in self.parts:
            L.orc_part_free(p._h)
        self.parts = []
        if self._w:
            L.orc_world_free(self._w)
            self._w = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Part:
    def __init__(self, world: World, handle, pid: int):
        self.world = world
        self._h = handle
        self.pid = pid

    @property
    def n_local(self) -> int:
        return int(lib().orc_n_local(self._h))

    @property
    def n_halo(self) -> int:
        return int(lib().orc_n_halo(self._h))

    @property
    def cap(self) -> int:
        return int(lib().orc_capacity(self._h))

    def halo(self):
        n = self.n_halo
        ids = np.zeros(n, np.int32)
        deg = np.zeros(n, np.int32)
        lib().orc_halo(self._h, _p(ids), _p(deg))
        return ids, deg

    def buffer_init(self, gamma, alpha, theta_r, delta, f_bp) -> None:
        rc = lib().orc_buffer_init(self._h, float(np.float32(gamma)), float(np.float32(alpha)),
                                   float(np.float32(theta_r)), int(delta), int(f_bp))
        if rc != 0:
            raise ValueError("orc_buffer_init: invalid policy")

    def set_expand_remote(self, on: bool) -> None:
        """NEXT-1: sample non-local frontier nodes from their owner's CSR (see orc.h)."""
        lib().orc_set_expand_remote(self._h, 1 if on else 0)

    def epoch_perm(self, run_seed: int, epoch: int, n_train: int) -> np.ndarray:
        out = np.zeros(n_train, np.int32)
        lib().orc_epoch_perm(self._h, run_seed, epoch, _p(out))
        return out

    def step(self, run_seed: int, step: int, fanouts: Sequence[int], batch: int,
             seeds: Optional[np.ndarray] = None) -> None:
        fo = np.array(fanouts, dtype=np.int32)
        sd = None if seeds is None else np.ascontiguousarray(seeds, dtype=np.int32)
        rc = lib().orc_step(self._h, run_seed, step, _p(fo), fo.shape[0], batch, _p(sd),
                            0 if sd is None else sd.shape[0])
        if rc != 0:
            raise ValueError(f"orc_step({step}) failed")
        self.L = len(fanouts)

    # results of the last step
    def counts(self) -> Dict[str, int]:
        c = np.zeros(7, np.int64)
        lib().orc_counts(self._h, _p(c))
        keys = ["n_nodes", "n_local", "n_hit", "n_miss", "n_evicted", "n_refilled", "rows_fetched"]
        return {k: int(v) for k, v in zip(keys, c)}

    def hop_sizes(self) -> List[int]:
        return [int(lib().orc_hop_size(self._h, i)) for i in range(self.L + 1)]

    def frontier(self) -> np.ndarray:
        n = self.hop_sizes()[-1]
        out = np.zeros(n, np.int32)
        lib().orc_frontier(self._h, _p(out))
        return out

    def hop_block(self, hop: int):
        nf = int(lib().orc_hop_size(self._h, hop))
        ne = int(lib().orc_hop_edges(self._h, hop))
        off = np.zeros(nf + 1, np.int64)
        cols = np.zeros(ne, np.int32)
        lib().orc_hop_block(self._h, hop, _p(off), _p(cols))
        return off, cols

    def features(self) -> np.ndarray:
        n = self.hop_sizes()[-1]
        out = np.zeros((n, self.world.D), np.float32)
        lib().orc_features_out(self._h, _p(out))
        return out

    def classes(self) -> np.ndarray:
        n = self.hop_sizes()[-1]
        out = np.zeros(n, np.int8)
        lib().orc_classes(self._h, _p(out))
        return out

    def buffer_state(self, rows: bool = False):
        cap, nh = self.cap, self.n_halo
        node = np.zeros(cap, np.int32)
        se = np.zeros(cap, np.float32)
        sa = np.zeros(nh, np.float32)
        slot = np.zeros(nh, np.int32)
        r = np.zeros((cap, self.world.D), np.float32) if rows else None
        lib().orc_buffer_state(self._h, _p(node), _p(se), _p(sa), _p(slot), _p(r))
        return {"node_of_slot": node, "se": se, "sa": sa, "slot_of": slot, "rows": r}

    def totals(self) -> Dict[str, int]:
        t = np.zeros(4, np.int64)
        lib().orc_totals(self._h, _p(t))
        return {"hits": int(t[0]), "misses": int(t[1]), "refills": int(t[2]), "init_fetch": int(t[3])}
