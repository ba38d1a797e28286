"""Thin Python front-end over the C ABI (include/mgnn.h).

Argument marshalling only: every step of the halo feature pipeline runs in
libmgnn.so's CUDA kernels.  PyTorch supplies streams, zero-copy device views
(via __cuda_array_interface__) and torch.distributed for the multi-GPU
plumbing (exchanging the CUDA IPC handles of the feature tables).
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import MgnnError, Policy, PartitionDesc, SageDesc, Window


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _stream(stream) -> C.c_void_p:
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class _DevArray:
    """__cuda_array_interface__ wrapper of a library-owned device buffer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def device_view(ptr: int, shape, dtype: str):
    """Zero-copy torch tensor over a library device pointer."""
    import torch
    typestr = {"f4": "<f4", "i4": "<i4", "i8": "<i8"}[dtype]
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device="cuda")


class Context:
    """One GPU's share of the partitioned graph (one or more trainers/partitions)."""

    def __init__(self, device: int, bounds: np.ndarray, feat_dim: int, feat_seed: int):
        self.L = _lib.load()
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        self.P = len(self.bounds) - 1
        self.n_global = int(self.bounds[-1])
        self.D = int(feat_dim)
        self.pitch = ((self.D + 3) // 4) * 4 or 4
        self._h = C.c_void_p()
        st = self.L.mgnn_ctx_create(device, self.P, self.n_global, _ptr(self.bounds), self.D, feat_seed,
                                    C.byref(self._h))
        if st != 0:
            raise MgnnError("mgnn_ctx_create", st, "cannot create context (CUDA device / arguments)")
        self.parts: List[int] = []       # part ids in local order
        self.n_steps = [0, 0]
        self.fanouts: List[int] = []
        self.batch = 0

    # ------------------------------------------------------------ helpers
    def _chk(self, fn: str, st: int):
        if st != 0:
            msg = self.L.mgnn_last_error(self._h)
            raise MgnnError(fn, st, msg.decode() if msg else "")

    def close(self):
        if self._h:
            self.L.mgnn_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ setup
    def load_partition(self, part_id: int, indptr: np.ndarray, cols: np.ndarray, train_ids: np.ndarray) -> int:
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        cl = np.ascontiguousarray(cols, dtype=np.int32)
        tr = np.ascontiguousarray(train_ids, dtype=np.int32)
        d = PartitionDesc(part_id, ip.ctypes.data, cl.ctypes.data, tr.ctypes.data, tr.shape[0])
        lp = C.c_int32(-1)
        self._chk("mgnn_partition_load", self.L.mgnn_partition_load(self._h, C.byref(d), C.byref(lp)))
        self.parts.append(part_id)
        return lp.value

    def export_table(self, part_id: int) -> bytes:
        buf = C.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        self._chk("mgnn_table_export", self.L.mgnn_table_export(self._h, part_id, buf))
        return buf.raw

    def import_table(self, part_id: int, handle: bytes) -> None:
        buf = C.create_string_buffer(bytes(handle), _lib.IPC_HANDLE_BYTES)
        self._chk("mgnn_table_import", self.L.mgnn_table_import(self._h, part_id, buf))

    def buffer_init(self, gamma: float, alpha: float, theta_r: float, delta: int, f_bp: int, stream=None):
        pol = Policy(gamma, alpha, theta_r, delta, f_bp)
        self.delta = delta
        self._chk("mgnn_buffer_init", self.L.mgnn_buffer_init(self._h, C.byref(pol), _stream(stream)))

    def load_global_csr(self, indptr: np.ndarray, cols: np.ndarray):
        """Replicated global CSR (NEXT-1 across GPUs)."""
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        cl = np.ascontiguousarray(cols, dtype=np.int32)
        self._chk("mgnn_graph_csr_load", self.L.mgnn_graph_csr_load(self._h, _ptr(ip), _ptr(cl)))

    def expand_remote(self, enable: bool = True):
        """NEXT-1: sample non-local frontier nodes from their owner's CSR (before sampler_config)."""
        self._chk("mgnn_sampler_expand_remote", self.L.mgnn_sampler_expand_remote(self._h, 1 if enable else 0))

    def sampler_config(self, fanouts: Sequence[int], batch: int, run_seed: int, max_window: int,
                       rows_bound: int = 0):
        """rows_bound > 0: realistic window arenas (mgnn_sampler_config_bounded); 0: static worst case."""
        fo = np.array(fanouts, dtype=np.int32)
        self._chk("mgnn_sampler_config_bounded",
                  self.L.mgnn_sampler_config_bounded(self._h, _ptr(fo), fo.shape[0], batch, run_seed, max_window,
                                                     int(rows_bound)))
        self.rows_bound = int(rows_bound)
        self.fanouts = list(fanouts)
        self.batch = batch
        self.max_window = max_window

    # ------------------------------------------------------------ the hot path
    def sample(self, slot: int, t0: int, n_steps: int, seeds: Optional[np.ndarray] = None,
               seed_counts: Optional[np.ndarray] = None, stream=None, seeds_on_host: bool = True):
        if seeds is None:
            st = self.L.mgnn_sample(self._h, slot, t0, n_steps, None, None, 0, _stream(stream))
        elif seeds_on_host:
            self._seeds_keep = (np.ascontiguousarray(seeds, np.int32), np.ascontiguousarray(seed_counts, np.int32))
            st = self.L.mgnn_sample(self._h, slot, t0, n_steps, _ptr(self._seeds_keep[0]),
                                    _ptr(self._seeds_keep[1]), 1, _stream(stream))
        else:   # torch device tensors
            st = self.L.mgnn_sample(self._h, slot, t0, n_steps, C.c_void_p(seeds.data_ptr()),
                                    C.c_void_p(seed_counts.data_ptr()), 0, _stream(stream))
        self._chk("mgnn_sample", st)
        self.n_steps[slot] = n_steps

    def sample_ptr(self, slot: int, t0: int, n_steps: int, seeds_ptr: int, counts_ptr: int, on_host: bool, stream=None):
        """mgnn_sample with raw (pinned host or device) seed pointers."""
        self._chk("mgnn_sample", self.L.mgnn_sample(self._h, slot, t0, n_steps, C.c_void_p(seeds_ptr),
                                                    C.c_void_p(counts_ptr), 1 if on_host else 0, _stream(stream)))
        self.n_steps[slot] = n_steps

    def defer_relabel(self, enable: bool = True):
        """mgnn_sampler_defer_relabel: mgnn_sample leaves the columns in rank space until relabel()."""
        self._chk("mgnn_sampler_defer_relabel", self.L.mgnn_sampler_defer_relabel(self._h, 1 if enable else 0))

    def sm_partition(self, gather_sms: int):
        """mgnn_sm_partition: gather + scoring on `gather_sms` SMs, sampling + relabel on the rest
        (green contexts; 0 = whole GPU).  Returns (gather-side SMs, prepare-side SMs)."""
        out = (C.c_int32 * 2)()
        self._chk("mgnn_sm_partition", self.L.mgnn_sm_partition(self._h, int(gather_sms), out))
        return int(out[0]), int(out[1])

    def relabel(self, slot: int, stream=None):
        self._chk("mgnn_relabel", self.L.mgnn_relabel(self._h, slot, _stream(stream)))

    def lookup_gather(self, slot: int, stream=None):
        self._chk("mgnn_lookup_gather", self.L.mgnn_lookup_gather(self._h, slot, _stream(stream)))

    def score(self, slot: int, stream=None):
        self._chk("mgnn_score_evict_refill", self.L.mgnn_score_evict_refill(self._h, slot, _stream(stream)))

    def prepare(self, slot: int, t0: int, n_steps: int, stream=None):
        """PREPARE_NEXT_MINIBATCH (Alg.1 l.9) for a window of steps."""
        s = _stream(stream)
        self.sample(slot, t0, n_steps, stream=s.value)
        self.lookup_gather(slot, stream=s.value)
        self.score(slot, stream=s.value)

    # ------------------------------------------------------------ A14: GraphSAGE-mean consumer
    def sage_config(self, dims: Sequence[int], w_self: Sequence[np.ndarray], w_neigh: Sequence[np.ndarray],
                    bias: Sequence[np.ndarray]):
        """Upload layer weights (nn.Linear layout [dims[l+1]][dims[l]], fp32) to the library."""
        L = len(dims) - 1
        keep = [np.ascontiguousarray(dims, np.int32)]
        arrs = []
        for group in (w_self, w_neigh, bias):
            ptrs = (C.c_void_p * L)()
            for l in range(L):
                a = np.ascontiguousarray(group[l], np.float32)
                keep.append(a)
                ptrs[l] = a.ctypes.data
            arrs.append(ptrs)
        d = SageDesc(L, keep[0].ctypes.data, C.cast(arrs[0], C.c_void_p), C.cast(arrs[1], C.c_void_p),
                     C.cast(arrs[2], C.c_void_p))
        self._chk("mgnn_sage_config", self.L.mgnn_sage_config(self._h, C.byref(d)))
        self.sage_dims = list(dims)

    def sage_forward(self, slot: int, logits, stream=None):
        """Forward pass of the window in `slot` into logits (torch CUDA tensor [n_inst][batch][pitch])."""
        assert logits.is_cuda and logits.dtype.itemsize == 4 and logits.is_contiguous()
        self._chk("mgnn_sage_forward", self.L.mgnn_sage_forward(self._h, slot, C.c_void_p(logits.data_ptr()),
                                                                logits.shape[-1], _stream(stream)))

    # ------------------------------------------------------------ NEXT-3: DDP training step
    def train_config(self, labels: np.ndarray):
        lab = np.ascontiguousarray(labels, np.int32)
        self._chk("mgnn_sage_train_config", self.L.mgnn_sage_train_config(self._h, _ptr(lab)))

    def train_step(self, slot: int, step_in_window: int, n_trainers: int, stream=None):
        self._chk("mgnn_sage_train_step",
                  self.L.mgnn_sage_train_step(self._h, slot, step_in_window, n_trainers, _stream(stream)))

    def grads(self):
        """Zero-copy torch view of the gradient buffer (the all-reduce operand)."""
        p = C.c_void_p()
        n = C.c_int64()
        self._chk("mgnn_sage_grads", self.L.mgnn_sage_grads(self._h, C.byref(p), C.byref(n)))
        return device_view(p.value, (n.value,), "f4")

    def sgd(self, lr: float, stream=None):
        self._chk("mgnn_sage_sgd", self.L.mgnn_sage_sgd(self._h, lr, _stream(stream)))

    def loss(self, stream=None) -> float:
        out = C.c_float()
        self._chk("mgnn_sage_loss", self.L.mgnn_sage_loss(self._h, C.byref(out), _stream(stream)))
        return out.value

    def params(self, l: int):
        d_in, d_out = self.sage_dims[l], self.sage_dims[l + 1]
        ws = np.zeros((d_out, d_in), np.float32)
        wn = np.zeros((d_out, d_in), np.float32)
        b = np.zeros(d_out, np.float32)
        self._chk("mgnn_sage_params", self.L.mgnn_sage_params(self._h, l, _ptr(ws), _ptr(wn), _ptr(b)))
        return ws, wn, b

    # ------------------------------------------------------------ outputs
    def window(self, slot: int) -> Window:
        w = Window()
        self._chk("mgnn_window_get", self.L.mgnn_window_get(self._h, slot, C.byref(w)))
        return w

    def counts(self, slot: int, stream=None) -> np.ndarray:
        n_inst = len(self.parts) * self.n_steps[slot]
        out = np.zeros((n_inst, _lib.C_N), dtype=np.int64)
        self._chk("mgnn_counts_read", self.L.mgnn_counts_read(self._h, slot, _ptr(out), _stream(stream)))
        return out

    def counts_async(self, slot: int, host_ptr: int, stream=None):
        """Enqueue the D2H copy of the window's counters into pinned host memory (no sync)."""
        self._chk("mgnn_counts_read_async",
                  self.L.mgnn_counts_read_async(self._h, slot, C.c_void_p(host_ptr), _stream(stream)))

    def instance(self, slot: int, m: int, with_x: bool = True) -> Dict[str, np.ndarray]:
        """Host copies of instance m of a window (tests; synchronises)."""
        import torch
        torch.cuda.synchronize()
        w = self.window(slot)
        L = w.n_layers
        hs = device_view(w.hop_size, (w.n_inst, _lib.MAX_LAYERS + 1), "i8")[m, :L + 1].cpu().numpy()
        U = int(hs[L])
        out = {"hop_size": hs}
        out["frontier"] = device_view(w.frontier, (w.n_inst, w.rows_stride), "i4")[m, :U].cpu().numpy()
        for i in range(L):
            off = device_view(w.offsets[i], (w.n_inst, w.off_stride[i]), "i8")[m, :hs[i] + 1].cpu().numpy()
            E = int(off[-1])
            cols = device_view(w.cols[i], (w.n_inst, w.col_stride[i]), "i4")[m, :E].cpu().numpy()
            out[f"off{i}"] = off
            out[f"cols{i}"] = cols
        if with_x:
            X = device_view(w.X, (w.n_inst, w.rows_stride, w.pitch), "f4")[m, :U, :self.D].cpu().numpy()
            out["X"] = X
        return out

    def snapshot(self, lp: int, rows: bool = False) -> Dict[str, np.ndarray]:
        info = self.part_info(lp)
        cap, nh = info["cap"], info["n_halo"]
        node = np.zeros(cap, np.int32)
        se = np.zeros(cap, np.float32)
        sa = np.zeros(nh, np.float32)
        slot = np.zeros(nh, np.int32)
        r = np.zeros((cap, self.D), np.float32) if rows else None
        self._chk("mgnn_buffer_snapshot", self.L.mgnn_buffer_snapshot(self._h, lp, _ptr(node), _ptr(se), _ptr(sa),
                                                                      _ptr(slot), _ptr(r)))
        return {"node_of_slot": node, "se": se, "sa": sa, "slot_of": slot, "rows": r}

    def part_info(self, lp: int) -> Dict[str, int]:
        info = np.zeros(5, np.int64)
        self._chk("mgnn_part_info", self.L.mgnn_part_info(self._h, lp, _ptr(info)))
        return dict(zip(["part_id", "n_local", "n_halo", "cap", "n_train"], (int(x) for x in info)))

    def halo(self, lp: int):
        nh = self.part_info(lp)["n_halo"]
        ids = np.zeros(nh, np.int32)
        deg = np.zeros(nh, np.int32)
        self._chk("mgnn_halo_get", self.L.mgnn_halo_get(self._h, lp, _ptr(ids), _ptr(deg)))
        return ids, deg

    def table_row(self, node: int) -> np.ndarray:
        out = np.zeros(self.D, np.float32)
        self._chk("mgnn_table_row", self.L.mgnn_table_row(self._h, node, _ptr(out)))
        return out

    def window_shape(self):
        """(rows_stride, pitch, n_inst_max) of the window arenas (mgnn_window_shape)."""
        r, p, m = C.c_int64(), C.c_int64(), C.c_int64()
        self._chk("mgnn_window_shape", self.L.mgnn_window_shape(self._h, C.byref(r), C.byref(p), C.byref(m)))
        return r.value, p.value, m.value

    def bind_x(self, slot: int, X) -> None:
        """Caller-owned X for window slot `slot` (mgnn_window_bind_x): a contiguous float32 CUDA tensor of
        at least n_inst_max * rows_stride * pitch elements; the caller keeps it alive."""
        assert X.is_cuda and X.dtype.itemsize == 4 and X.is_contiguous()
        self._chk("mgnn_window_bind_x", self.L.mgnn_window_bind_x(self._h, slot, C.c_void_p(X.data_ptr()), X.numel()))
        self._x_keep = getattr(self, "_x_keep", {})
        self._x_keep[slot] = X

    def next_step(self) -> int:
        """mgnn_next_step: first step of the next window the library will gather."""
        out = C.c_uint64()
        self._chk("mgnn_next_step", self.L.mgnn_next_step(self._h, C.byref(out)))
        return int(out.value)

    def launch_count(self) -> int:
        return int(self.L.mgnn_launch_count(self._h))

    def profile(self, enable, gather_only: bool = False):
        """mgnn_profile_enable: events around every stage (1), around the gather launch only (2,
        gather_only=True: the other stages keep their programmatic launch overlap), or off."""
        level = (2 if gather_only else 1) if enable else 0
        self._chk("mgnn_profile_enable", self.L.mgnn_profile_enable(self._h, level))

    def profile_stages(self) -> Dict[str, float]:
        """mgnn_profile_stages: per-stage event times and sampled units since the last read."""
        out = np.zeros(_lib.PROF_N, np.float64)
        self._chk("mgnn_profile_stages", self.L.mgnn_profile_stages(self._h, _ptr(out), _lib.PROF_N))
        keys = ["sample_ms", "sample_calls", "edges", "frontier", "unique", "gather_ms", "gather_calls",
                "gather_rows", "score_ms", "score_calls", "hits", "misses", "relabel_ms", "relabel_calls",
                "relabel_probes"]
        return {k: float(out[i]) for i, k in enumerate(keys)}

    def profile_read(self):
        ms = C.c_double()
        n = C.c_int64()
        b = C.c_int64()
        self._chk("mgnn_profile_read", self.L.mgnn_profile_read(self._h, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value


def estimate_rows_bound(ctx: "Context", fanouts: Sequence[int], batch: int, run_seed: int, pilot_steps=(1, 2),
                        slack: float = 1.25, stream=None) -> int:
    """A realistic arena bound for mgnn_sampler_config_bounded: the largest |F_L| of a pilot
    (one-step windows at `pilot_steps`, every hosted partition, static arenas for one step) times
    `slack`, rounded up to 1024 rows.  Sampling reads no buffer state, so the pilot changes nothing
    the run depends on; the caller reconfigures the sampler afterwards."""
    import torch
    ctx.sampler_config(fanouts, batch, run_seed, 1)
    u_max = 0
    for t in pilot_steps:
        ctx.sample(0, int(t), 1, stream=stream)
        w = ctx.window(0)
        hs = device_view(w.hop_size, (w.n_inst, _lib.MAX_LAYERS + 1), "i8")[:, w.n_layers]
        torch.cuda.synchronize()
        u_max = max(u_max, int(hs.max().item()))
    return int(-(-int(u_max * slack) // 1024) * 1024)


def alpha_default(gamma: float, delta: int) -> float:
    """Eq.1 threshold as the iterated fp32 product (computed by the library)."""
    return float(_lib.load().mgnn_alpha_default(gamma, delta))


def build_context(device: int, parts_in, feat_dim: int, feat_seed: int, hosted: Optional[Sequence[int]] = None,
                  dense: bool = False) -> Context:
    """Context hosting the partitions `hosted` (default: all) of a partitioned graph.
    dense: NEXT-1's dense S_A (every non-local node scorable)."""
    p0 = parts_in[0]
    ctx = Context(device, p0.bounds, feat_dim, feat_seed)
    if dense:
        ctx._chk("mgnn_ctx_set_dense_scores", ctx.L.mgnn_ctx_set_dense_scores(ctx._h, 1))
    for pi in parts_in:
        if hosted is None or pi.part_id in hosted:
            ctx.load_partition(pi.part_id, pi.indptr, pi.cols, pi.train_ids)
    return ctx


def exchange_tables(ctx: Context, group=None) -> None:
    """Multi-GPU: share every hosted table's CUDA IPC handle over torch.distributed
    and map all remote tables (miss / refill rows are then NVLink peer loads)."""
    import torch.distributed as dist
    mine = {pid: ctx.export_table(pid) for pid in ctx.parts}
    allh: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    for d in allh:
        for pid, h in d.items():
            if pid not in ctx.parts:
                ctx.import_table(pid, h)


def ddp_step(ctx: Context, slot: int, step_in_window: int, n_trainers: int, lr: float, stream=None,
             group=None) -> None:
    """One DDP training step (Alg.1 l.6-8): forward and backward
    of every local trainer's minibatch (library kernels), sum-all-reduce of the gradient buffer
    across ranks (NCCL through torch.distributed, on the same stream), then SGD."""
    import torch
    import torch.distributed as dist
    if isinstance(stream, int):        # a raw cudaStream_t: the all-reduce must be ordered on it too
        stream = torch.cuda.ExternalStream(stream)
    ctx.train_step(slot, step_in_window, n_trainers, stream)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        g = ctx.grads()
        if stream is not None:
            with torch.cuda.stream(stream):
                dist.all_reduce(g, group=group)
        else:                          # the current stream, which train_step / sgd also use
            dist.all_reduce(g, group=group)
    ctx.sgd(lr, stream)

