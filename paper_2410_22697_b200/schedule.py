"""The prepare-ahead schedule of the halo feature pipeline on two CUDA streams.

PAPER.md Alg.1 l.5-9 overlaps PREPARE_NEXT_MINIBATCH with the
training of the current one, with a queue depth of one.  Here the unit
is a WINDOW of steps and the overlap is between the two halves
of the path that do not share state:

  stream A : mgnn_sample of window w+1 (partition-local sampling reads no
             buffer state, R#1),
  stream B : mgnn_lookup_gather + mgnn_score_evict_refill of window w
             (classification, gather, tally, decay, eviction round).

One `iteration()` is one bench step: (optional L2 flush) -> start event on B ->
A waits for it -> sample(w+1) on A || consume(w) on B -> B joins A -> end event.
A window slot is resampled only after the window it held was consumed (event
ev_done).  This module is product code: bench.py times exactly this loop, and the
GPU test suite (tests/test_gpu_schedule.py) drives exactly this loop in its parity check.
Argument marshalling and stream/event plumbing only -- every step of the path
runs in libmgnn.so's kernels.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch


class PrepareAhead:
    """Two-stream window pipeline over one mgnn context (all its hosted partitions)."""

    def __init__(self, ctx, window: int, t0: int = 1, stream_b: Optional[torch.cuda.Stream] = None,
                 flush_bytes: int = 256 << 20,
                 host_seeds: Optional[Callable[[int, int], Tuple[int, int]]] = None, serial: bool = False,
                 relabel_stream: bool = False, relabel_after_gather: bool = False, score_after_sample: bool = False,
                 sampling_priority: int = 0, score_priority: Optional[int] = None):
        """window: steps per window (a window may end on an eviction step, never contain one earlier);
        t0: first global step (1-based, R#8); flush_bytes: L2 flush buffer written before every
        iteration (0 = none; B200 L2 is 126 MB); host_seeds(slot, t) -> (seeds_ptr, counts_ptr) of
        pinned host buffers makes mgnn_sample copy the window's seeds host -> device (the e2e path);
        serial=True runs everything on stream B: consume(w), then sample(w+1) (no overlap);
        relabel_stream=True defers the columns' relabelling (mgnn_sampler_defer_relabel): window w's
        k_relabel runs on a third stream C beside its gather (L2-bound beside HBM-bound) and stream B
        joins C before the iteration ends, so the window's blocks are final when its end event fires;
        relabel_after_gather=True starts that relabel only when window w's gather is done, i.e. beside its
        scoring / eviction round (both latency-bound) instead of beside the HBM-bound gather."""
        self.ctx = ctx
        self.W = int(window)
        self.t = int(t0)
        self.slot = 0
        self.sB = stream_b if stream_b is not None else torch.cuda.current_stream()
        self.serial = serial
        self.sA = self.sB if serial else torch.cuda.Stream(device=self.sB.device, priority=sampling_priority)
        self.ev_sampled = [torch.cuda.Event(), torch.cuda.Event()]
        self.ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        self.flush = torch.empty(flush_bytes, dtype=torch.uint8, device=self.sB.device) if flush_bytes else None
        self.host_seeds = host_seeds
        self.primed = False
        self.relabel_stream = relabel_stream and not serial
        # the relabel stream takes stream B's priority: both carry window w, which the iteration waits for;
        # stream A (the next window's sampling) has the slack
        self.sC = (torch.cuda.Stream(device=self.sB.device, priority=self.sB.priority) if self.relabel_stream
                   else None)
        self.ev_relabeled = [torch.cuda.Event(), torch.cuda.Event()]
        self.relabel_after_gather = relabel_after_gather and self.relabel_stream
        self.ev_gathered = [torch.cuda.Event(), torch.cuda.Event()]
        self.score_after_sample = score_after_sample and not serial
        # score_priority: the eviction round of window w on its own stream D at this priority (a chain of
        # short latency-bound launches that would otherwise queue behind the next window's sampling)
        self.sD = (torch.cuda.Stream(device=self.sB.device, priority=score_priority)
                   if score_priority is not None and not serial else None)
        self.ev_gdone = [torch.cuda.Event(), torch.cuda.Event()]
        self.ev_sdone = [torch.cuda.Event(), torch.cuda.Event()]
        self._next_sampled = False
        ctx.defer_relabel(self.relabel_stream)

    # ---------------------------------------------------------------- the two halves
    def _sample(self, sl: int, tt: int) -> None:
        self.sA.wait_event(self.ev_done[sl])          # slot free once its previous window was consumed
        if self.relabel_stream:
            self.sA.wait_event(self.ev_relabeled[sl])
        if self.host_seeds is None:
            self.ctx.sample(sl, tt, self.W, stream=self.sA)
        else:
            sp, cp = self.host_seeds(sl, tt)
            self.ctx.sample_ptr(sl, tt, self.W, sp, cp, True, self.sA)
        self.ev_sampled[sl].record(self.sA)

    def _consume(self, sl: int) -> None:
        self.sB.wait_event(self.ev_sampled[sl])
        self.ctx.lookup_gather(sl, self.sB)
        if self.relabel_after_gather:
            self.ev_gathered[sl].record(self.sB)
            self.sC.wait_event(self.ev_gathered[sl])
            self._relabel(sl)
        if self.score_after_sample and self._next_sampled:
            self.sB.wait_event(self.ev_sampled[sl ^ 1])   # the eviction round after the next window's sampling
        if self.sD is not None:
            self.ev_gdone[sl].record(self.sB)
            self.sD.wait_event(self.ev_gdone[sl])
            self.ctx.score(sl, self.sD)
            self.ev_sdone[sl].record(self.sD)
            self.sB.wait_event(self.ev_sdone[sl])
        else:
            self.ctx.score(sl, self.sB)
        self.ev_done[sl].record(self.sB)

    def _relabel(self, sl: int) -> None:
        self.sC.wait_event(self.ev_sampled[sl])
        self.ctx.relabel(sl, self.sC)
        self.ev_relabeled[sl].record(self.sC)

    # ---------------------------------------------------------------- public
    def prime(self) -> None:
        """Sample the first window (before the first iteration)."""
        if not self.primed:
            self._sample(self.slot, self.t)
            self.primed = True

    def iteration(self, events: Optional[Tuple[torch.cuda.Event, torch.cuda.Event]] = None,
                  after_consume: Optional[Callable[[int, int, torch.cuda.Stream], None]] = None,
                  prepare_next: bool = True) -> Tuple[int, int]:
        """One bench step.  `events` (start, end) bracket the iteration on stream B (the flush is
        outside them).  after_consume(slot, t0, stream_b) is called after the window is consumed and
        before the join (it may enqueue work on stream B that reads the window).  prepare_next=False
        skips sampling the next window (the last iteration of a run).  Returns (slot, t0) of the
        consumed window; its outputs stay valid until that slot is sampled again, i.e. until the
        end of the next iteration."""
        self.prime()
        sA, sB = self.sA, self.sB
        if self.flush is not None:
            with torch.cuda.stream(sB):
                self.flush.zero_()
        if events is not None:
            events[0].record(sB)
        ev_go = torch.cuda.Event()
        ev_go.record(sB)
        sA.wait_event(ev_go)
        if self.serial:
            self._consume(self.slot)
            if prepare_next:
                self._sample(self.slot ^ 1, self.t + self.W)
        else:
            self._next_sampled = prepare_next
            if prepare_next:
                self._sample(self.slot ^ 1, self.t + self.W)  # window w+1: sampling stream
            if self.relabel_stream and not self.relabel_after_gather:
                self._relabel(self.slot)                      # window w's blocks: third stream
            self._consume(self.slot)                          # window w: buffer stream
            if self.relabel_stream:
                sB.wait_event(self.ev_relabeled[self.slot])
        consumed = (self.slot, self.t)
        if after_consume is not None:
            after_consume(self.slot, self.t, sB)
        sB.wait_stream(sA)
        if events is not None:
            events[1].record(sB)
        self.t += self.W
        self.slot ^= 1
        if not prepare_next:
            self.primed = False
        return consumed
