"""Straight-line reference of the buffer policy, for pinning the oracle.

Written directly from PAPER.md Alg.1 INITIALIZE_PREFETCHER,
Alg.2 l.2-9, l.21, EVICT_AND_REPLACE l.25-34 and the swap
paragraph of §3.2, with python sets/dicts and full rescans --
no sorting networks, no index maps, no shared code with oracle/orc.c.
fp32 arithmetic is numpy.float32 (IEEE binary32, RN, denormals kept).
SPEC.md acceptance criterion 2 asks for exactly this comparison.
"""
from __future__ import annotations

import numpy as np

F32 = np.float32


class PolicyRef:
    def __init__(self, halo_ids, deg_in, f_bp, gamma, alpha, theta_r, delta):
        self.halo = [int(x) for x in halo_ids]
        self.deg = {int(h): int(d) for h, d in zip(halo_ids, deg_in)}
        self.gamma, self.alpha, self.theta_r, self.delta = F32(gamma), F32(alpha), F32(theta_r), int(delta)
        n_h = len(self.halo)
        cap = -(-(f_bp * n_h) // 10000)                  # ceil(f * |V_p^h|)
        ranked = sorted(self.halo, key=lambda n: (-self.deg[n], n))   # top-f by degree, ties by id
        self.slot = {}                                    # BUF: node -> slot
        self.se = {}                                      # S_E over BUF
        self.sa = {n: F32(0.0) for n in self.halo}        # S_A[m] = 0 for halo nodes not in BUF
        for s, n in enumerate(ranked[:cap]):
            self.slot[n] = s
            self.se[n] = F32(1.0)                         # S_E[n] = 1
            self.sa[n] = F32(-1.0)                        # S_A[n] = -1
        self.cap = cap

    def step(self, step: int, sampled_nodes):
        halo_s = {int(n) for n in sampled_nodes if int(n) in self.sa}       # V^{h|s}
        hits = {n for n in halo_s if n in self.slot}
        misses = halo_s - hits
        for n in list(self.slot):                         # decay unused buffer entries
            if n not in halo_s:
                self.se[n] = F32(self.se[n] * self.gamma)
        for n in misses:                                  # S_A += 1 per miss (every step)
            self.sa[n] = F32(self.sa[n] + F32(1.0))
        k = 0
        if self.delta > 0 and step % self.delta == 0:
            E = [n for n in self.slot if self.se[n] < self.alpha]
            E.sort(key=lambda n: (float(self.se[n]), n))
            R = [n for n in self.halo if n not in self.slot and self.sa[n] >= self.theta_r]
            R.sort(key=lambda n: (-float(self.sa[n]), -self.deg[n], n))
            k = min(len(E), len(R))
            for e, r in zip(E[:k], R[:k]):
                s = self.slot.pop(e)
                se_e = self.se.pop(e)
                sa_r = self.sa[r]
                self.sa[e] = se_e
                self.slot[r] = s
                self.se[r] = sa_r
                self.sa[r] = F32(-1.0)
        return len(hits), len(misses), k

    def arrays(self):
        """(node_of_slot, se per slot, sa in halo-id order) for comparison with the oracle."""
        node_of = np.full(self.cap, -1, np.int32)
        se = np.zeros(self.cap, np.float32)
        for n, s in self.slot.items():
            node_of[s] = n
            se[s] = self.se[n]
        sa = np.array([self.sa[n] for n in self.halo], dtype=np.float32)
        return node_of, se, sa
