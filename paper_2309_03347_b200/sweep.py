"""ALS double sweep over a TT (BASELINE.json configs[4]):
for k = 1..d-1 (left-to-right) als_local_apply + left interface update, then
for k = d..2 (right-to-left) als_local_apply + right interface update — the
K7 + K8 skeleton of an AMEn sweep without the local solve.  Every contraction
is a libtt C-ABI call (DMMA GEMM chains); this module only sequences them."""
from __future__ import annotations

import numpy as np
import torch

from .tt import TTVec, als_local_apply, als_update_interfaces, tt_normalize


class SweepProblem:
    def __init__(self, A_cores, X_cores, device="cuda"):
        self.d = len(X_cores)
        self.n = [c.shape[1] for c in X_cores]
        self.r = [c.shape[0] for c in X_cores] + [1]
        self.R = [c.shape[0] for c in A_cores] + [1]
        dev = torch.device(device)
        f = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a).reshape(-1, order="F"))).to(dev)
        self.X = [f(c) for c in X_cores]
        self.A = [f(c) for c in A_cores]
        # interfaces at every bond (left Phi and right Psi), [r, R, r]
        self.Phi = [torch.zeros(self.r[k] * self.R[k] * self.r[k], dtype=torch.float64, device=dev)
                    for k in range(self.d + 1)]
        self.Psi = [torch.zeros(self.r[k] * self.R[k] * self.r[k], dtype=torch.float64, device=dev)
                    for k in range(self.d + 1)]
        self.Phi[0].fill_(1.0)
        self.Psi[self.d].fill_(1.0)
        mx = max(self.r[k] * self.n[k] * self.r[k + 1] for k in range(self.d))
        self.y = torch.zeros(mx, dtype=torch.float64, device=dev)

    def dims_apply(self, k):
        r0, r1, n = self.r[k], self.r[k + 1], self.n[k]
        return (r0, self.R[k], r0, n, n, r1, self.R[k + 1], r1)

    def build_right(self, normalize=True):
        """Untimed setup: right interfaces Psi_k for k = d-1..1 (Z25: normalised)."""
        for k in range(self.d - 1, 0, -1):
            als_update_interfaces(-1, self.dims_apply(k), self.Psi[k + 1], self.X[k], self.A[k], self.X[k],
                                  self.Psi[k])
            if normalize:   # Z25, by libtt (the interface viewed as a one-core TT-vector)
                v = TTVec([self.Psi[k].numel()], [1, 1], self.X[0].device)
                v.data = self.Psi[k]
                v._c.data = self.Psi[k].data_ptr()
                tt_normalize(v)

    def double_sweep(self, two_streams=False):
        if two_streams:
            return self._double_sweep_2s()
        for k in range(self.d - 1):
            als_local_apply(self.dims_apply(k), self.Phi[k], self.A[k], self.Psi[k + 1], self.X[k], self.y)
            als_update_interfaces(+1, self.dims_apply(k), self.Phi[k], self.X[k], self.A[k], self.X[k],
                                  self.Phi[k + 1])
        for k in range(self.d - 1, 0, -1):
            als_local_apply(self.dims_apply(k), self.Phi[k], self.A[k], self.Psi[k + 1], self.X[k], self.y)
            als_update_interfaces(-1, self.dims_apply(k), self.Psi[k + 1], self.X[k], self.A[k], self.X[k],
                                  self.Psi[k])

    def _double_sweep_2s(self):
        """The same double sweep with the local applies off the critical path: the
        interface updates (the dependent chain Phi_k -> Phi_{k+1}) stay on the
        current stream, each apply runs on a side stream as soon as the interface
        it reads is complete (an event per core), with its own workspace; the
        side stream joins at the end (graph-capturable fork/join)."""
        from . import _lib
        main = torch.cuda.current_stream()
        if getattr(self, "side", None) is None:
            need = max(_lib.lib().als_workspace(*self.dims_apply(k)) for k in range(self.d))
            self.side = torch.cuda.Stream(device=self.X[0].device)
            self.ws_side = torch.empty(need, dtype=torch.uint8, device=self.X[0].device)
            self.ws_main = torch.empty(need, dtype=torch.uint8, device=self.X[0].device)
        side = self.side

        def apply_async(k):
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            with torch.cuda.stream(side):
                als_local_apply(self.dims_apply(k), self.Phi[k], self.A[k], self.Psi[k + 1], self.X[k], self.y,
                                stream=side, ws=self.ws_side)

        for k in range(self.d - 1):
            apply_async(k)
            als_update_interfaces(+1, self.dims_apply(k), self.Phi[k], self.X[k], self.A[k], self.X[k],
                                  self.Phi[k + 1], stream=main, ws=self.ws_main)
        for k in range(self.d - 1, 0, -1):
            apply_async(k)
            als_update_interfaces(-1, self.dims_apply(k), self.Psi[k + 1], self.X[k], self.A[k], self.X[k],
                                  self.Psi[k], stream=main, ws=self.ws_main)
        main.wait_stream(side)

    def capture(self, two_streams=True):
        """Record one double sweep into a CUDA graph (the sequence of libtt launches
        is fixed for fixed shapes); replay with self.graph.replay()."""
        from .tt import workspace
        from . import _lib
        need = max(_lib.lib().als_workspace(*self.dims_apply(k)) for k in range(self.d))
        workspace(need, self.X[0].device)          # allocate before capture
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.double_sweep(two_streams)         # warm (cudaFuncSetAttribute etc.)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.double_sweep(two_streams)
        return self.graph

    def flops(self):
        """Algorithmic flops of one double sweep."""
        tot = 0
        visits = list(range(self.d - 1)) + list(range(self.d - 1, 0, -1))
        for k in visits:
            rA, R, rB, m, n, rAp, Rp, rBp = self.dims_apply(k)
            apply = 2 * (n * rB * rBp * rAp * Rp + m * n * rB * rAp * R * Rp + m * rA * rAp * rB * R)
            upd = 2 * (m * rA * rB * rAp * R + m * n * rB * rAp * R * Rp + n * rB * rBp * rAp * Rp)
            tot += apply + upd
        return tot
