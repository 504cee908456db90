"""One multi-layer decode step as a CUDA graph: host inputs in, host outputs out.

A decode step over ``DecodeKvCache`` is, per layer: copy that layer's q / k / v rows from
pinned host memory, run the fused attention (prepare -> split -> combine, with the new
token appended to the tail by the combine kernel), copy the output back.  Launching this
from Python costs ~10 us of host time per op, more than the GPU needs for a layer, so the
step is captured once and replayed:

- host-to-device copies run ahead on one side stream (layer groups of 1, 2, 4, ...: each group
  lands while the groups before it compute, whatever the box's PCIe rate -- groups of 1, 3
  and the rest stalled layer 4 on a box whose uploads ran at ~25 GB/s: 3.0 against 2.24 ms
  per C2 step) and device-to-host copies trail on another (groups of ..., 4, 2, 1 layers, so
  one layer's output is left after the last kernel).  The compute stream waits for an upload group before the group's first layer and
  records a download group after its last: every such cross-stream edge turns the programmatic
  launch edge into the next layer's prepare kernel into a full dependency.  One edge per layer
  measured 2.55 ms per C2 step against 2.34 ms grouped (`scripts/e2e_probe.py`, round robin);
- the kernels keep their programmatic dependent launch edges inside a group;
- the host keeps the cache's token counters in step (``DecodeKvCache._after_append``).

A replay that would seal a tail chunk (which re-plans the layer's segment table) is
refused; call ``recapture()`` after sealing steps run eagerly.  Every layer's plan
generation (``_Layer.gen``, bumped by a seal and by a re-plan) is recorded at capture:
a replay after any re-plan raises instead of replaying stale segment tables, and the
captured tables (``_Layer.keep``) are held by the graph so they outlive a re-plan.
"""

from __future__ import annotations

import torch

from .attention import DecodeKvCache
from .errors import ShapeMismatch


class _StepGraph:
    """A captured decode step over every layer of ``cache`` (``_body`` records one step)."""

    cache: DecodeKvCache

    def _body(self):
        raise NotImplementedError

    def _sealing_ahead(self) -> bool:
        return any(lay.tail_len + 1 >= self.cache.chunk_len for lay in self.cache._layers)

    def recapture(self):
        """(Re)build the graph: one eager step (it is a real decode step), then the capture."""
        self.cache._flush_seals()  # full tails of an eager sealing step are compressed first
        if self._sealing_ahead():
            raise ShapeMismatch("a tail chunk seals on the next token: run that step eagerly first")
        self._body()  # eager step: builds every layer's segment table outside the capture
        torch.cuda.synchronize()
        if self._sealing_ahead():
            raise ShapeMismatch("a tail chunk seals on the next token: run that step eagerly first")
        tails = [lay.tail_len for lay in self.cache._layers]
        self.gens = [lay.gen for lay in self.cache._layers]
        self.keep = [list(lay.keep) for lay in self.cache._layers]  # device tables the graph points at
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._body()
        for lay, t in zip(self.cache._layers, tails):  # the capture ran no device work
            lay.tail_len = t
        if [lay.gen for lay in self.cache._layers] != self.gens:
            raise ShapeMismatch("a layer was re-planned during the capture")

    def replay(self):
        """One decode step for every layer."""
        if self._sealing_ahead():
            raise ShapeMismatch("a tail chunk seals on this token: run the step eagerly, then recapture()")
        if [lay.gen for lay in self.cache._layers] != self.gens:
            raise ShapeMismatch("a layer was re-planned (sealed chunk) since the capture: recapture()")
        self.graph.replay()
        for layer in range(self.cache.layers):
            self.cache._after_append(layer)


class DeviceStepGraph(_StepGraph):
    """The decode step on device-resident q (layers, units, g, 128), k / v (layers, units, 128)
    and out (like q), captured once: every layer's prepare -> split -> combine (+ append) with
    the programmatic launch edges of the whole step in one graph."""

    def __init__(self, cache: DecodeKvCache, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor):
        self.cache, self.q, self.k, self.v, self.out = cache, q, k, v, out
        self.graph = None
        self.recapture()

    def _body(self):
        for layer in range(self.cache.layers):
            self.cache.attend(layer, self.q[layer], self.out[layer], append=(self.k[layer], self.v[layer]))


class DecodeStepGraph(_StepGraph):
    """Captured decode step for every layer of ``cache``.

    q_h: (layers, units, g, 128), k_h / v_h: (layers, units, 128), out_h like q_h: pinned
    host fp16 tensors the caller refills / reads between replays.
    """

    def __init__(self, cache: DecodeKvCache, q_h: torch.Tensor, k_h: torch.Tensor, v_h: torch.Tensor,
                 out_h: torch.Tensor, up_sizes=None, down_sizes=None):
        L, U, g, D = cache.layers, cache.units, cache.g, cache.dim
        if q_h.shape != (L, U, g, D) or out_h.shape != q_h.shape or k_h.shape != (L, U, D) or v_h.shape != (L, U, D):
            raise ShapeMismatch("host buffers must be q/out (layers, units, g, 128) and k/v (layers, units, 128)")
        for t in (q_h, k_h, v_h, out_h):
            if t.dtype != torch.float16 or not t.is_pinned():
                raise ShapeMismatch("host buffers must be pinned fp16")
        self.cache = cache
        self.q_h, self.k_h, self.v_h, self.out_h = q_h, k_h, v_h, out_h
        dev = cache.device
        self.q_d = torch.empty(q_h.shape, dtype=torch.float16, device=dev)
        self.k_d = torch.empty(k_h.shape, dtype=torch.float16, device=dev)
        self.v_d = torch.empty(v_h.shape, dtype=torch.float16, device=dev)
        self.o_d = torch.empty(q_h.shape, dtype=torch.float16, device=dev)
        self.up = torch.cuda.Stream(device=dev)    # host -> device, runs ahead
        self.down = torch.cuda.Stream(device=dev)  # device -> host, trails the layers
        if up_sizes is None:  # 1, 2, 4, ... layers: each group lands while the groups before it compute
            up_sizes, n, left = [], 1, L
            while left > 0:
                up_sizes.append(min(n, left))
                left -= n
                n *= 2
        self.up_groups = self._groups(L, up_sizes)
        if down_sizes is None:  # ..., 4, 2, 1 layers: the outputs left after the last layer are one layer's
            down_sizes, n, left = [], 1, L
            while left > 0:
                down_sizes.insert(0, min(n, left))
                left -= n
                n *= 2
        self.down_groups = self._groups(L, down_sizes)
        self.h2d = [torch.cuda.Event() for _ in self.up_groups]
        self.done = [torch.cuda.Event() for _ in self.down_groups]
        self.graph = None
        self.recapture()

    def _body(self):
        cache, L = self.cache, self.cache.layers
        compute = torch.cuda.current_stream()
        self.up.wait_stream(compute)
        self.down.wait_stream(compute)
        with torch.cuda.stream(self.up):
            for gi, (a, b) in enumerate(self.up_groups):
                self.q_d[a:b].copy_(self.q_h[a:b], non_blocking=True)
                self.k_d[a:b].copy_(self.k_h[a:b], non_blocking=True)
                self.v_d[a:b].copy_(self.v_h[a:b], non_blocking=True)
                self.h2d[gi].record(self.up)
        starts = {a: gi for gi, (a, _) in enumerate(self.up_groups)}
        ends = {b - 1: gi for gi, (_, b) in enumerate(self.down_groups)}
        for layer in range(L):
            if layer in starts:
                compute.wait_event(self.h2d[starts[layer]])
            cache.attend(layer, self.q_d[layer], self.o_d[layer], append=(self.k_d[layer], self.v_d[layer]))
            if layer in ends:
                gi = ends[layer]
                a, b = self.down_groups[gi]
                self.done[gi].record(compute)
                with torch.cuda.stream(self.down):
                    self.down.wait_event(self.done[gi])
                    self.out_h[a:b].copy_(self.o_d[a:b], non_blocking=True)
        compute.wait_stream(self.up)
        compute.wait_stream(self.down)

    @staticmethod
    def _groups(L: int, sizes) -> list[tuple[int, int]]:
        """Layer groups [start, stop) of the given sizes, the rest of the layers in one more."""
        out, start = [], 0
        for n in sizes:
            if start >= L:
                break
            out.append((start, min(L, start + n)))
            start += n
        if start < L:
            out.append((start, L))
        return out
