"""Multi-step generation driver on the device.

Mirrors the reference's ``run_generation`` (harness.cpp:123-224) and
``resolve_schedule`` (schedule.cpp:44-87): the latent is voxel-ordered once, every
step runs the block stack densely or sparsely (or is skipped inside the step-cache
window, reusing the previous model output), the latent advances by
``x += (1/T) * model_output`` (harness.cpp:200), and the final latent is decoded
back to grid order.  Per-step latent R^2 against the dense-baseline trajectory
(harness.cpp:154-163, metrics.cpp:5-30) is computed on the device.

Device residency: the fp32 master latent, its bf16 shadow (PROD block input), the
layer outputs and the block caches stay in HBM for the whole run; in PROD each step
kind (dense / sparse / skipped) is one CUDA graph replay.  Nothing here computes on
the CPU except the schedule (a few integers).

Cache offload (``offload=True``, memory.cpp:33-58 "optimized double-buffers two layers while
the rest live off-device"): every layer's persistent caches are one arena
(csd_block_bind_cache_arena); two device arenas serve the whole stack (layer l uses slot
l % 2) and the others live in pinned host memory.  While layer l computes, the previous user
of the other slot is copied out on one copy stream and the next layer's arena copied in on
another, so the device holds 2 / L of the caches (plus one layer's per-step scratch each).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import List, Optional

import torch

from . import _capi as capi
from . import ops
from .errors import raise_for

DENSE, SPARSE, SKIPPED = 0, 1, 2
MODE_NAMES = {DENSE: "dense", SPARSE: "sparse", SKIPPED: "skipped"}  # schedule.cpp:9-16


@dataclass
class ScheduleParams:
    """harness.hpp:19-25"""
    total_steps: int = 20
    dense_interval: int = 10
    step_cache: bool = False
    window: int = 0
    stride: int = 1


def resolve_schedule(total_steps: int, dense_interval: int, use_step_cache: bool = False,
                     window: int = 0, stride: int = 1) -> List[int]:
    """schedule.cpp:44-87 through csd_resolve_schedule: per-step DENSE / SPARSE / SKIPPED.

    Raises ConfigError for the reference's ConfigError cases."""
    lib = capi.lib()
    modes = (C.c_int32 * max(int(total_steps), 1))()
    raise_for(lib, lib.csd_resolve_schedule(total_steps, dense_interval, int(bool(use_step_cache)), window, stride, modes))
    return [int(m) for m in modes[:total_steps]]


def latent_axpy(latent: torch.Tensor, a: float, y: torch.Tensor,
                shadow: Optional[torch.Tensor] = None) -> None:
    """latent += a * y in place (harness.cpp:24-30); fp32 latent, y fp32 (CHECK) or bf16 (PROD)."""
    if latent.dtype != torch.float32:
        raise TypeError("the latent is an fp32 master tensor")
    mode = capi.MODE_PROD if y.dtype == torch.bfloat16 else capi.MODE_CHECK
    lib = ops.context().lib
    raise_for(lib, lib.csd_latent_axpy(ops.context().h, mode, ops._ptr(latent), float(a), ops._ptr(y),
                      latent.numel(), ops._ptr(shadow), ops._stream()))


def r_squared(truth: torch.Tensor, approx: torch.Tensor,
              origin: Optional[torch.Tensor] = None) -> float:
    """R^2 of (truth - origin) vs (approx - origin) (metrics.cpp:5-30), device reduction."""
    if truth.shape != approx.shape or (origin is not None and origin.shape != truth.shape):
        from .errors import ShapeError
        raise ShapeError(f"r_squared shapes disagree: {list(truth.shape)} vs {list(approx.shape)}")
    lib = ops.context().lib
    out = C.c_double(0.0)
    raise_for(lib, lib.csd_r_squared(ops.context().h, ops._ptr(truth), ops._ptr(approx), ops._ptr(origin),
                      truth.numel(), C.byref(out), ops._stream()))
    return out.value


@dataclass
class StepReport:
    """harness.hpp:37-43 (latent R^2 only; the per-layer probes are host instrumentation)."""
    step: int
    mode: int
    latent_r2: Optional[float] = None


@dataclass
class RunReport:
    modes: List[int]
    steps: List[StepReport] = field(default_factory=list)
    end_to_end_r2: Optional[float] = None
    final_latent: Optional[torch.Tensor] = None  # decoded grid order [B, T, H, W, D], fp32
    device_ms: float = 0.0                       # the step loop, CUDA events
    wall_ms: float = 0.0


class Generation:
    """run_generation (harness.cpp:123-224, RunMode::SparseDelta) over a stack of Blocks.

    ``layers``: the model's blocks in order (ops.Block, all CHECK or all PROD).  ``baseline``:
    an independent stack with the same weights for the dense trajectory the R^2 figures are
    measured against (model_forward_dense per step); None skips the R^2 report."""

    def __init__(self, layers: List[ops.Block], layout: ops.VoxelLayout,
                 baseline: Optional[List[ops.Block]] = None, use_graphs: Optional[bool] = None,
                 offload: bool = False):
        if not layers:
            raise ValueError("a generation needs at least one layer")
        self.layers = layers
        self.baseline = baseline
        self.layout = layout
        self.prod = layers[0].mode == capi.MODE_PROD
        if any((blk.mode == capi.MODE_PROD) != self.prod for blk in layers):
            raise ValueError("all layers must run in the same mode")
        self.use_graphs = self.prod if use_graphs is None else bool(use_graphs)
        if self.use_graphs and not self.prod:
            # CHECK mode double-buffers the softmax stats on the host side (block.cpp): a
            # captured dense step would bake one buffer index and replay stale stats
            raise ValueError("CUDA graphs are PROD-only; CHECK generations run eagerly")
        c = layers[0].cfg
        self.shape = (c.batch, c.seq, c.dim)
        dt = torch.bfloat16 if self.prod else torch.float32
        dev = torch.device("cuda")
        self.latent = torch.empty(self.shape, dtype=torch.float32, device=dev)
        self.shadow = torch.empty(self.shape, dtype=torch.bfloat16, device=dev) if self.prod else None
        self.outs = [torch.empty(self.shape, dtype=dt, device=dev) for _ in layers]
        self._graphs = {}
        self.offload = bool(offload) and len(layers) > 2
        if self.offload:
            nbytes = max(blk.cache_arena()[1] for blk in layers)
            self._slots = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
            self._host = []
            for l, blk in enumerate(layers):
                blk.bind_cache_arena(self._slots[l % 2])
                self._host.append(torch.zeros(nbytes, dtype=torch.uint8, pin_memory=True))
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
            self._ready = [None] * len(layers)  # H2D of layer l's arena into its slot done
            self.arena_bytes = nbytes

    def memory_report(self) -> dict:
        """Cache bytes on the device, resident vs offloaded (memory.cpp:47-53 act_naive /
        act_resident, here measured from the arenas)."""
        n = max(blk.cache_arena()[1] for blk in self.layers)
        resident = (2 if self.offload else len(self.layers)) * n
        return {"arena_bytes_per_layer": n, "layers": len(self.layers),
                "cache_naive_bytes": len(self.layers) * n, "cache_device_bytes": resident,
                "cache_host_bytes": len(self.layers) * n if self.offload else 0}

    def _next_user(self, l: int) -> int:
        """The layer that uses slot l % 2 next after layer l (the stack repeats every step)."""
        L = len(self.layers)
        for k in range(1, L + 1):
            m = (l + k) % L
            if m % 2 == l % 2:
                return m
        return l

    def _prefetch(self, l: int, after=None):
        """H2D of layer l's arena into its slot on the copy stream (after `after`)."""
        with torch.cuda.stream(self._h2d):
            if after is not None:
                self._h2d.wait_event(after)
            self._slots[l % 2].copy_(self._host[l], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._h2d)
            self._ready[l] = ev

    def _input(self):
        return self.shadow if self.prod else self.latent

    def _forward(self, dense: bool):
        cur = self._input()
        if not self.offload:
            for blk, out in zip(self.layers, self.outs):
                blk.step(cur, dense, out=out)
                cur = out
            return
        stream = torch.cuda.current_stream()
        L = len(self.layers)
        # the first two layers' arenas come in before the stack starts (a step's last copies
        # are joined below, so every step -- and every captured graph -- is self-contained)
        for l in range(min(2, L)):
            self._prefetch(l, after=self._mark(stream))
        for l, (blk, out) in enumerate(zip(self.layers, self.outs)):
            stream.wait_event(self._ready[l])
            blk.step(cur, dense, out=out)
            cur = out
            done = self._mark(stream)
            with torch.cuda.stream(self._d2h):  # this layer's caches back to host memory
                self._d2h.wait_event(done)
                self._host[l].copy_(self._slots[l % 2], non_blocking=True)
                saved = torch.cuda.Event()
                saved.record(self._d2h)
            n = self._next_user(l)
            if n > l:  # a later layer of this step reuses the slot
                self._prefetch(n, after=saved)
        stream.wait_stream(self._d2h)
        stream.wait_stream(self._h2d)

    @staticmethod
    def _mark(stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev

    def _step(self, mode: int, scale: float):
        if mode != SKIPPED:
            self._forward(mode == DENSE)
        latent_axpy(self.latent, scale, self.outs[-1], self.shadow)

    def _graph(self, mode: int, scale: float):
        key = (mode, scale)
        g = self._graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._step(mode, scale)
            self._graphs[key] = g
        return g

    def _dense_trajectory(self, x0: torch.Tensor, total: int, scale: float) -> List[torch.Tensor]:
        """harness.cpp:154-163: latent_b += scale * model_forward_dense(latent_b) per step."""
        lat = x0.clone()
        dt = torch.bfloat16 if self.prod else torch.float32
        shadow = lat.to(dt)
        outs = [torch.empty(self.shape, dtype=dt, device=lat.device) for _ in self.baseline]
        traj = []
        for _ in range(total):
            cur = shadow if self.prod else lat
            for blk, out in zip(self.baseline, outs):
                blk.forward_dense(cur, out=out)  # model_forward_dense: exact attention + MLP
                cur = out
            latent_axpy(lat, scale, outs[-1], shadow if self.prod else None)
            traj.append(lat.clone())
        return traj

    def prepare(self, scale: float):
        """PROD: run each step kind once eagerly (workspaces, tensor maps, cuBLAS plans), then
        record one CUDA graph per kind.  The block caches this touches are rebuilt by the
        run's first step, which is always dense (schedule.cpp:21-41); run() starts the
        warm-up from the run's own x0 so the stale softmax stats equal fresh ones."""
        for mode in (DENSE, SPARSE, SKIPPED):
            self._step(mode, scale)
        torch.cuda.synchronize()
        for mode in (DENSE, SPARSE, SKIPPED):
            self._graph(mode, scale)

    def run(self, grid0: torch.Tensor, schedule: ScheduleParams) -> RunReport:
        """grid0: seeded latent [B, T, H, W, D] fp32 (harness.cpp:16-22) on the device."""
        import numpy as np
        modes = resolve_schedule(schedule.total_steps, schedule.dense_interval, schedule.step_cache,
                                 schedule.window, schedule.stride)
        total = len(modes)
        scale = float(np.float32(1.0) / np.float32(total))  # harness.cpp:149, fp32 division
        x0, _ = ops.voxel_order(grid0.to(torch.float32).contiguous(), self.layout)
        for blk in self.layers + (self.baseline or []):  # fresh ModelStates (harness.cpp:180)
            blk.reset()
        base = self._dense_trajectory(x0, total, scale) if self.baseline else None

        def reset():
            self.latent.copy_(x0)
            if self.prod:
                self.shadow.copy_(x0.to(torch.bfloat16))
        if self.use_graphs:
            # warm-up from x0 itself: its dense step leaves exactly the softmax stats the
            # reference's first dense step computes fresh (attention.cpp:122-137), which the
            # captured dense step then reads as its "previous" stats
            reset()
            self.prepare(scale)
        reset()
        snaps = [torch.empty_like(self.latent) for _ in modes] if base is not None else None
        rep = RunReport(modes=modes)
        stream = torch.cuda.current_stream()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record(stream)
        have_output = False
        for s, mode in enumerate(modes):
            if mode == SKIPPED and not have_output:
                from .errors import StateError
                raise StateError(f"skipped step {s} has no previous model output to reuse")
            if self.use_graphs:
                self._graphs[(mode, scale)].replay()
            else:
                self._step(mode, scale)
            have_output = have_output or mode != SKIPPED
            if snaps is not None:
                snaps[s].copy_(self.latent, non_blocking=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        rep.device_ms = ev0.elapsed_time(ev1)
        rep.wall_ms = (time.perf_counter() - t0) * 1e3
        from .errors import NumericError
        for s, mode in enumerate(modes):
            r2 = None
            if base is not None:
                try:
                    r2 = r_squared(base[s], snaps[s], x0)
                except NumericError:  # zero-variance true delta: the reference reports nothing
                    r2 = None
            rep.steps.append(StepReport(step=s, mode=mode, latent_r2=r2))
        if base is not None:
            try:
                rep.end_to_end_r2 = r_squared(base[-1], self.latent, x0)
            except NumericError:
                rep.end_to_end_r2 = None
        rep.final_latent = ops.reverse_voxel_order(self.latent, self.layout)
        return rep
