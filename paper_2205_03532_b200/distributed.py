"""Environment sharding across GPUs.

Envs never interact, so each rank owns a contiguous env block, holds its own
replica of the (small, immutable) SDF and mesh assets, and runs collide on its
shard with no data-path communication. The only collective is one all-gather
of the per-env stats [n_cand, n_patch, n_kept, max_penetration] (16 B/env), the
batched counterpart of StepReport.contacts_before / contacts_after / patches /
max_penetration (dynamics/scene.py:28-37,155-161).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .scenes import shard_range


def env_shard(n_envs: int, rank: int | None = None, world: int | None = None) -> tuple[int, int]:
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    return shard_range(n_envs, rank, world)


def gather_env_stats(local_stats: torch.Tensor, n_envs: int, group=None) -> torch.Tensor:
    """All-gather per-env stats (E_local, 4) float32 into (n_envs, 4) on every rank.

    Shards may differ by one env; they are padded to the largest shard for the
    collective and trimmed after (one all_gather_into_tensor call)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return local_stats
    sizes = [shard_range(n_envs, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((width, local_stats.shape[1]), dtype=local_stats.dtype, device=local_stats.device)
    pad[: local_stats.shape[0]] = local_stats
    out = torch.empty((world * width, local_stats.shape[1]), dtype=local_stats.dtype, device=local_stats.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    return torch.cat(parts, dim=0)


class StatsGather:
    """The per-step stats all-gather with its buffers allocated once (the step loop
    allocates nothing) and, on CUDA, issued on a side stream so it stays off the
    collide's critical path: `launch(stats, after=stream)` makes the side stream wait
    for the step (an event), copies the local stats into the padded send buffer and
    all-gathers into a persistent (world * width, 4) buffer; `wait(stream)` orders a
    consumer after it; `result()` is the (n_envs, 4) view in env order."""

    def __init__(self, n_envs: int, cols: int = 4, device=None, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.n_envs = n_envs
        self.sizes = [shard_range(n_envs, r, self.world) for r in range(self.world)]
        self.width = max(hi - lo for lo, hi in self.sizes)
        dev = torch.device(device) if device is not None else torch.device("cpu")
        self.send = torch.zeros((self.width, cols), dtype=torch.float32, device=dev)
        self.out = torch.zeros((self.world * self.width, cols), dtype=torch.float32, device=dev)
        contiguous = all(hi - lo == self.width for lo, hi in self.sizes)
        self._view = self.out if contiguous else None
        self.side = torch.cuda.Stream(device=dev) if dev.type == "cuda" else None
        self._done = None

    def launch(self, local_stats: torch.Tensor, after=None) -> None:
        if self.side is not None:
            ev = torch.cuda.Event()
            ev.record(after if after is not None else torch.cuda.current_stream(self.send.device))
            self.side.wait_event(ev)
            ctx = torch.cuda.stream(self.side)
        else:
            import contextlib

            ctx = contextlib.nullcontext()
        with ctx:
            self.send[: local_stats.shape[0]].copy_(local_stats, non_blocking=True)
            if self.world > 1:
                dist.all_gather_into_tensor(self.out, self.send, group=self.group)
            else:
                self.out[: local_stats.shape[0]].copy_(self.send[: local_stats.shape[0]])
            if self.side is not None:
                self._done = torch.cuda.Event()
                self._done.record(self.side)

    def wait(self, stream=None) -> None:
        if self._done is not None:
            (stream if stream is not None else torch.cuda.current_stream(self.send.device)).wait_event(self._done)

    def result(self) -> torch.Tensor:
        if self._view is not None:
            return self._view[: self.n_envs]
        return torch.cat([self.out[r * self.width: r * self.width + (hi - lo)] for r, (lo, hi) in
                          enumerate(self.sizes)], dim=0)


def step_report(stats: torch.Tensor) -> dict:
    """Scene-level totals from gathered stats (StepReport fields, scene.py:155-161)."""
    s = stats.double()
    return {
        "contacts_before": int(s[:, 0].sum().item()),
        "patches": int(s[:, 1].sum().item()),
        "contacts_after": int(s[:, 2].sum().item()),
        "max_penetration": float(s[:, 3].max().item()) if len(s) else 0.0,
    }
