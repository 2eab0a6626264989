"""Process/GPU placement of the m model-averaging workers and the
hierarchical average (parallel.cpp:26-59, 61-77, 163-181).

One process per GPU hosts a contiguous block of worker ranks (config 5 runs
4 virtual workers per GPU). For power-of-two counts the reference's
midpoint tree over [0, m) splits exactly at the process boundaries, so
"local subtree sum -> cross-process sum -> x 1/m" reproduces the reference's
summation grouping. The average itself runs on the device
(Averager, csrc/parallel.cu); this module holds the host-side placement plan.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import parnn as P


@dataclass(frozen=True)
class WorkerLayout:
    workers: int      # m
    world: int        # processes (= GPUs)
    rank: int         # this process
    rank0: int        # first global worker rank hosted here
    local: int        # workers hosted here

    @property
    def ranks(self) -> range:
        return range(self.rank0, self.rank0 + self.local)


def worker_layout(workers: int, world: int, rank: int) -> WorkerLayout:
    """Contiguous ranks per process: process p hosts [p*m/world, (p+1)*m/world)."""
    if workers < 1:
        raise P.ParnnError("train_parallel: workers must be >= 1")
    if world < 1 or not 0 <= rank < world:
        raise P.ParnnError(f"worker_layout: rank {rank} outside world {world}")
    if workers % world != 0:
        raise P.ParnnError(f"worker_layout: {workers} workers do not split evenly over {world} processes")
    local = workers // world
    return WorkerLayout(workers, world, rank, rank * local, local)


def shard_rows(n: int, layout: WorkerLayout, base_seed: int) -> np.ndarray:
    """Dataset row ids of every worker this process hosts (partition_data)."""
    return P.partition_rows(n, layout.workers, base_seed)[layout.rank0:layout.rank0 + layout.local]


def epoch_orders(shard_size: int, minibatch: int, layout: WorkerLayout, base_seed: int, epochs: int):
    """Per hosted worker, per epoch: shard positions in minibatch order.
    Worker r draws its epoch seeds from Rng(base_seed + r) (parallel.cpp:99,180)."""
    out = []
    for r in layout.ranks:
        seeds = P.rng_u64(base_seed + r, epochs)
        out.append([P.minibatch_rows(shard_size, minibatch, int(s)) for s in seeds])
    return out
