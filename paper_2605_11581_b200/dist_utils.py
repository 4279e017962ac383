"""Multi-GPU plumbing of the benchmark / serving harness (one process per GPU).

BASELINE.json configs[1] (Qwen2.5-1.5B, 2 KV heads) does not shard usefully:
N GPUs run N independent replicas ("replicas only"), so the data
path has no collective.  ``torch.distributed`` is used only to line the ranks
up (barrier) and to take the maximum of their device-side timings.
"""

from __future__ import annotations

import os

import torch


class RankGroup:
    """Thin wrapper over torch.distributed that also works for a single process."""

    def __init__(self, backend: str | None = None):
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            kw = {}
            if backend == "nccl":
                kw["device_id"] = torch.device("cuda", self.local_rank)
            dist.init_process_group(backend, rank=self.rank, world_size=self.world, **kw)
            self.dist = dist
            self.backend = backend

    def barrier(self) -> None:
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, values, device="cpu") -> list:
        """Element-wise maximum of a list of floats over all ranks."""
        t = torch.tensor(list(values), dtype=torch.float64, device=device)
        if self.dist is not None:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def aggregate_throughput(self, units_per_rank: float, seconds_local: float, device="cpu") -> float:
        """Whole-job throughput: units of ALL ranks / max-over-ranks time."""
        (t_max,) = self.max_over_ranks([seconds_local], device=device)
        return self.world * units_per_rank / t_max

    def close(self) -> None:
        if self.dist is not None:
            self.dist.destroy_process_group()
            self.dist = None
