"""Multi-GPU plumbing of the benchmark / serving harness (one process per GPU).

BASELINE.json configs[1] (Qwen2.5-1.5B, 2 KV heads) does not shard usefully:
N GPUs run N independent replicas ("replicas only"), so the data
path has no collective.  ``torch.distributed`` is used only to line the ranks
up (barrier) and to take the maximum of their device-side timings.

Tensor parallelism (configs[3], Qwen3-8B) keeps the step a single launch per rank: the kernel stores its
partial rows straight into every peer's workspace over NVLink.  ``torch.distributed`` is used once, at
start-up, to exchange the CUDA IPC handles of the workspaces (``share_workspaces``).
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


def share_workspaces(group: RankGroup, workspace: torch.Tensor) -> list[torch.Tensor]:
    """Map every rank's workspace into this process (same node, NVLink / NVSwitch peers).

    Each rank exports its workspace allocation as a CUDA IPC handle (``UntypedStorage._share_cuda_``), the
    handles are all-gathered as Python objects, and every rank opens its peers' handles
    (``cudaIpcOpenMemHandle`` with lazy peer access).  Returns uint8 tensors in rank order, this rank's own
    tensor at index ``group.rank``; keep them alive as long as the plugin runs.  Exercised on hardware by
    tools/tp_two_process.py (tests/test_gpu_decode.py::test_tensor_parallel_across_processes_with_ipc_workspaces):
    two processes, IPC handles over gloo, in-kernel exchange across the two address spaces."""
    if group.world == 1:
        return [workspace]
    assert workspace.is_cuda and workspace.dtype == torch.uint8 and workspace.is_contiguous()
    storage = workspace.untyped_storage()
    handle = storage._share_cuda_()
    meta = (handle, workspace.storage_offset(), workspace.numel())
    metas: list = [None] * group.world
    group.dist.all_gather_object(metas, meta)
    out = []
    for r, (h, off, n) in enumerate(metas):
        if r == group.rank:
            out.append(workspace)
            continue
        st = torch.UntypedStorage._new_shared_cuda(*h)
        t = torch.empty(0, dtype=torch.uint8, device=torch.device("cuda", st.device.index))
        t.set_(st, off, (n,))
        out.append(t)
    group.barrier()
    return out
