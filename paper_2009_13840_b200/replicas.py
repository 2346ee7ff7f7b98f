"""Multi-GPU plumbing for bench.py: independent replicas, one process per GPU.

The 2-D solver path does not shard ("replicas only"): every
rank solves its own copy of the system and the only collectives are the
timing barrier and the max-over-ranks of the step time. Backend "nccl" on
GPUs, "gloo" for the CPU tests (tests/test_replicas.py).
"""
from __future__ import annotations

import os


def dist_env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Replicas:
    def __init__(self, backend: str = "nccl"):
        self.ws, self.rank, self.local = dist_env()
        self.backend = backend
        if self.ws > 1:
            import torch
            import torch.distributed as dist

            if not dist.is_initialized():
                if backend == "nccl":
                    torch.cuda.set_device(self.local)
                    dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
                else:
                    dist.init_process_group(backend)

    def barrier(self):
        if self.ws > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        """Max of a per-rank device time (the job's step time)."""
        if self.ws == 1:
            return x
        import torch
        import torch.distributed as dist

        dev = torch.device("cuda", self.local) if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.ws > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.destroy_process_group()
