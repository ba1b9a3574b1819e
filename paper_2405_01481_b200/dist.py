"""The experience step's single collective: the 6 fp64
whitening / metric partials {n_tokens, sum adv, sum adv^2, kl_sum,
reward_sum, n_seqs} are ALL-GATHERED from every rank and summed in rank order
on every rank, so all ranks hold bit-identical statistics.  torch.distributed
is the plumbing (NCCL over NVLink on B200 ranks, gloo for the CPU tests)."""
from __future__ import annotations

import ctypes

import numpy as np


class _CudaArray:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


def allgather_sum_fn(group=None, device=None, stage_on_host=False):
    """fn(ptr, n, stream) for ExperienceMaker(allreduce=...): replaces the n
    doubles at ptr (device memory on `device`, or host memory when device is
    None/cpu) by their sum over the ranks of `group`, in rank order.
    stage_on_host: gather through host tensors (a gloo group over device
    buffers, e.g. several ranks sharing one GPU in the tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)

    def fn(ptr: int, n: int, stream=None):
        if device is None or torch.device(device).type == "cpu":
            host = np.ctypeslib.as_array((ctypes.c_double * n).from_address(ptr))
            buf = torch.from_numpy(host)
        else:
            buf = torch.as_tensor(_CudaArray(ptr, n), device=device)
        src = buf.cpu() if stage_on_host else buf.clone()
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src, group=group)
        total = parts[0].clone()
        for p in parts[1:]:  # fixed rank order
            total += p
        buf.copy_(total.to(buf.device))
        if buf.is_cuda:
            torch.cuda.current_stream(buf.device).synchronize()

    return fn
