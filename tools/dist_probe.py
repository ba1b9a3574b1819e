import os, sys, time
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_01481_b200.dist import allgather_sum_fn
local = int(os.environ["LOCAL_RANK"]); rank = int(os.environ["RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
print(rank, "init ok", flush=True)
buf = torch.full((6,), float(rank + 1), dtype=torch.float64, device=dev)
allgather_sum_fn(device=dev)(buf.data_ptr(), 6, None)
print(rank, "allgather ok", buf.tolist(), flush=True)
dist.barrier(); print(rank, "barrier ok", flush=True)
dist.destroy_process_group()
