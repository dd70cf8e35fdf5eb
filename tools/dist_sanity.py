# torchrun --nproc-per-node 1 --master-addr 127.0.0.1 tools/dist_sanity.py: the mixed
# gloo/NCCL group and the NCCL-backed count exchange callback on one GPU.
import os
import sys

sys.path.insert(0, ".")
import torch
import torch.distributed as dist

from paper_2512_16896_b200.dist import init_group, nccl_allgather_dev, torch_allgather

dev = init_group(int(os.environ.get("LOCAL_RANK", "0")))
ag = torch_allgather(dist.get_world_size(), dev)
print("device", dev, "gather", ag([1, 2, (1 << 64) - 1]))
agd = nccl_allgather_dev(dist.get_world_size(), dev)
send = torch.tensor([7, 8], dtype=torch.int64, device=dev)
recv = torch.zeros(2 * dist.get_world_size(), dtype=torch.int64, device=dev)
s = torch.cuda.Stream(device=dev)
agd(send.data_ptr(), 2, recv.data_ptr(), s.cuda_stream)
s.synchronize()
print("device gather", recv.tolist())
t = torch.tensor([1.5], dtype=torch.float64)
dist.all_reduce(t)
dist.barrier()
print("cpu all_reduce", t.item())
dist.destroy_process_group()
