"""Probe torch symmetric memory on this box: rendezvous, peer pointers, P2P copy."""
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
t = symm.empty(1024, dtype=torch.float32, device=dev)
t.fill_(rank)
h = symm.rendezvous(t, dist.group.WORLD)
print(rank, "backend", symm.get_backend(dev), "ptrs", [hex(p) for p in h.buffer_ptrs],
      "t", hex(t.data_ptr()), "offset", h.offset, file=sys.stderr)
dist.barrier()
peer = (rank + 1) % world
rt = h.get_remote_tensor(peer, (1024,), torch.float32)
print(rank, "remote view of", peer, float(rt[0]), "ptr", hex(rt.data_ptr()), file=sys.stderr)
# write into the peer through its pointer with a plain copy kernel
rt[1:2].fill_(100 + rank)
torch.cuda.synchronize()
dist.barrier()
print(rank, "after peer write", float(t[1]), file=sys.stderr)
dist.destroy_process_group()
