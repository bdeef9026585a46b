"""Probe: CUDA IPC mapping of a neighbour rank's tensor through torch's own reductions
(the mechanism the slab driver uses for peer-memory halo stores).  Two processes on one
GPU, gloo for the handle exchange."""
import os, sys
import torch, torch.distributed as dist, torch.multiprocessing as mp
from torch.multiprocessing.reductions import reduce_tensor


def worker(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    big = torch.zeros((1 << 20, 4), dtype=torch.float32, device="cuda:0")   # sub-allocated or not
    mine = torch.full((1000, 4), -1.0, dtype=torch.float32, device="cuda:0")
    fn, args = reduce_tensor(mine)
    handles = [None] * world
    dist.all_gather_object(handles, (fn, args))
    pfn, pargs = handles[(rank + 1) % world]
    peer = pfn(*pargs)
    peer[10:20] = float(rank + 100)          # a kernel of this process writes the neighbour's memory
    torch.cuda.synchronize()
    dist.barrier()
    got = mine[10:20, 0].tolist()
    print(f"rank {rank}: peer ptr {peer.data_ptr():#x} mine {mine.data_ptr():#x} got {got[:3]}", flush=True)
    assert all(v == float((rank - 1) % world + 100) for v in got)
    dist.barrier()
    del peer
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2, 29571), nprocs=2, join=True)
    print("ipc ok")
