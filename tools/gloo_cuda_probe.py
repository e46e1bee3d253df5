"""Does the gloo backend move CUDA tensors (send/recv batch, all_reduce, all_gather_object)?
Two ranks on one GPU (torch.multiprocessing)."""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def work(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    x = torch.full((4,), float(rank + 1), device="cuda")
    dist.all_reduce(x)
    buf = torch.zeros(8, dtype=torch.complex128, device="cuda")
    if rank == 1:
        buf += 3 + 1j
    ops = [dist.P2POp(dist.isend if rank == 1 else dist.irecv, buf, 1 - rank)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    print(rank, x.tolist(), buf[:2].tolist(), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(work, args=(port,), nprocs=2)
