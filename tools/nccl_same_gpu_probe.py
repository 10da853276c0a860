"""Probe: can two NCCL ranks share one GPU here (for testing the library's NCCL paths)?"""
import os, sys
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def w(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
        t = torch.ones(4, device="cuda:0") * (rank + 1)
        dist.all_reduce(t)
        torch.cuda.synchronize()
        q.put((rank, "ok", t.tolist()))
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, "fail", repr(e)[:300]))


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=w, args=(r, 2, 29533, q)) for r in range(2)]
    for p in ps: p.start()
    for _ in range(2):
        try:
            print(q.get(timeout=120))
        except Exception as e:
            print("timeout", e)
    for p in ps: p.join(timeout=30)
