"""Experiment: can two NCCL ranks share one GPU (for 1-GPU testing of the multi-rank path)?"""
import os
import sys
import pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
import torch.multiprocessing as mp


def worker(rank, world, q):
    import paper_2310_01882_b200 as st
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29555")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = st.Comm.from_process_group(0)
        f = torch.full((6, 8), float(rank), dtype=torch.float64, device="cuda")
        st.st_halo_exchange(comm, [f], 4, 8, 1)
        torch.cuda.synchronize()
        q.put((rank, "ok", f[0, 0].item(), f[-1, 0].item()))
        comm.close()
    except Exception as e:  # noqa
        q.put((rank, "fail", repr(e)[:300]))
    dist.destroy_process_group()


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, q)) for r in range(2)]
    [p.start() for p in ps]
    [p.join(120) for p in ps]
    while not q.empty():
        print(q.get())
