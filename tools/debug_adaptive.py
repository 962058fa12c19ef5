#!/usr/bin/env python
"""Run the adaptive-completion worker on every rank (torchrun) and print per-rank outcomes."""

import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_13085_b200 as L  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    n = 100_003
    comm = L.P2PCommunicator(n, nblocks=16, timeout_s=20.0)
    x0 = np.random.default_rng(7).standard_normal(n).astype(np.float32)
    g = torch.empty(n, device="cuda")
    for tau_max in (1, 3):
        try:
            x = torch.from_numpy(x0.copy()).cuda()
            w = L.LASGDWorker(x, g, comm=comm, sync_period=tau_max, lr=0.05, mode="pull", adaptive=True,
                              tau_max=tau_max)
            for t in range(12):
                if rank == 1:
                    torch.cuda._sleep(2_000_000)
                g.copy_(torch.from_numpy(np.random.default_rng(t * 10 + rank).standard_normal(n).astype(np.float32)))
                w.step()
            st = w._native_state()
            print(f"rank {rank} tau_max {tau_max}: before drain seq={st.seq} hist={dict(w.tau_hist)}", flush=True)
            w.drain()
            torch.cuda.synchronize()
            print(f"rank {rank} tau_max {tau_max}: ok hist={dict(w.tau_hist)} finite={np.isfinite(x.cpu().numpy()).all()}",
                  flush=True)
        except Exception:
            print(f"rank {rank} tau_max {tau_max}: FAILED\n{traceback.format_exc()}", flush=True)
        dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
