"""Probe: the multi-process P2P workers with every rank on cuda:0 (contexts time-sliced)."""
import os
import socket
import sys
import time

import torch.multiprocessing as mp

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import test_gpu_multigpu as M  # noqa: E402


def port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


if __name__ == "__main__":
    names = sys.argv[1].split(",")
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for name in names:
        t0 = time.time()
        try:
            mp.spawn(getattr(M, name), args=(world, port()), nprocs=world, join=True)
            print(f"{name} world={world}: ok {time.time() - t0:.1f}s", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name} world={world}: FAIL {time.time() - t0:.1f}s {str(e)[-800:]}", flush=True)
