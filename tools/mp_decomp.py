"""Run the multi-process decomposition test workers directly (faulthandler on)."""
import faulthandler
import socket
import sys

import torch.multiprocessing as mp

sys.path.insert(0, ".")


def worker(rank, world, port, travel, path):
    faulthandler.enable()
    from tests.test_gpu_decomp import _mp_worker
    _mp_worker(rank, world, port, travel, path)


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    travel = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0008
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, world, port, travel, "/tmp/r0.npz")) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        print("exit", p.exitcode, flush=True)
