"""Diagnose the multi-process sharded filter on one GPU (gloo): each rank logs
its progress to gpurun_out/shard_rank<r>.log."""
import os
import socket
import sys
import time
import traceback

import torch.multiprocessing as mp


def worker(rank, world, port, P):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.getcwd())
    log = open(f"gpurun_out/shard_rank{rank}.log", "w", buffering=1)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=__import__("datetime").timedelta(seconds=60))
    try:
        from paper_1306_3277_b200 import LORENZ96, RngStream
        from paper_1306_3277_b200.inference import sharded as S
        from tests.test_gpu_sharded import _problem

        theta, grid = _problem()
        log.write("start\n")
        orig = S.PeerArena.__init__

        def init(self, t, shard):
            log.write(f"arena {t.shape}\n")
            orig(self, t, shard)
            log.write(f"arena ptrs {self.ptrs}\n")
        S.PeerArena.__init__ = init
        t0 = time.time()
        ll, traj = S.particle_filter_sharded(LORENZ96, theta, grid, RngStream(31), P, resampler="systematic")
        log.write(f"done {ll} {time.time() - t0:.2f}s traj0 {traj[0][:3]}\n")
    except Exception:
        log.write(traceback.format_exc())
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 15
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, 2, port, P)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(180)
        if p.is_alive():
            p.kill()
    print("exitcodes", [p.exitcode for p in ps])
