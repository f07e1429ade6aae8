"""Distributed (2D block-cyclic) factorization of a full config on one GPU over gloo,
checked bitwise against the single-GPU engine:  python scripts/dist_check.py C2 2"""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, cfg, out):
    import torch.distributed as dist

    import bench
    from paper_2512_04389_b200.parallel import DistEngine

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, f, g, t = bench.build_case(cfg)
    de = DistEngine(g, t)
    de.upload()
    t0 = time.perf_counter()
    ms, st = de.run()
    wall = time.perf_counter() - t0
    vals, perms = de.gather_values()
    if rank == 0:
        np.save(out, vals)
        print(f"[rank0] grid {de.pg.pr}x{de.pg.pc} segments {de.eng.n_segments} messages {de.messages} "
              f"sent {de.bytes_out / 1e9:.2f} GB status {st.code} device ms {ms:.1f} wall {wall:.1f}s", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = f"/tmp/dist_{cfg}.npy"
    mp.spawn(worker, args=(world, port, cfg, out), nprocs=world, join=True)
    import bench
    from paper_2512_04389_b200.numeric import Engine

    a, f, g, t = bench.build_case(cfg)
    eng = Engine(g, t)
    eng.upload()
    eng.run_device()
    ref, _ = eng.download()
    got = np.load(out)
    print(f"{cfg} world {world}: bitwise equal to single GPU: {got.tobytes() == ref.tobytes()} "
          f"(max |diff| {np.abs(got - ref).max():.3e}, {len(ref)} factor entries)", flush=True)
