"""N>1 path of bench.py on CPU: world-size-2 gloo ranks shard the batch (weak scaling, no
data-path collective) and reduce only the timing (max) and the unit count (sum)."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import synthetic as sy
    cfg = dict(sy.CONFIGS[2], n=24, batch=3)
    systems = bench.shard_systems(cfg["batch"], rank)
    k = sy.make_k(cfg, systems=systems)
    units, ms = bench.reduce_over_ranks(100.0 * (rank + 1), 10.0 + rank)
    out[rank] = (systems, units, ms, float(k.sum()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_reduction():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    s0, u0, t0, k0 = out[0]
    s1, u1, t1, k1 = out[1]
    assert s0 == [0, 1, 2] and s1 == [3, 4, 5]          # disjoint shards of one seeded stream
    assert u0 == u1 == 300.0                             # units summed over ranks
    assert t0 == t1 == 11.0                              # time = max over ranks
    assert k0 != k1                                      # each rank solves different systems


def test_single_process_identity():
    import bench
    assert bench.reduce_over_ranks(5.0, 2.0) == (5.0, 2.0)
    assert bench.shard_systems(4, 0) == [0, 1, 2, 3]
