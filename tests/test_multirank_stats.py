"""CPU, world_size 2 over gloo: the multi-GPU path shards requests (no
data-path collective); the only collective is the statistics reduction of
bench.reduce_over_ranks — max of step times, sum of hit / lookup / eviction
counters.  Each rank also builds its own, disjoint request set."""
import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    reqs = bench.setup_workload(rank, 8)
    toks = sum(r.suffix_len for r in reqs)
    first = int(reqs[0].prefix_tokens[2048 + 5])  # past the shared system prompt
    mx, sm = bench.reduce_over_ranks([100.0 + rank, float(toks), float(rank + 1)])
    q.put((rank, mx, sm, toks, first))
    dist.destroy_process_group()


def test_stats_reduction_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, mx0, sm0, t0, f0), (r1, mx1, sm1, t1, f1) = res
    assert mx0 == mx1 and sm0 == sm1
    assert mx0[0] == 101.0  # max over ranks of the step time
    assert sm0[1] == t0 + t1 and sm0[2] == 3.0
    assert f0 != f1  # ranks serve different requests (weak scaling)
