"""CPU: host-side pieces of bench.py and the workloads — pool sizing, the
configs[2] request shape, the committed ncu evidence the bench line cites,
and the stats all-gather used by the sharded trace metrics (world_size 2,
gloo)."""
import json
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from paper_2601_12967_b200 import workload as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_configs2_requests():
    reqs = W.long_prefix_continuation_batch(8)
    lens = [r.prefix_len for r in reqs]
    assert lens[0] == 8192 and lens[-1] == 32768 and lens == sorted(lens)
    assert all(l % 16 == 0 for l in lens) and all(r.suffix_len == 1024 for r in reqs)
    # shared system prompt: identical first 2048 tokens
    assert all(np.array_equal(r.prefix_tokens[:2048], reqs[0].prefix_tokens[:2048]) for r in reqs)
    assert len({int(r.prefix_tokens[2048]) for r in reqs}) == len(reqs)


def test_capacity_for_counts_shared_prefix_once():
    reqs = W.agentic_continuation_batch(4, seed=1)
    pre, suf, cap = bench.capacity_for(reqs)
    assert pre == sum(r.prefix_len // 16 for r in reqs) - 3 * (2048 // 16)
    assert suf == sum((r.suffix_len + 15) // 16 for r in reqs) + len(reqs)  # + one response block per call
    assert cap == pre + int(1.25 * suf) + 1


def test_attention_traffic_from_committed_ncu():
    t = bench.ncu_traffic(bench.ATTN_NCU)
    m = json.load(open(bench.ATTN_NCU))
    assert "continuation_attention" in m["kernel"]
    assert 1e9 < t < 1e10  # bytes per launch, read + write


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # bench.gather_rows: ragged per-rank tables (one trace shard per rank)
    rows = np.array([[10.0 * rank + i, float(i)] for i in range(3 + rank)])
    out = bench.gather_rows(rows, world)
    q.put((rank, out.tolist()))
    dist.destroy_process_group()


def test_trace_stats_gather_world2():
    """The configs[3] gather: rank r's shard rows, in rank order, ragged."""
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
    exp = [[0.0, 0.0], [1.0, 1.0], [2.0, 2.0], [10.0, 0.0], [11.0, 1.0], [12.0, 2.0], [13.0, 3.0]]
    assert res[0][1] == res[1][1] == exp


def test_trace_summary_tool_share():
    tab = np.array([[100, 200, 16, 64, 50, 10, 30, 10], [200, 300, 0, 64, 20, 100, 60, 20]], np.float64)
    s = bench.trace_summary(tab, 7, 1.5)
    assert s["p50_ftr_ms"] == 100 and s["hit_rate"] == 16 / 128 and s["evictions"] == 7
    assert s["tool_share_of_ftr"]["frac_in_30_80pct"] == 0.5


def test_clock_sampler_parses_power_and_reasons():
    """nvidia-smi rows -> median SM clock, power draw and limit, the throttle
    reasons the timing rules reject or note (no GPU needed)."""
    s = bench.ClockSampler(0)
    s.proc = type("P", (), {"terminate": lambda self: None, "wait": lambda self, timeout=None: 0})()
    # index, clocks.sm, clocks.max.sm, power.draw, active, hw_slow, hw_thermal, sw_thermal, sw_power_cap, power.limit
    s.rows = [["0", "1520", "1965", "990.5", "0x4", "Not Active", "Not Active", "Not Active", "Active", "1000.00"],
              ["0", "1540", "1965", "985.0", "0x4", "Not Active", "Not Active", "Not Active", "Active", "1000.00"],
              ["0", "1530", "1965", "995.0", "0x0", "Not Active", "Not Active", "Not Active", "Not Active", "1000.00"]]
    import time as _t
    sleep, _t.sleep = _t.sleep, lambda x: None
    try:
        c = s.stop()
    finally:
        _t.sleep = sleep
    assert c["sm_mhz"] == 1530.0 and c["sm_max_mhz"] == 1965.0 and c["samples"] == 3
    assert c["power_w"] == 990.5 and c["power_limit_w"] == 1000.0
    assert c["reasons"] == ["sw_power_cap"]
