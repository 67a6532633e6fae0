"""Engine-side KV work of the configs[1] step in isolation: the same 64
agentic continuations and pool as bench.py, with a 1-layer / 1-kv-head
model shape so the step is dominated by the pool's op programs (admission
lookups, pin_partial, complete_prefill, finish_decode) instead of attention.

    python bench_engine_ops.py [--steps 10] [--requests 64]

Prints one JSON line: ms per step (CUDA events), launches, and with
SB_PROG_PROFILE=1 the op program's per-phase cycle counters on stderr."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--requests", type=int, default=64)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2601_12967_b200 import workload as W
    from paper_2601_12967_b200.engine import ContinuationEngine, ModelShape
    from paper_2601_12967_b200.kv_cache import TIERED

    reqs = W.agentic_continuation_batch(args.requests, seed=1)
    _, _, cap = bench.capacity_for(reqs)
    eng = ContinuationEngine(ModelShape(1, 1, 1, 128), cap, TIERED)
    batch = eng.make_batch([r.prefix_tokens for r in reqs], [r.prefix_tags for r in reqs],
                           [r.suffix_len for r in reqs])
    sfx = [torch.from_numpy(np.concatenate([W.fresh_suffix_tokens(r, s) for r in reqs]).view(np.int64)).cuda()
           for s in range(args.warmup + args.steps)]
    for s in range(args.warmup):
        batch.stage_suffix_device(sfx[s])
        batch.run(10 + s)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in range(args.warmup, args.warmup + args.steps):
        batch.stage_suffix_device(sfx[s])
        batch.run(10 + s)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    hits, st, _ = batch.results()
    print(json.dumps({"ms_per_step": ms, "requests": args.requests, "pool_blocks": cap,
                      "launches_per_step": batch.launches_per_step, "hit_rate": float(hits.sum()) / sum(batch.full_lens),
                      "evicted_total": eng.cache.total_evicted()}))
    del batch, eng


if __name__ == "__main__":
    main()
