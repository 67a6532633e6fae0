"""BASELINE configs[4]: KV-pool pressure sweep — hint-aware (Sutradhara
preset: tiered eviction + request-aware scheduling + prompt splitting) vs the
LRU baseline on the reference's synthetic agent trace, every KV decision on
the B200 pool (csrc/replay.cu), timing rules of the reference simulator.

The pool is swept from well below to above the trace's working set (the
smallest swept capacity with zero evictions under LRU); one JSON line per
(capacity, preset) with hit rate, p50 FTR, p50 end-to-end time, evictions,
plus a summary line.

    python bench_pressure.py [--requests 60] [--seed 1]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    from paper_2601_12967_b200.replay import replay

    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=60)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--caps", default="4096,8192,16384,32768,65536,131072,262144,524288")
    args = ap.parse_args()
    caps = [int(c) for c in args.caps.split(",")]
    rows = []
    for cap in caps:
        for preset in ("baseline", "sutradhara"):
            t0 = time.perf_counter()
            r = replay(args.requests, seed=args.seed, preset=preset, capacity_blocks=cap)
            row = {"capacity_blocks": cap, "preset": preset, "policy": "tiered (hint-aware)" if preset == "sutradhara"
                   else "LRU", "hit_rate": r.hit_rate, "p50_ftr_ms": r.p50(), "p50_e2e_ms": r.p50(r.e2e_ms),
                   "evictions": r.evictions, "replay_wall_s": time.perf_counter() - t0}
            rows.append(row)
            print(json.dumps(row), flush=True)
    ws = next((c for c in caps if all(r["evictions"] == 0 for r in rows
                                       if r["capacity_blocks"] == c and r["preset"] == "baseline")), None)
    summary = {"summary": "pressure sweep", "requests": args.requests, "seed": args.seed,
               "working_set_blocks": ws, "points": []}
    for cap in caps:
        b = next(r for r in rows if r["capacity_blocks"] == cap and r["preset"] == "baseline")
        s = next(r for r in rows if r["capacity_blocks"] == cap and r["preset"] == "sutradhara")
        summary["points"].append({"capacity_blocks": cap, "pool_frac_of_working_set": cap / ws if ws else None,
                                  "hit_rate_lru": b["hit_rate"], "hit_rate_hint_aware": s["hit_rate"],
                                  "p50_ftr_lru_ms": b["p50_ftr_ms"], "p50_ftr_hint_aware_ms": s["p50_ftr_ms"],
                                  "ftr_speedup": b["p50_ftr_ms"] / s["p50_ftr_ms"] if s["p50_ftr_ms"] else None})
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
