#!/bin/bash
for d in 0 1 2; do echo dbg=$d
SB_SELECT_DBG=$d SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict > /dev/null 2> gpurun_out/sel_prof_w.err
grep "SB_SELECT_PROF " gpurun_out/sel_prof_w.err | tail -1 | cut -c1-300
grep "SB_SELECT_PROF_WARPS" gpurun_out/sel_prof_w.err | tail -1 | cut -c1-120
done
