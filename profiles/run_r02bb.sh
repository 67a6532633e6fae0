#!/bin/bash
SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict_big > /dev/null 2> gpurun_out/sel_prof_16m.err
grep "SB_SELECT_PROF " gpurun_out/sel_prof_16m.err | awk 'NR%4==0' | tail -2 | cut -c1-330
grep "SB_SELECT_PROF_CTA" gpurun_out/sel_prof_16m.err | tail -2 | cut -c1-900
