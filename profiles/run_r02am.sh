#!/bin/bash
# phase timestamps of the cooperative evict (SB_SELECT_PROF=1): where k_select_coop's time goes
SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict_small,evict,probe > gpurun_out/sel_prof.jsonl 2> gpurun_out/sel_prof.err
echo rc=$?
grep SB_SELECT_PROF gpurun_out/sel_prof.err | awk 'NR%3==0' | head -60
