#!/bin/bash
# phase timestamps of the fused cooperative evict at 4M blocks (SB_SELECT_PROF=1; diagnostic, not a bench value)
mkdir -p gpurun_out
SB_SELECT_PROF=1 timeout 300 python bench_kv.py --only evict > gpurun_out/kv_prof.jsonl 2> gpurun_out/kv_prof.err; echo rc=$?
grep "SB_SELECT_PROF mode" gpurun_out/kv_prof.err | tail -4
grep "SB_SELECT_PROF_CTA" gpurun_out/kv_prof.err | tail -2 | cut -c1-600
