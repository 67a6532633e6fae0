#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kvcache_gpu.py tests/test_dropin_gpu.py tests/test_engine_gpu.py tests/test_program_fastpath_gpu.py -x -q > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_probe.log
for m in 1 0; do SB_PROBE_SPEC=$m timeout 600 python bench_kv.py --only probe,probe_big 2>/dev/null | grep probe_rows | cut -c1-200; done
SB_PROBE_SPEC=0 timeout 900 python -m pytest tests/test_kvcache_gpu.py tests/test_dropin_gpu.py -x -q 2>&1 | tail -1
