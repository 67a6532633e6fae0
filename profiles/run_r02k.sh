#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kvcache_gpu.py tests/test_dropin_gpu.py tests/test_engine_gpu.py -x -q > gpurun_out/pytest_probe.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_probe.log
for m in 0 2; do SB_PROBE_PER=$m timeout 600 python bench_kv.py --only probe,probe_big 2>/dev/null | grep probe_rows; done
