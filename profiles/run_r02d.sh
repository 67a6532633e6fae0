#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tests/fastpath_diff.py > gpurun_out/fastdiff.json 2>gpurun_out/fastdiff.err; echo diff_rc=$?
python -c "import json; d=json.load(open('gpurun_out/fastdiff.json')); print(d['stats'])"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
