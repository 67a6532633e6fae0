#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dense_launches.csv \
   python tests/cuda/dense_once.py > gpurun_out/dense_ncu.log 2>&1; echo rc=$?
