#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/pytest_dist_e8.log 2>&1; tail -15 gpurun_out/pytest_dist_e8.log
