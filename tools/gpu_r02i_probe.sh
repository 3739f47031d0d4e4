#!/bin/bash
# Probe: health (GPU tests), shard timing, and per-launch lists of c5s8 / c2 / c4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_probe.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_probe.log
timeout 300 python tools/exp_shard.py 8 > gpurun_out/shard_probe.jsonl 2>&1
for c in c5s8 c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
    --log-file gpurun_out/launches_$c.csv python tools/profile_run.py --config $c > /dev/null 2>&1
  echo "$c ncu exit $?"
done
