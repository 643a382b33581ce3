#!/bin/bash
# 8 stages on 4 GPUs (one process), three repeats with the full measured profiles dumped
cd "$(dirname "$0")/.."
O=gpurun_out/s8reps; rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
for r in 1 2 3; do
  timeout 900 python scripts/run_stages.py --stages 8 --gpus 4 --no-links > $O/s8_profiles_rep$r.log 2>&1
done
echo done > $O/done
