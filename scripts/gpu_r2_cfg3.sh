#!/bin/bash
# BASELINE config 3 (Qwen2-72B shape, 8 stages, 256 requests 512/256, max_batched_tokens 131072)
# in one process on a 4-GPU box (two stages per GPU), per-GPU roofline fraction
cd "$(dirname "$0")/.."
O=gpurun_out/cfg3
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
timeout 2400 python scripts/run_stages.py --stages 8 --gpus 4 --model qwen2-72b-shape --batch 256 --prompt 512 \
  --decode 256 --max-batched 131072 --no-links > $O/cfg3_s8_g4.log 2>&1
echo done > $O/done
