#!/bin/bash
# compute-sanitizer --tool synccheck on one small invocation of every kernel family
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/san
python -m paper_2507_05043_b200.build > gpurun_out/san/build.log 2>&1
timeout 600 python scripts/sanitize_kernels.py > gpurun_out/san/plain_synccheck.log 2>&1 && \
timeout 2400 compute-sanitizer --tool synccheck --print-limit 100 python scripts/sanitize_kernels.py > gpurun_out/san/synccheck.log 2>&1
echo "rc=$?" >> gpurun_out/san/synccheck.log
