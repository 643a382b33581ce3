#!/bin/bash
# round 2 validation: GPU test suite, smoke, N=1 bench (parity object included)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m paper_2507_05043_b200.build > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2a.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_r2a.log
