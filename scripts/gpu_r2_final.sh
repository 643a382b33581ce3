#!/bin/bash
# round-2 validation on one B200: GPU suite, smoke, N=1 bench, then the ncu launch list
cd "$(dirname "$0")/.."
O=gpurun_out/final
rm -rf $O; mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
echo "pytest rc=$?" >> $O/pytest.log
timeout 600 python __graft_entry__.py smoke > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_n1.log 2>&1
echo "bench rc=$?" >> $O/bench_n1.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --decode 4 --no-cpu-baseline --no-parity"
timeout 600 $CMD > $O/prof_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 14000 -c 1500 --csv \
    --log-file $O/launches.csv $CMD > $O/launches_run.log 2>&1
echo done > $O/done
