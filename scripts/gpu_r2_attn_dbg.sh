#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/attn_dbg
mkdir -p $O
python -m paper_2507_05043_b200.build > $O/build.log 2>&1
for c in "2 1 128,128" "2 1 256" "2 1 200" "2 1 64,64" "2 1 1,63" "2 1 65" "4 2 128,128" "4 2 256" "4 2 1,63,64,65,200" "8 1 256" "8 8 256" "32 8 512" "2 1 1000"; do
  timeout 60 python scripts/attn_debug.py 2 $c >> $O/cases.log 2>&1 || echo "FAILED: $c" >> $O/cases.log
done
timeout 300 compute-sanitizer --tool memcheck python scripts/attn_debug.py 2 4 2 1,63,64,65,200 > $O/memcheck.log 2>&1
echo done > $O/done
