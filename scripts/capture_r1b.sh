#!/usr/bin/env bash
# ncu --set full of the kernels added late in round 1 (run on a GPU box, one GPU):
#   the cluster split-K QKV GEMM (decode, T = 64) and the CTA-pair prefill gate_up GEMM.
set -u
OUT=gpurun_out
export PYTHONPATH=$PWD
python scripts/profile_decode.py --layers 4 --iters 2 --last 0 > $OUT/prof_r1b_decode_plain.log 2>&1 || exit 1
# 4 gemm_tc launches per layer (qkv, o, gate_up, down): index 8 = layer 2's QKV (cluster split-K)
ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 8 -c 1 \
    -o $OUT/prof_r1b_qkv_csk python scripts/profile_decode.py --layers 4 --iters 2 --last 0 \
    > $OUT/prof_r1b_qkv_csk.log 2>&1
PF="import torch; from paper_2507_05043_b200 import ops
x = torch.randn(16384, 4096, device='cuda').to(torch.bfloat16)
w = (torch.randn(28672, 4096, device='cuda') * 0.02).to(torch.bfloat16)
for _ in range(3): ops.gemm(x, w, ops.EPI_SWIGLU)
torch.cuda.synchronize(); print('ok')"
python -c "$PF" > $OUT/prof_r1b_pair_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:gemm_pair -s 2 -c 1 \
    -o $OUT/prof_r1b_pair_gate_up python -c "$PF" > $OUT/prof_r1b_pair.log 2>&1
echo done
