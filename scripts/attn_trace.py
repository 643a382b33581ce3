"""Timeline of CTA 0 of the tcgen05 prefill attention kernel (experiment build with
-DPL_AT_TRACE, loaded through PL_LIB_PATH): per step, when the MMA warp got V, each
tile's P, and when each tile's softmax got S / finished loading it / published P.

    PL_LIB_PATH=.../_lib_trace/libb200link.so python scripts/attn_trace.py HQ HKV L1,L2,...
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    from paper_2507_05043_b200 import _native as N, ops

    Hq, Hkv = int(sys.argv[1]), int(sys.argv[2])
    lens = [int(x) for x in sys.argv[3].split(",")]
    hd, T = 128, sum(lens)
    qkv = torch.randn(T, (Hq + 2 * Hkv) * hd, device="cuda").to(torch.bfloat16)
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32, device="cuda")
    for _ in range(3):
        ops.attn_prefill(qkv, cu, max(lens), Hq, Hkv, hd, impl=2)
    torch.cuda.synchronize()
    buf = np.zeros((64, 12), dtype=np.uint64)
    lib = N.lib()
    lib.pl_attn_trace_read.argtypes = [C.c_void_p]
    assert lib.pl_attn_trace_read(buf.ctypes.data) == 0
    t0 = buf[0, 0]
    rel = (buf.astype(np.int64) - int(t0)) / 1000.0  # us
    names = ["mma:v_wait", "mma:v_ok", "mma:pA_ok", "mma:step_end", "mma:pB_ok", "-",
             "smA:s_ok", "smA:ld_done", "smA:p_done", "smB:s_ok", "smB:ld_done", "smB:p_done"]
    print("step " + " ".join(f"{n:>11}" for n in names))
    for i in range(64):
        if buf[i, 0] == 0:
            break
        print(f"{i:4d} " + " ".join(f"{rel[i, k]:11.2f}" for k in range(12)))
    d = np.diff(rel[:, 3][rel[:, 3] > 0])
    print(f"median step {np.median(d):.2f} us; softmax A (s_ok -> p_done) "
          f"{np.median(rel[:, 8] - rel[:, 6]):.2f} us, of which S load {np.median(rel[:, 7] - rel[:, 6]):.2f}; "
          f"softmax B {np.median(rel[:, 11] - rel[:, 9]):.2f} us; "
          f"P_A published -> MMA sees it {np.median(rel[:, 2] - rel[:, 8]):.2f} us")


if __name__ == "__main__":
    main()
