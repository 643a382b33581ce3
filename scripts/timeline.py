"""Kernel timeline of a decode forward (experiment build with -DPL_TIMELINE).

    PL_BUILD_VARIANT=tl PL_NVCC_EXTRA=-DPL_TIMELINE python -m paper_2507_05043_b200.build
    PL_LIB_PATH=paper_2507_05043_b200/_lib_tl/libb200link.so \
        python scripts/timeline.py [--layers 4] [--T 64] [--ctx 640]

Every CTA of the decode GEMMs, the residual+norm reduce and the decode attention
appends %globaltimer stamps at its start and end; one forward (PDL chain, no events
between kernels) is recorded after warm-up.  Prints, per launch in issue order: the
first CTA start, last CTA start, first and last CTA end (us from the forward's first
stamp), the span, the overlap with / gap after the previous launch, and the
algorithmic bytes over the launch's busy window.
"""

import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_05043_b200 import LLAMA3_8B, _native  # noqa: E402
from paper_2507_05043_b200.executor import StageExecutor  # noqa: E402
from paper_2507_05043_b200.profiler import time_forward  # noqa: E402


def name_of(tag, spec):
    kind = tag >> 24
    if kind == 2:
        return "reduce+norm"
    if kind == 3:
        return "attn_decode"
    n, kb = ((tag >> 12) & 0xFFF) * 128, tag & 0xFFF
    k = kb * 64
    names = {(spec.qkv_dim, spec.d): "qkv", (spec.d, spec.attn_dim): "o", (2 * spec.ffn, spec.d): "gate_up",
             (spec.d, spec.ffn): "down", (spec.vocab, spec.d): "lm_head"}
    return names.get((n, k), f"gemm N{n} K{k}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--T", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=640)
    ap.add_argument("--last", type=int, default=0)
    a = ap.parse_args()
    spec = LLAMA3_8B.with_(num_layers=a.layers)
    exe = StageExecutor(spec, 0, (0, a.layers), True, bool(a.last), torch.device("cuda", 0),
                        max_tokens=a.T, max_reqs=max(a.T, 1), max_ctx=a.ctx + 1,
                        num_blocks=a.T * (-(-(a.ctx + 1) // 64)) + 64, n_slots=1)
    for _ in range(5):
        time_forward(exe, a.T, True, ctx=a.ctx, reps=1)
    L = _native.lib()
    f = L.pl_timeline_set
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32]
    f.restype = C.c_int32
    cap = 1 << 20
    buf = torch.zeros(2 * cap, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    assert f(buf.data_ptr(), cnt.data_ptr(), cap) == 0
    time_forward(exe, a.T, True, ctx=a.ctx, reps=0)  # one recorded forward
    torch.cuda.synchronize()
    assert f(None, None, 0) == 0
    n = int(cnt.item())
    rec = buf[: 2 * n].view(n, 2).cpu().numpy().astype(np.uint64)
    tags = (rec[:, 0] >> np.uint64(32)).astype(np.int64)
    blocks = ((rec[:, 0] >> np.uint64(3)) & np.uint64(0x1FFFFFFF)).astype(np.int64)
    ends = (rec[:, 0] & np.uint64(7)).astype(np.int64)
    ts = rec[:, 1].astype(np.int64)
    order = np.argsort(ts, kind="stable")
    tags, blocks, ends, ts = tags[order], blocks[order], ends[order], ts[order]
    # launches: group records by tag into runs separated by a change of launch; a start
    # record of block b that was already started in the current run of that tag opens a new run
    runs = []  # list of dicts
    open_run = {}
    for tg, b, e, t_ in zip(tags, blocks, ends, ts):
        r = open_run.get(tg)
        if e == 0 and (r is None or b in r["started"]):
            r = {"tag": tg, "started": set(), "s": [], "e": [], **{f"p{k}": [] for k in range(2, 8)}}
            runs.append(r)
            open_run[tg] = r
        if r is None:
            continue
        if e == 0:
            r["started"].add(b)
            r["s"].append(t_)
        elif e == 1:
            r["e"].append(t_)
        else:
            r[f"p{e}"].append(t_)
    runs = [r for r in runs if r["s"] and r["e"]]
    runs.sort(key=lambda r: min(r["s"]))
    t0 = min(runs[0]["s"])
    d, qkv, attn, ffn = spec.d, spec.qkv_dim, spec.attn_dim, spec.ffn
    wbytes = {"qkv": qkv * d * 2, "o": d * attn * 2, "gate_up": 2 * ffn * d * 2, "down": d * ffn * 2,
              "attn_decode": a.T * a.ctx * spec.Hkv * spec.hd * 2 * 2, "lm_head": spec.vocab * d * 2}
    print(f"decode T={a.T} ctx={a.ctx} layers={a.layers}: "
          f"{len(runs)} launches recorded")
    print("phases (us from the forward start): p2 = GEMM: first weight+activation k-block in smem / "
          "attention: predecessor complete; p3 = GEMM: accumulator complete / attention: last page in")
    print(f"{'kernel':<12} {'ctas':>5} {'start0':>8} {'startN':>8} {'end0':>8} {'endN':>8} {'span':>7} "
          f"{'vs prev':>8} {'GB/s busy':>9} {'p2 min':>7} {'p2 max':>7} {'p3 min':>7} {'p3 max':>7}  "
          "(p4-p6: cluster split-K park / sync / reduced; other GEMMs p4 = warp 2 epilogue done, p5 = thread 0 at the final barrier)")
    prev_end = None
    tot = {}
    for r in runs:
        nm = name_of(int(r["tag"]), spec)
        s0, sN, e0, eN = (min(r["s"]) - t0) / 1e3, (max(r["s"]) - t0) / 1e3, (min(r["e"]) - t0) / 1e3, \
            (max(r["e"]) - t0) / 1e3
        span = eN - s0
        rel = "" if prev_end is None else f"{s0 - prev_end:+.1f}"
        bw = wbytes.get(nm)
        gbs = f"{bw / ((eN - sN) * 1e3):.0f}" if bw and eN > sN else ""
        ph = []
        for k in ("p2", "p3", "p4", "p5", "p6"):
            v = r[k]
            if v or k in ("p2", "p3"):
                ph += [f"{(min(v) - t0) / 1e3:7.1f}", f"{(max(v) - t0) / 1e3:7.1f}"] if v else ["", ""]
        print(f"{nm:<12} {len(r['s']):>5} {s0:8.1f} {sN:8.1f} {e0:8.1f} {eN:8.1f} {span:7.1f} {rel:>8} {gbs:>9} "
              + " ".join(f"{x:>7}" for x in ph))
        prev_end = eN
        tot.setdefault(nm, []).append((sN, eN))
    end = max(max(r["e"]) for r in runs)
    print(f"total {(end - t0) / 1e3:.1f} us; per layer {(end - t0) / 1e3 / a.layers:.1f} us")
    # critical-path attribution: time between consecutive launches' last ends
    print("per kernel (avg of last-end minus previous launch's last-end, i.e. its share of the chain):")
    shares = {}
    pe = t0
    for r in runs:
        nm = name_of(int(r["tag"]), spec)
        eN = max(r["e"])
        shares.setdefault(nm, []).append((eN - pe) / 1e3)
        pe = eN
    for nm, v in shares.items():
        print(f"  {nm:<12} {np.mean(v):7.1f} us  (n={len(v)})")


if __name__ == "__main__":
    main()
