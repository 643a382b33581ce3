"""Live S-stage NVLink pipeline (run_device_demo) vs the virtual engine and the CPU oracle.

    torchrun --nproc-per-node S scripts/check_live.py      (S = 2 or 4 stages, one per rank)

Criterion-11 analog (test_acceptance.py:367-381): per-request token counts of the
live run equal the virtual run's; additionally the generated ids equal the CPU
oracle's (margin-engineered init).  The head's RuntimeMonitor rebuilds the stage /
link profiles every 8 micro-batches from measured forwards and round trips; the
profiles it ended with are printed.  Exit code 0 = parity holds.
"""

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import faulthandler

    faulthandler.dump_traceback_later(150, exit=True, file=sys.stdout)  # a hang prints every thread's stack
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group(backend="cuda:nccl,cpu:gloo")
    from paper_2507_05043_b200 import TINY, deploy
    from paper_2507_05043_b200.live import run_device_demo
    from paper_2507_05043_b200.spec import prompt_tokens
    import pipelink as PL

    S = dist.get_world_size()  # one stage per rank
    spec = TINY.with_(peaked=True)
    cluster = deploy.b200_cluster(S)
    plan = deploy.plan(cluster, spec, S)
    cfg = deploy.engine_config(plan, spec, PL.ControllerConfig(max_batched_tokens=256, max_batch_size=8),
                               chunk_size=4096)
    trace = PL.Trace(requests=[PL.Request(i, 0.0, 40 + 7 * i, 6 + (i % 5)) for i in range(20)])
    profiles = [PL.synth_profile(hi - lo, 1e-6, 2e-5, stage_id=i) for i, (_, (lo, hi)) in enumerate(plan.stages)]
    res = run_device_demo(cfg, cluster, profiles, trace, decoder=spec, monitor_epoch=8)
    ok = True
    if dist.get_rank() == 0:
        virtual = PL.PipelineEngine(cfg, cluster, profiles).run(trace)
        counts_ok = res.tokens_by_request == virtual.tokens_by_request()
        from oracle import decoder as OD

        model = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=256)
        bad = 0
        for r in trace.requests:
            want, _ = model.greedy([torch.from_numpy(prompt_tokens(0, r.id, r.input_len, spec.vocab))],
                                   r.output_len)
            bad += not np.array_equal(res.tokens[r.id], want[0].numpy())
        print(f"live {S}-stage NVLink run: {res.microbatches} micro-batches in {res.wall_s:.2f} s; "
              f"token counts {'==' if counts_ok else '!='} virtual; "
              f"{len(trace.requests) - bad}/{len(trace.requests)} requests identical to the oracle", flush=True)
        # runtime monitoring: the profiles the head ended with (measured on the device clock)
        dec = {s: [(t, round(sec * 1e6, 1)) for t, sec in p.points(PL.Phase.DECODE)]
               for s, p in enumerate(res.stage_profiles)}
        links = [(lp.name, round(lp.latency_s * 1e6, 1), round(lp.bandwidth_bps / 1e9, 1)) for lp in res.link_profiles]
        print(f"monitor: {res.monitor_updates} profile updates; decode points (tokens, us) {dec}; "
              f"links (us, GB/s) {links}", flush=True)
        ok = counts_ok and bad == 0
    t = torch.tensor([0 if ok else 1])
    dist.all_reduce(t)
    dist.destroy_process_group()
    sys.exit(int(t.item() != 0))


if __name__ == "__main__":
    try:
        main()
    except SystemExit:
        raise
    except BaseException:
        import traceback

        traceback.print_exc(file=sys.stdout)
        sys.stdout.flush()
        raise
