"""Single-box deployment helpers built on the reference's planning API.

One B200 box is registered as S single-GPU ``NodeDescriptor``s joined by
NVLink ``LinkProfile``s, and the reference's own ``plan_deployment``
(placement.py:417-425 -> select_nodes + partition_layers) produces the
S-stage layer split, exactly as a pipelink user would plan a weak-link
deployment.  ``partition_layers`` is capacity-proportional with largest
remainder (placement.py:378-414): uniform nodes give L3 [8]x4 / [4]x8,
Q2 [10]x8, tiny [2,2].
"""

from __future__ import annotations

from ._pipelink import pipelink
from .spec import DecoderSpec

GPU_TYPE = "b200"
B200_MEM = 180 * (1 << 30)
NVLINK = (2e-6, 9e11)            # measured-class one-way latency (s), bytes/s per direction
WEAK_LINK = (0.015, 12.5e6)      # 100 Mbps, 30 ms RTT (BASELINE config 5)


def b200_cluster(S: int, latency_s: float = NVLINK[0], bandwidth_bps: float = NVLINK[1]):
    names = [f"b200-{i}" for i in range(S)]
    nodes = {
        n: pipelink.NodeDescriptor(name=n, platform=pipelink.Platform.LINUX, gpu_type=GPU_TYPE,
                                   gpu_count=1, gpu_mem_bytes=B200_MEM, capacity_score=1.0,
                                   cpu_score=1.0, network_score=1.0)
        for n in names
    }
    links = {}
    for a in names:
        for b in names:
            if a != b:
                links[(a, b)] = pipelink.LinkProfile(a, b, latency_s, bandwidth_bps)
    return pipelink.ClusterSpec(nodes=nodes, links=links)


def plan(cluster, decoder: DecoderSpec, S: int):
    return pipelink.plan_deployment(cluster, decoder.model_spec(), GPU_TYPE, S)


def engine_config(plan_, decoder: DecoderSpec, controller, chunk_size="default", **kw):
    if chunk_size == "default":
        chunk_size = pipelink.DEFAULT_CHUNK_SIZE
    return pipelink.EngineConfig(partition=plan_, model=decoder.model_spec(), controller=controller,
                                 chunk_size=chunk_size, **kw)


def uniform_trace(n: int, input_len: int, output_len: int, arrival_s: float = 0.0):
    return pipelink.Trace(requests=[
        pipelink.Request(id=i, arrival_time=arrival_s, input_len=input_len, output_len=output_len)
        for i in range(n)])
