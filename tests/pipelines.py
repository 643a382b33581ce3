"""Small builders for schedule-level tests (clusters, plans, profiles, traces)."""

import pipelink
from pipelink import ClusterSpec, LinkProfile, NodeDescriptor, PartitionPlan, Platform, Request, Trace


def make_node(name, gpu_count=1, capacity=1.0, mem=180 << 30, gpu_type="b200"):
    return NodeDescriptor(name=name, platform=Platform.LINUX, gpu_type=gpu_type, gpu_count=gpu_count,
                          gpu_mem_bytes=mem, capacity_score=capacity, cpu_score=1.0, network_score=1.0)


def ring_cluster(S, latency_s, bandwidth):
    """S single-GPU nodes b0..b{S-1} with forward hops and the return hop."""
    names = [f"b{i}" for i in range(S)]
    links = {}
    if S > 1:
        for src, dst in list(zip(names, names[1:])) + [(names[-1], names[0])]:
            links[(src, dst)] = LinkProfile(src, dst, latency_s, bandwidth)
    return names, ClusterSpec(nodes={n: make_node(n) for n in names}, links=links)


def uniform_pipeline(S, compute_s, latency_s, bandwidth=1e18, hidden_dim=1, dtype_bytes=1):
    names, cluster = ring_cluster(S, latency_s, bandwidth)
    model = pipelink.ModelSpec("test", S, hidden_dim, dtype_bytes, 1)
    plan = PartitionPlan(stages=tuple((names[i], (i, i + 1)) for i in range(S)), head=names[0])
    return cluster, model, plan, [pipelink.flat_profile(compute_s, stage_id=i) for i in range(S)]


def decode_trace(n, output_len=10**6, input_len=1):
    return Trace(requests=[Request(id=i, arrival_time=0.0, input_len=input_len, output_len=output_len)
                           for i in range(n)])
