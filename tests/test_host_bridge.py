"""Cross-host hops (§8(f)4): the reference's socket framing carrying device payloads.

On CPU the bodies are host tensors; the framing, chunking and decode-priority
preemption are the reference's own (pipelink/wire.py), so a decode payload sent
behind a large prefill payload overtakes it at a chunk boundary, as in
pkg/tests/test_wire.py."""

import threading

import torch

import pipelink
import pipelink.wire  # noqa: F401
from paper_2507_05043_b200.wire import HostBridgeLinkReceiver, HostBridgeLinkSender


def test_loopback_roundtrip_and_decode_overtake():
    a, b = pipelink.wire.loopback_pair()
    got, done = [], threading.Event()

    def on_payload(p):
        got.append(p)
        if len(got) == 3:
            done.set()

    rx = HostBridgeLinkReceiver(b, on_payload)
    rx.start()
    tx = HostBridgeLinkSender(a, chunk_size=4096)
    big = torch.arange(200_000, dtype=torch.int32).view(torch.uint8)        # 800 KB prefill
    small = torch.full((64,), 7, dtype=torch.int64)                          # 512 B decode
    P = pipelink.Payload
    tx.send(P(id=1, phase_class=pipelink.PayloadClass.PREFILL, size_bytes=big.numel(), micro_batch_id=1,
              enqueue_time=0), big)
    tx.send(P(id=2, phase_class=pipelink.PayloadClass.DECODE, size_bytes=512, micro_batch_id=2,
              enqueue_time=0), small)
    tx.send(P(id=3, phase_class=pipelink.PayloadClass.PREFILL, size_bytes=16, micro_batch_id=3,
              enqueue_time=0), torch.arange(16, dtype=torch.uint8))
    tx.start()
    assert done.wait(30)
    tx.close()
    tx.join(10)
    rx.join(10)
    assert not rx.failed
    by_id = {p.payload_id: p for p in got}
    assert [p.payload_id for p in got][0] == 2          # decode overtook the 800 KB payload
    assert torch.equal(by_id[1].body, big) and torch.equal(by_id[2].body.view(torch.int64), small)
    assert by_id[2].phase_class is pipelink.PayloadClass.DECODE
