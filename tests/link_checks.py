"""Invariants of a REALIZED link log (device clock), after pkg/tests/test_transport.py:136-211.

The reference's check_link_invariants judges a virtual-time log.  On the device
clock a link may idle while the producing forward is still running, so its
work-conservation rule does not apply; what must hold for every realized link:

* the emitted chunk sequence (payload, index, size) is exactly the LinkQueue's
  virtual sequence (decode priority and class FIFO are decided there);
* bytes are conserved: a payload's emitted chunks sum to its enqueued size;
* chunks never overlap on a link: emit_{k+1} >= sent_k (one copy / ncclSend stream);
* no chunk leaves before its payload exists (emit >= enqueue, 1 us event slack);
* within a class, payloads complete in enqueue order (FIFO by completion).
"""

from __future__ import annotations


def check_realized_link(real_events, virtual_events, link_name: str) -> dict:
    real = [e for e in real_events if e.link == link_name]
    virt = [e for e in virtual_events if e.link == link_name]
    emits = [e for e in real if e.event == "emit"]
    sents = [e for e in real if e.event == "sent"]
    v_emits = [(e.payload_id, e.chunk_index, e.size_bytes) for e in virt if e.event == "emit"]
    assert [(e.payload_id, e.chunk_index, e.size_bytes) for e in emits] == v_emits, \
        f"{link_name}: realized chunk sequence differs from the LinkQueue's"
    sizes = {}
    for e in emits:
        sizes[e.payload_id] = sizes.get(e.payload_id, 0) + e.size_bytes
    v_sizes = {e.payload_id: e.size_bytes for e in virt if e.event == "enqueue"}
    assert sizes == v_sizes, f"{link_name}: bytes not conserved"
    for a, b in zip(sents, emits[1:]):
        assert b.time_ns >= a.time_ns, f"{link_name}: two chunks in flight"
    enq = {e.payload_id: e.time_ns for e in real if e.event == "enqueue"}
    for e in emits:
        assert e.time_ns >= enq[e.payload_id] - 1000, f"{link_name}: chunk before its payload existed"
    done = {}
    for e in sents:
        done[e.payload_id] = e.time_ns
    cls = {e.payload_id: e.phase_class for e in virt if e.event == "enqueue"}
    v_enq = {e.payload_id: e.time_ns for e in virt if e.event == "enqueue"}
    for c in set(cls.values()):
        pids = [p for p in done if cls[p] == c]
        by_enq = sorted(pids, key=lambda p: (v_enq[p], p))
        by_done = sorted(pids, key=lambda p: (done[p], p))
        assert by_enq == by_done, f"{link_name}: {c} payloads reordered"
    busy = sum(b.time_ns - a.time_ns for a, b in zip(emits, sents))
    span = (sents[-1].time_ns - emits[0].time_ns) if emits else 0
    return {"chunks": len(emits), "payloads": len(sizes), "bytes": sum(sizes.values()),
            "busy_us": round(busy / 1e3, 1), "span_us": round(span / 1e3, 1)}
