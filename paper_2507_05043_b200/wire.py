"""NVLink twin of the reference's real-bytes link backend (pipelink/wire.py:28-199).

Same contract as ``SocketLinkSender`` / ``SocketLinkReceiver``:

  sender = DeviceLinkSender(comm, peer, chunk_size, policy, name)
  sender.start(); sender.send(payload, body); ...; sender.close(); sender.join()
  receiver = DeviceLinkReceiver(comm, peer, on_payload, name); receiver.start()

* the sender owns an unchanged reference ``LinkQueue`` (transport.py:70-160) and
  a worker thread drains it one chunk per frame, so decode payloads preempt
  prefill payloads at chunk boundaries exactly as on the socket backend;
* a frame is a 40-byte header (payload id, chunk index, flags, chunk bytes,
  payload bytes) and the chunk's bytes, each one ``ncclSend`` on the sender's stream -- the body
  goes GPU to GPU over NVLink straight from the payload tensor;
* flags are the socket backend's (``FLAG_LAST`` / ``FLAG_DECODE`` /
  ``FLAG_SHUTDOWN``, wire.py:31-33); ``send`` raises ``ProtocolError`` on a size
  mismatch, a duplicate id or while closing (wire.py:93-105); the sender holds
  the body until its last chunk is on the wire (wire.py:103, 142-146);
* the receiver lands every chunk at its offset of one device tensor (no
  re-copy, no torch kernel while NCCL kernels spin) and calls
  ``on_payload(ReceivedDevicePayload)`` on its own thread; transport failures
  set ``failed`` (wire.py:160-185).

The communicator is a 2-rank NCCL comm per direction (sender = rank 0).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._pipelink import pipelink

LinkQueue = pipelink.LinkQueue
LinkPolicy = pipelink.LinkPolicy
PayloadClass = pipelink.PayloadClass
ProtocolError = pipelink.ProtocolError

FLAG_LAST = 1
FLAG_DECODE = 2
FLAG_SHUTDOWN = 4
HEADER_WORDS = 5  # int64: payload id, chunk index, flags, chunk bytes, payload bytes
HEADER_BYTES = HEADER_WORDS * 8


@dataclass
class ReceivedDevicePayload:
    payload_id: int
    phase_class: object
    body: torch.Tensor  # uint8, on the receiver's device


class DeviceLinkSender(threading.Thread):
    """Worker draining a LinkQueue onto an NCCL link, one chunk per frame."""

    def __init__(self, comm, peer: int, chunk_size, policy=LinkPolicy.DECODE_PRIORITY,
                 name: str = "link-sender", device=None):
        super().__init__(name=name, daemon=True)
        self._comm, self._peer = comm, peer
        self._queue = LinkQueue(chunk_size=chunk_size, policy=policy)
        self._bodies: dict = {}
        self._offsets: dict = {}
        self._cond = threading.Condition()
        self._closing = False
        self.device = torch.device(device if device is not None else torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self._stream = torch.cuda.Stream(self.device)
            self._hdr_dev = torch.empty(HEADER_WORDS, dtype=torch.int64, device=self.device)
        self._hdr_host = torch.empty(HEADER_WORDS, dtype=torch.int64).pin_memory()
        self.failed = False
        self.frames = 0

    def send(self, payload, body: torch.Tensor, ready: torch.cuda.Event | None = None) -> None:
        """Queue `payload` whose bytes are the CUDA tensor `body` (kept alive until sent).
        `ready` (optional) is an event the link stream waits on before reading `body`."""
        if not body.is_cuda or not body.is_contiguous():
            raise ProtocolError(f"payload {payload.id}: body must be a contiguous CUDA tensor")
        nbytes = body.numel() * body.element_size()
        if nbytes != payload.size_bytes:
            raise ProtocolError(f"payload {payload.id}: body is {nbytes} bytes, "
                                f"declared {payload.size_bytes}")
        with self._cond:
            if self._closing:
                raise ProtocolError("sender is closing")
            self._queue.enqueue(payload)  # ProtocolError on a duplicate id (transport.py:104-105)
            self._bodies[payload.id] = (body.view(torch.uint8).reshape(-1), ready)
            self._offsets[payload.id] = 0
            self._cond.notify()

    def close(self) -> None:
        """Stop accepting payloads; the sender thread drains what is queued, posts the
        end-of-stream frame and exits (wire.py:107-111 semantics)."""
        with self._cond:
            self._closing = True
            self._cond.notify_all()

    def _next_chunk(self):
        """Block until the LinkQueue yields a chunk; False once closed and drained."""
        with self._cond:
            chunk = self._queue.next_chunk()
            while chunk is None and not self._closing:
                self._cond.wait()
                chunk = self._queue.next_chunk()
            return chunk if chunk is not None else False

    def _frame(self, payload_id: int, index: int, flags: int, piece: torch.Tensor | None,
               total: int = 0) -> None:
        size = 0 if piece is None else piece.numel()
        self._stream.synchronize()  # the pinned header staging buffer is reused per frame
        self._hdr_host.numpy()[:] = np.array([payload_id, index, flags, size, total], dtype=np.int64)
        lib = N.lib()
        st = self._stream.cuda_stream
        N.check(lib.pl_memcpy_async(self._hdr_dev.data_ptr(), self._hdr_host.data_ptr(), HEADER_BYTES, st),
                "pl_memcpy_async")
        N.check(lib.pl_p2p_send(self._comm, self._hdr_dev.data_ptr(), HEADER_BYTES, self._peer, st),
                "pl_p2p_send")
        if size:
            N.check(lib.pl_p2p_send(self._comm, piece.data_ptr(), size, self._peer, st), "pl_p2p_send")
        self.frames += 1

    def run(self) -> None:
        try:
            torch.cuda.set_device(self.device)
            while True:
                chunk = self._next_chunk()
                if chunk is False:
                    break
                body, ready = self._bodies[chunk.payload_id]
                off = self._offsets[chunk.payload_id]
                if ready is not None and off == 0:
                    self._stream.wait_event(ready)
                flags = (FLAG_LAST if chunk.is_last else 0) | (
                    FLAG_DECODE if chunk.phase_class is PayloadClass.DECODE else 0)
                self._frame(chunk.payload_id, chunk.index, flags, body[off:off + chunk.size_bytes],
                            body.numel())
                if chunk.is_last:
                    self._stream.synchronize()  # ownership ends once the last chunk is on the wire
                    del self._bodies[chunk.payload_id]
                    del self._offsets[chunk.payload_id]
                else:
                    self._offsets[chunk.payload_id] = off + chunk.size_bytes
            self._frame(0, 0, FLAG_SHUTDOWN, None)
            self._stream.synchronize()
        except Exception:  # the receiver surfaces the failure (wire.py:148-149)
            self.failed = True


class DeviceLinkReceiver(threading.Thread):
    """Reassembles NCCL frames into payloads and hands them to `on_payload` in order."""

    def __init__(self, comm, peer: int, on_payload, name: str = "link-receiver", device=None):
        super().__init__(name=name, daemon=True)
        self._comm, self._peer = comm, peer
        self._on_payload = on_payload
        self._partial: dict = {}
        self.device = torch.device(device if device is not None else torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self._stream = torch.cuda.Stream(self.device)
            self._hdr_dev = torch.empty(HEADER_WORDS, dtype=torch.int64, device=self.device)
        self._hdr_host = torch.empty(HEADER_WORDS, dtype=torch.int64).pin_memory()
        self.failed = False
        self.error: Exception | None = None

    def run(self) -> None:
        lib = N.lib()
        st = self._stream.cuda_stream
        try:
            torch.cuda.set_device(self.device)
            with torch.cuda.stream(self._stream):  # allocations and the final cat stay stream-ordered
                self._loop(lib, st)
        except Exception as e:  # noqa: BLE001 -- mirror wire.py: failures surface via `failed`
            self.error = e
            self.failed = True

    def _loop(self, lib, st) -> None:
        while True:
            N.check(lib.pl_p2p_recv(self._comm, self._hdr_dev.data_ptr(), HEADER_BYTES, self._peer, st),
                    "pl_p2p_recv")
            N.check(lib.pl_memcpy_async(self._hdr_host.data_ptr(), self._hdr_dev.data_ptr(), HEADER_BYTES,
                                        st), "pl_memcpy_async")
            self._stream.synchronize()
            pid, index, flags, size, total = (int(v) for v in self._hdr_host.numpy())
            if flags & FLAG_SHUTDOWN:
                self.failed = bool(self._partial)
                return
            if size < 0 or total < size:
                raise ProtocolError(f"bad frame length {size} of {total}")
            if index == 0:
                if pid in self._partial:
                    raise ProtocolError(f"payload {pid}: duplicate first chunk")
                self._partial[pid] = [torch.empty(total, dtype=torch.uint8, device=self.device), 0, 0]
            state = self._partial.get(pid)
            if state is None or index != state[2]:
                raise ProtocolError(f"payload {pid}: chunk {index} out of order")
            body, off, _ = state
            if off + size > body.numel():
                raise ProtocolError(f"payload {pid}: chunks overrun {body.numel()} bytes")
            if size:
                N.check(lib.pl_p2p_recv(self._comm, body.data_ptr() + off, size, self._peer, st),
                        "pl_p2p_recv")
            state[1], state[2] = off + size, index + 1
            if flags & FLAG_LAST:
                del self._partial[pid]
                if state[1] != body.numel():
                    raise ProtocolError(f"payload {pid}: {state[1]} of {body.numel()} bytes arrived")
                self._stream.synchronize()
                phase = PayloadClass.DECODE if flags & FLAG_DECODE else PayloadClass.PREFILL
                self._on_payload(ReceivedDevicePayload(pid, phase, body))


# ------------------------------------------------------------ cross-host hops
# A pipeline spanning boxes (the paper's deployment: consumer GPUs over the Internet,
# PAPER.md:50) crosses hosts on TCP.  These wrap the reference's own socket backend
# unchanged -- its framing (u32 length + <QII> payload id / chunk index / flags header +
# body, wire.py:3-15, 28-65), LinkQueue draining and reassembly (wire.py:75-185) --
# and add only the device staging at both ends: one device-to-pinned-host copy when
# the producing forward is done, one host-to-device copy of the reassembled payload.

def _ref_wire():
    import importlib

    return importlib.import_module("pipelink.wire")


class HostBridgeLinkSender:
    """``SocketLinkSender`` for a device payload (same contract: start / send / close /
    join; ``send`` raises ProtocolError on a size mismatch or while closing)."""

    def __init__(self, sock, chunk_size, policy=LinkPolicy.DECODE_PRIORITY, name: str = "host-link-sender"):
        self._inner = _ref_wire().SocketLinkSender(sock, chunk_size, policy, name)

    def start(self) -> None:
        self._inner.start()

    def send(self, payload, body: torch.Tensor, ready: torch.cuda.Event | None = None) -> None:
        if body.numel() * body.element_size() != payload.size_bytes:
            raise ProtocolError(f"payload {payload.id}: body is {body.numel() * body.element_size()} bytes, "
                                f"declared {payload.size_bytes}")
        flat = body.reshape(-1).view(torch.uint8)
        if flat.is_cuda:
            host = torch.empty(flat.numel(), dtype=torch.uint8, pin_memory=True)
            st = torch.cuda.current_stream(flat.device)
            if ready is not None:
                st.wait_event(ready)
            host.copy_(flat, non_blocking=True)
            st.synchronize()
        else:
            host = flat
        self._inner.send(payload, host.numpy().tobytes())

    def close(self) -> None:
        self._inner.close()

    def join(self, timeout: float | None = None) -> None:
        self._inner.join(timeout)


class HostBridgeLinkReceiver:
    """``SocketLinkReceiver`` delivering ``ReceivedDevicePayload`` (body on `device`)."""

    def __init__(self, sock, on_payload, name: str = "host-link-receiver", device=None):
        self.device = torch.device(device) if device is not None else torch.device("cpu")

        def deliver(p):
            body = torch.frombuffer(bytearray(p.body), dtype=torch.uint8)
            if self.device.type == "cuda":
                body = body.pin_memory().to(self.device, non_blocking=False)
            on_payload(ReceivedDevicePayload(p.payload_id, p.phase_class, body))

        self._inner = _ref_wire().SocketLinkReceiver(sock, deliver, name)

    @property
    def failed(self) -> bool:
        return self._inner.failed

    def start(self) -> None:
        self._inner.start()

    def run(self) -> None:
        self._inner.run()

    def join(self, timeout: float | None = None) -> None:
        self._inner.join(timeout)
