"""Per-stage decoder executor: resident weights, paged KV cache, C-ABI forward.

``StageExecutor.forward`` is what the reference's simulated compute call
``compute_time(stage.profile, phase, mb.batched_tokens)`` (engine.py:384)
becomes: one ``pl_stage_forward`` call that launches the whole layer range of
the stage on the stage's compute stream.

HBM layout per stage (bf16 unless noted):
  weights        per layer w_qkv [(Hq+2Hkv)hd, d], w_o [d, Hq hd],
                 w_gate_up [2ffn, d] (64-row gate|up blocks), w_down [d, ffn],
                 2 norm vectors (+ qkv bias); embed [V, d] on the first stage,
                 final norm + lm_head [V, d] on the last.  After creation the
                 projection weights and lm_head are repacked in place into
                 pre-swizzled 16 KB tiles [N/128][K/64] (pl_stage_pack_weights)
  KV cache       per layer k/v [num_blocks, Hkv, 64, hd]  (paged, 64-token blocks)
  hidden[slot]   [max_tokens, d] residual stream per in-flight micro-batch slot
                 (the payload buffer the inter-stage links read and write)
  workspace      activations + split-K / attention partials (pl_stage_workspace_bytes)
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import ops
from .spec import (
    BLOCK_SIZE,
    T_ATTN_NORM,
    T_DOWN,
    T_EMBED,
    T_FINAL_NORM,
    T_GATE_UP,
    T_LM_HEAD,
    T_MLP_NORM,
    T_O,
    T_QKV,
    T_QKV_BIAS,
    DecoderSpec,
    layer_tensor_id,
    rope_table,
)

BF16 = torch.bfloat16


def meta_len(T: int, R: int, max_blocks: int) -> int:
    return 3 * T + 3 * R + 1 + R * max_blocks


class StageExecutor:
    """Weights + KV cache + workspace of one pipeline stage on one GPU."""

    def __init__(self, spec: DecoderSpec, stage_idx: int, layers: tuple[int, int], is_first: bool,
                 is_last: bool, device: torch.device, *, seed: int = 0, max_tokens: int,
                 max_reqs: int, max_ctx: int, num_blocks: int, n_slots: int = 1,
                 pack_weights: bool = True):
        self.spec = spec
        self.stage_idx = stage_idx
        self.lo, self.hi = layers
        self.is_first, self.is_last = is_first, is_last
        self.device = torch.device(device)
        self.max_tokens, self.max_reqs, self.max_ctx = max_tokens, max_reqs, max_ctx
        self.max_blocks = (max_ctx + BLOCK_SIZE - 1) // BLOCK_SIZE
        self.num_blocks = num_blocks
        self.n_slots = n_slots
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(self.device)
            self._alloc(seed)
            self._create()
            # projection weights -> pre-swizzled 16 KB tiles (one bulk copy per k-block);
            # afterwards the weight tensors are only meaningful to this stage
            self.packed = bool(pack_weights)
            if self.packed:
                N.call("pl_stage_pack_weights", self.handle, self.stream.cuda_stream)

    # ------------------------------------------------------------- setup
    def _alloc(self, seed: int) -> None:
        s, dev = self.spec, self.device
        e = lambda *shape: torch.empty(*shape, dtype=BF16, device=dev)  # noqa: E731
        self.layers = []
        with torch.cuda.stream(self.stream):
            for l in range(self.lo, self.hi):
                tid = lambda k: layer_tensor_id(l, k)  # noqa: E731
                L = {
                    "attn_norm": ops.fill_hash_(e(s.d), seed, tid(T_ATTN_NORM), s.norm_jitter, 1.0),
                    "w_qkv": ops.fill_hash_(e(s.qkv_dim, s.d), seed, tid(T_QKV), s.weight_scale),
                    "b_qkv": ops.fill_hash_(e(s.qkv_dim), seed, tid(T_QKV_BIAS), s.bias_scale)
                    if s.qkv_bias else None,
                    "w_o": ops.fill_hash_(e(s.d, s.attn_dim), seed, tid(T_O), s.weight_scale),
                    "mlp_norm": ops.fill_hash_(e(s.d), seed, tid(T_MLP_NORM), s.norm_jitter, 1.0),
                    "w_gate_up": ops.fill_hash_(e(2 * s.ffn, s.d), seed, tid(T_GATE_UP), s.weight_scale),
                    "w_down": ops.fill_hash_(e(s.d, s.ffn), seed, tid(T_DOWN), s.weight_scale),
                    "k_cache": torch.zeros(self.num_blocks, s.Hkv, BLOCK_SIZE, s.hd, dtype=BF16, device=dev),
                    "v_cache": torch.zeros(self.num_blocks, s.Hkv, BLOCK_SIZE, s.hd, dtype=BF16, device=dev),
                }
                self.layers.append(L)
            self.embed = self.final_norm = self.lm_head = None
            embed_scale = s.peaked_embed_scale if s.peaked else s.embed_scale
            if self.is_first:
                self.embed = ops.fill_hash_(e(s.vocab, s.d), seed, T_EMBED, embed_scale)
            if self.is_last:
                self.final_norm = ops.fill_hash_(e(s.d), seed, T_FINAL_NORM, s.norm_jitter, 1.0)
                if s.peaked:
                    emb = self.embed if self.embed is not None else ops.fill_hash_(
                        e(s.vocab, s.d), seed, T_EMBED, embed_scale)
                    self.lm_head = (torch.roll(emb, shifts=-1, dims=0).float() * s.lm_alpha).to(BF16)
                    del emb
                else:
                    self.lm_head = ops.fill_hash_(e(s.vocab, s.d), seed, T_LM_HEAD, s.weight_scale)
            self.max_pos = max(self.max_ctx, 1)
            self.cos_sin = rope_table(s, self.max_pos).to(dev)
            # per-slot residual-stream payload buffers and per-slot token outputs
            self.hidden = [e(self.max_tokens, s.d) for _ in range(self.n_slots)]
            self.out_ids = [torch.zeros(self.max_reqs, dtype=torch.int64, device=dev)
                            for _ in range(self.n_slots)] if self.is_last else None
            self.meta_dev = torch.empty(meta_len(self.max_tokens, self.max_reqs, self.max_blocks),
                                        dtype=torch.int32, device=dev)
            self.ids_dev = torch.empty(self.max_tokens, dtype=torch.int64, device=dev) if self.is_first else None
        self.stream.synchronize()

    def _create(self) -> None:
        s = self.spec
        cfg = N.StageConfig()
        cfg.d, cfg.Hq, cfg.Hkv, cfg.hd, cfg.ffn = s.d, s.Hq, s.Hkv, s.hd, s.ffn
        cfg.num_layers = self.hi - self.lo
        cfg.vocab, cfg.eps = s.vocab, s.eps
        cfg.block_size, cfg.max_blocks_per_req, cfg.max_pos = BLOCK_SIZE, self.max_blocks, self.max_pos
        cfg.num_blocks = self.num_blocks
        cfg.is_first, cfg.is_last = int(self.is_first), int(self.is_last)
        cfg.max_tokens, cfg.max_reqs, cfg.max_ctx = self.max_tokens, self.max_reqs, self.max_ctx
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        cfg.embed, cfg.final_norm, cfg.lm_head = ptr(self.embed), ptr(self.final_norm), ptr(self.lm_head)
        cfg.cos_sin = ptr(self.cos_sin)
        self._cfg = cfg
        arr = (N.LayerWeights * max(1, len(self.layers)))()
        for i, L in enumerate(self.layers):
            for k in ("attn_norm", "w_qkv", "b_qkv", "w_o", "mlp_norm", "w_gate_up", "w_down",
                      "k_cache", "v_cache"):
                setattr(arr[i], k, ptr(L[k]))
        self._layer_arr = arr
        lib = N.lib()
        ws_bytes = lib.pl_stage_workspace_bytes(C.byref(cfg))
        self.workspace = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=self.device)
        h = C.c_void_p()
        N.check(lib.pl_stage_create(C.byref(cfg), arr, self.workspace.data_ptr(), self.workspace.numel(),
                                    C.byref(h)), "pl_stage_create")
        self.handle = h
        self._mb = N.MicroBatch()
        self._stream_ptr = C.c_void_p(self.stream.cuda_stream)
        self._forward = lib.pl_stage_forward

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib().pl_stage_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- forward
    def forward(self, slot: int, T: int, R: int, decode: bool, max_seqlen: int, max_ctx: int,
                last_token: torch.Tensor | None = None, n_decode: int = 0) -> None:
        """Launch the stage forward for the micro-batch whose metadata sits in meta_dev
        (and prompt ids in ids_dev) on self.stream; hidden[slot] in, hidden[slot] out,
        out_ids[slot] on the last stage.  n_decode > 0 with decode=False: a mixed batch
        whose first n_decode requests decode one token each."""
        mb = self._mb
        mixed = (not decode) and n_decode > 0
        mb.T, mb.R, mb.phase = T, R, 2 if mixed else (1 if decode else 0)
        mb.n_decode = n_decode if mixed else 0
        mb.max_seqlen, mb.max_ctx = max_seqlen, max_ctx
        mb.meta = self.meta_dev.data_ptr()
        mb.token_ids = self.ids_dev.data_ptr() if (self.is_first and not decode) else None
        mb.last_token = last_token.data_ptr() if (self.is_first and (decode or mixed)) else None
        mb.hidden = self.hidden[slot].data_ptr()
        mb.out_ids = self.out_ids[slot].data_ptr() if self.is_last else None
        rc = self._forward(self.handle, C.byref(mb), self._stream_ptr)
        if rc:
            N.check(rc, "pl_stage_forward")

    # --------------------------------------------------- direct requests
    def greedy(self, prompts: list, n_steps: int, slot: int = 0):
        """Greedy generation for explicit requests without the scheduler (whole model in
        this stage: first and last): one prefill micro-batch of every prompt, then
        n_steps - 1 decode micro-batches, each fed this stage's own argmax ids.  Returns
        (ids [R, n_steps] int64, hn [n_steps, R, d] bf16 on the host), hn = the final
        RMSNorm of each request's newest row -- what the lm_head / argmax read."""
        if not (self.is_first and self.is_last):
            raise ValueError("greedy() needs a stage holding the whole model")
        lens = [len(p) for p in prompts]
        R, T = len(lens), sum(lens)
        if T > self.max_tokens or R > self.max_reqs or max(lens) + n_steps > self.max_ctx:
            raise ValueError("requests exceed the stage's capacity")
        mb_ = self.max_blocks
        need = [-(-(n + n_steps) // BLOCK_SIZE) for n in lens]
        if sum(need) > self.num_blocks:
            raise ValueError("paged KV cache too small")
        rows = np.zeros((R, mb_), dtype=np.int32)
        b = 0
        for r, k in enumerate(need):
            rows[r, :k] = np.arange(b, b + k)
            b += k
        cu = np.concatenate([[0], np.cumsum(lens)])
        pos = np.concatenate([np.arange(n) for n in lens])
        req_of = np.repeat(np.arange(R), lens)
        slots = rows[req_of, pos // BLOCK_SIZE] * BLOCK_SIZE + pos % BLOCK_SIZE
        last_token = torch.zeros(R, dtype=torch.int64, device=self.device)
        ids_out, hn_out = [], []
        with torch.cuda.device(self.device):
            for step in range(n_steps):
                if step == 0:
                    meta = build_meta(T, R, mb_, pos, slots, req_of, cu, lens, cu[1:] - 1, rows)
                    ids = np.concatenate([np.asarray(p, dtype=np.int64) for p in prompts])
                    self.ids_dev[:T].copy_(torch.from_numpy(ids))
                    last = torch.tensor(cu[1:] - 1, dtype=torch.int32, device=self.device)
                else:
                    p = np.array([lens[r] + step - 1 for r in range(R)])
                    ds = rows[np.arange(R), p // BLOCK_SIZE] * BLOCK_SIZE + p % BLOCK_SIZE
                    meta = build_meta(R, R, mb_, p, ds, np.arange(R), np.arange(R + 1), p + 1,
                                      np.arange(R), rows)
                    last = torch.arange(R, dtype=torch.int32, device=self.device)
                self.meta_dev[: meta.size].copy_(torch.from_numpy(meta))
                torch.cuda.synchronize(self.device)
                if step == 0:
                    self.forward(slot, T, R, False, max(lens), max(lens))
                else:
                    self.forward(slot, R, R, True, 1, max(lens) + step, last_token=last_token)
                self.stream.synchronize()
                out = self.out_ids[slot][:R].clone()
                last_token.copy_(out)
                hn = ops.rmsnorm(self.hidden[slot], self.final_norm, self.spec.eps, row_idx=last)
                ids_out.append(out.cpu())
                hn_out.append(hn.cpu())
        return torch.stack(ids_out, 1).numpy(), torch.stack(hn_out)

    # ------------------------------------------------------------- probe
    def probe(self, layer: int) -> None:
        N.call("pl_stage_probe", self.handle, layer)

    def probe_read(self, cap: int = 65536) -> tuple[np.ndarray, np.ndarray]:
        """(ms [n, 5], meta [n, 3] = (phase, T, kind)); see pl_stage_probe_read."""
        ms = np.zeros(cap * 5, dtype=np.float32)
        meta = np.zeros(cap * 3, dtype=np.int32)
        n = C.c_int32()
        N.call("pl_stage_probe_read", self.handle, ms.ctypes.data_as(C.POINTER(C.c_float)),
               meta.ctypes.data_as(C.POINTER(C.c_int32)), cap, C.byref(n))
        k = n.value
        return ms[: k * 5].reshape(k, 5), meta[: k * 3].reshape(k, 3)

    def weight_bytes(self) -> int:
        n = sum(t.numel() * t.element_size() for L in self.layers for k, t in L.items()
                if t is not None and not k.endswith("cache"))
        for t in (self.embed, self.final_norm, self.lm_head):
            if t is not None:
                n += t.numel() * t.element_size()
        return n


def build_meta(T: int, R: int, max_blocks: int, pos, slot, req_slot, cu, ctx, last, bt) -> np.ndarray:
    """Pack the int32 micro-batch metadata in the layout pl_stage_forward expects."""
    out = np.empty(meta_len(T, R, max_blocks), dtype=np.int32)
    o = 0
    for arr, n in ((pos, T), (slot, T), (req_slot, T), (cu, R + 1), (ctx, R), (last, R),
                   (bt, R * max_blocks)):
        out[o:o + n] = np.asarray(arr, dtype=np.int32).reshape(-1)[:n]
        o += n
    return out
