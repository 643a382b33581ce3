"""Pin the CPU decoder oracle against the public architecture definition it restates.

The reference pins no decoder arithmetic ("parity unpinned" by
pipelink itself, MoLink runs vLLM).  The oracle follows HF transformers'
LlamaForCausalLM / Qwen2ForCausalLM (transformers 5.5.0 in this image), so it
is checked here against those very modules loaded with the same synthetic
weights: logits agree within the bf16 tolerance below (HF's eager attention
rounds QK^T and P to bf16 where the oracle keeps fp32) and greedy ids agree
exactly under the margin-engineered init.  Skipped where transformers is absent
(the GPU box has the same image).
"""

import pytest
import torch

from oracle import decoder as OD

transformers = pytest.importorskip("transformers")

from paper_2507_05043_b200.spec import TINY  # noqa: E402


def hf_model(spec, seed=0, bias=False):
    o = OD.OracleSpec.from_spec(spec)
    common = dict(hidden_size=spec.d, intermediate_size=spec.ffn, num_attention_heads=spec.Hq,
                  num_key_value_heads=spec.Hkv, head_dim=spec.hd, num_hidden_layers=spec.num_layers,
                  vocab_size=spec.vocab, rms_norm_eps=spec.eps, tie_word_embeddings=False,
                  max_position_embeddings=4096,
                  rope_parameters={"rope_theta": spec.rope_theta, "rope_type": "default"})
    if bias:
        cfg = transformers.Qwen2Config(**common)
        model = transformers.Qwen2ForCausalLM(cfg)
    else:
        cfg = transformers.LlamaConfig(attention_bias=False, mlp_bias=False, **common)
        model = transformers.LlamaForCausalLM(cfg)
    cfg._attn_implementation = "eager"
    model = model.to(torch.bfloat16).eval()
    emb = OD.make_embed(o, seed)
    fn, lm = OD.make_head(o, seed)
    with torch.no_grad():
        model.model.embed_tokens.weight.copy_(emb)
        model.model.norm.weight.copy_(fn)
        model.lm_head.weight.copy_(lm)
        for l, layer in enumerate(model.model.layers):
            W = OD.make_layer(o, l, seed)
            at = layer.self_attn
            at.q_proj.weight.copy_(W.w_q)
            at.k_proj.weight.copy_(W.w_k)
            at.v_proj.weight.copy_(W.w_v)
            if bias:
                at.q_proj.bias.copy_(W.b_q)
                at.k_proj.bias.copy_(W.b_k)
                at.v_proj.bias.copy_(W.b_v)
            at.o_proj.weight.copy_(W.w_o)
            layer.input_layernorm.weight.copy_(W.attn_norm)
            layer.post_attention_layernorm.weight.copy_(W.mlp_norm)
            layer.mlp.gate_proj.weight.copy_(W.w_gate)
            layer.mlp.up_proj.weight.copy_(W.w_up)
            layer.mlp.down_proj.weight.copy_(W.w_down)
    return model


@pytest.mark.parametrize("bias", [False, True])
def test_oracle_logits_match_hf(bias):
    spec = TINY.with_(qkv_bias=bias)
    hf = hf_model(spec, bias=bias)
    ora = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=512)
    ids = OD.prompt(0, 3, 96, spec.vocab)
    with torch.no_grad():
        ref = hf(ids[None]).logits[0].float()                      # [T, V]
    got = ora.teacher_forced(ids[:1], ids[1:])                    # rows 0..T-2
    ref = ref[:-1]
    span = (ref.max() - ref.min()).item()
    err = (got - ref).abs().max().item()
    assert err <= 0.02 + 0.03 * span, f"max |dlogit| {err:.4f}, span {span:.3f}"


def test_oracle_greedy_matches_hf_peaked():
    spec = TINY.with_(peaked=True)
    hf = hf_model(spec)
    ora = OD.OracleModel(OD.OracleSpec.from_spec(spec), seed=0, max_pos=512)
    prompt = OD.prompt(0, 1, 64, spec.vocab)
    toks, _ = ora.greedy([prompt], 12)
    with torch.no_grad():
        seq = prompt.clone()
        out = []
        for _ in range(12):
            nxt = hf(seq[None]).logits[0, -1].float().argmax()
            out.append(int(nxt))
            seq = torch.cat([seq, nxt[None]])
    assert toks[0].tolist() == out
