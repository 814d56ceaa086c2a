"""CPU ORACLE for the LLM fusion scorer -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU legs may import this module.

What it restates: the reference sidecar's scoring convention
(`/root/reference/pkg/sidecar/src/model.ts:35-47` sentence case + BOS tokenisation,
`:116-127` scoreText = sum of natural-log next-token probabilities over the full sequence,
empty text -> 0, `:130-137` scoreEos = best of text + ".", "?", "!" with strict `>`), behind the
reference scorer protocol (`pkg/src/lightbeam/scorer.py:93-163`: `submit`/`next_request_id`,
kinds "score" and "score_eos").  The sidecar's own model is a char-level TypeScript toy that
cannot run here (no Node); the north star names random-init GPT-2/Llama-architecture models,
so the model is transformers' `LlamaForCausalLM` / `GPT2LMHeadModel` in fp32 on the CPU, loaded
with exactly the weights of the GPU scorer.  Tokens: one per word, FNV-1a-64 of the utf-8 word mod (V - 8) + 8,
BOS = 1, ".?!" = 2, 3, 4 (restated here independently of the product's tokenizer).

Parity status: LLM numerics are "parity unpinned" (no reference test pins LLM
scores).  Pinned are the protocol properties the reference tests: chunk invariance, eos ties
-> ".", eos score = score(text + punct), empty text -> 0.
"""

from __future__ import annotations

import itertools

PUNCTS = (".", "?", "!")
PUNCT_IDS = (2, 3, 4)


def fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for x in data:
        h = ((h ^ x) * 0x100000001B3) % (1 << 64)
    return h


def tokens(text: str, vocab: int) -> list[int]:
    sc = text[:1].upper() + text[1:]
    return [1] + [8 + fnv1a64(w.encode("utf-8")) % (vocab - 8) for w in sc.split()]


def hf_model(cfg, state_dict, device="cpu"):
    """transformers LlamaForCausalLM / GPT2LMHeadModel (fp32) with the given weights.  `device`
    "cuda" builds it on the GPU (TF32 off: plain fp32 FMA GEMMs) for the 8B-class shape, which
    does not fit a CPU-speed test budget."""
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    if device != "cpu":
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False

    if getattr(cfg, "arch", "llama") == "gpt2":
        from transformers import GPT2Config, GPT2LMHeadModel

        g = GPT2Config(vocab_size=cfg.vocab_size, n_positions=state_dict["transformer.wpe.weight"].shape[0],
                       n_embd=cfg.hidden, n_layer=cfg.layers, n_head=cfg.heads, n_inner=cfg.ffn,
                       activation_function="gelu_new", layer_norm_epsilon=cfg.rms_eps,
                       resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0, tie_word_embeddings=True)
        m = GPT2LMHeadModel(g).float().eval()
        missing, unexpected = m.load_state_dict(state_dict, strict=False)
        assert not unexpected and all(k.endswith(".attn.bias") or k.endswith("masked_bias")
                                      for k in missing), (missing, unexpected)
        torch.set_grad_enabled(False)
        return m

    kw = dict(vocab_size=cfg.vocab_size, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
              num_hidden_layers=cfg.layers, num_attention_heads=cfg.heads,
              num_key_value_heads=cfg.kv_heads, head_dim=cfg.head_dim, rope_theta=cfg.rope_theta,
              rms_norm_eps=cfg.rms_eps, tie_word_embeddings=True, max_position_embeddings=131072,
              attention_bias=False, mlp_bias=False)
    if cfg.rope_scaling:
        kw["rope_scaling"] = dict(rope_type="llama3", **cfg.rope_scaling)
    with torch.device(device):
        m = LlamaForCausalLM(LlamaConfig(**kw)).float().eval()
    missing, unexpected = m.load_state_dict(state_dict, strict=False, assign=device != "cpu")
    assert not unexpected and all("rotary" in k for k in missing), (missing, unexpected)
    torch.set_grad_enabled(False)
    return m


class OracleLlmScorer:
    """Reference-protocol scorer over a CPU fp32 transformers Llama."""

    def __init__(self, cfg, state_dict, device="cpu"):
        self.cfg = cfg
        self.device = device
        self.model = hf_model(cfg, state_dict, device)
        self._ids = itertools.count(1)
        self.evaluations = 0

    def next_request_id(self) -> int:
        return next(self._ids)

    def _logprobs(self, text: str):
        import torch

        ids = tokens(text, self.cfg.vocab_size)
        out = self.model(torch.tensor([ids], device=self.device)).logits[0].float()
        return ids, torch.log_softmax(out, -1).double().cpu()

    def score(self, text: str) -> float:
        if not text:
            return 0.0
        ids, lsm = self._logprobs(text)
        total = 0.0
        for t in range(len(ids) - 1):  # model.ts:121-125, left-to-right sum
            total += float(lsm[t, ids[t + 1]])
        return total

    def score_eos(self, text: str) -> tuple[str, float]:
        ids, lsm = self._logprobs(text)
        base = 0.0
        for t in range(len(ids) - 1):
            base += float(lsm[t, ids[t + 1]])
        best_p, best = ".", None
        for p, pid in zip(PUNCTS, PUNCT_IDS):  # model.ts:130-137: strict >, ties keep "."
            s = base + float(lsm[len(ids) - 1, pid])
            if best is None or s > best:
                best_p, best = p, s
        return best_p, best

    def submit(self, request):
        from paper_2603_14002_b200.scorer import ScoreResponse

        self.evaluations += len(request.texts)
        if request.kind == "score":
            return ScoreResponse(request.id, tuple(self.score(t) for t in request.texts))
        pairs = [self.score_eos(t) for t in request.texts]
        return ScoreResponse(request.id, tuple(s for _, s in pairs), tuple(p for p, _ in pairs))

    def close(self):
        pass
