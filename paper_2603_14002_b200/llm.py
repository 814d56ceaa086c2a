"""LLM scorer for delayed fusion: a random-init Llama-architecture model on the GPU.

Plugin contract (the reference's, `pkg/src/lightbeam/scorer.py:93-163,269-325`): `LlamaScorer`
has `submit(ScoreRequest) -> ScoreResponse` and `next_request_id()`, so any caller of the
reference protocol (including the reference decoder itself) can use it with host strings.

Scoring convention (the reference sidecar, `pkg/sidecar/src/model.ts:35-47,116-137`, at word
rather than character granularity): tokens = [BOS] + tokens(sentenceCase(text)); score = sum over
positions of the natural-log next-token probability; empty text scores 0; `score_eos` returns
the best of `text + "."`, `"?"`, `"!"` with strict `>` (ties keep "."), where the punctuation is
one more token after the text: score_eos(text, p) = score(text) + log P(p | text).

Tokenizer (synthetic -- there is no Llama tokenizer offline): one token per
whitespace-separated word, id = 8 + FNV-1a-64(utf-8 word) mod (vocab - 8); BOS = 1; ".", "?",
"!" = 2, 3, 4.  Sentence case upper-cases the first character of the text (model.ts:35-38), so
the first word has its own token.

Two execution paths share the weights:
  * `submit()` -- every text is a full forward pass (plain torch, bf16, SDPA), no KV reuse: the
    "CPU search + GPU LLM" split of the paper and the reference arm of bench.py;
  * the device path (`DeviceLlmSession`) the decoder drives when it decodes on the GPU: texts are
    paths of one prefix trie whose nodes are evaluated once (lb_llm_* in csrc/lb_llm.cu); the
    transformer body's GEMMs run on the tensor cores through torch (cuBLAS, bf16 in, fp32
    accumulate), everything around them is hand-written kernels.
"""

from __future__ import annotations

import ctypes as C
import itertools
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DeviceError, ScorerError
from .scorer import PUNCTS, ScoreRequest, ScoreResponse

BOS_ID = 1
PUNCT_IDS = (2, 3, 4)
FIRST_WORD_ID = 8


@dataclass(frozen=True)
class LlmConfig:
    name: str
    vocab_size: int
    hidden: int
    layers: int
    heads: int
    kv_heads: int
    ffn: int
    head_dim: int
    rope_theta: float = 500000.0
    rope_scaling: dict | None = None  # llama3 rope parameters
    rms_eps: float = 1e-5
    init_std: float = 0.02
    arch: str = "llama"  # "llama" | "gpt2" (learned positions, LayerNorm, GELU, biases, MHA)
    #                      | "tinychar" (the reference sidecar's TinyCausalLM, charlm.py)
    identifier: str = ""  # tinychar: the model identifier its weights derive from (model.ts:93)

    def n_params(self) -> int:
        att = self.hidden * (self.heads + 2 * self.kv_heads) * self.head_dim
        att += self.heads * self.head_dim * self.hidden
        mlp = (3 if self.arch == "llama" else 2) * self.hidden * self.ffn
        return self.vocab_size * self.hidden + self.layers * (att + mlp + 2 * self.hidden) + self.hidden

    def flops_per_token(self) -> float:
        """2 x (body + LM head) multiply-adds per forwarded token (attention over the short
        prefix excluded)."""
        att = self.hidden * (self.heads + 2 * self.kv_heads) * self.head_dim
        att += self.heads * self.head_dim * self.hidden
        mlp = (3 if self.arch == "llama" else 2) * self.hidden * self.ffn
        return 2.0 * (self.layers * (att + mlp) + self.vocab_size * self.hidden)


_LLAMA3_1B_ROPE = {"factor": 32.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
                   "original_max_position_embeddings": 8192}
_LLAMA3_8B_ROPE = {"factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
                   "original_max_position_embeddings": 8192}

PRESETS = {
    # config 1 of BASELINE.json: the tiny GPT-2-style model (2 layers, d = 64)
    "tiny-gpt2": LlmConfig("tiny-gpt2", 4096, 64, 2, 1, 1, 256, 64, arch="gpt2"),
    # a tiny Llama-architecture model (fast tests of the Llama kernels)
    "tiny": LlmConfig("tiny", 4096, 128, 2, 2, 1, 512, 64),
    # config 1 with the reference's own scorer model: the sidecar's TinyCausalLM (model.ts:20-26:
    # char-level, dim 32, 2 heads of 16 -- padded to 64 on the device, q pre-scaled by 2 so the
    # 1/sqrt(64) softmax scale equals model.ts's 1/sqrt(16) exactly -- 2 layers, untied head)
    "tiny-char-lm": LlmConfig("tiny-char-lm", 97, 32, 2, 2, 2, 128, 64, rms_eps=1e-5,
                              arch="tinychar", identifier="tiny-char-lm-v1"),
    # config 3: Llama-3.2-1B architecture
    "llama-3.2-1b": LlmConfig("llama-3.2-1b", 128256, 2048, 16, 32, 8, 8192, 64,
                              rope_scaling=_LLAMA3_1B_ROPE),
    # config 5: 8B-class = Llama-3.1-8B architecture
    "llama-3.1-8b": LlmConfig("llama-3.1-8b", 128256, 4096, 32, 32, 8, 14336, 128,
                              rope_scaling=_LLAMA3_8B_ROPE),
}


def get_config(cfg) -> LlmConfig:
    if isinstance(cfg, LlmConfig):
        return cfg
    if cfg not in PRESETS:
        raise ValueError(f"unknown LLM preset {cfg!r}; choose from {sorted(PRESETS)}")
    return PRESETS[cfg]


# ------------------------------------------------------------------------------ tokenizer
def _fnv1a64(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for x in data:
        h ^= x
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def sentence_case(text: str) -> str:
    """model.ts:35-38: upper-case the first character."""
    return text[:1].upper() + text[1:] if text else text


class WordTokenizer:
    def __init__(self, vocab_size: int):
        if vocab_size <= FIRST_WORD_ID:
            raise ValueError("vocab too small")
        self.vocab_size = vocab_size
        self.bos = BOS_ID
        self.punct = dict(zip(PUNCTS, PUNCT_IDS))
        self._cache: dict[str, int] = {}

    def word_id(self, word: str) -> int:
        got = self._cache.get(word)
        if got is None:
            got = FIRST_WORD_ID + _fnv1a64(word.encode("utf-8")) % (self.vocab_size - FIRST_WORD_ID)
            self._cache[word] = got
        return got

    def encode(self, text: str) -> list[int]:
        """[BOS] + one id per word of the sentence-cased text."""
        return [self.bos] + [self.word_id(w) for w in sentence_case(text).split()]

    def surface_tables(self, surfaces) -> tuple[np.ndarray, np.ndarray]:
        """(token mid-sentence, token as the first word) per lexicon surface."""
        low = np.fromiter((self.word_id(s) for s in surfaces), dtype=np.int32, count=len(surfaces))
        cap = np.fromiter((self.word_id(sentence_case(s)) for s in surfaces), dtype=np.int32,
                          count=len(surfaces))
        return low, cap


# ------------------------------------------------------------------------------ weights
def rope_inv_freq(cfg: LlmConfig):
    """Llama rotary frequencies, llama3 frequency scaling when configured (the formula of the
    Llama-3 release, as implemented by transformers' `_compute_llama3_parameters`)."""
    import torch

    hd = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    rs = cfg.rope_scaling
    if not rs:
        return inv
    factor, lo, hi = rs["factor"], rs["low_freq_factor"], rs["high_freq_factor"]
    old = rs["original_max_position_embeddings"]
    lo_wl, hi_wl = old / lo, old / hi
    wl = 2 * math.pi / inv
    inv_l = torch.where(wl > lo_wl, inv / factor, inv)
    smooth = (old / wl - lo) / (hi - lo)
    smoothed = (1 - smooth) * inv_l / factor + smooth * inv_l
    medium = ~(wl < hi_wl) * ~(wl > lo_wl)
    return torch.where(medium, smoothed, inv_l)


class LlamaWeights:
    """Random-init weights (normal(0, init_std) for every linear/embedding, ones for RMSNorm --
    the Llama initialisation) as bf16 device tensors; q/k/v and gate/up are stored fused."""

    def __init__(self, cfg: LlmConfig, seed: int = 0, device: str = "cuda:0", max_pos: int = 4096):
        import torch

        self.cfg = cfg
        self.device = torch.device(device)
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        std = cfg.init_std

        def rnd(*shape):
            w = torch.empty(shape, dtype=torch.float32, device=self.device)
            w.normal_(0.0, std, generator=g)
            return w.to(torch.bfloat16)

        H, hd = cfg.hidden, cfg.head_dim
        self.layers = []
        if cfg.arch == "tinychar":
            self._init_tinychar(max_pos)
            return
        self.emb = rnd(cfg.vocab_size, H)
        if cfg.arch == "gpt2":
            self._init_gpt2(rnd, max_pos)
            return
        for _ in range(cfg.layers):
            wq = rnd(cfg.heads * hd, H)
            wk = rnd(cfg.kv_heads * hd, H)
            wv = rnd(cfg.kv_heads * hd, H)
            wo = rnd(H, cfg.heads * hd)
            wg = rnd(cfg.ffn, H)
            wu = rnd(cfg.ffn, H)
            wd = rnd(H, cfg.ffn)
            self.layers.append({
                "ln1": torch.ones(H, dtype=torch.float32, device=self.device),
                "wqkv": torch.cat([wq, wk, wv], 0).contiguous(),
                "wo": wo,
                "ln2": torch.ones(H, dtype=torch.float32, device=self.device),
                "wgu": torch.cat([wg, wu], 0).contiguous(),
                "wd": wd,
            })
        self.norm = torch.ones(H, dtype=torch.float32, device=self.device)
        inv = rope_inv_freq(cfg)
        pos = torch.arange(max_pos, dtype=torch.float32)
        freqs = pos[:, None] * inv[None, :]
        self.cos = freqs.cos().to(self.device).contiguous()
        self.sin = freqs.sin().to(self.device).contiguous()
        self.max_pos = max_pos

    def _init_gpt2(self, rnd, max_pos):
        """GPT-2 layout: learned positions, pre-LayerNorm blocks, fused q/k/v with biases, GELU
        MLP; every weight, bias and position row ~ N(0, init_std) (biases and LayerNorm shifts
        random too, so the kernels' bias paths are exercised), LayerNorm gains 1."""
        import torch

        cfg, H, dev = self.cfg, self.cfg.hidden, self.device
        f32 = lambda t: t.float().contiguous()  # noqa: E731  (bf16-valued fp32 vectors)
        self.wpe = f32(rnd(max(max_pos, 1024), H))
        for _ in range(cfg.layers):
            self.layers.append({
                "ln1": torch.ones(H, dtype=torch.float32, device=dev), "ln1b": f32(rnd(H)),
                "wqkv": rnd(3 * H, H), "bqkv": f32(rnd(3 * H)),
                "wo": rnd(H, H), "bo": f32(rnd(H)),
                "ln2": torch.ones(H, dtype=torch.float32, device=dev), "ln2b": f32(rnd(H)),
                "wfc": rnd(cfg.ffn, H), "bfc": f32(rnd(cfg.ffn)),
                "wd": rnd(H, cfg.ffn), "bd": f32(rnd(H)),
            })
        self.norm = torch.ones(H, dtype=torch.float32, device=dev)
        self.normb = f32(rnd(H))
        half = cfg.head_dim // 2  # no rotary embedding: identity tables for the shared kernel
        self.cos = torch.ones((max_pos, half), dtype=torch.float32, device=dev)
        self.sin = torch.zeros((max_pos, half), dtype=torch.float32, device=dev)
        self.max_pos = max_pos

    def _init_tinychar(self, max_pos):
        """TinyCausalLM (charlm.tiny_char_weights, model.ts:93-117) on the GPT-2-style kernels:
        LayerNorm gain 1 / shift 0 (model.ts:220-236 has no affine), no biases, tanh GELU,
        learned positions, MHA with head_dim padded 16 -> 64 (zero rows / columns; q x 2 so the
        kernel's 1/sqrt(64) scale is model.ts's 1/sqrt(16)), untied LM head.  The float64
        weights are not bf16-exact, so every GEMM weight is a bf16 hi + lo pair (the lo term is
        one more GEMM against the hi half of the activation), the input rows are fp32 and the
        next-token dot products read an fp32 copy of the head."""
        import torch

        from .charlm import VOCAB, tiny_char_weights

        cfg, H, dev = self.cfg, self.cfg.hidden, self.device
        nh, hdp = cfg.heads, cfg.head_dim
        w = tiny_char_weights(cfg.identifier or "tiny-char-lm-v1", H, nh, cfg.layers, 1024)
        hd = H // nh
        self.f64 = w

        def hilo(a):
            t = torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
            hi = t.to(torch.bfloat16)
            return hi.contiguous(), (t - hi.double()).to(torch.bfloat16).contiguous()

        f32 = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float32, device=dev)  # noqa: E731
        self.emb_in = f32(w["embed"])
        self.wpe = f32(w["pos"])
        vpad = (VOCAB + 7) // 8 * 8  # GEMM row pitch; the log-sum-exp reads the first VOCAB
        head = np.zeros((vpad, H))
        head[:VOCAB] = w["wout"].T
        self.emb, self.head_lo = hilo(head)
        self.head32 = f32(w["wout"].T)
        ones = lambda n: torch.ones(n, dtype=torch.float32, device=dev)  # noqa: E731
        zeros = lambda n: torch.zeros(n, dtype=torch.float32, device=dev)  # noqa: E731
        for li in range(cfg.layers):
            wqkv = np.zeros((3 * nh * hdp, H))
            for h in range(nh):
                for part, name, sc in ((0, "wq", 2.0), (1, "wk", 1.0), (2, "wv", 1.0)):
                    r0 = part * nh * hdp + h * hdp
                    wqkv[r0:r0 + hd] = sc * w[f"{name}.{li}"][:, h * hd:(h + 1) * hd].T
            wo = np.zeros((H, nh * hdp))
            for h in range(nh):
                wo[:, h * hdp:h * hdp + hd] = w[f"wo.{li}"][h * hd:(h + 1) * hd, :].T
            L = {"ln1": ones(H), "ln1b": zeros(H), "ln2": ones(H), "ln2b": zeros(H),
                 "bqkv": None, "bo": None, "bfc": None, "bd": None}
            for k, m in (("wqkv", wqkv), ("wo", wo), ("wfc", w[f"w1.{li}"].T),
                         ("wd", w[f"w2.{li}"].T)):
                L[k], L[k + "_lo"] = hilo(m)
            self.layers.append(L)
        self.norm, self.normb = ones(H), zeros(H)
        self.cos = torch.ones((max_pos, hdp // 2), dtype=torch.float32, device=dev)
        self.sin = torch.zeros((max_pos, hdp // 2), dtype=torch.float32, device=dev)
        self.max_pos = max_pos

    def hf_state_dict(self, device="cpu") -> dict:
        """fp32 tensors (on `device`) under transformers' LlamaForCausalLM / GPT2LMHeadModel
        names (for the test oracle)."""
        cfg = self.cfg
        if cfg.arch == "gpt2":
            c = lambda t: t.float().to(device)  # noqa: E731
            sd = {"transformer.wte.weight": c(self.emb), "transformer.wpe.weight": c(self.wpe),
                  "transformer.ln_f.weight": c(self.norm), "transformer.ln_f.bias": c(self.normb),
                  "lm_head.weight": c(self.emb)}
            for i, L in enumerate(self.layers):
                p = f"transformer.h.{i}."
                sd[p + "ln_1.weight"], sd[p + "ln_1.bias"] = c(L["ln1"]), c(L["ln1b"])
                sd[p + "ln_2.weight"], sd[p + "ln_2.bias"] = c(L["ln2"]), c(L["ln2b"])
                sd[p + "attn.c_attn.weight"] = c(L["wqkv"]).t().contiguous()  # Conv1D: [in, out]
                sd[p + "attn.c_attn.bias"] = c(L["bqkv"])
                sd[p + "attn.c_proj.weight"] = c(L["wo"]).t().contiguous()
                sd[p + "attn.c_proj.bias"] = c(L["bo"])
                sd[p + "mlp.c_fc.weight"] = c(L["wfc"]).t().contiguous()
                sd[p + "mlp.c_fc.bias"] = c(L["bfc"])
                sd[p + "mlp.c_proj.weight"] = c(L["wd"]).t().contiguous()
                sd[p + "mlp.c_proj.bias"] = c(L["bd"])
            return sd
        qn, kn = cfg.heads * cfg.head_dim, cfg.kv_heads * cfg.head_dim
        sd = {"model.embed_tokens.weight": self.emb.float().to(device),
              "model.norm.weight": self.norm.float().to(device),
              "lm_head.weight": self.emb.float().to(device)}
        for i, L in enumerate(self.layers):
            p = f"model.layers.{i}."
            w = L["wqkv"].float().to(device)
            sd[p + "self_attn.q_proj.weight"] = w[:qn]
            sd[p + "self_attn.k_proj.weight"] = w[qn: qn + kn]
            sd[p + "self_attn.v_proj.weight"] = w[qn + kn:]
            sd[p + "self_attn.o_proj.weight"] = L["wo"].float().to(device)
            gu = L["wgu"].float().to(device)
            sd[p + "mlp.gate_proj.weight"] = gu[: cfg.ffn]
            sd[p + "mlp.up_proj.weight"] = gu[cfg.ffn:]
            sd[p + "mlp.down_proj.weight"] = L["wd"].float().to(device)
            sd[p + "input_layernorm.weight"] = L["ln1"].float().to(device)
            sd[p + "post_attention_layernorm.weight"] = L["ln2"].float().to(device)
        return sd


# ------------------------------------------------------------------------------ scorer
class LlamaScorer:
    """Delayed-fusion scorer backed by a random-init Llama-architecture model on one GPU."""

    PRECISIONS = ("bf16x2", "bf16")

    def __init__(self, config="tiny", seed: int = 0, device: int = 0, max_slots: int | None = None,
                 max_depth: int = 1023, row_chunk: int = 16384, lm_chunk: int = 2048,
                 precision: str = "bf16x2", lm_head: str = "fused", fused_swiglu: bool = False,
                 fused_swiglu_min_rows: int = 4096, graphs: bool | None = None,
                 lse_split: bool = False):
        """precision: "bf16x2" (default) feeds every body GEMM the activation as a hi+lo pair of
        bf16 values against duplicated bf16 weights -- fp32-equivalent activations on the bf16
        tensor cores, scores within ~1e-3 of an fp32 forward even for 40-token texts -- and keeps
        q/K/V in fp32; "bf16" is one bf16 operand per activation (half the body FLOPs; measured
        per-text error vs fp32 grows to ~0.1 at 40 tokens on the random-init 1B model).
        lse_split: in bf16x2, also run the LM-head log-sum-exp GEMM on hi|lo activations.  Off by
        default: a token's log-prob is h.E[token] with the fp32 final hidden state (lp kernel)
        minus the row's LSE, and the LSE -- a softmax-weighted average of logits -- barely feels
        the hi-only rounding (tools/prec_lse.py: 39-token text error max 1.1e-3 on the 1B model,
        2.1e-3 on the 8B one, against 5.6e-4 / 1.7e-3 with hi|lo), for half the head FLOPs."""
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("LlamaScorer needs a CUDA device (no CPU path)")
        torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
        self.cfg = get_config(config)
        self.device = device
        self.seed = seed
        if self.cfg.arch == "tinychar":
            max_depth = min(max_depth, 1023)  # model.ts:25 maxContext 1024 positions
            lm_head = "cublas"  # untied 97-token head: hi/lo GEMM + log-sum-exp kernel
        self.weights = LlamaWeights(self.cfg, seed, f"cuda:{device}", max_pos=max(max_depth + 2, 1100))
        if self.cfg.arch == "tinychar":
            from .charlm import CharTokenizer

            self.tokenizer = CharTokenizer()
        else:
            self.tokenizer = WordTokenizer(self.cfg.vocab_size)
        self.max_slots = max_slots
        self.max_depth = max_depth
        self.row_chunk = row_chunk
        self.lm_chunk = lm_chunk
        self.evaluations = 0
        self._ids = itertools.count(1)
        if precision not in self.PRECISIONS:
            raise ValueError(f"precision must be one of {self.PRECISIONS}")
        if self.cfg.arch == "tinychar" and precision != "bf16x2":
            raise ValueError("the TinyCausalLM runs in bf16x2 only (float64 weights as hi+lo)")
        if lm_head not in ("fused", "cublas"):
            raise ValueError("lm_head must be 'fused' (tcgen05 GEMM + log-sum-exp) or 'cublas'")
        self.lm_head = lm_head
        self.precision = precision
        self.split = precision == "bf16x2"
        self.lse_split = bool(lse_split) and self.split
        # gate/up rows interleaved in 128-row blocks for the tcgen05 GEMM with the SwiGLU epilogue
        # (opt-in, for waves of >= fused_swiglu_min_rows rows).  On the 13.4k-row final wave of
        # config 3 its 128x256 tiles keep the tensor pipe ~81% busy and the gate/up product never
        # reaches HBM, but measured per step it only ties cuBLAS + the SwiGLU kernel (and loses
        # on small waves to cuBLAS's per-shape tiles), so it is off by default.
        self.fused_swiglu = fused_swiglu and self.cfg.arch == "llama" and self.cfg.ffn % 128 == 0
        self.fused_swiglu_min_rows = fused_swiglu_min_rows
        if self.fused_swiglu:
            F, H = self.cfg.ffn, self.cfg.hidden
            for L in self.weights.layers:
                g, u = L["wgu"][:F].view(F // 128, 128, H), L["wgu"][F:].view(F // 128, 128, H)
                L["wgui"] = torch.stack([g, u], 1).reshape(2 * F, H).contiguous()
        if self.split:  # [W | W]: one GEMM computes hi @ W^T + lo @ W^T with fp32 accumulation
            for L in self.weights.layers:
                for k in ("wqkv", "wo", "wgu", "wgui", "wfc", "wd"):
                    if k in L:
                        L[k + "2"] = torch.cat([L[k], L[k]], 1).contiguous()
            if self.lse_split or lm_head == "cublas":
                self.emb2 = torch.cat([self.weights.emb, self.weights.emb], 1).contiguous()
        self.device_llm_scorer = self  # the GPU decoder drives this scorer on the device
        # graph mode: whole decodes replay as one CUDA graph (events padded to a fixed row
        # capacity, no host round trip per event) -- for small models, where an event is
        # launch-bound; big models keep the eager path (exact row counts, large GEMMs)
        self.graphs = (self.cfg.hidden <= 256) if graphs is None else bool(graphs)
        # the weights were built on the legacy default stream; decodes may run on non-blocking
        # streams that do not order after it
        torch.cuda.synchronize(device)

    # ---- reference protocol (host strings, one full forward per text, no KV reuse)
    def executed_flops_per_token(self) -> float:
        """FLOPs the tensor cores execute per forwarded token: bf16x2 runs every body GEMM on
        hi|lo activations (twice the algorithmic work) and the LM head once (or twice with
        lse_split)."""
        c = self.cfg
        head = 2.0 * c.vocab_size * c.hidden
        body = c.flops_per_token() - head
        k = 2 if self.split else 1
        return k * body + (2 if self.lse_split else 1) * head

    def next_request_id(self) -> int:
        return next(self._ids)

    def submit(self, request: ScoreRequest) -> ScoreResponse:
        self.evaluations += len(request.texts)
        if request.kind == "score":
            return ScoreResponse(request.id, tuple(self.score_texts_dense(list(request.texts))))
        if request.kind == "score_eos":
            pairs = self.score_eos_dense(list(request.texts))
            return ScoreResponse(request.id, tuple(s for _, s in pairs), tuple(p for p, _ in pairs))
        raise ScorerError(f"unknown request kind {request.kind!r}", request.id)

    def close(self):
        pass

    def score_texts_dense(self, texts: list[str]) -> list[float]:
        return [s for s, _ in self._dense(texts, eos=False)]

    def score_eos_dense(self, texts: list[str]) -> list[tuple[str, float]]:
        out = []
        for s, plp in self._dense(texts, eos=True):
            best, bs = 0, s + plp[0]
            for j in (1, 2):
                v = s + plp[j]
                if v > bs:
                    best, bs = j, v
            out.append((PUNCTS[best], bs))
        return out

    def _dense(self, texts: list[str], eos: bool, batch_tokens: int = 1 << 16):
        """Full-sequence forward per text (plain torch: bf16 GEMMs, SDPA, fp32 log-softmax)."""
        import torch

        if self.cfg.arch == "tinychar":  # float64, as the sidecar computes (model.ts:119-209)
            return self._dense_tinychar(texts, eos)
        res: list = [None] * len(texts)
        toks = [self.tokenizer.encode(t) for t in texts]
        order = sorted(range(len(texts)), key=lambda i: len(toks[i]))
        i = 0
        while i < len(order):
            S = len(toks[order[i]])
            j = i
            while j < len(order) and (j - i + 1) * len(toks[order[j]]) <= batch_tokens:
                j += 1
            j = max(j, i + 1)
            idx = order[i:j]
            S = max(len(toks[k]) for k in idx)
            if S > self.weights.max_pos:
                raise ScorerError(f"text longer than {self.weights.max_pos} tokens")
            ids = torch.zeros((len(idx), S), dtype=torch.long)
            for r, k in enumerate(idx):
                ids[r, : len(toks[k])] = torch.tensor(toks[k])
            with torch.no_grad():
                lp_all, plp = self._dense_forward(ids.to(self.weights.device), [len(toks[k]) for k in idx],
                                                  eos)
            for r, k in enumerate(idx):
                res[k] = (lp_all[r], plp[r] if eos else None)
            i = j
        return res

    def _dense_tinychar(self, texts, eos):
        from .charlm import dense_scores

        return dense_scores(self.weights.f64, texts, self.weights.device, eos)

    def _dense_forward(self, ids, lens, eos):
        split = frozenset(("qkv", "o", "gu", "down", "attn", "lm")) if self.split else frozenset()
        return dense_forward(self.weights, ids, lens, eos, split=split)

    # ---- device path
    def session(self, batch) -> "DeviceLlmSession":
        if batch.dm.device != self.device:
            raise DeviceError(f"LlamaScorer lives on cuda:{self.device} but the decode runs on "
                              f"cuda:{batch.dm.device}; build one scorer per device")
        sess = getattr(batch, "_llm_session", None)
        if sess is None or sess.scorer is not self:
            if sess is not None:
                sess.destroy()
            sess = DeviceLlmSession(self, batch)
            batch._llm_session = sess
        return sess


def dense_forward(W: LlamaWeights, ids, lens, eos: bool, exact_fp32: bool = False,
                  split: frozenset = frozenset()):
    """Full-sequence Llama forward of a padded [B, S] batch (plain torch: bf16 GEMMs with fp32
    outputs and an fp32 residual stream; `exact_fp32` runs everything in fp32 -- the CPU
    semantic check against transformers).  Returns (sum of next-token log-probs per row,
    log-probs of ".?!" after each row's last token if `eos`)."""
    import torch
    import torch.nn.functional as F

    cfg = W.cfg
    B, S = ids.shape
    hd, nh, nkv = cfg.head_dim, cfg.heads, cfg.kv_heads
    opd = torch.float32 if exact_fp32 else torch.bfloat16

    def mm(a, w, tag=None):
        a2 = a.reshape(-1, a.shape[-1])
        if exact_fp32:
            out = a2.float() @ w.float().t()
        elif tag in split:  # bf16 hi/lo split of the activation: two bf16 GEMMs, fp32 accumulate
            hi = a2.float().to(torch.bfloat16)
            lo = (a2.float() - hi.float()).to(torch.bfloat16)
            out = torch.mm(hi, w.t(), out_dtype=torch.float32) + torch.mm(lo, w.t(), out_dtype=torch.float32)
        else:
            out = torch.mm(a2.to(torch.bfloat16), w.t(), out_dtype=torch.float32)
        return out.view(*a.shape[:-1], -1)

    if cfg.arch == "gpt2":
        return _dense_forward_gpt2(W, ids, lens, eos, exact_fp32, split)
    x = W.emb[ids].float()
    cos = W.cos[:S].repeat(1, 2)[None, None]
    sin = W.sin[:S].repeat(1, 2)[None, None]

    def keep(tag):  # activation precision kept for a split GEMM input
        return torch.float32 if (exact_fp32 or tag in split) else torch.bfloat16

    def norm(v, w, tag=None):
        return (v * torch.rsqrt(v.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * w).to(keep(tag))

    attd = torch.float32 if ("attn" in split or exact_fp32) else opd

    def rope(t):
        t1, t2 = t[..., : hd // 2], t[..., hd // 2:]
        return (t * cos + torch.cat([-t2, t1], -1) * sin).to(attd)

    for L in W.layers:
        h = norm(x, L["ln1"], "qkv")
        qkv = mm(h, L["wqkv"], "qkv")
        q = qkv[..., : nh * hd].view(B, S, nh, hd).transpose(1, 2)
        k = qkv[..., nh * hd: (nh + nkv) * hd].view(B, S, nkv, hd).transpose(1, 2)
        v = qkv[..., (nh + nkv) * hd:].view(B, S, nkv, hd).transpose(1, 2).to(attd)
        q, k = rope(q), rope(k)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        x = x + mm(a.transpose(1, 2).reshape(B, S, nh * hd).to(keep("o")), L["wo"], "o")
        h = norm(x, L["ln2"], "gu")
        gu = mm(h, L["wgu"], "gu").to(keep("down"))
        g, u = gu[..., : cfg.ffn], gu[..., cfg.ffn:]
        x = x + mm((F.silu(g.float()) * u.float()).to(keep("down")), L["wd"], "down")
    hn = (x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * W.norm)
    out_lp, out_p = [], []
    for r in range(B):
        n = lens[r]
        logits = (mm(hn[r, :n], W.emb, "lm") if "lm" in split else mm(hn[r, :n].to(opd), W.emb)) \
            if not exact_fp32 else hn[r, :n] @ W.emb.float().t()
        lsm = torch.log_softmax(logits.float(), -1).double()
        tgt = ids[r, 1:n]
        total = 0.0
        for t, v in enumerate(lsm[: n - 1].gather(1, tgt[:, None])[:, 0].tolist()):
            total += v
        out_lp.append(total)
        if eos:
            out_p.append([float(lsm[n - 1, p]) for p in PUNCT_IDS])
    return out_lp, out_p


def _dense_forward_gpt2(W, ids, lens, eos, exact_fp32, split):
    """GPT-2 block structure (transformers' GPT2LMHeadModel): x = wte + wpe; per layer
    x += c_proj(attn(ln_1(x))) and x += mlp_proj(gelu_tanh(c_fc(ln_2(x)))); ln_f; tied head."""
    import torch
    import torch.nn.functional as F

    cfg = W.cfg
    B, S = ids.shape
    hd, nh = cfg.head_dim, cfg.heads
    opd = torch.float32 if exact_fp32 else torch.bfloat16

    def mm(a, w, tag=None):
        a2 = a.reshape(-1, a.shape[-1])
        if exact_fp32:
            out = a2.float() @ w.float().t()
        elif tag in split:
            hi = a2.float().to(torch.bfloat16)
            lo = (a2.float() - hi.float()).to(torch.bfloat16)
            out = torch.mm(hi, w.t(), out_dtype=torch.float32) + torch.mm(lo, w.t(), out_dtype=torch.float32)
        else:
            out = torch.mm(a2.to(torch.bfloat16), w.t(), out_dtype=torch.float32)
        return out.view(*a.shape[:-1], -1)

    def keep(tag):
        return torch.float32 if (exact_fp32 or tag in split) else torch.bfloat16

    def ln(v, w, b, tag=None):
        return F.layer_norm(v, (v.shape[-1],), w, b, cfg.rms_eps).to(keep(tag))

    attd = torch.float32 if ("attn" in split or exact_fp32) else opd
    x = W.emb[ids].float() + W.wpe[:S][None]
    for L in W.layers:
        h = ln(x, L["ln1"], L["ln1b"], "qkv")
        qkv = mm(h, L["wqkv"], "qkv") + L["bqkv"]
        q, k, v = (qkv[..., i * nh * hd: (i + 1) * nh * hd].view(B, S, nh, hd).transpose(1, 2).to(attd)
                   for i in range(3))
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + mm(a.transpose(1, 2).reshape(B, S, nh * hd).to(keep("o")), L["wo"], "o") + L["bo"]
        h = ln(x, L["ln2"], L["ln2b"], "gu")
        f = mm(h, L["wfc"], "gu") + L["bfc"]
        act = F.gelu(f.float(), approximate="tanh").to(keep("down"))
        x = x + mm(act, L["wd"], "down") + L["bd"]
    hn = F.layer_norm(x, (x.shape[-1],), W.norm, W.normb, cfg.rms_eps)
    out_lp, out_p = [], []
    for r in range(B):
        n = lens[r]
        logits = (mm(hn[r, :n], W.emb, "lm") if "lm" in split else mm(hn[r, :n].to(opd), W.emb)) \
            if not exact_fp32 else hn[r, :n] @ W.emb.float().t()
        lsm = torch.log_softmax(logits.float(), -1).double()
        total = 0.0
        for v in lsm[: n - 1].gather(1, ids[r, 1:n][:, None])[:, 0].tolist():
            total += v
        out_lp.append(total)
        if eos:
            out_p.append([float(lsm[n - 1, p]) for p in PUNCT_IDS])
    return out_lp, out_p


def _surface_tokens(dm, tok):
    """Per-surface token tables of the tokenizer: (low, cap) one token each (word level) or
    (low, low_off, cap, cap_off) CSR (char level), cached on the device model."""
    key = ("llm_tokens", type(tok).__name__, tok.vocab_size)
    cache = dm.__dict__.setdefault("_tok_cache", {})
    if key not in cache:
        cache[key] = tok.surface_tables(dm.surfaces)
    return cache[key]


class DeviceLlmSession:
    """The prefix-trie KV cache of one DeviceBatch plus the transformer body that fills it."""

    def __init__(self, scorer: LlamaScorer, batch):
        import torch

        self.scorer = scorer
        self.batch = batch
        cfg, W = scorer.cfg, scorer.weights
        tabs = _surface_tokens(batch.dm, scorer.tokenizer)
        if len(tabs) == 2:
            low, cap = tabs
            low_off = cap_off = None
        else:
            low, low_off, cap, cap_off = tabs
        self._low, self._cap = low, cap  # (word level: token per surface)
        self._tabs = tabs
        esz = 4 if scorer.split else 2
        per_slot = cfg.layers * 2 * cfg.kv_heads * cfg.head_dim * esz + cfg.hidden * 4 + 96
        if scorer.max_slots:
            max_slots = int(scorer.max_slots)
        else:
            # measured on the synthetic B2T worlds: slots per utterance ~ T k (1 + 20/r) / 96
            # (T=500: 743 at k=64 r=20, 3725 at k=256 r=10); sized 2x that, capped at half the
            # free memory (the 1B model's T=2000 k=256 r=10 sweep point needs ~1.1M slots)
            c = batch.cfg
            per_trial = batch.max_frames * c.beam_size * (1 + 20 / c.llm_rescore_interval) / 48
            want = max(1 << 16, int(batch.max_trials * per_trial))
            free, _ = torch.cuda.mem_get_info(scorer.device)
            max_slots = int(min(want, 0.5 * free / per_slot, 1 << 26))
        self.max_slots = max_slots
        self.pitch = scorer.max_depth + 1
        d = N.LbLlmDesc()
        d.n_layers, d.n_heads, d.n_kv_heads = cfg.layers, cfg.heads, cfg.kv_heads
        d.head_dim, d.hidden, d.vocab = cfg.head_dim, cfg.hidden, cfg.vocab_size
        d.max_slots = max_slots
        d.max_depth = scorer.max_depth
        tok = scorer.tokenizer
        d.bos_token = tok.bos
        pids = getattr(tok, "punct_ids", PUNCT_IDS)
        for j in range(3):
            d.punct_tokens[j] = pids[j]
        d.surface_tokens = low.ctypes.data
        d.surface_tokens_first = cap.ctypes.data
        d.n_surfaces = len(batch.dm.surfaces)
        d.surface_token_off = low_off.ctypes.data if low_off is not None else None
        d.surface_token_off_first = cap_off.ctypes.data if cap_off is not None else None
        d.embedding = W.emb.data_ptr()
        head32 = getattr(W, "head32", None)
        d.head_f32 = head32.data_ptr() if head32 is not None else None
        d.precision = 1 if scorer.split else 0
        h = C.c_void_p()
        N.check(N.lib().lb_llm_create(batch.h, C.byref(d), C.byref(h)))
        self.h = h
        self._ws = {}
        self.waves_log: list = []
        self.graphs: dict = {}  # decode shape -> captured CUDA graph (LLM graph mode)

    def destroy(self):
        getattr(self, "graphs", {}).clear()  # captured graphs point into this session's buffers
        if getattr(self, "h", None):
            N.lib(False).lb_llm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def reset(self):
        N.check(N.lib().lb_llm_reset(self.h))
        self.waves_log = []
        if getattr(self, "_timing", None) is not None:
            self._timing = []

    def _work(self, n: int):
        cap = self._ws.get("n", 0)
        if cap < n:
            self._ws = {}  # free the old buffers first
            self._ws = self._alloc_work(max(n, 256))
        return self._ws

    def graph_workspace(self, n: int) -> dict:
        """Buffers owned by one captured graph (never reallocated under it)."""
        return self._alloc_work(n)

    def _alloc_work(self, cap: int) -> dict:
        import torch

        if True:
            dev = self.scorer.weights.device
            cfg = self.scorer.cfg
            k = 2 if self.scorer.split else 1
            i32 = dict(dtype=torch.int32, device=dev)
            bf = dict(dtype=torch.bfloat16, device=dev)
            return {
                "n": cap,
                "tok": torch.empty(cap, **i32),
                "pos": torch.empty(cap, **i32),
                "slot": torch.empty(cap, **i32),
                "chain": torch.empty((cap, self.pitch), **i32),
                "q": torch.empty((cap, cfg.heads * cfg.head_dim),
                                 dtype=torch.float32 if k == 2 else torch.bfloat16, device=dev),
                "att": torch.empty((cap, k * cfg.heads * cfg.head_dim), **bf),
                "hn": torch.empty((cap, k * cfg.hidden), **bf),
                "act": torch.empty((cap, k * cfg.ffn), **bf),
            }

    def enable_timing(self, on: bool = True):
        """Record CUDA events around every fusion event (device ms spent in the LLM step)."""
        self._timing = [] if on else None

    def llm_ms(self) -> float:
        import torch

        if not getattr(self, "_timing", None):
            return 0.0
        torch.cuda.synchronize()
        return float(sum(a.elapsed_time(b) for a, b in self._timing))

    def event(self, final: bool, min_frames: int):
        import contextlib

        import torch

        # torch's GEMMs must run on the batch's stream, in order with the lb_llm kernels
        ptr = getattr(self.batch, "stream_ptr", 0)
        ctx = (torch.cuda.stream(torch.cuda.ExternalStream(ptr, device=self.scorer.weights.device))
               if ptr else contextlib.nullcontext())
        with ctx:
            timing = getattr(self, "_timing", None)
            if timing is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            self._event(final, min_frames)
            if timing is not None:
                ev[1].record()
                timing.append(ev)

    def _event(self, final: bool, min_frames: int):
        lib = N.lib()
        nw = C.c_int32()
        rows = np.zeros(N.LLM_MAX_WAVES, dtype=np.int64)
        N.check(lib.lb_llm_plan(self.h, int(final), int(min_frames), C.byref(nw), N.ptr(rows)))
        sizes = [int(x) for x in rows[: nw.value]]
        self.waves_log.append(sizes)
        for w, m in enumerate(sizes):
            for r0 in range(0, m, self.scorer.row_chunk):
                self._forward_rows(w, r0, min(self.scorer.row_chunk, m - r0))
        N.check(lib.lb_llm_finish(self.h, int(final), int(min_frames)))

    def event_async(self, final: bool, min_frames: int, rows_cap: int, ws: dict):
        """One fusion event without host synchronisation (CUDA-graph capturable): planning
        kernels, a forward over `rows_cap` rows (the event's rows + BOS-only padding), the
        fusion kernels.  Overflow is flagged on the device (`check`)."""
        lib = N.lib()
        N.check(lib.lb_llm_plan_async(self.h, int(final), int(min_frames), int(rows_cap)))
        self._forward_rows(0, 0, rows_cap, ws=ws)
        N.check(lib.lb_llm_finish(self.h, int(final), int(min_frames)))

    def check(self):
        """Synchronise and raise DeviceError if a graph-mode event overflowed its rows."""
        N.check(N.lib().lb_llm_check(self.h))

    def _forward_rows(self, wave: int, row0: int, n: int, ws: dict | None = None):
        import torch

        lib = N.lib()
        cfg, W = self.scorer.cfg, self.scorer.weights
        graph_rows = ws is not None
        ws = ws if graph_rows else self._work(n)
        tok, pos, slot, chain = ws["tok"][:n], ws["pos"][:n], ws["slot"][:n], ws["chain"][:n]
        if graph_rows:
            N.check(lib.lb_llm_wave_rows_async(self.h, n, tok.data_ptr(), pos.data_ptr(),
                                               slot.data_ptr(), chain.data_ptr()))
        else:
            N.check(lib.lb_llm_wave_rows(self.h, wave, row0, n, tok.data_ptr(), pos.data_ptr(),
                                         slot.data_ptr(), chain.data_ptr()))
        if cfg.arch in ("gpt2", "tinychar"):
            return self._forward_rows_gpt2(tok, pos, slot, chain, n, ws)
        x = W.emb.index_select(0, tok.long()).float()
        hn, q, att, act = ws["hn"][:n], ws["q"][:n], ws["att"][:n], ws["act"][:n]
        eps = cfg.rms_eps
        sfx = "2" if self.scorer.split else ""
        f32 = torch.float32
        N.check(lib.lb_llm_rmsnorm(self.h, x.data_ptr(), None, W.layers[0]["ln1"].data_ptr(), eps, n,
                                   hn.data_ptr(), None))
        for li, L in enumerate(W.layers):
            qkv = torch.mm(hn, L["wqkv" + sfx].t(), out_dtype=f32)
            N.check(lib.lb_llm_rope_kv(self.h, li, qkv.data_ptr(), n, pos.data_ptr(), slot.data_ptr(),
                                       W.cos.data_ptr(), W.sin.data_ptr(), q.data_ptr()))
            del qkv
            N.check(lib.lb_llm_attention(self.h, li, q.data_ptr(), n, chain.data_ptr(), pos.data_ptr(),
                                         att.data_ptr()))
            # residual add in the GEMM epilogue: x += att @ Wo^T (fp32 C/D, bf16 A/B)
            torch.addmm(x, att, L["wo" + sfx].t(), out_dtype=f32, out=x)
            N.check(lib.lb_llm_rmsnorm(self.h, x.data_ptr(), None, L["ln2"].data_ptr(), eps, n,
                                       hn.data_ptr(), None))
            if self.scorer.fused_swiglu and n >= self.scorer.fused_swiglu_min_rows:
                # gate/up GEMM + SwiGLU in one tcgen05 kernel
                wi = L["wgui" + sfx]
                N.check(lib.lb_llm_gateup_swiglu(self.h, hn.data_ptr(), n, hn.stride(0), wi.shape[1],
                                                 wi.data_ptr(), wi.stride(0), cfg.ffn, act.data_ptr()))
            else:
                gu = torch.mm(hn, L["wgu" + sfx].t(), out_dtype=f32) if sfx else torch.mm(hn, L["wgu"].t())
                N.check(lib.lb_llm_swiglu(self.h, gu.data_ptr(), n, cfg.ffn, act.data_ptr()))
                del gu
            torch.addmm(x, act, L["wd" + sfx].t(), out_dtype=f32, out=x)
            last = li + 1 == cfg.layers
            wnext = W.norm if last else W.layers[li + 1]["ln1"]
            N.check(lib.lb_llm_rmsnorm(self.h, x.data_ptr(), None, wnext.data_ptr(), eps, n,
                                       hn.data_ptr(), slot.data_ptr() if last else None))
        self._lm_head(hn, slot, n)

    def _lm_head(self, hn, slot, n: int):
        import torch

        lib = N.lib()
        W = self.scorer.weights
        sfx = "2" if self.scorer.split else ""
        f32 = torch.float32
        if self.scorer.lm_head == "fused":  # K6 on tcgen05: logits never leave TMEM
            # bf16x2: the LSE GEMM reads only the hi half of hn (first H columns) unless lse_split
            E = self.scorer.emb2 if (sfx and self.scorer.lse_split) else W.emb
            nt = (E.shape[0] + 255) // 256
            partial = torch.empty((n, nt, 2), dtype=torch.float32, device=hn.device)
            N.check(lib.lb_llm_lmhead_lse(self.h, hn.data_ptr(), n, hn.stride(0), E.shape[1],
                                          E.data_ptr(), E.stride(0), E.shape[0], slot.data_ptr(),
                                          partial.data_ptr()))
            return
        # rows per LM-head GEMM: large enough for full tensor-core tiles (measured: 2048 rows bf16 /
        # 1024 rows bf16x2 beat L2-resident 256-row chunks by ~15% of the LLM step)
        chunk = self.scorer.lm_chunk // (2 if sfx else 1)
        for c0 in range(0, n, chunk):
            c1 = min(n, c0 + chunk)
            head_lo = getattr(W, "head_lo", None)
            if sfx or head_lo is not None:  # hi|lo against [E | E], fp32 logits
                logits = (torch.mm(hn[c0:c1], self.scorer.emb2.t(), out_dtype=f32) if sfx
                          else torch.mm(hn[c0:c1], W.emb.t(), out_dtype=f32))
                if head_lo is not None:  # + hi @ E_lo^T (head weights not bf16-exact)
                    torch.addmm(logits, hn[c0:c1, : head_lo.shape[1]], head_lo.t(), out_dtype=f32,
                                out=logits)
            else:
                logits = torch.mm(hn[c0:c1], W.emb.t())
            N.check(lib.lb_llm_lse(self.h, logits.data_ptr(), c1 - c0, logits.stride(0),
                                   slot[c0:].data_ptr()))

    def _forward_rows_gpt2(self, tok, pos, slot, chain, n: int, ws: dict):
        """GPT-2 blocks on the same kernels: LayerNorm (+bias), fused q/k/v GEMM + bias, identity
        rotary tables (learned positions were added at the input), MHA chain attention, GELU."""
        import torch

        lib = N.lib()
        cfg, W = self.scorer.cfg, self.scorer.weights
        hn, q, att, act = ws["hn"][:n], ws["q"][:n], ws["att"][:n], ws["act"][:n]
        eps, f32 = cfg.rms_eps, torch.float32
        sfx = "2" if self.scorer.split else ""
        emb_in = getattr(W, "emb_in", None)  # tinychar: fp32 input rows
        x = (emb_in.index_select(0, tok.long()) if emb_in is not None
             else W.emb.index_select(0, tok.long()).float()) + W.wpe.index_select(0, pos.long())

        def lo_fix(out, a, L, k):  # weights that are bf16 hi + lo pairs: out += a_hi @ W_lo^T
            wl = L.get(k + "_lo")
            if wl is not None:
                torch.addmm(out, a[:, : wl.shape[1]], wl.t(), out_dtype=f32, out=out)

        L0 = W.layers[0]
        N.check(lib.lb_llm_layernorm(self.h, x.data_ptr(), None, L0["ln1"].data_ptr(),
                                     L0["ln1b"].data_ptr(), eps, n, hn.data_ptr(), None))
        for li, L in enumerate(W.layers):
            qkv = torch.mm(hn, L["wqkv" + sfx].t(), out_dtype=f32)
            lo_fix(qkv, hn, L, "wqkv")
            if L["bqkv"] is not None:
                qkv += L["bqkv"]
            N.check(lib.lb_llm_rope_kv(self.h, li, qkv.data_ptr(), n, pos.data_ptr(), slot.data_ptr(),
                                       W.cos.data_ptr(), W.sin.data_ptr(), q.data_ptr()))
            del qkv
            N.check(lib.lb_llm_attention(self.h, li, q.data_ptr(), n, chain.data_ptr(), pos.data_ptr(),
                                         att.data_ptr()))
            o = torch.mm(att, L["wo" + sfx].t(), out_dtype=f32)
            lo_fix(o, att, L, "wo")
            if L["bo"] is not None:
                o += L["bo"]
            N.check(lib.lb_llm_layernorm(self.h, x.data_ptr(), o.data_ptr(), L["ln2"].data_ptr(),
                                         L["ln2b"].data_ptr(), eps, n, hn.data_ptr(), None))
            del o
            f = torch.mm(hn, L["wfc" + sfx].t(), out_dtype=f32)
            lo_fix(f, hn, L, "wfc")
            N.check(lib.lb_llm_gelu(self.h, f.data_ptr(),
                                    L["bfc"].data_ptr() if L["bfc"] is not None else None, n,
                                    cfg.ffn, act.data_ptr()))
            del f
            dn = torch.mm(act, L["wd" + sfx].t(), out_dtype=f32)
            lo_fix(dn, act, L, "wd")
            if L["bd"] is not None:
                dn += L["bd"]
            last = li + 1 == cfg.layers
            nw, nb = (W.norm, W.normb) if last else (W.layers[li + 1]["ln1"], W.layers[li + 1]["ln1b"])
            N.check(lib.lb_llm_layernorm(self.h, x.data_ptr(), dn.data_ptr(), nw.data_ptr(),
                                         nb.data_ptr(), eps, n, hn.data_ptr(),
                                         slot.data_ptr() if last else None))
            del dn
        self._lm_head(hn, slot, n)

    def stats(self) -> dict:
        out = np.zeros(8, dtype=np.int64)
        N.check(N.lib().lb_llm_stats(self.h, N.ptr(out)))
        return {"slots": int(out[0]), "events": int(out[1]), "waves": int(out[2]),
                "forward_rows": int(out[3]), "max_wave_rows": int(out[4]), "cache_bytes": int(out[5]),
                "scores": int(out[6]), "grouped_attention_launches": int(out[7])}

    def export(self) -> dict:
        """Slot table for parity checks: parent, token, depth, state bits, score, punct lps."""
        n = C.c_int64()
        N.check(N.lib().lb_llm_export(self.h, 0, C.byref(n), None, None, None, None, None, None))
        k = n.value
        par = np.empty(k, np.int32)
        tok = np.empty(k, np.int32)
        dep = np.empty(k, np.int32)
        st = np.empty(k, np.int32)
        cum = np.empty(k, np.float64)
        plp = np.empty((k, 3), np.float64)
        N.check(N.lib().lb_llm_export(self.h, k, C.byref(n), N.ptr(par), N.ptr(tok), N.ptr(dep),
                                      N.ptr(st), N.ptr(cum), N.ptr(plp)))
        return {"parent": par, "token": tok, "depth": dep, "state": st, "cum": cum, "punct_lp": plp}

    def replay_table(self) -> "ReplayTable":
        return ReplayTable(self.export(), self.scorer.tokenizer)


class ReplayTable:
    """text -> the score the device assigned it (score-replay scorer of SURVEY.md §8c(3))."""

    def __init__(self, ex: dict, tok: WordTokenizer):
        self.tok = tok
        self.child = {}
        for s in range(1, len(ex["parent"])):
            if ex["parent"][s] >= 0:  # -2: spare slot of a lost insert race, never referenced
                self.child[(int(ex["parent"][s]), int(ex["token"][s]))] = s
        self.ex = ex

    def slot_of(self, text: str) -> int:
        ids = self.tok.encode(text)
        s = 0
        for t in ids[1:]:
            s = self.child[(s, t)]
        return s

    def score(self, text: str) -> float:
        s = self.slot_of(text)
        if not self.ex["state"][s] & 2:
            raise KeyError(f"text never scored on the device: {text!r}")
        return float(self.ex["cum"][s])

    def score_eos(self, text: str) -> tuple[str, float]:
        s = self.slot_of(text)
        if not self.ex["state"][s] & 4:
            raise KeyError(f"text never eos-scored on the device: {text!r}")
        base = float(self.ex["cum"][s])
        best, bs = 0, base + float(self.ex["punct_lp"][s][0])
        for j in (1, 2):
            v = base + float(self.ex["punct_lp"][s][j])
            if v > bs:
                best, bs = j, v
        return PUNCTS[best], bs


class ReplayScorer:
    """Reference-protocol scorer answering from a device ReplayTable (parity harness)."""

    def __init__(self, table: ReplayTable):
        self.table = table
        self._ids = itertools.count(1)

    def next_request_id(self) -> int:
        return next(self._ids)

    def submit(self, request: ScoreRequest) -> ScoreResponse:
        if request.kind == "score":
            return ScoreResponse(request.id, tuple(self.table.score(t) for t in request.texts))
        pairs = [self.table.score_eos(t) for t in request.texts]
        return ScoreResponse(request.id, tuple(s for _, s in pairs), tuple(p for p, _ in pairs))

    def close(self):
        pass
