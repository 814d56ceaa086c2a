"""CPU ORACLE of the reference sidecar's scorer model -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and bench.py's CPU legs may import this module.

A float64 numpy restatement of `TinyCausalLM` (`/root/reference/pkg/sidecar/src/model.ts`), the
model behind the reference's LLM scorer slot (the TypeScript sidecar cannot run here: no Node):
- tokenizer `sentenceCase` + `tokenize` (model.ts:35-47): printable ASCII -> code - 32, else
  UNK = 95, BOS = 96 first;
- weights (model.ts:50-117): `hashSeed(identifier)` seeds `mulberry32`; matrices drawn in
  constructor order (embed, pos, per layer wq wk wv wo w1 w2, wOut), each entry
  `(rng() * 2 - 1) * scale`, scale 1/sqrt(dim) (w2: 1/sqrt(4 dim));
- `forward` (model.ts:141-209): x = embed + pos; per layer LayerNorm (no affine, eps 1e-5),
  q/k/v, per-head causal softmax attention scaled by 1/sqrt(headDim), residual through wo,
  LayerNorm, w1, tanh-GELU, w2, residual; final LayerNorm; logits = x @ wOut;
- `score_text` (model.ts:119-129): sum over positions of logit[next] - logSumExp(row), left to
  right; empty text -> 0; `score_eos` (model.ts:131-139): best of text+".", "?", "!" with
  strict `>` (ties keep ".").
Written loop-by-loop after the TypeScript (JS numbers are float64; `Math.imul`/`>>>` are
32-bit).  Parity status: no reference test pins numbers (model.test.ts checks properties only:
determinism, identifier dependence, finite negative scores, empty -> 0, nonsense suffix lowers
the score, eos = score(text + punct), argmax) -- tests/test_tiny_char_lm.py re-checks exactly
those properties here, so the restatement is pinned to the reference's own test strategy.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

DIM, HEADS, LAYERS, MAX_CONTEXT = 32, 2, 2, 1024
N_CHARS = 126 - 32 + 1
UNK, BOS = N_CHARS, N_CHARS + 1
VOCAB_SIZE = N_CHARS + 2
PUNCTS = (".", "?", "!")


def sentence_case(text: str) -> str:
    if len(text) == 0:
        return text
    return text[0].upper() + text[1:]


def tokenize(text: str) -> list[int]:
    toks = [BOS]
    for ch in sentence_case(text):
        code = ord(ch)
        toks.append(code - 32 if 32 <= code <= 126 else UNK)
    return toks


def _u32(x: int) -> int:
    return x % 4294967296


def _hash_seed(text: str) -> int:
    h = 0x9E3779B9
    raw = text.encode("utf-16-le")
    for k in range(len(raw) // 2):
        c = raw[2 * k] + 256 * raw[2 * k + 1]
        h = _u32((h ^ c) * 0x85EBCA6B)
        h = _u32((h << 13) | (h >> 19))
    return h


class _Mulberry32:
    def __init__(self, seed: int):
        self.a = _u32(seed)

    def __call__(self) -> float:
        self.a = _u32(self.a + 0x6D2B79F5)
        t = self.a
        t = _u32((t ^ (t >> 15)) * (t | 1))
        t = t ^ _u32(t + _u32((t ^ (t >> 7)) * (t | 61)))
        return _u32(t ^ (t >> 14)) / 4294967296.0


def _init_matrix(rng, rows, cols, scale):
    return np.array([(rng() * 2 - 1) * scale for _ in range(rows * cols)]).reshape(rows, cols)


class TinyCharLM:
    def __init__(self, identifier: str = "tiny-char-lm-v1", dim=DIM, heads=HEADS, layers=LAYERS,
                 max_context=MAX_CONTEXT):
        if dim % heads:
            raise ValueError("dim must be divisible by heads")
        self.dim, self.heads, self.max_context = dim, heads, max_context
        rng = _Mulberry32(_hash_seed(identifier))
        scale = 1 / math.sqrt(dim)
        self.embed = _init_matrix(rng, VOCAB_SIZE, dim, scale)
        self.pos = _init_matrix(rng, max_context, dim, scale)
        self.layers = []
        for _ in range(layers):
            self.layers.append({
                "wq": _init_matrix(rng, dim, dim, scale), "wk": _init_matrix(rng, dim, dim, scale),
                "wv": _init_matrix(rng, dim, dim, scale), "wo": _init_matrix(rng, dim, dim, scale),
                "w1": _init_matrix(rng, dim, 4 * dim, scale),
                "w2": _init_matrix(rng, 4 * dim, dim, 1 / math.sqrt(4 * dim)),
            })
        self.w_out = _init_matrix(rng, dim, VOCAB_SIZE, scale)

    @staticmethod
    def _layer_norm(x):
        out = np.empty_like(x)
        for i in range(x.shape[0]):
            mean = x[i].sum() / x.shape[1]
            d = x[i] - mean
            var = (d * d).sum() / x.shape[1]
            out[i] = d * (1 / math.sqrt(var + 1e-5))
        return out

    def forward(self, tokens):
        n = min(len(tokens), self.max_context)
        seq = tokens[len(tokens) - n:]
        hd = self.dim // self.heads
        x = self.embed[seq] + self.pos[:n]
        for w in self.layers:
            h = self._layer_norm(x)
            q, k, v = h @ w["wq"], h @ w["wk"], h @ w["wv"]
            att = np.zeros_like(x)
            inv = 1 / math.sqrt(hd)
            for hh in range(self.heads):
                o = hh * hd
                for t in range(n):
                    sc = (k[: t + 1, o:o + hd] @ q[t, o:o + hd]) * inv
                    e = np.exp(sc - sc.max())
                    att[t, o:o + hd] = (e / e.sum()) @ v[: t + 1, o:o + hd]
            x = x + att @ w["wo"]
            h = self._layer_norm(x)
            f = h @ w["w1"]
            g = 0.5 * f * (1 + np.tanh(math.sqrt(2 / math.pi) * (f + 0.044715 * f * f * f)))
            x = x + g @ w["w2"]
        return self._layer_norm(x) @ self.w_out

    def score_text(self, text: str) -> float:
        toks = tokenize(text)
        if len(toks) == 1:
            return 0.0
        logits = self.forward(toks[:-1])
        total = 0.0
        for t in range(len(toks) - 1):
            row = logits[t]
            m = row.max()
            total += row[toks[t + 1]] - (m + math.log(np.exp(row - m).sum()))
        return total

    def score_eos(self, text: str) -> tuple[str, float]:
        best_p, best = ".", -math.inf
        for p in PUNCTS:
            s = self.score_text(text + p)
            if s > best:
                best_p, best = p, s
        return best_p, best


class OracleTinyCharScorer:
    """The reference scorer protocol (scorer.py:93-163) over TinyCharLM."""

    def __init__(self, identifier: str = "tiny-char-lm-v1"):
        self.lm = TinyCharLM(identifier)
        self._ids = itertools.count(1)

    def next_request_id(self) -> int:
        return next(self._ids)

    def submit(self, request):
        from paper_2603_14002_b200.scorer import ScoreResponse

        if request.kind == "score":
            return ScoreResponse(request.id, tuple(self.lm.score_text(t) for t in request.texts))
        pairs = [self.lm.score_eos(t) for t in request.texts]
        return ScoreResponse(request.id, tuple(s for _, s in pairs), tuple(p for p, _ in pairs))

    def close(self):
        pass
