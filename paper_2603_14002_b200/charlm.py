"""The reference sidecar's own scorer model, on the device path.

`pkg/sidecar/src/model.ts` (the LLM slot of the reference, reached through the JSONL scorer
protocol) is `TinyCausalLM`: a character-level pre-LayerNorm transformer whose weights are
derived deterministically from its identifier (`mulberry32(hashSeed(identifier))`,
model.ts:50-76,93-117), so "the same model" means the same numbers on every machine.  This
module rebuilds it for the GPU decoder:

- `CharTokenizer` -- model.ts:27-47: printable ASCII 32..126 -> 0..94, anything else -> UNK 95,
  BOS 96; texts are sentence-cased first.  A lexicon surface is a multi-token word: " w o r d"
  after an earlier word, "W o r d" as the first word (the device trie holds one slot per token).
- `tiny_char_weights` -- the float64 weights of model.ts:93-117 in the generation order of the
  constructor (embed, pos, per layer wq wk wv wo w1 w2, wOut), as numpy arrays laid out like the
  TypeScript ones (row-major [in][out] for every matmul).
- `dense_scores` -- a float64 torch forward of full texts (model.ts:119-209) for the scorer
  protocol's `submit()` (the reference arm: one forward per text, no KV reuse).

The device body maps the model onto the GPT-2-style kernels of llm.py (learned positions,
LayerNorm without affine = gain 1 / shift 0, zero biases, tanh GELU, MHA, untied head); see
`LlamaWeights._init_tinychar` for the head-dim padding and the hi/lo weight split.
"""

from __future__ import annotations

import numpy as np

CHAR_LO, CHAR_HI = 32, 126
N_CHARS = CHAR_HI - CHAR_LO + 1
UNK = N_CHARS
BOS = N_CHARS + 1
VOCAB = N_CHARS + 2  # 97
PUNCT_TOKENS = tuple(ord(p) - CHAR_LO for p in ".?!")
M32 = 0xFFFFFFFF


def sentence_case(text: str) -> str:
    return text[:1].upper() + text[1:] if text else text


def char_token(ch: str) -> int:
    c = ord(ch)
    return c - CHAR_LO if CHAR_LO <= c <= CHAR_HI else UNK


class CharTokenizer:
    """model.ts:39-47 behind the interface of llm.WordTokenizer."""

    vocab_size = VOCAB
    bos = BOS
    punct_ids = PUNCT_TOKENS

    def encode(self, text: str) -> list[int]:
        return [BOS] + [char_token(ch) for ch in sentence_case(text)]

    def surface_tables(self, surfaces):
        """CSR token tables per lexicon surface: (tokens after an earlier word = " " + word,
        offsets, tokens as the sentence-cased first word, offsets)."""
        low, cap = [], []
        low_off, cap_off = [0], [0]
        for s in surfaces:
            low.extend(char_token(ch) for ch in " " + s)
            low_off.append(len(low))
            cap.extend(char_token(ch) for ch in sentence_case(s))
            cap_off.append(len(cap))
        as32 = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
        return as32(low), as32(low_off), as32(cap), as32(cap_off)


def _imul(a: int, b: int) -> int:
    return (a * b) & M32


def hash_seed(text: str) -> int:
    """model.ts:50-57 over UTF-16 code units."""
    h = 0x9E3779B9
    units = text.encode("utf-16-le")
    for i in range(0, len(units), 2):
        h = _imul(h ^ (units[i] | units[i + 1] << 8), 0x85EBCA6B)
        h = ((h << 13) | (h >> 19)) & M32
    return h


def _mulberry32_stream(seed: int, n: int) -> np.ndarray:
    """model.ts:60-68: n successive draws in [0, 1) (uint32 / 2^32, exact in float64).  JS
    coerces every bitwise operand to 32 bits, so the arithmetic is mod 2^32 throughout."""
    out = np.empty(n, dtype=np.float64)
    a = seed & M32
    for i in range(n):
        a = (a + 0x6D2B79F5) & M32
        t = _imul(a ^ (a >> 15), a | 1)
        t = (t ^ ((t + _imul(t ^ (t >> 7), t | 61)) & M32)) & M32
        out[i] = ((t ^ (t >> 14)) & M32) / 4294967296.0
    return out


def tiny_char_weights(identifier: str = "tiny-char-lm-v1", dim: int = 32, heads: int = 2,
                      layers: int = 2, max_context: int = 1024) -> dict:
    """model.ts:93-117: every matrix (rng() * 2 - 1) * scale in constructor order."""
    if dim % heads:
        raise ValueError("dim must be divisible by heads")
    shapes = [("embed", VOCAB, dim, dim), ("pos", max_context, dim, dim)]
    for li in range(layers):
        for name, r, c, sc in (("wq", dim, dim, dim), ("wk", dim, dim, dim), ("wv", dim, dim, dim),
                               ("wo", dim, dim, dim), ("w1", dim, 4 * dim, dim),
                               ("w2", 4 * dim, dim, 4 * dim)):
            shapes.append((f"{name}.{li}", r, c, sc))
    shapes.append(("wout", dim, VOCAB, dim))
    total = sum(r * c for _, r, c, _ in shapes)
    draws = _mulberry32_stream(hash_seed(identifier), total)
    out, pos = {"dim": dim, "heads": heads, "layers": layers, "max_context": max_context}, 0
    for name, r, c, sc in shapes:
        scale = 1.0 / np.sqrt(sc)
        out[name] = ((draws[pos:pos + r * c] * 2.0 - 1.0) * scale).reshape(r, c)
        pos += r * c
    return out


def dense_scores(w: dict, texts, device, eos: bool):
    """float64 full-text forward (model.ts:141-209) per text: the protocol path of the device
    scorer.  Returns [(sum of next-token log-probs, [lp(".") lp("?") lp("!")] | None)]."""
    import torch

    dev = torch.device(device)
    t = lambda a: torch.as_tensor(a, dtype=torch.float64, device=dev)  # noqa: E731
    dim, heads, L = w["dim"], w["heads"], w["layers"]
    hd = dim // heads
    emb, pos, wout = t(w["embed"]), t(w["pos"]), t(w["wout"])
    lay = [{k: t(w[f"{k}.{i}"]) for k in ("wq", "wk", "wv", "wo", "w1", "w2")} for i in range(L)]
    tok = CharTokenizer()

    def ln(x):
        m = x.mean(-1, keepdim=True)
        v = ((x - m) ** 2).mean(-1, keepdim=True)
        return (x - m) / torch.sqrt(v + 1e-5)

    res = []
    for text in texts:
        ids = tok.encode(text)
        seq = ids if eos else ids[:-1]  # eos: one more position (the punctuation after the text)
        if not seq or (not eos and len(ids) == 1):
            res.append((0.0, None))
            continue
        n = min(len(seq), w["max_context"])
        seq = seq[len(seq) - n:]
        x = emb[seq] + pos[:n]
        mask = torch.ones(n, n, dtype=torch.bool, device=dev).tril()
        for p in lay:
            h = ln(x)
            q, k, v = h @ p["wq"], h @ p["wk"], h @ p["wv"]
            q = q.view(n, heads, hd).transpose(0, 1)
            k = k.view(n, heads, hd).transpose(0, 1)
            v = v.view(n, heads, hd).transpose(0, 1)
            s = (q @ k.transpose(1, 2)) * (1.0 / np.sqrt(hd))
            s = s.masked_fill(~mask, float("-inf"))
            a = torch.softmax(s, -1) @ v
            x = x + a.transpose(0, 1).reshape(n, dim) @ p["wo"]
            h = ln(x)
            f = h @ p["w1"]
            g = 0.5 * f * (1 + torch.tanh(np.sqrt(2 / np.pi) * (f + 0.044715 * f ** 3)))
            x = x + g @ p["w2"]
        lsm = torch.log_softmax(ln(x) @ wout, -1)
        total = 0.0
        for j in range(len(ids) - 1):
            total += float(lsm[j, ids[j + 1]])
        plp = [float(lsm[len(ids) - 1, pt]) for pt in PUNCT_TOKENS] if eos else None
        res.append((total, plp))
    return res
