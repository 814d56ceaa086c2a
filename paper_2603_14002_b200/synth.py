"""Seeded synthetic worlds for parity tests and the benchmark.

Everything here is new code that only *produces inputs* in the reference's formats:
- the 41-token vocabulary `<blank>, P00..P38, <sp>` (blank 0, space 40) of
  `pkg/tests/test_acceptance.py:363-366`;
- lexicons of U{2..8}-phoneme words over phones 1..39 with a homophone fraction (same
  pronunciation, new surface) and no adjacent duplicate phonemes (those are unreachable:
  a repeat never emits, `decoder.py:276`);
- a 4-gram ARPA model with the section sizes / log10 ranges / back-offs of §8d, built as
  an `NGramModel` directly or rendered as ARPA text (identical values: `float(repr(x))==x`);
- N(0, 2) fp32 logits, trial i seeded with `base + i` (`test_acceptance.py:413-416`).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lexicon import Lexicon, LexiconEntry, build_transition_table
from .ngram import LN10, NGramModel, parse_arpa_text
from .vocab import Vocabulary


def vocab41() -> Vocabulary:
    return Vocabulary(("<blank>",) + tuple(f"P{i:02d}" for i in range(39)) + ("<sp>",), 0, 40)


def make_lexicon(n_words: int, seed: int = 12345, homophone_frac: float = 0.1,
                 min_len: int = 2, max_len: int = 8, n_phones: int = 39) -> Lexicon:
    """`n_words` entries; the last `homophone_frac` share an earlier pronunciation."""
    rng = np.random.default_rng(seed)
    n_homo = int(round(n_words * homophone_frac))
    n_base = n_words - n_homo
    lens = rng.integers(min_len, max_len + 1, size=n_base)
    total = int(lens.sum())
    # draw phones 1..n_phones with no adjacent repeats: p_i = p_{i-1} + U{1..n-1} (mod n)
    steps = rng.integers(1, n_phones, size=total)
    firsts = rng.integers(0, n_phones, size=n_base)
    entries = []
    pos = 0
    for i in range(n_base):
        ln = int(lens[i])
        ph = np.empty(ln, dtype=np.int64)
        ph[0] = firsts[i]
        if ln > 1:
            ph[1:] = (firsts[i] + np.cumsum(steps[pos + 1:pos + ln])) % n_phones
        pos += ln
        entries.append(LexiconEntry(f"w{i}", f"w{i}", tuple(int(x) + 1 for x in ph)))
    src = rng.integers(0, n_base, size=n_homo)
    for j in range(n_homo):
        i = n_base + j
        entries.append(LexiconEntry(f"w{i}", f"w{i}", entries[int(src[j])].phonemes))
    return Lexicon(tuple(entries))


@dataclass
class NgramSpec:
    words: list  # LM word strings (index = position)
    grams: list  # per order n (1..4): int array [count, n] of word indices, -1 = <s>
    logp10: list  # per order: float array [count]
    bo10: list  # per order: float array or None


SPECIAL_BOS, SPECIAL_EOS, SPECIAL_UNK = "<s>", "</s>", "<unk>"


def make_ngram_spec(words: list, n2: int, n3: int, n4: int, seed: int = 4242,
                    bos_frac: float = 0.05) -> NgramSpec:
    """4-gram spec in the shape of §8d: unigrams U(-4.5,-2) bo -0.3; bigrams U(-2,-0.5)
    bo -0.2 (a `bos_frac` share with `<s>` history); trigrams U(-1.5,-0.3) bo -0.1
    extending listed bigrams; 4-grams U(-1,-0.2) extending listed trigrams."""
    rng = np.random.default_rng(seed)
    w = len(words)
    bos = w  # index of <s> in the combined id space
    n_bos = int(n2 * bos_frac)
    a = np.concatenate([np.full(n_bos, bos), rng.integers(0, w, size=n2 - n_bos)])
    b = rng.integers(0, w, size=n2)
    key2 = np.unique(a.astype(np.int64) * (w + 1) + b)
    g2 = np.stack([key2 // (w + 1), key2 % (w + 1)], axis=1)

    def extend(prev, count):
        pick = prev[rng.integers(0, len(prev), size=count)]
        nxt = rng.integers(0, w, size=count)
        g = np.concatenate([pick, nxt[:, None]], axis=1)
        return np.unique(g, axis=0)

    g3 = extend(g2, n3)
    g4 = extend(g3, n4)
    r4 = lambda lo, hi, n: np.round(rng.uniform(lo, hi, size=n), 4)  # noqa: E731
    return NgramSpec(
        words=list(words),
        grams=[np.arange(w)[:, None], g2, g3, g4],
        logp10=[r4(-4.5, -2.0, w), r4(-2.0, -0.5, len(g2)), r4(-1.5, -0.3, len(g3)),
                r4(-1.0, -0.2, len(g4))],
        bo10=[np.full(w, -0.3), np.full(len(g2), -0.2), np.full(len(g3), -0.1), None],
    )


def _name(spec: NgramSpec, idx: int) -> str:
    return SPECIAL_BOS if idx == len(spec.words) else spec.words[idx]


def ngram_model_from_spec(spec: NgramSpec) -> NGramModel:
    """Same values `load_arpa` would produce from `arpa_text_from_spec(spec)`."""
    probs: dict = {(SPECIAL_BOS,): -99.0 * LN10, (SPECIAL_EOS,): -1.5 * LN10,
                   (SPECIAL_UNK,): -2.5 * LN10}
    backoffs: dict = {(SPECIAL_BOS,): -0.3 * LN10}
    names = spec.words + [SPECIAL_BOS]
    for n in range(4):
        g = spec.grams[n]
        lp = spec.logp10[n]
        bo = spec.bo10[n]
        for row in range(len(g)):
            key = tuple(names[i] for i in g[row])
            probs[key] = float(lp[row]) * LN10
            if bo is not None:
                backoffs[key] = float(bo[row]) * LN10
    return NGramModel(order=4, probs=probs, backoffs=backoffs, unk_present=True)


def arpa_text_from_spec(spec: NgramSpec) -> str:
    names = spec.words + [SPECIAL_BOS]
    sections = []
    head = [((SPECIAL_BOS,), -99.0, -0.3), ((SPECIAL_EOS,), -1.5, None), ((SPECIAL_UNK,), -2.5, None)]
    for n in range(4):
        rows = head if n == 0 else []
        g, lp, bo = spec.grams[n], spec.logp10[n], spec.bo10[n]
        lines = [f"{repr(float(p))}\t{' '.join(k)}" + (f"\t{repr(float(b))}" if b is not None else "")
                 for k, p, b in rows]
        for r in range(len(g)):
            line = f"{repr(float(lp[r]))}\t{' '.join(names[i] for i in g[r])}"
            if bo is not None:
                line += f"\t{repr(float(bo[r]))}"
            lines.append(line)
        sections.append(lines)
    out = ["\\data\\"] + [f"ngram {n + 1}={len(s)}" for n, s in enumerate(sections)] + [""]
    for n, s in enumerate(sections):
        out.append(f"\\{n + 1}-grams:")
        out.extend(s)
        out.append("")
    out.append("\\end\\")
    return "\n".join(out) + "\n"


def make_logits(n_trials: int, n_frames: int, vocab_size: int = 41, base_seed: int = 1000,
                scale: float = 2.0) -> np.ndarray:
    out = np.empty((n_trials, n_frames, vocab_size), dtype=np.float32)
    for i in range(n_trials):
        rng = np.random.default_rng(base_seed + i)
        out[i] = rng.normal(scale=scale, size=(n_frames, vocab_size)).astype(np.float32)
    return out


@dataclass
class World:
    vocab: Vocabulary
    lexicon: Lexicon
    table: object
    model: NGramModel


def make_world(n_words: int = 100_000, n2: int = 500_000, n3: int = 250_000, n4: int = 150_000,
               seed: int = 12345, homophone_frac: float = 0.1) -> World:
    """BASELINE config-2 world at defaults (~1M n-grams, 100k words); smaller for tests."""
    vocab = vocab41()
    lex = make_lexicon(n_words, seed=seed, homophone_frac=homophone_frac)
    surfaces = [e.surface for e in lex.entries]
    spec = make_ngram_spec(surfaces, n2, n3, n4, seed=seed + 1)
    return World(vocab, lex, build_transition_table(lex, vocab), ngram_model_from_spec(spec))


def toy_world(n_words: int = 2000, seed: int = 7) -> World:
    """Config-1-sized world (2k words, ~11k n-grams) through real ARPA text parsing."""
    vocab = vocab41()
    lex = make_lexicon(n_words, seed=seed)
    spec = make_ngram_spec([e.surface for e in lex.entries], 5 * n_words // 2, 3 * n_words // 2,
                           n_words, seed=seed + 1)
    model = parse_arpa_text(arpa_text_from_spec(spec))
    return World(vocab, lex, build_transition_table(lex, vocab), model)


def _successors(model: NGramModel) -> dict:
    """word -> (successor words, weights 10^log10p) from the listed bigrams (cached)."""
    cache = getattr(model, "_synth_succ", None)
    if cache is None:
        tmp: dict = {}
        for key, lp in model.probs.items():
            if len(key) == 2:
                tmp.setdefault(key[0], []).append((key[1], lp))
        cache = {}
        for w, lst in tmp.items():
            words = [x for x, _ in lst]
            p = np.exp(np.array([lp for _, lp in lst]))
            cache[w] = (words, p / p.sum())
        model._synth_succ = cache
    return cache


def make_wer_trials(world: World, n_trials: int, seed: int = 777, sigma: float = 2.0,
                    mu: float = 10.0, min_words: int = 8, max_words: int = 20):
    """Ground-truth sentences and CTC-shaped logits for WER measurement:
    sentence = a walk over the LM's listed bigrams from `<s>` (uniform word when a history
    has no listed continuation); each word -> its lexicon phonemes, each phoneme held
    U{1..3} frames with U{0..2} blank frames before it, one `<sp>` frame after each word;
    logits = N(0, sigma) + mu on the true token (mu = 10 puts the CPU reference's WER in the
    5-25% band §8d asks for: 15% on the 2k-word world at beam 16).  Returns (list of word
    lists, list of fp32 (T_i, 41) arrays)."""
    rng = np.random.default_rng(seed)
    succ = _successors(world.model)
    pron = {e.surface: e.phonemes for e in world.lexicon.entries}
    vocab_words = [e.surface for e in world.lexicon.entries]
    sentences, logits = [], []
    for _ in range(n_trials):
        n_w = int(rng.integers(min_words, max_words + 1))
        words, prev = [], SPECIAL_BOS
        while len(words) < n_w:
            cand = succ.get(prev)
            if cand is not None and rng.random() < 0.8:
                w = cand[0][int(rng.choice(len(cand[0]), p=cand[1]))]
            else:
                w = vocab_words[int(rng.integers(0, len(vocab_words)))]
            if w not in pron:
                continue
            words.append(w)
            prev = w
        labels = []
        for w in words:
            for ph in pron[w]:
                labels.extend([0] * int(rng.integers(0, 3)))
                labels.extend([ph] * int(rng.integers(1, 4)))
            labels.append(40)
        lab = np.asarray(labels, dtype=np.int64)
        x = rng.normal(scale=sigma, size=(len(lab), 41)).astype(np.float32)
        x[np.arange(len(lab)), lab] += np.float32(mu)
        sentences.append(words)
        logits.append(x)
    return sentences, logits
