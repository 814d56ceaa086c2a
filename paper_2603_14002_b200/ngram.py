"""ARPA back-off n-gram model: host parsing plus the host-side scoring contract.

The parse semantics follow the reference `load_arpa` (`pkg/src/lightbeam/ngram.py:90-174`):
log10 values are converted to natural log at load (`float(x) * ln 10`, one fp64 rounding),
the model order is the highest populated section, declared counts must match.  Scoring
(`score_word`, `ngram.py:187-236`) is restated here because the scorer protocol's n-gram
stub (`scorer.StubScorer(ngram_model=...)`) needs it on the host; the *decoder's* n-gram
probes run on the GPU against the hashed image built by `images.compile_ngram`.

Registry/cache (`LmStateRegistry`, `LmSession`) exist for API compatibility with callers of
the reference: the device path identifies LM states by packed word ids, not session ids.
"""

from __future__ import annotations

import gzip
import math
import re
from dataclasses import dataclass, field
from pathlib import Path

from .errors import FormatError

BOS = "<s>"
EOS = "</s>"
UNK = "<unk>"
LN10 = math.log(10.0)
NEG_INF = -1.0e30  # finite log(0): additions never produce NaN
NEG_INF_GUARD = -1.0e29  # anything at or below is treated as pruned

_COUNT_LINE = re.compile(r"^ngram (\d+)=(\d+)$")
_SECTION_LINE = re.compile(r"^\\(\d+)-grams:$")


@dataclass
class NGramModel:
    order: int
    probs: dict[tuple[str, ...], float]
    backoffs: dict[tuple[str, ...], float]
    unk_present: bool
    prob_lookups: int = 0  # diagnostic counter, as in the reference

    def vocabulary(self) -> list[str]:
        return sorted(g[0] for g in self.probs if len(g) == 1)


@dataclass
class LmStateRegistry:
    histories: list[tuple[str, ...]] = field(default_factory=lambda: [(BOS,)])
    index: dict[tuple[str, ...], int] = field(default_factory=lambda: {(BOS,): 0})

    def state_of(self, history: tuple[str, ...]) -> int:
        sid = self.index.get(history)
        if sid is None:
            sid = len(self.histories)
            self.index[history] = sid
            self.histories.append(history)
        return sid

    def history(self, state: int) -> tuple[str, ...]:
        if not 0 <= state < len(self.histories):
            raise IndexError(f"unregistered LM state id {state}")
        return self.histories[state]


@dataclass
class LmSession:
    model: NGramModel
    registry: LmStateRegistry = field(default_factory=LmStateRegistry)
    cache: dict = field(default_factory=dict)

    @property
    def bos_state(self) -> int:
        return 0


class _ArpaReader:
    """Line-driven ARPA state machine; errors carry `path:line`."""

    def __init__(self, path):
        self.path = path
        self.declared: dict[int, int] = {}
        self.found: dict[int, int] = {}
        self.probs: dict[tuple[str, ...], float] = {}
        self.backoffs: dict[tuple[str, ...], float] = {}
        self.section = None  # None | "data" | n
        self.saw_data = False
        self.saw_end = False

    def fail(self, lineno, msg):
        raise FormatError(f"{self.path}:{lineno}: {msg}")

    def feed(self, lineno: int, line: str) -> None:
        if line == "\\data\\":
            self.saw_data, self.section = True, "data"
            return
        sect = _SECTION_LINE.match(line)
        if sect:
            n = int(sect.group(1))
            if n not in self.declared:
                self.fail(lineno, f"section \\{n}-grams: not declared")
            self.section = n
            return
        if line == "\\end\\":
            self.saw_end, self.section = True, None
            return
        if self.section == "data":
            m = _COUNT_LINE.match(line)
            if not m:
                self.fail(lineno, f"bad count line {line!r}")
            self.declared[int(m.group(1))] = int(m.group(2))
            return
        if isinstance(self.section, int):
            self.entry(lineno, line, self.section)
            return
        if self.saw_data:
            self.fail(lineno, f"unexpected line outside any section: {line!r}")
        # free-form preamble before \data\ is tolerated

    def entry(self, lineno: int, line: str, n: int) -> None:
        cols = line.split()
        if len(cols) != n + 1 and len(cols) != n + 2:
            self.fail(lineno, f"malformed {n}-gram line {line!r}")
        try:
            logp = float(cols[0])
        except ValueError:
            self.fail(lineno, f"bad probability {cols[0]!r}")
        gram = tuple(cols[1 : n + 1])
        self.probs[gram] = logp * LN10
        if len(cols) == n + 2:
            try:
                self.backoffs[gram] = float(cols[n + 1]) * LN10
            except ValueError:
                self.fail(lineno, f"bad backoff {cols[n + 1]!r}")
        self.found[n] = self.found.get(n, 0) + 1

    def finish(self) -> NGramModel:
        if not self.saw_data:
            raise FormatError(f"{self.path}: missing \\data\\ section")
        if not self.saw_end:
            raise FormatError(f"{self.path}: missing \\end\\ marker")
        for n, want in self.declared.items():
            have = self.found.get(n, 0)
            if have != want:
                raise FormatError(f"{self.path}: declared {want} {n}-grams but found {have}")
        populated = [n for n, c in self.found.items() if c > 0]
        if not populated:
            raise FormatError(f"{self.path}: no n-gram entries")
        return NGramModel(max(populated), self.probs, self.backoffs, (UNK,) in self.probs)


def parse_arpa_text(text: str, path="<string>") -> NGramModel:
    reader = _ArpaReader(path)
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.strip()
        if line:
            reader.feed(lineno, line)
    return reader.finish()


def load_arpa(path: str | Path) -> NGramModel:
    blob = Path(path).read_bytes()
    if blob[:2] == b"\x1f\x8b":
        blob = gzip.decompress(blob)
    return parse_arpa_text(blob.decode("utf-8"), path)


def backoff_logprob(model: NGramModel, history: tuple[str, ...], word: str) -> float:
    """P(word | history) with right-nested back-off: bo(h0) + (bo(h1) + (... + p))."""
    chain = []
    h = history
    while True:
        model.prob_lookups += 1
        p = model.probs.get(h + (word,))
        if p is not None:
            break
        if not h:
            p = NEG_INF
            break
        chain.append(model.backoffs.get(h, 0.0))
        h = h[1:]
    for bo in reversed(chain):
        p = bo + p
    return p


def successor_history(model: NGramModel, history: tuple[str, ...], word: str):
    """Longest suffix of (history + word), capped at order-1 words, that is a listed n-gram."""
    if model.order <= 1:
        return ()
    h = (history + (word,))[-(model.order - 1) :]
    while h:
        model.prob_lookups += 1
        if h in model.probs:
            break
        h = h[1:]
    return h


def score_word(model: NGramModel, registry: LmStateRegistry, cache: dict, state: int, word: str):
    """(natural-log increment, successor registry id); OOV -> <unk> or NEG_INF."""
    key = (state, word)
    hit = cache.get(key)
    if hit is not None:
        return hit
    history = registry.history(state)
    model.prob_lookups += 1
    if (word,) in model.probs:
        effective = word
    elif model.unk_present:
        effective = UNK
    else:
        result = (NEG_INF, registry.state_of(()))
        cache[key] = result
        return result
    result = (
        backoff_logprob(model, history, effective),
        registry.state_of(successor_history(model, history, effective)),
    )
    cache[key] = result
    return result


def score_sequence(model: NGramModel, words: list[str], include_eos: bool = False) -> float:
    """Left-to-right sum of increments from `<s>` (reference `ngram.py:239-250`)."""
    session = LmSession(model)
    state, total = session.bos_state, 0.0
    for w in list(words) + ([EOS] if include_eos else []):
        inc, state = score_word(model, session.registry, session.cache, state, w)
        total += inc
    return total
