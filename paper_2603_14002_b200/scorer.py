"""Sentence-scorer plugin contract (host side) for delayed LLM fusion.

The duck-typed contract is the reference's (`pkg/src/lightbeam/scorer.py:34-45,93-163,
269-325`): a scorer exposes `submit(ScoreRequest) -> ScoreResponse` and
`next_request_id()`; requests carry `kind` "score" or "score_eos"; `score_texts` /
`score_eos` dedupe order-preservingly and chunk by `llm_chunk_size`.  Any such object --
including the reference's own `StubScorer`/`SubprocessScorer` -- can be passed to
`decoder.decode`; the decoder then moves word-history texts device->host at each fusion
event and the scores host->device.

Scorers that also carry a device-native evaluation (`DeviceNgramScorer` below) are driven
without leaving the GPU: the decoder evaluates them inside its own kernels.
"""

from __future__ import annotations

import itertools
import json
import time
from dataclasses import dataclass

from .errors import ScorerError
from .ngram import NGramModel, score_sequence

PUNCTS = (".", "?", "!")


@dataclass(frozen=True)
class ScoreRequest:
    id: int
    kind: str  # "score" | "score_eos"
    texts: tuple[str, ...]


@dataclass(frozen=True)
class ScoreResponse:
    id: int
    scores: tuple[float, ...]
    puncts: tuple[str, ...] | None = None


def encode_request(req: ScoreRequest) -> str:
    return json.dumps({"id": req.id, "kind": req.kind, "texts": list(req.texts)})


def decode_request(line: str) -> ScoreRequest:
    obj = json.loads(line)
    return ScoreRequest(int(obj["id"]), str(obj["kind"]), tuple(obj["texts"]))


def encode_response(resp: ScoreResponse) -> str:
    obj: dict = {"id": resp.id, "scores": list(resp.scores)}
    if resp.puncts is not None:
        obj["puncts"] = list(resp.puncts)
    return json.dumps(obj)


def decode_response(line: str, expect_id: int | None = None) -> ScoreResponse:
    try:
        obj = json.loads(line)
    except json.JSONDecodeError as exc:
        raise ScorerError(f"malformed scorer reply: {exc}", expect_id) from exc
    if "error" in obj:
        raise ScorerError(f"scorer error: {obj['error']}", obj.get("id", expect_id))
    if "id" not in obj or "scores" not in obj:
        raise ScorerError("scorer reply missing id/scores", expect_id)
    resp = ScoreResponse(
        int(obj["id"]),
        tuple(float(s) for s in obj["scores"]),
        tuple(obj["puncts"]) if "puncts" in obj else None,
    )
    if expect_id is not None and resp.id != expect_id:
        raise ScorerError(f"scorer reply id {resp.id} != request id {expect_id}", expect_id)
    return resp


class StubScorer:
    """Deterministic in-process scorer (reference `scorer.py:93-163`).

    Table mode: `scale * table[text]`, unknown text -> `scale * -(#words)`; eos picks the best
    of `text+"."`, `text+"?"`, `text+"!"` with strict `>` (ties -> "."). N-gram mode:
    `scale * score_sequence(words)`; eos appends `</s>` and always answers ".".
    """

    def __init__(self, table=None, ngram_model: NGramModel | None = None, scale: float = 1.0,
                 delay_per_text_s: float = 0.0):
        if (table is None) == (ngram_model is None):
            raise ValueError("provide exactly one of table or ngram_model")
        self.table = table
        self.ngram_model = ngram_model
        self.scale = scale
        self.delay_per_text_s = delay_per_text_s
        self.evaluations = 0
        self._ids = itertools.count(1)

    def next_request_id(self) -> int:
        return next(self._ids)

    def _table_score(self, text: str) -> float:
        raw = self.table[text] if text in self.table else -1.0 * len(text.split())
        return self.scale * raw

    def score_one(self, text: str) -> float:
        if self.table is not None:
            return self._table_score(text)
        return self.scale * score_sequence(self.ngram_model, text.split())

    def score_eos_one(self, text: str) -> tuple[str, float]:
        if self.table is None:
            total = score_sequence(self.ngram_model, text.split(), include_eos=True)
            return PUNCTS[0], self.scale * total
        best_p, best = None, None
        for p in PUNCTS:
            s = self._table_score(text + p)
            if best is None or s > best:
                best_p, best = p, s
        return best_p, best

    def submit(self, request: ScoreRequest) -> ScoreResponse:
        if self.delay_per_text_s > 0:
            time.sleep(self.delay_per_text_s * len(request.texts))
        self.evaluations += len(request.texts)
        if request.kind == "score":
            return ScoreResponse(request.id, tuple(self.score_one(t) for t in request.texts))
        if request.kind == "score_eos":
            pairs = [self.score_eos_one(t) for t in request.texts]
            return ScoreResponse(request.id, tuple(s for _, s in pairs), tuple(p for p, _ in pairs))
        raise ScorerError(f"unknown request kind {request.kind!r}", request.id)

    def close(self):
        pass


def _unique_in_order(texts, chunk_size):
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    slot: dict[str, int] = {}
    uniq: list[str] = []
    where = []
    for t in texts:
        if t not in slot:
            slot[t] = len(uniq)
            uniq.append(t)
        where.append(slot[t])
    return uniq, where


def score_texts(scorer, texts: list[str], chunk_size: int) -> list[float]:
    if not texts:
        return []
    uniq, where = _unique_in_order(texts, chunk_size)
    got: list[float] = []
    for lo in range(0, len(uniq), chunk_size):
        chunk = tuple(uniq[lo : lo + chunk_size])
        resp = scorer.submit(ScoreRequest(scorer.next_request_id(), "score", chunk))
        if len(resp.scores) != len(chunk):
            raise ScorerError(
                f"scorer returned {len(resp.scores)} scores for {len(chunk)} texts", resp.id
            )
        got.extend(resp.scores)
    return [got[i] for i in where]


def score_eos(scorer, texts: list[str], chunk_size: int = 256) -> list[tuple[str, float]]:
    if not texts:
        return []
    uniq, where = _unique_in_order(texts, chunk_size)
    got: list[tuple[str, float]] = []
    for lo in range(0, len(uniq), chunk_size):
        chunk = tuple(uniq[lo : lo + chunk_size])
        resp = scorer.submit(ScoreRequest(scorer.next_request_id(), "score_eos", chunk))
        if resp.puncts is None or len(resp.scores) != len(chunk) or len(resp.puncts) != len(chunk):
            raise ScorerError("score_eos reply missing puncts or wrong length", resp.id)
        for p, s in zip(resp.puncts, resp.scores):
            if p not in PUNCTS:
                raise ScorerError(f"scorer chose invalid punctuation {p!r}", resp.id)
            got.append((p, s))
    return [got[i] for i in where]


class DeviceNgramScorer:
    """Device-native twin of `StubScorer(ngram_model=model, scale=scale)`.

    Same scores by construction: the stub's `scale * score_sequence(words)` is the
    left-to-right sum of the n-gram increments from `<s>` (`ngram.py:239-250`), which is exactly
    the sum the decoder already formed when it created each word-history node (same start
    state, same `score_word` chain, same fp64 order).  The device keeps that running sum per
    node, so an interval event costs one load per entry and the final pass one extra
    `</s>` probe (`scorer.py:136-139`: eos appends `</s>`, punctuation is always ".").

    `decode` drives it on the GPU when `model` is the decode's own LM and every lexicon
    surface is a single whitespace-free token (otherwise `text.split()` could regroup words);
    `submit()` keeps the host protocol for any other caller.
    """

    def __init__(self, model: NGramModel, scale: float = 1.0):
        self.device_ngram_model = model
        self.scale = float(scale)
        self._host = StubScorer(ngram_model=model, scale=scale)

    def next_request_id(self) -> int:
        return self._host.next_request_id()

    def submit(self, request: ScoreRequest) -> ScoreResponse:
        return self._host.submit(request)

    def close(self):
        pass
