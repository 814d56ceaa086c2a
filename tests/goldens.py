"""Loaders turning tests/golden/*.json.gz (made from the reference by make_golden.py) into our
host objects.  Never imports the reference: these fixtures are how its behaviour travels."""

from __future__ import annotations

import gzip
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2603_14002_b200 import (
    DecodeConfig,
    Lexicon,
    LexiconEntry,
    NGramModel,
    StubScorer,
    Vocabulary,
    build_transition_table,
)
from paper_2603_14002_b200.ngram import parse_arpa_text

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt", encoding="utf-8") as fh:
        return json.load(fh)


def vocab_of(v) -> Vocabulary:
    return Vocabulary(tuple(v["tokens"]), v["blank"], v["space"])


def lexicon_of(rows) -> Lexicon:
    return Lexicon(tuple(LexiconEntry(k, s, tuple(p)) for k, s, p in rows))


def model_of(inst) -> NGramModel:
    if inst.get("arpa"):
        return parse_arpa_text(inst["arpa"])
    probs = {tuple(k): v for k, v in inst["probs"]}
    backoffs = {tuple(k): v for k, v in inst["backoffs"]}
    return NGramModel(inst["order"], probs, backoffs, inst["unk"])


def config_of(d) -> DecodeConfig:
    return DecodeConfig(**d)


TINY_VOCAB = {"tokens": ["<blank>", "AE", "N", "T", "<sp>"], "blank": 0, "space": 4}


def instance_world(inst):
    vocab = vocab_of(inst.get("vocab", TINY_VOCAB))
    tt = build_transition_table(lexicon_of(inst["lexicon"]), vocab)
    return vocab, tt, model_of(inst)


def scorer_for(run, inst, model, cfg):
    if run.get("ngram_stub"):
        return StubScorer(ngram_model=model, scale=cfg.ngram_weight / cfg.llm_weight)
    return StubScorer(table=dict(inst.get("stub_table") or {}))


def d_of(inst) -> np.ndarray:
    return np.asarray(inst["D"], dtype=np.float64).reshape(len(inst["D"]), -1)


def same_result(got, want) -> str | None:
    """None if `got` (text, score, nbest, llm_events | exception) equals the golden exactly."""
    if "error" in want:
        if not isinstance(got, Exception):
            return f"expected {want['error']}({want['message']}), got result {got}"
        if type(got).__name__ not in (want["error"], "OracleEmptyBeam", "OracleEmptyInput"):
            return f"expected {want['error']}, got {type(got).__name__}"
        if str(got) != want["message"]:
            return f"message {str(got)!r} != {want['message']!r}"
        return None
    if isinstance(got, Exception):
        return f"expected result, got {type(got).__name__}: {got}"
    if got.text != want["text"]:
        return f"text {got.text!r} != {want['text']!r}"
    if got.score != want["score"]:
        return f"score {got.score!r} != {want['score']!r}"
    nb = [(t, s) for t, s in want["nbest"]]
    if list(got.nbest) != nb:
        return f"nbest {got.nbest[:4]} != {nb[:4]}"
    if got.llm_events != want["llm_events"]:
        return f"llm_events {got.llm_events} != {want['llm_events']}"
    return None


def trace_rows(tr):
    return [[(int(a), int(b), p, la, s) for a, b, p, la, s in frame] for frame in tr]
