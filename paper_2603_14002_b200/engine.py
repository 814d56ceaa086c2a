"""Engine: a loaded component set ready to decode utterances on the GPU.

Mirrors the reference's orchestration API (`pkg/src/lightbeam/engine.py:41-177`):
`build_engine(vocab_path, arpa_path, scorer_spec, lexicon_path | table_path, config...)` and
`Engine.decode_matrix / decode_raw / decode_path / close` with the same arguments and return
values (`DecodeResult`, and `(DecodeResult, RtfSample)` for raw logits), so a service or CLI
built on the reference engine can switch by import.  Added for the GPU: `decode_batch` /
`decode_batch_raw` / `decode_paths`, which decode many utterances in one device batch (one
CTA per utterance) and return a result or the exception per utterance.

Scorer specs: the reference kinds `stub_table` and `stub_ngram` behave identically;
`device_ngram` is the device twin of `stub_ngram` (fusion events never leave the GPU); `llama`
builds a `LlamaScorer` (random-init Llama architecture on the GPU, prefix-trie KV cache).
The JSONL `subprocess`/`tcp` transports are outside the B200 path: pass the
reference's own `SubprocessScorer`/`TcpScorer` object as `ScorerSpec(kind="object", obj=...)`
and it is driven through its `submit()` protocol.
"""

from __future__ import annotations

import hashlib
import json
import time
from dataclasses import dataclass, field
from pathlib import Path

from .config import DecodeConfig, config_from_dict, load_config
from .decoder import DecodeResult, decode, decode_batch, decode_batch_raw
from .errors import ConfigError
from .lexicon import TransitionTable, build_transition_table, load_lexicon, load_table
from .logits import LogProbMatrix, RawLogits, load_logits, load_logits_batch
from .metrics import RtfSample, rtf
from .ngram import LmSession, NGramModel, load_arpa
from .scorer import DeviceNgramScorer, StubScorer
from .vocab import Vocabulary, load_vocab


def sha256_of(path: str | Path) -> str:
    digest = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 20), b""):
            digest.update(chunk)
    return digest.hexdigest()


@dataclass
class ScorerSpec:
    """How to construct the fusion scorer of an engine (engine.py:41-74)."""

    kind: str  # "stub_table" | "stub_ngram" | "device_ngram" | "llama" | "object"
    table: dict | None = None
    table_path: str | None = None
    scale: float = 1.0
    delay_per_text_s: float = 0.0
    model: str = "llama-3.2-1b"  # llama: preset name
    precision: str = "bf16x2"  # llama: "bf16x2" | "bf16"
    seed: int = 0
    obj: object = None  # kind "object": any submit() scorer
    options: dict = field(default_factory=dict)

    def build(self, ngram_model: NGramModel):
        if self.kind == "stub_table":
            table = self.table
            if table is None and self.table_path:
                table = json.loads(Path(self.table_path).read_text(encoding="utf-8"))
            return StubScorer(table=dict(table or {}), scale=self.scale,
                              delay_per_text_s=self.delay_per_text_s)
        if self.kind == "stub_ngram":
            return StubScorer(ngram_model=ngram_model, scale=self.scale,
                              delay_per_text_s=self.delay_per_text_s)
        if self.kind == "device_ngram":
            return DeviceNgramScorer(ngram_model, self.scale)
        if self.kind == "llama":
            from .llm import LlamaScorer

            return LlamaScorer(self.model, seed=self.seed, precision=self.precision, **self.options)
        if self.kind == "object":
            if self.obj is None or not hasattr(self.obj, "submit"):
                raise ConfigError("object scorer needs an instance with submit()")
            return self.obj
        if self.kind in ("subprocess", "tcp"):
            raise ConfigError(f"{self.kind} transport is not part of the B200 decoder; construct "
                              "the reference scorer and pass it as ScorerSpec(kind='object', obj=...)")
        raise ConfigError(f"unknown scorer kind {self.kind!r}")


class Engine:
    """Immutable components (vocab, table, n-gram model, config) plus a scorer; the device
    images of the table and n-gram model are built on first use and shared by every decode."""

    def __init__(self, vocab: Vocabulary, table: TransitionTable, ngram_model: NGramModel,
                 config: DecodeConfig, scorer, components: dict, device: int = 0):
        self.vocab = vocab
        self.table = table
        self.ngram_model = ngram_model
        self.config = config
        self.scorer = scorer
        self.components = components
        self.device = device

    # ---- reference API (engine.py:113-126)
    def decode_matrix(self, d: LogProbMatrix, final_llm_only: bool = False) -> DecodeResult:
        lm = LmSession(self.ngram_model)
        return decode(d, self.config, self.table, lm, self.scorer, final_llm_only=final_llm_only)

    def decode_raw(self, raw: RawLogits, final_llm_only: bool = False):
        """Raw fp32 logits -> (DecodeResult, RtfSample); the log-softmax prologue runs on the
        device (kernel K1, within a few ulps of numpy's)."""
        res = self.decode_batch_raw([raw], final_llm_only)[0]
        if isinstance(res, Exception):
            raise res
        return res, rtf(res.wall_time_s, res.frame_count, raw.frame_duration_ms)

    def decode_path(self, path: str | Path, final_llm_only: bool = False):
        return self.decode_raw(load_logits(path, self.vocab), final_llm_only=final_llm_only)

    def close(self):
        if hasattr(self.scorer, "close"):
            self.scorer.close()

    # ---- batched GPU API
    def decode_batch(self, ds, final_llm_only: bool = False) -> list:
        return decode_batch(ds, self.config, self.table, self.ngram_model, self.scorer,
                            final_llm_only=final_llm_only, device=self.device)

    def decode_batch_raw(self, raws, final_llm_only: bool = False) -> list:
        return decode_batch_raw(raws, self.config, self.table, self.ngram_model, self.scorer,
                                final_llm_only=final_llm_only, device=self.device)

    def decode_paths(self, paths, final_llm_only: bool = False) -> list:
        """[(DecodeResult, RtfSample) | exception] per file, decoded as one device batch; the
        LBLT payloads are read straight into one page-locked staging array."""
        paths = list(paths)
        if not paths:
            return []
        arr, frames, frame_ms, errors = load_logits_batch(paths, self.vocab)
        err = dict(errors)
        ok = [i for i in range(len(paths)) if i not in err]
        t0 = time.perf_counter()
        if len(ok) == len(paths):  # keep the page-locked staging array (no gather copy)
            res = self.decode_batch_raw((arr, frames), final_llm_only)
        else:
            res = self.decode_batch_raw((arr[ok], frames[ok]), final_llm_only) if ok else []
        wall = time.perf_counter() - t0
        out: list = [None] * len(paths)
        for i, e in err.items():
            out[i] = e
        for j, i in enumerate(ok):
            r = res[j]
            out[i] = r if isinstance(r, Exception) else (
                r, rtf(wall / max(len(ok), 1), r.frame_count, frame_ms[i]))
        return out


def build_engine(vocab_path, arpa_path, scorer_spec: ScorerSpec, lexicon_path=None,
                 table_path=None, config: DecodeConfig | None = None, config_path=None,
                 config_overrides: dict | None = None, device: int = 0) -> Engine:
    """engine.py:132-177 with the same argument rules (exactly one of lexicon/table, a config
    from an object, a file or overrides)."""
    if (lexicon_path is None) == (table_path is None):
        raise ConfigError("provide exactly one of lexicon_path or table_path")
    if config is None:
        if config_path is not None:
            config = load_config(config_path)
        elif config_overrides is not None:
            config = config_from_dict(config_overrides)
        else:
            raise ConfigError("no decoding config given")
    elif config_overrides:
        config = config.replace(**config_overrides)
    vocab = load_vocab(vocab_path)
    components = {"vocab": {"path": str(vocab_path), "sha256": sha256_of(vocab_path)}}
    if lexicon_path is not None:
        table = build_transition_table(load_lexicon(lexicon_path, vocab), vocab)
        components["lexicon"] = {"path": str(lexicon_path), "sha256": sha256_of(lexicon_path)}
    else:
        table = load_table(table_path, vocab)
        components["table"] = {"path": str(table_path), "sha256": sha256_of(table_path)}
    ngram_model = load_arpa(arpa_path)
    components["arpa"] = {"path": str(arpa_path), "sha256": sha256_of(arpa_path)}
    if scorer_spec.table_path:
        components["stub_table"] = {"path": str(scorer_spec.table_path),
                                    "sha256": sha256_of(scorer_spec.table_path)}
    return Engine(vocab, table, ngram_model, config, scorer_spec.build(ngram_model), components,
                  device)
