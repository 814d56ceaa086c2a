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
    """Hex sha256 of a component file (recorded in `Engine.components`, as the reference's
    run manifests do)."""
    with open(path, "rb") as fh:
        return hashlib.file_digest(fh, "sha256").hexdigest()


def _stub_table(spec: "ScorerSpec", _model):
    table = spec.table
    if table is None and spec.table_path:
        table = json.loads(Path(spec.table_path).read_text(encoding="utf-8"))
    return StubScorer(table=dict(table or {}), scale=spec.scale,
                      delay_per_text_s=spec.delay_per_text_s)


def _llama(spec: "ScorerSpec", _model):
    from .llm import LlamaScorer

    return LlamaScorer(spec.model, seed=spec.seed, precision=spec.precision, **spec.options)


def _instance(spec: "ScorerSpec", _model):
    if not hasattr(spec.obj, "submit"):
        raise ConfigError("object scorer needs an instance with submit()")
    return spec.obj


def _transport(spec: "ScorerSpec", _model):
    raise ConfigError(f"{spec.kind} transport is not part of the B200 decoder; construct the "
                      "reference scorer and pass it as ScorerSpec(kind='object', obj=...)")


_BUILDERS = {
    "stub_table": _stub_table,
    "stub_ngram": lambda spec, model: StubScorer(ngram_model=model, scale=spec.scale,
                                                 delay_per_text_s=spec.delay_per_text_s),
    "device_ngram": lambda spec, model: DeviceNgramScorer(model, spec.scale),
    "llama": _llama,
    "object": _instance,
    "subprocess": _transport,
    "tcp": _transport,
}


@dataclass
class ScorerSpec:
    """How to construct the fusion scorer of an engine (the reference's kinds, engine.py:41-74,
    plus the device kinds); `build` dispatches on `kind` through `_BUILDERS`."""

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
        builder = _BUILDERS.get(self.kind)
        if builder is None:
            raise ConfigError(f"unknown scorer kind {self.kind!r}")
        return builder(self, ngram_model)


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

    # ---- reference API (engine.py:113-126), routed through the batched device path
    def decode_matrix(self, d: LogProbMatrix, final_llm_only: bool = False) -> DecodeResult:
        return decode(d, self.config, self.table, self.ngram_model, self.scorer,
                      final_llm_only=final_llm_only)

    def decode_raw(self, raw: RawLogits, final_llm_only: bool = False):
        """Raw fp32 logits -> (DecodeResult, RtfSample); the log-softmax prologue runs on the
        device (kernel K1, within a few ulps of numpy's)."""
        (res,) = self.decode_batch_raw([raw], final_llm_only)
        if isinstance(res, Exception):
            raise res
        return res, rtf(res.wall_time_s, res.frame_count, raw.frame_duration_ms)

    def decode_path(self, path: str | Path, final_llm_only: bool = False):
        return self.decode_raw(load_logits(path, self.vocab), final_llm_only=final_llm_only)

    def close(self):
        """Close the scorer (if it has a transport) and drop this engine's device images."""
        getattr(self.scorer, "close", lambda: None)()
        from .decoder import release_device_model

        release_device_model(self.table, self.ngram_model, self.device)

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


def _resolve_config(config, config_path, overrides) -> DecodeConfig:
    """An explicit config (with overrides applied), else a config file, else overrides alone."""
    if config is not None:
        return config.replace(**overrides) if overrides else config
    if config_path is not None:
        return load_config(config_path)
    if overrides is not None:
        return config_from_dict(overrides)
    raise ConfigError("no decoding config given")


def build_engine(vocab_path, arpa_path, scorer_spec: ScorerSpec, lexicon_path=None,
                 table_path=None, config: DecodeConfig | None = None, config_path=None,
                 config_overrides: dict | None = None, device: int = 0,
                 image_cache=None) -> Engine:
    """Load the component set (the argument rules of the reference's `build_engine`,
    engine.py:132-177: exactly one of lexicon/table; a config object, file or overrides) and
    record every component file's path and sha256.  `image_cache` (a directory): the compiled
    device images are kept there under the components' combined sha256, so the next engine
    over the same files uploads them instead of compiling."""
    if (lexicon_path is None) == (table_path is None):
        raise ConfigError("provide exactly one of lexicon_path or table_path")
    cfg = _resolve_config(config, config_path, config_overrides)
    vocab = load_vocab(vocab_path)
    if lexicon_path is not None:
        table = build_transition_table(load_lexicon(lexicon_path, vocab), vocab)
    else:
        table = load_table(table_path, vocab)
    ngram_model = load_arpa(arpa_path)
    files = {"vocab": vocab_path, "lexicon": lexicon_path, "table": table_path,
             "arpa": arpa_path, "stub_table": scorer_spec.table_path}
    components = {name: {"path": str(p), "sha256": sha256_of(p)}
                  for name, p in files.items() if p}
    if image_cache is not None:
        from .decoder import register_image_path

        digest = hashlib.sha256("".join(
            f"{n}={components[n]['sha256']};" for n in ("vocab", "lexicon", "table", "arpa")
            if n in components).encode()).hexdigest()
        Path(image_cache).mkdir(parents=True, exist_ok=True)
        path = Path(image_cache) / f"lb_images_{digest[:32]}.npz"
        register_image_path(table, ngram_model, path)
        components["device_images"] = {"path": str(path), "sha256_of_components": digest}
    return Engine(vocab, table, ngram_model, cfg, scorer_spec.build(ngram_model), components,
                  device)
