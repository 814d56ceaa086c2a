"""TEST INFRASTRUCTURE — never imported by the product package.

Loads the *unmodified* reference package `lightbeam` (pkg/src/lightbeam, installed with
`pip install --no-index --no-deps --target baseline/_ref <copy of /root/reference/pkg>`, see
DESIGN.md §6) and builds the reference's own objects for a synthetic world, so that tests and
the CPU legs of bench.py can run `lightbeam.decoder.decode` itself (`decoder.py:408-460`) on the
same inputs as the GPU path:

- `Vocabulary(tokens, blank_id, space_id)` (`vocab.py:15-40`)
- `Lexicon` / `LexiconEntry` (`lexicon.py:36-51`) -> the reference's own
  `build_transition_table` (`lexicon.py:149-209`, BFS prefix ids)
- `NGramModel(order, probs, backoffs, unk_present)` (`ngram.py:34-47`) from the same natural-log
  dictionaries `load_arpa` produces, or through the reference's own `load_arpa` on ARPA text
- `LmSession(model)` (`ngram.py:78-88`), `DecodeConfig` / `PROFILES` (`config.py:14-94`),
  `StubScorer` (`scorer.py:93-163`), `LogProbMatrix` (`logits.py:40-52`).

Search order for the package: an importable `lightbeam`, then `<repo>/baseline/_ref` (travels
to the GPU box with the snapshot), then `/root/reference/pkg/src` (this container only).
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
_CANDIDATES = (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))


def reference():
    """The reference package namespace (a module with decoder/lexicon/ngram/... loaded), or
    None when it is not available anywhere."""
    try:
        return _load()
    except ImportError:
        return None


def _load():
    try:
        lb = importlib.import_module("lightbeam")
    except ImportError:
        for c in _CANDIDATES:
            if (c / "lightbeam" / "decoder.py").exists():
                sys.path.insert(0, str(c))
                break
        else:
            raise
        lb = importlib.import_module("lightbeam")
    for sub in ("decoder", "lexicon", "ngram", "vocab", "config", "scorer", "logits", "errors"):
        importlib.import_module(f"lightbeam.{sub}")
    return lb


class RefWorld:
    """The reference-typed twin of a `paper_2603_14002_b200.synth.World`."""

    def __init__(self, world, arpa_text: str | None = None):
        lb = _load()
        self.lb = lb
        v = world.vocab
        self.vocab = lb.vocab.Vocabulary(tuple(v.tokens), v.blank_id, v.space_id)
        self.lexicon = lb.lexicon.Lexicon(tuple(
            lb.lexicon.LexiconEntry(e.key, e.surface, tuple(e.phonemes))
            for e in world.lexicon.entries))
        self.table = lb.lexicon.build_transition_table(self.lexicon, self.vocab)
        if arpa_text is not None:
            import tempfile

            with tempfile.NamedTemporaryFile("w", suffix=".arpa", delete=False) as f:
                f.write(arpa_text)
            self.model = lb.ngram.load_arpa(f.name)
            Path(f.name).unlink()
        else:
            m = world.model
            self.model = lb.ngram.NGramModel(order=m.order, probs=dict(m.probs),
                                             backoffs=dict(m.backoffs), unk_present=m.unk_present)

    def config(self, cfg):
        """The reference DecodeConfig with the same field values as `cfg`."""
        return self.lb.config.DecodeConfig(**cfg.as_dict())

    def session(self):
        return self.lb.ngram.LmSession(self.model)

    def stub(self, scale: float):
        return self.lb.scorer.StubScorer(ngram_model=self.model, scale=scale)

    def logprobs(self, d, cfg, frame_ms: float = 80.0):
        return self.lb.logits.LogProbMatrix(d, cfg.acoustic_scale, frame_ms)

    def scale_log_softmax(self, raw, cfg, frame_ms: float = 80.0):
        """The reference prologue (`logits.py:119-130`) on fp32 logits -> fp64 [T, V]."""
        lg = self.lb.logits
        return lg.scale_log_softmax(lg.RawLogits(raw, frame_ms), cfg.acoustic_scale).frames

    def decode(self, d, cfg, scorer, final_llm_only=False):
        """`lightbeam.decoder.decode` on an fp64 [T, V] matrix; returns its DecodeResult or the
        reference exception instance it raised."""
        rc = cfg if isinstance(cfg, self.lb.config.DecodeConfig) else self.config(cfg)
        try:
            return self.lb.decoder.decode(self.logprobs(d, rc), rc, self.table, self.session(),
                                          scorer, final_llm_only=final_llm_only)
        except self.lb.errors.LightBeamError as exc:
            return exc
