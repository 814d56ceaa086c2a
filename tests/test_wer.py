"""WER measurement support: the restated metric against the reference's (when its tree is
present) and hand cases; WER-parity trials (ragged, speech-shaped) decode identically on the
GPU and in the oracle."""

import os
import sys

import pytest

from paper_2603_14002_b200 import PROFILES, StubScorer, synth
from paper_2603_14002_b200.metrics import corpus_wer, wer

REF = "/root/reference/pkg/src"


def test_wer_hand_cases():
    b = wer(["a", "b", "c"], ["a", "x", "c", "d"])
    assert (b.substitutions, b.insertions, b.deletions, b.reference_words) == (1, 1, 0, 3)
    assert wer(["A", "b."], ["a", "b"]).wer == 0.0
    assert wer(["a", "b"], []).deletions == 2
    assert corpus_wer([["a", "b"], ["c"]], [["a"], ["c"]]) == pytest.approx(1 / 3)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")
def test_wer_matches_reference_metric():
    import numpy as np

    sys.path.insert(0, REF)
    try:
        from lightbeam.metrics import wer as ref_wer
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(3)
    for _ in range(300):
        r = [f"w{x}" for x in rng.integers(0, 5, size=rng.integers(1, 8))]
        h = [f"w{x}" for x in rng.integers(0, 5, size=rng.integers(0, 8))]
        a, b = wer(r, h), ref_wer(r, h)
        assert (a.substitutions, a.insertions, a.deletions, a.wer) == (
            b.substitutions, b.insertions, b.deletions, b.wer)


def test_wer_trials_shape():
    w = synth.toy_world(n_words=300, seed=3)
    sents, logs = synth.make_wer_trials(w, 4, seed=1)
    assert len(sents) == 4 and all(x.shape[1] == 41 for x in logs)
    assert len({x.shape[0] for x in logs}) > 1  # ragged


@pytest.mark.gpu
def test_wer_trials_gpu_equals_oracle():
    from oracle import lightbeam_oracle as O
    from paper_2603_14002_b200 import decode_batch_raw

    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=16)
    sc = StubScorer(ngram_model=w.model, scale=cfg.ngram_weight / cfg.llm_weight)
    sents, logs = synth.make_wer_trials(w, 12, seed=5)
    got = decode_batch_raw(logs, cfg, w.table, w.model, sc, final_llm_only=True)
    want = [O.decode(O.log_softmax_scaled(x, cfg.acoustic_scale), cfg, w.table, w.model, sc,
                     final_llm_only=True).text for x in logs]
    assert [g.text for g in got] == want
    assert corpus_wer(sents, [g.text.split() for g in got]) < 0.3
