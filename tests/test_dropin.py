"""Drop-in boundary on CPU: the reference's own objects (`TransitionTable`, `NGramModel` /
`LmSession`, `DecodeConfig`, `StubScorer`, built by the unmodified reference package) go
through this package's host preparation and produce exactly the device images, config and
fusion-score batches the mirror objects produce; with `lightbeam` loaded, this package's
errors are reference exceptions and its results are the reference's `DecodeResult`."""

import dataclasses
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import refbridge
from paper_2603_14002_b200 import PROFILES, StubScorer, images, synth
from paper_2603_14002_b200.config import coerce_config
from paper_2603_14002_b200.scorer import score_eos, score_texts

REF = refbridge.reference()
needs_ref = pytest.mark.skipif(REF is None, reason="reference package not installed")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def worlds():
    w = synth.toy_world(n_words=1500, seed=11)
    return w, refbridge.RefWorld(w, arpa_text=None)


def _same_dataclass(a, b):
    for f in dataclasses.fields(a):
        x, y = getattr(a, f.name), getattr(b, f.name)
        if isinstance(x, np.ndarray):
            assert x.dtype == y.dtype and np.array_equal(x, y), f.name
        elif isinstance(x, dict):
            assert x == y, f.name
        else:
            assert x == y, f.name


@needs_ref
def test_reference_objects_compile_to_identical_device_images(worlds):
    w, rw = worlds
    # the reference's own BFS numbering == the mirror builder's (prefix ids)
    assert np.array_equal(rw.table.table, w.table.table)
    ng_ref, ng_ours = images.compile_ngram(rw.model), images.compile_ngram(w.model)
    _same_dataclass(ng_ref, ng_ours)
    _same_dataclass(images.compile_table(rw.table, rw.model, ng_ref),
                    images.compile_table(w.table, w.model, ng_ours))
    # LmSession is accepted where the reference passes it (decode(..., lm, ...)): its .model
    sess = rw.session()
    assert getattr(sess, "model", sess) is rw.model


@needs_ref
def test_reference_config_and_profiles_coerce(worlds):
    _, rw = worlds
    for name, prof in REF.config.PROFILES.items():
        ours = coerce_config(prof.replace(beam_size=33))
        assert ours == PROFILES[name].replace(beam_size=33)
        assert ours.as_dict() == prof.replace(beam_size=33).as_dict()


@needs_ref
def test_host_fusion_batches_with_reference_scorer(worlds):
    """The host fusion path sends texts through the scorer protocol with this package's
    score_texts/score_eos; with the reference's StubScorer they return what the reference's
    own helpers return (scorer.py:269-325: dedupe, chunks, eos punctuation)."""
    w, rw = worlds
    texts = ["w1 w2", "w3", "", "w1 w2", "w7 w8 w9", "w4"]
    for scale in (0.5, 1.0):
        a, b = rw.stub(scale), rw.stub(scale)
        assert score_texts(a, texts, 2) == REF.scorer.score_texts(b, texts, 2)
        assert score_eos(a, texts, 3) == REF.scorer.score_eos(b, texts, 3)
        assert a.evaluations == b.evaluations
    ours = StubScorer(ngram_model=w.model, scale=0.5)
    assert score_texts(ours, texts, 4) == REF.scorer.score_texts(rw.stub(0.5), texts, 4)


@needs_ref
def test_error_and_result_types_are_the_reference_types():
    """In a process where `lightbeam` is importable, the package's exception classes derive
    from the reference's and DecodeResult is the reference's dataclass (errors.py:4-45,
    decoder.py:86-93)."""
    lb_dir = os.path.dirname(os.path.dirname(REF.__file__))
    code = (
        "import lightbeam, paper_2603_14002_b200 as P\n"
        "names = ['LightBeamError','FormatError','ShapeError','DataValueError','ConfigError',"
        "'ScorerError','EmptyBeamError','MetricError','InstanceTooLargeError','BuilderError']\n"
        "for n in names:\n"
        "    assert issubclass(getattr(P, n), getattr(lightbeam, n)), n\n"
        "    assert issubclass(getattr(P, n), P.LightBeamError), n\n"
        "assert issubclass(P.DeviceError, lightbeam.LightBeamError)\n"
        "assert P.DecodeResult is lightbeam.DecodeResult\n"
        "try:\n"
        "    raise P.EmptyBeamError('all candidates pruned at frame 3')\n"
        "except lightbeam.EmptyBeamError as e:\n"
        "    assert str(e) == 'all candidates pruned at frame 3'\n"
        "e = P.ScorerError('bad', request_id=7)\n"
        "assert isinstance(e, lightbeam.ScorerError) and e.request_id == 7\n"
        "try:\n"
        "    P.decode(__import__('numpy').zeros((0, 41)), None, None, None, None)\n"
        "except lightbeam.DataValueError as e:\n"
        "    assert 'empty' in str(e)\n"
        "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([lb_dir, ROOT]))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr[-2000:]
    # and standalone (no reference importable): plain package classes
    env = dict(os.environ, PYTHONPATH=ROOT, LIGHTBEAM_B200_STANDALONE="1")
    code = ("import paper_2603_14002_b200 as P\n"
            "assert P.errors.REFERENCE_ERRORS is None\n"
            "assert P.EmptyBeamError.__mro__[2] is Exception\n"
            "assert P.DecodeResult.__module__ == 'paper_2603_14002_b200.decoder'\nprint('ok')\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr[-2000:]
