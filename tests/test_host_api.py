"""CPU tests of the host-side mirror of the reference API and of the C-ABI library surface
(no compute calls: there is no GPU in the build container)."""

import gzip
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import goldens as G
from paper_2603_14002_b200 import (
    PROFILES,
    ConfigError,
    DecodeConfig,
    DeviceError,
    FormatError,
    LmSession,
    ScoreRequest,
    ScoreResponse,
    StubScorer,
    Vocabulary,
    build_transition_table,
    config_from_dict,
    decode,
    load_arpa,
    load_table,
    save_table,
    score_eos,
    score_sequence,
    score_texts,
    synth,
)
from paper_2603_14002_b200 import _native, images
from paper_2603_14002_b200.ngram import LN10, NEG_INF_GUARD, parse_arpa_text
from paper_2603_14002_b200.scorer import decode_request, decode_response, encode_request, encode_response

ROOT = Path(__file__).resolve().parents[1]


def test_table5_profiles():
    b24, b25 = PROFILES["b2t24"], PROFILES["b2t25"]
    assert (b24.acoustic_scale, b24.beam_size, b24.beam_prune_threshold, b24.ortho_beams,
            b24.homophone_prune_threshold, b24.token_insertion_bonus, b24.word_boundary_bonus,
            b24.ngram_weight, b24.llm_weight, b24.llm_rescore_interval, b24.llm_chunk_size) == (
        0.6, 1000, 22.0, 3, 4.0, 1.5, 1.0, 0.8, 1.2, 10, 256)
    assert (b25.acoustic_scale, b25.beam_size, b25.beam_prune_threshold, b25.ngram_weight,
            b25.llm_rescore_interval) == (0.4, 900, 18.0, 1.0, 15)


@pytest.mark.parametrize("bad", [
    dict(beam_size=0), dict(ortho_beams=0), dict(beam_prune_threshold=0.0),
    dict(homophone_prune_threshold=-1.0), dict(ngram_weight=-0.1), dict(llm_rescore_interval=0),
    dict(llm_chunk_size=0), dict(acoustic_scale=float("nan")), dict(acoustic_scale=0.0)])
def test_config_validation(bad):
    with pytest.raises(ConfigError):
        PROFILES["b2t25"].replace(**bad)


def test_config_from_dict():
    assert config_from_dict({"profile": "b2t24", "beam_size": 16}).beam_size == 16
    with pytest.raises(ConfigError):
        config_from_dict({"profile": "nope"})
    with pytest.raises(ConfigError):
        config_from_dict({"beam_size": 3})
    with pytest.raises(ConfigError):
        config_from_dict({"profile": "b2t24", "bogus": 1})


def test_lexicon_table_semantics():
    vocab = Vocabulary(("<blank>", "AE", "N", "T", "<sp>"), 0, 4)
    lex = G.lexicon_of([["ant", "ant", [1, 2, 3]], ["aunt", "aunt", [1, 2, 3]],
                        ["at", "at", [1, 3]], ["an", "an", [1, 2]]])
    tt = build_transition_table(lex, vocab)
    # BFS numbering: root 0; children of root in token order; sink last
    assert tt.advance(0, 1) == 1
    assert tt.table[tt.sink].tolist() == [tt.sink] * 5
    assert tt.completions_at(tt.advance(tt.advance(tt.advance(0, 1), 2), 3)) == (0, 1)
    s = tt.advance(tt.advance(0, 1), 2)
    assert tt.advance(s, 4) == 0  # "an" completes: space returns to the root
    assert tt.advance(1, 4) == tt.sink
    m = tt.valid_mask(np.array([0, 1]), np.array([0, 1]))
    assert m[0].tolist() == [True, True, False, False, False]
    assert m[1].tolist() == [True, True, True, True, False]


def test_lbtt_roundtrip(tmp_path):
    w = synth.toy_world(n_words=300, seed=3)
    p = tmp_path / "t.lbtt"
    save_table(p, w.table)
    back = load_table(p, w.vocab)
    assert np.array_equal(back.table, w.table.table)
    assert back.completion_states() == w.table.completion_states()
    assert [e.surface for e in back.entries] == [e.surface for e in w.table.entries]


def test_arpa_parse_and_errors(tmp_path):
    g = G.load("hand_ngram")
    p = tmp_path / "m.arpa"
    p.write_text(g["arpa"])
    m = load_arpa(p)
    assert m.order == 3 and m.unk_present
    assert m.probs[("a",)] == -0.47712 * LN10
    gz = tmp_path / "m.arpa.gz"
    gz.write_bytes(gzip.compress(g["arpa"].encode()))
    assert load_arpa(gz).probs == m.probs
    bad = {
        "no data": "\\1-grams:\n-1.0 a\n\\end\\\n",
        "count": "\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0 a\n\\end\\\n",
        "no end": "\\data\\\nngram 1=1\n\n\\1-grams:\n-1.0 a\n",
        "bad prob": "\\data\\\nngram 1=1\n\n\\1-grams:\nxx a\n\\end\\\n",
        "undeclared": "\\data\\\nngram 1=1\n\n\\2-grams:\n-1.0 a b\n\\end\\\n",
    }
    for name, text in bad.items():
        with pytest.raises(FormatError):
            parse_arpa_text(text)


def test_host_score_sequence_matches_hand():
    g = G.load("hand_ngram")
    m = parse_arpa_text(g["arpa"])
    total = score_sequence(m, ["a", "b", "a"], include_eos=True)
    s = LmSession(m)
    from paper_2603_14002_b200 import score_word

    st, acc = 0, 0.0
    for w in ["a", "b", "a", "</s>"]:
        inc, st = score_word(m, s.registry, s.cache, st, w)
        acc += inc
    assert total == acc


def test_scorer_protocol():
    req = ScoreRequest(7, "score", ("a b", "c"))
    assert decode_request(encode_request(req)) == req
    resp = ScoreResponse(7, (-1.5, -2.0))
    assert decode_response(encode_response(resp), expect_id=7) == resp
    stub = StubScorer(table={"a": -0.5, "c": -2.5})
    texts = ["a", "b b", "c", "a", "long text here"] * 3
    ref = score_texts(stub, texts, 256)
    for chunk in (1, 2, 7):
        assert score_texts(StubScorer(table={"a": -0.5, "c": -2.5}), texts, chunk) == ref
    assert score_eos(StubScorer(table={}), ["hello there"]) == [(".", -2.0)]
    assert score_eos(StubScorer(table={"x?": -1.0, "x.": -3.0}), ["x"]) == [("?", -1.0)]


def test_ngram_image_compile():
    m = parse_arpa_text(G.load("hand_ngram")["arpa"])
    img = images.compile_ngram(m)
    keys = set()
    for row in range(len(img.probs)):
        g = tuple(int(x) for x in img.words[row] if x != images.WORD_PAD)
        keys.add(g)
    names = {v: k for k, v in img.word_id.items()}
    assert {tuple(names[i] for i in g) for g in keys} == set(m.probs) | set(m.backoffs)
    assert img.eos_eff == img.word_id["</s>"]


def test_table_image_completion_csr():
    vocab = Vocabulary(("<blank>", "AE", "N", "T", "<sp>"), 0, 4)
    lex = G.lexicon_of([["ant", "ant", [1, 2, 3]], ["aunt", "aunt", [1, 2, 3]],
                        ["ant(2)", "ant", [1, 2, 3]], ["zz", "zz", [1]]])
    tt = build_transition_table(lex, vocab)
    m = parse_arpa_text("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0 ant\n-2.0 <unk>\n\\end\\\n")
    ng = images.compile_ngram(m)
    tab = images.compile_table(tt, m, ng)
    s = tt.advance(tt.advance(tt.advance(0, 1), 2), 3)
    lo, hi = tab.comp_off[s], tab.comp_off[s + 1]
    assert [tab.surfaces[i] for i in tab.comp_surface[lo:hi]] == ["ant", "aunt"]  # deduped
    assert tab.comp_lmword[lo:hi].tolist() == [ng.word_id["ant"], ng.word_id["<unk>"]]


def test_synth_determinism():
    a = synth.toy_world(n_words=500, seed=11)
    b = synth.toy_world(n_words=500, seed=11)
    assert np.array_equal(a.table.table, b.table.table)
    assert a.model.probs == b.model.probs
    assert np.array_equal(synth.make_logits(2, 10, base_seed=5), synth.make_logits(2, 10, base_seed=5))
    for e in a.lexicon.entries:  # no adjacent duplicate phonemes (unreachable in the search)
        assert all(x != y for x, y in zip(e.phonemes, e.phonemes[1:]))


def test_synth_arpa_text_equals_direct_model():
    lex = synth.make_lexicon(300, seed=4)
    spec = synth.make_ngram_spec([e.surface for e in lex.entries], 400, 200, 100, seed=5)
    direct = synth.ngram_model_from_spec(spec)
    parsed = parse_arpa_text(synth.arpa_text_from_spec(spec))
    assert direct.probs == parsed.probs and direct.backoffs == parsed.backoffs
    assert direct.order == parsed.order == 4


def _header_symbols():
    text = (ROOT / "include" / "lightbeam_b200.h").read_text()
    return sorted(set(re.findall(r"\b(lb_[a-z_0-9]+)\s*\(", text)))


def test_c_abi_exports_every_header_symbol():
    _native.build()
    syms = _header_symbols()
    assert len(syms) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(syms) == set(_native.exported_symbols())
    lib = _native.lib(require_device=False)
    for s in syms:
        assert getattr(lib, s) is not None


def test_sass_is_sm100a_with_tma_bulk():
    _native.build()
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    full = subprocess.run(["cuobjdump", "-sass", str(_native.LIB_PATH)], capture_output=True,
                          text=True).stdout
    funcs = {}
    cur = None
    for line in full.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    frames = [f for f in funcs if "frames_kernel" in f]
    assert len(frames) == 6  # {256,512,1024} threads x {all-shared, spilled} layouts
    sass = "\n".join(funcs[frames[0]])
    assert "UBLKCP" in sass  # cp.async.bulk (1-D TMA) staging of the log-prob frame chunks
    assert "LDGSTS" in sass  # cp.async lexicon-row gathers


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    w = synth.toy_world(n_words=100, seed=1)
    d = np.zeros((3, 41))
    with pytest.raises(DeviceError):
        decode(d, PROFILES["b2t25"].replace(beam_size=4), w.table, w.model, StubScorer(table={}))


def _engine_files(tmp_path):
    import json

    from paper_2603_14002_b200 import save_vocab, synth
    from paper_2603_14002_b200.synth import arpa_text_from_spec, make_ngram_spec

    w = synth.toy_world(n_words=200, seed=5)
    vp = tmp_path / "vocab.txt"
    save_vocab(vp, w.vocab)
    lp = tmp_path / "lexicon.txt"
    lp.write_text("".join(f"{e.key}\t{' '.join(w.vocab.tokens[p] for p in e.phonemes)}\n"
                          for e in w.lexicon.entries))
    spec = make_ngram_spec([e.surface for e in w.lexicon.entries], 400, 200, 100, seed=6)
    ap = tmp_path / "lm.arpa"
    ap.write_text(arpa_text_from_spec(spec))
    return vp, lp, ap


def test_build_engine_argument_rules(tmp_path):
    from paper_2603_14002_b200 import PROFILES, ConfigError, ScorerSpec, build_engine

    vp, lp, ap = _engine_files(tmp_path)
    with pytest.raises(ConfigError):
        build_engine(vp, ap, ScorerSpec("stub_table"), config=PROFILES["b2t25"])
    with pytest.raises(ConfigError):
        build_engine(vp, ap, ScorerSpec("stub_table"), lexicon_path=lp)
    with pytest.raises(ConfigError):
        ScorerSpec("subprocess").build(None)
    eng = build_engine(vp, ap, ScorerSpec("stub_ngram", scale=0.5), lexicon_path=lp,
                       config=PROFILES["b2t25"], config_overrides={"beam_size": 8})
    assert eng.config.beam_size == 8 and set(eng.components) == {"vocab", "lexicon", "arpa"}
    assert eng.table.num_states > 1


@pytest.mark.gpu
def test_engine_decode_paths_matches_oracle(tmp_path):
    import numpy as np

    from oracle import lightbeam_oracle as O
    from paper_2603_14002_b200 import PROFILES, RawLogits, ScorerSpec, build_engine, save_logits

    vp, lp, ap = _engine_files(tmp_path)
    eng = build_engine(vp, ap, ScorerSpec("stub_ngram", scale=0.5), lexicon_path=lp,
                       config=PROFILES["b2t25"].replace(beam_size=16))
    paths = []
    for i in range(4):
        x = np.random.default_rng(i).normal(scale=2.0, size=(60 + 10 * i, 41)).astype(np.float32)
        p = tmp_path / f"u{i}.lblt"
        save_logits(p, RawLogits(x, 80.0))
        paths.append(p)
    got = eng.decode_paths(paths)
    for p, g in zip(paths, got):
        res, sample = g
        raw = eng.decode_path(p)[0]
        assert (res.text, res.score, res.nbest) == (raw.text, raw.score, raw.nbest)
        assert sample.utterance_duration_s == res.frame_count * 80.0 / 1000.0
    from paper_2603_14002_b200 import load_logits

    d = O.log_softmax_scaled(load_logits(paths[0], eng.vocab).frames, eng.config.acoustic_scale)
    want = O.decode(d, eng.config, eng.table, eng.ngram_model, eng.scorer)
    r = eng.decode_matrix(d)
    assert (r.text, r.score, r.nbest) == (want.text, want.score, want.nbest)


def test_load_logits_batch_matches_single_loads(tmp_path):
    import numpy as np

    from paper_2603_14002_b200 import RawLogits, load_logits, save_logits, synth
    from paper_2603_14002_b200.logits import load_logits_batch

    vocab = synth.vocab41()
    paths = []
    for i, t in enumerate([5, 9, 3]):
        p = tmp_path / f"u{i}.lblt"
        save_logits(p, RawLogits(np.random.default_rng(i).normal(size=(t, 41)).astype(np.float32), 80.0))
        paths.append(p)
    bad = tmp_path / "bad.lblt"
    bad.write_bytes(b"LBLT" + b"\\x00" * 4)
    paths.insert(1, bad)
    arr, frames, ms, errors = load_logits_batch(paths, vocab, pinned=False)
    assert [i for i, _ in errors] == [1] and list(frames) == [5, 0, 9, 3]
    for i in (0, 2, 3):
        want = load_logits(paths[i], vocab).frames
        assert np.array_equal(arr[i, : frames[i]], want) and ms[i] == 80.0


def test_results_binding_builds_objects_from_a_view():
    """The CPython result binding (csrc/lb_pyresults.c) on a hand-made lb_results_view: texts by
    offset (utf-8, no separators needed), None for failed trials, n-best pairs in order."""
    import ctypes as C

    import numpy as np

    from paper_2603_14002_b200 import _native as N

    texts = ["héllo world", "héllo word.", "hello", "x y z?"]
    blob = b"".join(t.encode() for t in texts)
    offs = np.cumsum([0] + [len(t.encode()) for t in texts])[:-1].astype(np.int64)
    lens = np.array([len(t.encode()) for t in texts], dtype=np.int32)
    buf = C.create_string_buffer(blob, len(blob))
    status = np.array([0, 2, 0], dtype=np.int32)
    best_off = np.array([offs[0], 0, offs[3]], dtype=np.int64)
    best_len = np.array([lens[0], 0, lens[3]], dtype=np.int32)
    best_sc = np.array([-1.5, 0.0, -7.25])
    cnt = np.array([2, 0, 1], dtype=np.int32)
    nb_off = np.array([offs[1], offs[2], offs[3]], dtype=np.int64)
    nb_len = np.array([lens[1], lens[2], lens[3]], dtype=np.int32)
    nb_sc = np.array([-1.5, -2.0, -7.25])
    v = N.LbResultsView(3, 3, len(blob), C.addressof(buf), status.ctypes.data, best_off.ctypes.data,
                        best_len.ctypes.data, best_sc.ctypes.data, cnt.ctypes.data,
                        nb_off.ctypes.data, nb_len.ctypes.data, nb_sc.ctypes.data)
    got = N.pyresults().assemble(C.addressof(v))
    assert got == [("héllo world", -1.5, [("héllo word.", -1.5), ("hello", -2.0)]), None,
                   ("x y z?", -7.25, [("x y z?", -7.25)])]


def test_bench_algorithmic_bytes_counts_consumed_pairs_only():
    """bench.algorithmic_bytes: n-gram probe bytes scale with the pairs the
    word-boundary beams consume, not with the kernel's speculative pairs."""
    import bench

    base = dict(frames=100, beams_in=5000, ngram_probes=4000, ngram_calls=1000,
                ngram_pairs_used=500, history_nodes=300, boundary_beams=80)
    got = bench.algorithmic_bytes(base)
    want = 8 * 41 * 100 + 4 * 41 * 5000 + 32 * 4000 * 500 / 1000 + 20 * 300 + 8 * 80
    assert got == want
    # without speculation (every computed pair consumed) the probe term is the raw count
    full = dict(base, ngram_pairs_used=1000)
    assert bench.algorithmic_bytes(full) - got == 32 * 2000


def test_device_image_file_round_trip(tmp_path):
    """Persisted device images: save -> load reproduces every array and field
    bit for bit (absent-prob NaN payloads included)."""
    import dataclasses

    from paper_2603_14002_b200 import images

    w = synth.toy_world(n_words=1500, seed=3)
    ng = images.compile_ngram(w.model)
    tab = images.compile_table(w.table, w.model, ng)
    p = tmp_path / "img.npz"
    images.save_images(p, tab, ng, -0.25)
    t2, n2, bo = images.load_images(p)
    assert bo == -0.25
    for a, b in ((tab, t2), (ng, n2)):
        for f in dataclasses.fields(a):
            x, y = getattr(a, f.name), getattr(b, f.name)
            if isinstance(x, np.ndarray):
                assert x.dtype == y.dtype and x.tobytes() == y.tobytes(), f.name
            else:
                assert x == y, f.name


@pytest.mark.gpu
def test_engine_image_cache_reuses_images(tmp_path):
    """build_engine(image_cache=dir): the first engine compiles and writes the images, a second
    engine over the same files loads them, and both decode identically."""
    from paper_2603_14002_b200 import ScorerSpec, build_engine
    from paper_2603_14002_b200.decoder import device_model

    vp, lp, ap = _engine_files(tmp_path)
    raws = synth.make_logits(4, 80, 41, base_seed=31)
    outs, sources = [], []
    for _ in range(2):
        eng = build_engine(vp, ap, ScorerSpec(kind="device_ngram", scale=0.8), lexicon_path=lp,
                           config=PROFILES["b2t25"].replace(beam_size=16),
                           image_cache=tmp_path / "cache")
        res = eng.decode_batch_raw(list(raws))
        sources.append(device_model(eng.table, eng.ngram_model).image_source)
        outs.append([(r.text, r.score, r.nbest) for r in res])
        eng.close()
    assert sources == ["compiled", "loaded"]
    assert outs[0] == outs[1]
    assert len(list((tmp_path / "cache").glob("lb_images_*.npz"))) == 1
