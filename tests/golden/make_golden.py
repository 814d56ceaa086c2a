"""Generate tests/golden/*.json.gz by running the UNMODIFIED reference in the build container.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

The reference tree does not exist on the GPU box, so its behaviour is frozen here as
fixtures: every instance stores its *inputs* (vocabulary, lexicon entries, ARPA text, stub
table, fp64 log-prob matrix, configs) and the reference's *outputs* (text, score, n-best,
llm_events or the exception message; per-frame beam traces for a subset).  Sources of the
instances are the reference's own test fixtures (`pkg/tests/conftest.py:43-191`,
`test_decoder.py`, `test_acceptance.py:93-130`, `test_ngram.py:22-43`) plus 41-token worlds
from `paper_2603_14002_b200.synth` (regenerated from seeds; the table digest is stored so a
drifting generator is caught).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
ROOT = Path(__file__).resolve().parents[2]
for p in (REF_SRC, REF_TESTS, str(ROOT)):
    if p not in sys.path:
        sys.path.insert(0, p)

import lightbeam as ref  # noqa: E402  (reference, read-only)
from conftest import TRIGRAM_SPEC, one_hot_logits, random_instance, scaled, sentence_bigram_spec  # noqa: E402
from lightbeam.decoder import apply_llm, init_beams, step  # noqa: E402
from test_acceptance import _fixture_20_words  # noqa: E402
from test_ngram import HAND_CASES  # noqa: E402

from paper_2603_14002_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def cfg_dict(cfg) -> dict:
    return {k: getattr(cfg, k) for k in (
        "acoustic_scale", "beam_size", "ortho_beams", "beam_prune_threshold",
        "homophone_prune_threshold", "token_insertion_bonus", "word_boundary_bonus",
        "ngram_weight", "llm_weight", "llm_rescore_interval", "llm_chunk_size")}


def run(d, cfg, tt, model, scorer, final_only=False):
    try:
        r = ref.decode(d, cfg, tt, ref.LmSession(model), scorer, final_llm_only=final_only)
    except ref.LightBeamError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}
    return {"text": r.text, "score": r.score, "nbest": [list(p) for p in r.nbest],
            "llm_events": r.llm_events, "frame_count": r.frame_count}


def trace(d, cfg, tt, model, scorer, final_only=False):
    """Per-frame ordered beams (h1, h2, prefix, last, score) after each step / fusion event."""
    lm = ref.LmSession(model)
    beams = init_beams(cfg, tt, lm.registry)
    out = []
    try:
        for t in range(d.num_frames):
            step(beams, d.frames[t], t, cfg, tt, lm)
            out.append(snap(beams))
            if t > 0 and t % cfg.llm_rescore_interval == 0 and not final_only:
                apply_llm(beams, scorer, cfg, final=False)
                out.append(snap(beams))
    except ref.EmptyBeamError:
        pass
    return out


def snap(beams):
    return [[str(int(beams.hash1[i])), str(int(beams.hash2[i])), int(beams.prefix_states[i]),
             int(beams.last_tokens[i]), float(beams.scores[i])] for i in range(beams.size)]


def lexicon_rows(entries):
    return [[e.key, e.surface, list(e.phonemes)] for e in entries]


def table_digest(tt) -> str:
    return hashlib.sha256(np.ascontiguousarray(tt.table, dtype="<i4").tobytes()).hexdigest()


def small_config(**kw):
    base = dict(beam_size=64, llm_rescore_interval=100, homophone_prune_threshold=4.0, ortho_beams=3)
    base.update(kw)
    return ref.PROFILES["b2t24"].replace(**base)


def random_sets():
    """conftest.random_instance instances (the reference's own generator)."""
    exhaustive = ref.PROFILES["b2t24"].replace(beam_size=256, beam_prune_threshold=1e9,
                                               homophone_prune_threshold=1e9, ortho_beams=4,
                                               llm_rescore_interval=2)
    cfgs_unsafe = [small_config(beam_size=8, llm_rescore_interval=3),
                   small_config(beam_size=2, llm_rescore_interval=1, beam_prune_threshold=3.0),
                   small_config(beam_size=16, llm_rescore_interval=2, beam_prune_threshold=1e9,
                                homophone_prune_threshold=1e9, ortho_beams=4)]
    items = []
    for seed in range(200):
        items.append(("safe", seed, True, 6, [exhaustive], True))
    for seed in range(150):
        items.append(("unsafe", seed, False, 8, cfgs_unsafe, seed < 40))
    out = []
    for tag, seed, safe, tmax, cfgs, with_trace in items:
        d, tt, model, scorer = random_instance(seed, exhaustive_safe=safe, t_max=tmax)
        inst = {
            "name": f"{tag}-{seed}",
            "vocab": {"tokens": ["<blank>", "AE", "N", "T", "<sp>"], "blank": 0, "space": 4},
            "lexicon": lexicon_rows(tt.entries),
            "probs": [[list(k), v] for k, v in model.probs.items()],
            "backoffs": [[list(k), v] for k, v in model.backoffs.items()],
            "order": model.order,
            "unk": model.unk_present,
            "stub_table": scorer.table,
            "D": d.frames.tolist(),
            "table_digest": table_digest(tt),
            "runs": [],
        }
        for cfg in cfgs:
            entry = {"config": cfg_dict(cfg), "final_only": False,
                     "result": run(d, cfg, tt, model, ref.StubScorer(table=dict(scorer.table)))}
            if with_trace:
                entry["trace"] = trace(d, cfg, tt, model, ref.StubScorer(table=dict(scorer.table)))
            inst["runs"].append(entry)
            # n-gram fixed-point stub, final pass only (the "no LLM fusion" mode of config 2)
            stub = ref.StubScorer(ngram_model=model, scale=cfg.ngram_weight / cfg.llm_weight)
            inst["runs"].append({"config": cfg_dict(cfg), "final_only": True, "ngram_stub": True,
                                 "result": run(d, cfg, tt, model, stub, final_only=True)})
            stub = ref.StubScorer(ngram_model=model, scale=cfg.ngram_weight / cfg.llm_weight)
            inst["runs"].append({"config": cfg_dict(cfg), "final_only": False, "ngram_stub": True,
                                 "result": run(d, cfg, tt, model, stub)})
        if tag == "safe":
            try:
                text, score = ref.exhaustive_decode(d, exhaustive, tt, ref.LmSession(model),
                                                    ref.StubScorer(table=dict(scorer.table)))
                inst["exhaustive"] = {"text": text, "score": score}
            except ref.EmptyBeamError as exc:
                inst["exhaustive"] = {"error": "EmptyBeamError", "message": str(exc)}
        out.append(inst)
    return out


def forced20():
    vocab, lexicon, table, model = _fixture_20_words()
    cfg = ref.PROFILES["b2t24"].replace(beam_size=32, llm_rescore_interval=7)
    insts = []
    for entry in lexicon.entries:
        d = scaled(one_hot_logits([*entry.phonemes, vocab.space_id], 41), cfg.acoustic_scale)
        insts.append({"D": d.frames.tolist(), "word": entry.surface,
                      "result": run(d, cfg, table, model, ref.StubScorer(table={}))})
    return {
        "vocab": {"tokens": list(vocab.tokens), "blank": vocab.blank_id, "space": vocab.space_id},
        "lexicon": lexicon_rows(lexicon.entries),
        "arpa": None,
        "probs": [[list(k), v] for k, v in model.probs.items()],
        "backoffs": [[list(k), v] for k, v in model.backoffs.items()],
        "order": model.order,
        "unk": model.unk_present,
        "table_digest": table_digest(table),
        "config": cfg_dict(cfg),
        "instances": insts,
    }


def hand_ngram():
    path = Path(tempfile.mkdtemp()) / "tri.arpa"
    text = ref.build_toy_arpa(TRIGRAM_SPEC)
    path.write_text(text)
    model = ref.load_arpa(path)
    session = ref.LmSession(model)
    cases = []
    for history, word, log10 in HAND_CASES:
        state = session.registry.state_of(history)
        score, succ = ref.score_word(model, session.registry, session.cache, state, word)
        cases.append({"history": list(history), "word": word, "log10": log10, "score": score,
                      "succ": list(session.registry.history(succ))})
    return {"arpa": text, "cases": cases}


def ant_fixtures():
    """test_decoder.py fixtures: ant/aunt lexicons, one-hot paths, uniform ties, OOV kill."""
    vocab = ref.Vocabulary(tokens=("<blank>", "AE", "N", "T", "<sp>"), blank_id=0, space_id=4)
    AE, N, T_, SP, BL = 1, 2, 3, 4, 0
    ant_only = [(("<s>",), -99.0, -0.1), (("</s>",), -0.8), (("ant",), -0.5, -0.2),
                (("<unk>",), -2.0), (("<s>", "ant"), -0.2)]
    homo = [(("<s>",), -99.0, -0.1), (("</s>",), -0.8), (("ant",), -0.9, -0.2),
            (("aunt",), -0.3, -0.2), (("<unk>",), -2.0), (("<s>", "ant"), -0.5),
            (("<s>", "aunt"), -0.1)]
    no_unk = [(("<s>",), -99.0, -0.1), (("</s>",), -0.8), (("b",), -0.5)]
    lex_ant = [("ant", "ant", (AE, N, T_))]
    lex_homo = [("ant", "ant", (AE, N, T_)), ("aunt", "aunt", (AE, N, T_))]
    lex_four = [("ant", "ant", (AE, N, T_)), ("aunt", "aunt", (AE, N, T_)), ("at", "at", (AE, T_)),
                ("an", "an", (AE, N))]
    paths = [[AE], [AE, AE], [AE, BL, AE], [AE, N, T_, SP], [AE, N, T_], [AE, N],
             [AE, N, T_, SP, SP], [AE, T_, SP, AE, N, SP], [BL, AE, N, T_, SP, BL, AE, T_]]
    cases = []
    for lname, lex in (("ant", lex_ant), ("homo", lex_homo), ("four", lex_four)):
        for sname, spec in (("ant_only", ant_only), ("homo", homo), ("no_unk", no_unk)):
            for pi, path in enumerate(paths):
                for cfg in (small_config(beam_size=16), small_config(beam_size=1),
                            small_config(beam_size=64, beam_prune_threshold=1e9),
                            small_config(beam_size=4, beam_prune_threshold=3.0,
                                         llm_rescore_interval=2),
                            small_config(beam_size=1, token_insertion_bonus=0.0,
                                         word_boundary_bonus=0.0, ngram_weight=0.0,
                                         llm_weight=0.0, beam_prune_threshold=1e9)):
                    cases.append((lname, lex, sname, spec, pi, path, cfg))
    stub_tables = [{}, {"ant": -0.5, "aunt": -7.0}, {"aunt?": -0.2, "aunt.": -3.0, "aunt!": -3.0,
                                                      "ant?": -9.0, "ant.": -9.5, "ant!": -9.5}]
    out = []
    for lname, lex, sname, spec, pi, path, cfg in cases:
        lexicon = ref.Lexicon(entries=tuple(ref.LexiconEntry(k, s, p) for k, s, p in lex))
        tt = ref.build_transition_table(lexicon, vocab)
        arpa = ref.build_toy_arpa(spec)
        fpath = Path(tempfile.mkdtemp()) / "m.arpa"
        fpath.write_text(arpa)
        model = ref.load_arpa(fpath)
        d = scaled(one_hot_logits(path, 5), cfg.acoustic_scale)
        for si, st in enumerate(stub_tables):
            out.append({"lexicon": [[k, s, list(p)] for k, s, p in lex], "arpa": arpa,
                        "path": path, "config": cfg_dict(cfg), "stub_table": st,
                        "D": d.frames.tolist(), "name": f"{lname}/{sname}/{pi}/{si}",
                        "result": run(d, cfg, tt, model, ref.StubScorer(table=dict(st)))})
    # uniform zero logits (test_decode_uniform_ties_deterministic) and random small logits
    lexicon = ref.Lexicon(entries=tuple(ref.LexiconEntry(k, s, p) for k, s, p in lex_four))
    tt = ref.build_transition_table(lexicon, vocab)
    arpa = ref.build_toy_arpa(ant_only)
    fpath = Path(tempfile.mkdtemp()) / "m.arpa"
    fpath.write_text(arpa)
    model = ref.load_arpa(fpath)
    for k in (1, 2, 3, 8, 64):
        for zero in (True, False):
            cfg = small_config(beam_size=k, token_insertion_bonus=0.0, word_boundary_bonus=0.0,
                               beam_prune_threshold=1e9, llm_rescore_interval=3)
            frames = np.zeros((6, 5), dtype=np.float32) if zero else \
                np.random.default_rng(k).normal(scale=0.5, size=(31, 5)).astype(np.float32)
            d = scaled(ref.RawLogits(frames=frames, frame_duration_ms=100.0), cfg.acoustic_scale)
            out.append({"lexicon": [[k_, s, list(p)] for k_, s, p in lex_four], "arpa": arpa,
                        "path": None, "config": cfg_dict(cfg), "stub_table": {},
                        "D": d.frames.tolist(), "name": f"uniform-{k}-{zero}",
                        "result": run(d, cfg, tt, model, ref.StubScorer(table={}))})
    return out


def worlds41():
    """41-token synthetic worlds (config-1/2 shape at small size) from our synth generator."""
    out = []
    specs = [
        ("toy2k", dict(n_words=2000, seed=7), [
            (dict(beam_size=10, llm_rescore_interval=20), "table", False),
            (dict(beam_size=64, llm_rescore_interval=15), "ngram", True),
            (dict(beam_size=16, llm_rescore_interval=10), "ngram", False),
            (dict(beam_size=64, llm_rescore_interval=7, ortho_beams=4), "table", False),
        ]),
    ]
    for wname, wkw, runs in specs:
        w = synth.toy_world(**wkw)
        lex = ref.Lexicon(entries=tuple(ref.LexiconEntry(e.key, e.surface, e.phonemes)
                                        for e in w.lexicon.entries))
        vocab = ref.Vocabulary(tokens=w.vocab.tokens, blank_id=0, space_id=40)
        tt = ref.build_transition_table(lex, vocab)
        spec = synth.make_ngram_spec([e.surface for e in w.lexicon.entries], 5 * 2000 // 2,
                                     3 * 2000 // 2, 2000, seed=wkw["seed"] + 1)
        fpath = Path(tempfile.mkdtemp()) / "w.arpa"
        fpath.write_text(synth.arpa_text_from_spec(spec))
        model = ref.load_arpa(fpath)
        rng = np.random.default_rng(99)
        surfaces = sorted({e.surface for e in w.lexicon.entries})
        stub = {}
        for _ in range(3000):
            a, b = rng.integers(0, len(surfaces), size=2)
            stub[f"{surfaces[a]} {surfaces[b]}"] = round(float(rng.uniform(-9, -1)), 4)
            stub[surfaces[a]] = round(float(rng.uniform(-5, -0.5)), 4)
        raws = synth.make_logits(6, 200, 41, base_seed=500)
        for kw, sk, final_only in runs:
            cfg = ref.PROFILES["b2t25"].replace(**kw)
            res = []
            traces = []
            for i in range(len(raws)):
                d = ref.scale_log_softmax(ref.RawLogits(raws[i], 80.0), cfg.acoustic_scale)
                if sk == "table":
                    sc = ref.StubScorer(table=dict(stub))
                else:
                    sc = ref.StubScorer(ngram_model=model, scale=cfg.ngram_weight / cfg.llm_weight)
                res.append(run(d, cfg, tt, model, sc, final_only=final_only))
                if i < 2:
                    sc2 = ref.StubScorer(table=dict(stub)) if sk == "table" else \
                        ref.StubScorer(ngram_model=model, scale=cfg.ngram_weight / cfg.llm_weight)
                    traces.append(trace(d, cfg, tt, model, sc2, final_only=final_only))
            out.append({"world": wname, "world_kw": wkw, "config": cfg_dict(cfg), "scorer": sk,
                        "final_only": final_only, "logit_seed": 500, "n_trials": len(raws),
                        "frames": 200, "results": res, "traces": traces})
        out_meta = {"table_digest": table_digest(tt), "stub_table": stub,
                    "n_probs": len(model.probs)}
    return {"runs": out, "meta": out_meta}


def prologue():
    rng = np.random.default_rng(3)
    raws = [rng.normal(scale=s, size=(64, v)).astype(np.float32) for s, v in ((2.0, 41), (5.0, 5),
                                                                              (30.0, 41), (1.0, 7))]
    return [{"x": r.tolist(), "alpha": a,
             "d": ref.scale_log_softmax(ref.RawLogits(r, 10.0), a).frames.tolist()}
            for r, a in zip(raws, (0.4, 0.6, 1.0, 0.25))]


def dump(name, obj):
    with gzip.open(OUT / f"{name}.json.gz", "wt", encoding="utf-8") as fh:
        json.dump(obj, fh)
    print(name, (OUT / f"{name}.json.gz").stat().st_size, "bytes")


if __name__ == "__main__":
    dump("hand_ngram", hand_ngram())
    dump("prologue", prologue())
    dump("forced20", forced20())
    dump("ant_fixtures", ant_fixtures())
    dump("random_instances", random_sets())
    dump("worlds41", worlds41())
