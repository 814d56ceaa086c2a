"""Pin the CPU oracle (oracle/lightbeam_oracle.py) to the reference's recorded behaviour.

Every fixture in tests/golden was produced by the unmodified reference (make_golden.py); the
oracle must reproduce texts, scores, n-best lists, event counts, error messages and per-frame
beam traces exactly.  Also pins our host builders (table numbering, ARPA parsing, stub
scorer) that both the oracle and the GPU path consume.
"""

import hashlib

import numpy as np
import pytest

import goldens as G
from oracle import lightbeam_oracle as O
from paper_2603_14002_b200 import synth
from paper_2603_14002_b200.ngram import LN10, LmSession, score_word


def oracle_run(d, cfg, tt, model, scorer, final_only):
    try:
        return O.decode(d, cfg, tt, model, scorer, final_llm_only=final_only)
    except (O.OracleEmptyBeam, O.OracleEmptyInput) as exc:
        return exc


def test_hand_ngram_cases():
    g = G.load("hand_ngram")
    model = G.model_of({"arpa": g["arpa"]})
    ng = O.NgramOracle(model)
    session = LmSession(model)
    for case in g["cases"]:
        h = tuple(case["history"])
        inc, succ = ng.increment(h, case["word"])
        assert inc == case["score"], case
        assert inc == pytest.approx(case["log10"] * LN10, abs=1e-9)
        assert list(succ) == case["succ"]
        # our host score_word (used by StubScorer n-gram mode) agrees too
        s2, st = score_word(model, session.registry, session.cache, session.registry.state_of(h),
                            case["word"])
        assert s2 == case["score"] and list(session.registry.history(st)) == case["succ"]


def test_prologue_matches_reference_numpy():
    for case in G.load("prologue"):
        x = np.asarray(case["x"], dtype=np.float32)
        got = O.log_softmax_scaled(x, case["alpha"])
        assert np.array_equal(got, np.asarray(case["d"]))


def test_forced20():
    g = G.load("forced20")
    vocab, tt, model = G.instance_world(g)
    assert hashlib.sha256(np.ascontiguousarray(tt.table, dtype="<i4").tobytes()).hexdigest() == g["table_digest"]
    cfg = G.config_of(g["config"])
    for inst in g["instances"]:
        got = oracle_run(np.asarray(inst["D"]), cfg, tt, model, G.StubScorer(table={}), False)
        assert G.same_result(got, inst["result"]) is None, inst["word"]


def test_ant_fixtures():
    for inst in G.load("ant_fixtures"):
        vocab, tt, model = G.instance_world(inst)
        cfg = G.config_of(inst["config"])
        got = oracle_run(G.d_of(inst), cfg, tt, model, G.StubScorer(table=dict(inst["stub_table"])), False)
        err = G.same_result(got, inst["result"])
        assert err is None, (inst["name"], err)


@pytest.mark.parametrize("part", range(4))
def test_random_instances(part):
    insts = G.load("random_instances")
    for inst in insts[part::4]:
        vocab, tt, model = G.instance_world(inst)
        digest = hashlib.sha256(np.ascontiguousarray(tt.table, dtype="<i4").tobytes()).hexdigest()
        assert digest == inst["table_digest"], inst["name"]
        for run in inst["runs"]:
            cfg = G.config_of(run["config"])
            sc = G.scorer_for(run, inst, model, cfg)
            got = oracle_run(G.d_of(inst), cfg, tt, model, sc, run["final_only"])
            err = G.same_result(got, run["result"])
            assert err is None, (inst["name"], run["config"], err)
            if "trace" in run:
                sc = G.scorer_for(run, inst, model, cfg)
                tr = _oracle_trace(G.d_of(inst), cfg, tt, model, sc)
                assert tr == G.trace_rows(run["trace"]), inst["name"]
        if "exhaustive" in inst and "text" in inst["exhaustive"]:
            # the reference's brute-force oracle agreed with its decoder; so must ours
            cfg = G.config_of(inst["runs"][0]["config"])
            got = oracle_run(G.d_of(inst), cfg, tt, model, G.StubScorer(table=dict(inst["stub_table"])), False)
            assert got.text == inst["exhaustive"]["text"]
            assert got.score == pytest.approx(inst["exhaustive"]["score"], abs=1e-6)


def _oracle_trace(d, cfg, tt, model, scorer):
    s = O.OracleSearch(cfg, tt, model, scorer)
    out = []
    try:
        for t in range(d.shape[0]):
            s.frame(d[t], t)
            out.append(s.snapshot())
            if t > 0 and t % cfg.llm_rescore_interval == 0:
                s.rescore(final=False)
                out.append(s.snapshot())
    except O.OracleEmptyBeam:
        pass
    return out


def test_worlds41():
    g = G.load("worlds41")
    w = synth.toy_world(**g["runs"][0]["world_kw"])
    digest = hashlib.sha256(np.ascontiguousarray(w.table.table, dtype="<i4").tobytes()).hexdigest()
    assert digest == g["meta"]["table_digest"]
    assert len(w.model.probs) == g["meta"]["n_probs"]
    stub = g["meta"]["stub_table"]
    for run in g["runs"]:
        cfg = G.config_of(run["config"])
        raws = synth.make_logits(run["n_trials"], run["frames"], 41, base_seed=run["logit_seed"])
        for i, want in enumerate(run["results"]):
            d = O.log_softmax_scaled(raws[i], cfg.acoustic_scale)
            sc = (G.StubScorer(table=dict(stub)) if run["scorer"] == "table"
                  else G.StubScorer(ngram_model=w.model, scale=cfg.ngram_weight / cfg.llm_weight))
            got = oracle_run(d, cfg, w.table, w.model, sc, run["final_only"])
            assert G.same_result(got, want) is None, (run["config"], i)
            if i < len(run["traces"]):
                sc = (G.StubScorer(table=dict(stub)) if run["scorer"] == "table"
                      else G.StubScorer(ngram_model=w.model, scale=cfg.ngram_weight / cfg.llm_weight))
                s = O.OracleSearch(cfg, w.table, w.model, sc)
                tr = []
                try:
                    for t in range(d.shape[0]):
                        s.frame(d[t], t)
                        tr.append(s.snapshot())
                        if t > 0 and t % cfg.llm_rescore_interval == 0 and not run["final_only"]:
                            s.rescore(final=False)
                            tr.append(s.snapshot())
                except O.OracleEmptyBeam:
                    pass
                assert tr == G.trace_rows(run["traces"][i])
