"""The reference sidecar's TinyCausalLM (pkg/sidecar/src/model.ts) as the LLM scorer (SURVEY.md
§8a a14): the oracle restatement (oracle/tiny_char_lm.py) against the properties the reference's
own tests check (pkg/sidecar/test/model.test.ts), the product's weights / tokenizer / float64
protocol path against the oracle, and on the GPU the device path (multi-token surfaces in the
prefix trie, hi/lo weights) within the north star's 1e-2 plus decode parity by score replay."""

import numpy as np
import pytest

from oracle import tiny_char_lm as TC

TOL = 1e-2


@pytest.fixture(scope="module")
def lm():
    return TC.TinyCharLM()


# ------------------------------------------------------------------ model.test.ts properties
def test_tokenizer_properties():
    assert TC.sentence_case("hello world") == "Hello world"
    assert TC.sentence_case("") == ""
    assert TC.tokenize("hello") == TC.tokenize("Hello")
    assert TC.tokenize("aé")[-1] == TC.VOCAB_SIZE - 2  # out of range -> UNK


def test_scoring_properties(lm):
    other = TC.TinyCharLM()
    assert other.score_text("hello world") == lm.score_text("hello world")  # deterministic
    assert TC.TinyCharLM("another-seed").score_text("hello world") != lm.score_text("hello world")
    s = lm.score_text("hello world")
    assert np.isfinite(s) and s < 0
    assert lm.score_text("") == 0
    for text in ["how are you", "fine", "the quick brown fox"]:
        assert lm.score_text(text + " zzqx") < lm.score_text(text)


def test_eos_properties(lm):
    p, s = lm.score_eos("how are you")
    assert p in (".", "?", "!")
    assert abs(s - lm.score_text("how are you" + p)) < 1e-10
    text = "see you later"
    assert lm.score_eos(text)[1] == max(lm.score_text(text + q) for q in ".?!")


# ------------------------------------------------------------------ product vs oracle (CPU)
def test_product_weights_and_tokenizer_match_oracle(lm):
    from paper_2603_14002_b200 import charlm

    w = charlm.tiny_char_weights()
    assert np.array_equal(w["embed"], lm.embed) and np.array_equal(w["pos"], lm.pos)
    for i, L in enumerate(lm.layers):
        for k in ("wq", "wk", "wv", "wo", "w1", "w2"):
            assert np.array_equal(w[f"{k}.{i}"], L[k]), (k, i)
    assert np.array_equal(w["wout"], lm.w_out)
    tok = charlm.CharTokenizer()
    for text in ["", "hello", "w12 w3", "aé b", "Zz ~"]:
        assert tok.encode(text) == TC.tokenize(text)
    low, low_off, cap, cap_off = tok.surface_tables(["ant", "bé"])
    assert list(low[low_off[0]:low_off[1]]) == TC.tokenize("x ant")[2:]
    assert list(cap[cap_off[1]:cap_off[2]]) == TC.tokenize("bé")[1:]


def test_product_float64_protocol_path_matches_oracle(lm):
    """charlm.dense_scores (the scorer protocol's submit() path) == the oracle to 1e-9."""
    pytest.importorskip("torch")
    from paper_2603_14002_b200 import charlm

    w = charlm.tiny_char_weights()
    texts = ["", "ant", "the quick brown fox", "w12 w3 w45"]
    for (s, plp), t in zip(charlm.dense_scores(w, texts, "cpu", eos=True), texts):
        assert abs(s - lm.score_text(t)) < 1e-9, t
        p, best = lm.score_eos(t)
        j = ".?!".index(p)
        assert abs(s + plp[j] - best) < 1e-9
        assert plp[j] == max(plp)


# ------------------------------------------------------------------ GPU
def _char_world(n_words=2000):
    from paper_2603_14002_b200 import PROFILES, synth

    w = synth.toy_world(n_words=n_words, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=10, llm_rescore_interval=20)
    return w, cfg


@pytest.mark.gpu
def test_device_tiny_char_lm_scores_and_replay_parity(lm):
    """BASELINE config 1 with the sidecar's own model: every device-scored text (one slot per
    character; word nodes and the prefixes inside words) within 1e-2 of the float64 oracle, and
    the oracle decoder replaying the device scores reproduces texts, scores, n-best and event
    counts bit for bit."""
    from oracle import lightbeam_oracle as O
    from paper_2603_14002_b200 import LlamaScorer, ReplayScorer, decode_batch, synth
    from paper_2603_14002_b200.decoder import device_model

    w, cfg = _char_world()
    sc = LlamaScorer("tiny-char-lm")
    raws = synth.make_logits(3, 500, 41, base_seed=2024)
    ds = [O.log_softmax_scaled(x, cfg.acoustic_scale) for x in raws]
    got = decode_batch(ds, cfg, w.table, w.model, sc)
    sess = device_model(w.table, w.model).batch(cfg, len(ds), 500)._llm_session
    replay = ReplayScorer(sess.replay_table())
    for i, d in enumerate(ds):
        want = O.decode(d, cfg, w.table, w.model, replay)
        g = got[i]
        assert (g.text, g.score, g.nbest, g.llm_events) == (want.text, want.score, want.nbest,
                                                            want.llm_events), i
    ex = sess.export()
    texts, devs = [], []
    for s in range(1, len(ex["parent"])):
        if ex["parent"][s] < 0 or not ex["state"][s] & 2:
            continue
        toks, cur = [], s
        while cur != 0:
            toks.append(int(ex["token"][cur]))
            cur = int(ex["parent"][cur])
        texts.append("".join(chr(t + 32) for t in reversed(toks)))
        devs.append(float(ex["cum"][s]))
    assert len(texts) >= 200
    rng = np.random.default_rng(0)
    pick = rng.choice(len(texts), size=min(300, len(texts)), replace=False)
    err = max(abs(lm.score_text(texts[i]) - devs[i]) for i in pick)
    assert err <= TOL, err
    # the protocol path (float64 dense forward) agrees with the oracle too
    some = [texts[i] for i in pick[:20]]
    for t, s in zip(some, sc.score_texts_dense(some)):
        assert abs(s - lm.score_text(t)) < 1e-9
