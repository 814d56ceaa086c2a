"""Parity at the BASELINE sizes (SURVEY.md §8c protocol, §8d workloads), on the GPU.

The world is the bench's own: 100k-word lexicon (+10% homophones, 234,882 prefix states),
~1M-n-gram 4-gram LM (997,140 entries in the cuckoo image), 256 utterances x T=500 x 41
classes, beam 64, b2t25 profile (bench.py `make_inputs`, rank 0).  The CPU side is the
*unmodified reference* `lightbeam.decoder.decode` (`decoder.py:408-460`, installed under
baseline/_ref, see oracle/refbridge.py) in a fork pool over the host cores, or the oracle
restatement when the reference is not installed.  Both sides search the same fp64 log-prob
matrices (the reference's own prologue, `logits.py:119-130`, fed through the D-input path).

Bar (north star): texts, fp64 scores, n-best lists and event counts bit-exact; per-frame
ordered beams bit-exact; LLM fusion scores within 1e-2 of an fp32 model of the same weights.
"""

import multiprocessing as mp
import os

import numpy as np
import pytest

from oracle import lightbeam_oracle as O
from oracle import refbridge
from paper_2603_14002_b200 import PROFILES, DeviceNgramScorer, StubScorer, decode_batch, synth

pytestmark = pytest.mark.gpu

B, T, K = 256, 500, 64
TOL = 1e-2


@pytest.fixture(scope="module")
def full():
    world = synth.make_world(n_words=100_000, n2=500_000, n3=250_000, n4=150_000, seed=12345)
    cfg = PROFILES["b2t25"].replace(beam_size=K)
    raws = synth.make_logits(B, T, 41, base_seed=1000)
    rw = refbridge.RefWorld(world) if refbridge.reference() is not None else None
    if (refbridge.ROOT / "baseline" / "_ref" / "lightbeam").exists():
        assert rw is not None, "baseline/_ref holds the reference but it did not load"
    if rw is not None:
        ds = np.stack([rw.scale_log_softmax(r, cfg) for r in raws])
    else:
        ds = np.stack([O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws])
    return world, cfg, raws, ds, rw


# ------------------------------------------------------------------ CPU side (fork pool)
_POOL = {}


def _cpu_decode(i):
    world, cfg, ds, rw, mk, final_only = (_POOL[k] for k in
                                          ("world", "cfg", "ds", "rw", "mk", "final_only"))
    scorer = mk()
    if rw is not None:
        r = rw.decode(ds[i], cfg, scorer, final_llm_only=final_only)
    else:
        try:
            r = O.decode(ds[i], cfg, world.table, world.model, scorer, final_llm_only=final_only)
        except O.OracleEmptyBeam as exc:
            return ("error", str(exc))
    if isinstance(r, Exception):
        return ("error", str(r))
    return (r.text, r.score, list(map(tuple, r.nbest)), r.llm_events, r.frame_count)


def cpu_results(world, cfg, ds, rw, make_scorer, idx, final_only):
    _POOL.update(world=world, cfg=cfg, ds=ds, rw=rw, mk=make_scorer, final_only=final_only)
    with mp.get_context("fork").Pool(min(len(idx), os.cpu_count() or 1)) as pool:
        return pool.map(_cpu_decode, list(idx), chunksize=1)


def gpu_key(r):
    if isinstance(r, Exception):
        return ("error", str(r))
    return (r.text, r.score, list(map(tuple, r.nbest)), r.llm_events, r.frame_count)


def _compare(got, want, idx):
    bad = [i for i, g, w in zip(idx, got, want) if g != w]
    assert not bad, (f"{len(bad)}/{len(idx)} utterances differ; first {bad[0]}: "
                     f"gpu {got[idx.index(bad[0])][:2]} cpu {want[idx.index(bad[0])][:2]}")


# ------------------------------------------------------------------ config 2
@pytest.mark.parametrize("scorer_kind", ["device_ngram", "host_stub"])
def test_config2_full_batch_bit_exact(full, scorer_kind):
    """All 256 utterances of the headline workload: (text, score, n-best, events, frames)
    bit-exact against the reference decoder with StubScorer(ngram_model, omega/phi) and
    final-only fusion (BASELINE config 2)."""
    world, cfg, raws, ds, rw = full
    scale = cfg.ngram_weight / cfg.llm_weight
    sc = (DeviceNgramScorer(world.model, scale) if scorer_kind == "device_ngram"
          else StubScorer(ngram_model=world.model, scale=scale))
    got = decode_batch((ds, np.full(B, T, np.int32)), cfg, world.table, world.model, sc,
                       final_llm_only=True)
    if rw is not None:
        mk = lambda: rw.stub(scale)  # noqa: E731
    else:
        mk = lambda: StubScorer(ngram_model=world.model, scale=scale)  # noqa: E731
    idx = list(range(B))
    want = cpu_results(world, cfg, ds, rw, mk, idx, True)
    _compare([gpu_key(g) for g in got], want, idx)
    assert sum(1 for w in want if w[0] != "error") >= B - 2
    assert sum(len(w[2]) for w in want if w[0] != "error") > B  # n-best lists are non-trivial


def _ref_trace(rw, cfg, d):
    """Per-frame ordered beams of the unmodified reference (`init_beams` + `step`,
    decoder.py:177-326)."""
    lb = rw.lb
    rc = rw.config(cfg)
    lm = rw.session()
    beams = lb.decoder.init_beams(rc, rw.table, lm.registry)
    out = []
    for t in range(d.shape[0]):
        lb.decoder.step(beams, d[t], t, rc, rw.table, lm)
        out.append([(int(beams.hash1[i]), int(beams.hash2[i]), int(beams.prefix_states[i]),
                     int(beams.last_tokens[i]), float(beams.scores[i])) for i in range(beams.size)])
    return out


def test_config2_full_per_frame_traces(full):
    """Frame-by-frame ordered beams (hash lanes, prefix ids, last token, fp64 score) of two
    full-size utterances equal the reference's BeamSet after every step."""
    from paper_2603_14002_b200.decoder import device_model

    world, cfg, raws, ds, rw = full
    cfg_nf = cfg.replace(llm_rescore_interval=10_000)  # no interval events: frames only
    dm = device_model(world.table, world.model)
    batch = dm.batch(cfg_nf, 2, T)
    batch.enable_dump(True)
    batch.load_logprobs(ds[:2], np.full(2, T, np.int32))
    batch.reset()
    batch.run(0, T)
    try:
        for i in range(2):
            if rw is not None:
                want = _ref_trace(rw, cfg_nf, ds[i])
            else:
                s = O.OracleSearch(cfg_nf, world.table, world.model, StubScorer(table={}))
                want = []
                for t in range(T):
                    s.frame(ds[i][t], t)
                    want.append(s.snapshot())
            for t in range(T):
                assert batch.dump_frame(i, t) == want[t], (i, t)
    finally:
        batch.enable_dump(False)


def test_config2_raw_logit_path_full_batch(full):
    """The fused-prologue path (K1 on the device) over all 256 utterances: texts equal the
    reference's (the device prologue agrees with numpy's SIMD exp only to a few ulps, so
    scores are compared at 1e-9 relative, not bit for bit)."""
    from paper_2603_14002_b200 import decode_batch_raw

    world, cfg, raws, ds, rw = full
    scale = cfg.ngram_weight / cfg.llm_weight
    got = decode_batch_raw((raws, np.full(B, T, np.int32)), cfg, world.table, world.model,
                           DeviceNgramScorer(world.model, scale), final_llm_only=True)
    want = decode_batch((ds, np.full(B, T, np.int32)), cfg, world.table, world.model,
                        DeviceNgramScorer(world.model, scale), final_llm_only=True)
    same_text = sum(g.text == w.text for g, w in zip(got, want))
    assert same_text >= B - 2, same_text
    for g, w in zip(got, want):
        if g.text == w.text:
            assert abs(g.score - w.score) <= 1e-9 * abs(w.score)


# ------------------------------------------------------------------ configs 3 and 5 (LLM)
def session_texts(sess):
    """(text, device cum score) of every scored slot of a session's prefix trie."""
    ex = sess.export()
    first = {int(t): s for s, t in zip(sess.batch.dm.surfaces, sess._cap)}
    mid = {int(t): s for s, t in zip(sess.batch.dm.surfaces, sess._low)}
    out = []
    for s in range(1, len(ex["parent"])):
        if ex["parent"][s] < 0 or not ex["state"][s] & 2:
            continue
        words, cur = [], s
        while cur != 0:
            words.append(int(ex["token"][cur]))
            cur = int(ex["parent"][cur])
        words.reverse()
        out.append((" ".join([first[words[0]]] + [mid[t] for t in words[1:]]), float(ex["cum"][s]),
                    int(ex["depth"][s])))
    return out


def _llm_run(full, preset, n_trials):
    from paper_2603_14002_b200 import LlamaScorer, ReplayScorer
    from paper_2603_14002_b200.decoder import device_model

    world, cfg, raws, ds, rw = full
    cfg3 = cfg.replace(llm_rescore_interval=20)
    sc = LlamaScorer(preset, seed=0, precision="bf16x2")
    got = decode_batch((ds[:n_trials], np.full(n_trials, T, np.int32)), cfg3, world.table,
                       world.model, sc)
    sess = device_model(world.table, world.model).batch(cfg3, n_trials, T)._llm_session
    replay = ReplayScorer(sess.replay_table())
    texts = session_texts(sess)
    return sc, cfg3, got, replay, texts


def _replay_parity(full, cfg3, got, replay, n_check):
    world, cfg, raws, ds, rw = full
    idx = list(np.linspace(0, len(got) - 1, n_check).astype(int))
    want = cpu_results(world, cfg3, ds, rw, lambda: replay, idx, False)
    _compare([gpu_key(got[i]) for i in idx], want, idx)
    assert all(w[3] == (T - 1) // 20 for w in want if w[0] != "error")


def _numerics(sc, texts, n, device):
    """Device bf16x2 fusion scores vs transformers fp32 with the same weights (1e-2 abs): the
    `n` deepest scored texts plus an even spread over the rest."""
    import torch

    from oracle import llm_oracle as LO

    texts = sorted(texts, key=lambda x: -x[2])
    pick = texts[: n // 2] + texts[n // 2:: max(1, (len(texts) - n // 2) // (n - n // 2))][: n - n // 2]
    oracle = LO.OracleLlmScorer(sc.cfg, sc.weights.hf_state_dict(device), device=device)
    errs = []
    with torch.no_grad():
        for text, cum, _ in pick:
            errs.append(abs(oracle.score(text) - cum))
    del oracle
    torch.cuda.empty_cache()
    assert len(pick) >= n * 0.9
    assert max(errs) <= TOL, (max(errs), pick[int(np.argmax(errs))][0])
    return max(errs)


def test_config3_llama_1b_replay_and_numerics(full):
    """BASELINE config 3 (256 utterances, Llama-3.2-1B architecture, r = 20, bf16x2): 32
    utterances bit-exact against the reference decoder replaying the device's per-text scores,
    and >= 200 device-scored texts (the deepest first) within 1e-2 of fp32."""
    import torch

    sc, cfg3, got, replay, texts = _llm_run(full, "llama-3.2-1b", B)
    _replay_parity(full, cfg3, got, replay, 32)
    assert len(texts) >= 200
    _numerics(sc, texts, 200, "cuda")
    from paper_2603_14002_b200.decoder import release_device_model

    release_device_model(full[0].table, full[0].model)
    del sc
    torch.cuda.empty_cache()


def test_config5_llama_8b_replay_and_numerics(full):
    """BASELINE config 5's per-GPU device batch (256 utterances, Llama-3.1-8B architecture,
    bf16x2): 32 utterances bit-exact under replay, and >= 20 deep texts within 1e-2 of the
    fp32 model at the real 8B shape (head_dim 128, GQA 4, 32 layers)."""
    import torch

    from paper_2603_14002_b200.decoder import release_device_model

    world = full[0]
    sc, cfg3, got, replay, texts = _llm_run(full, "llama-3.1-8b", B)
    _replay_parity(full, cfg3, got, replay, 32)
    release_device_model(world.table, world.model)  # drop the prefix cache before the fp32 model
    torch.cuda.empty_cache()
    _numerics(sc, texts, 24, "cuda")
    del sc
    torch.cuda.empty_cache()
