"""GPU parity: the CUDA decoder (through the C ABI) against the oracle and the reference's
golden fixtures.  Bar: bit-exact texts, fp64 scores, n-best lists, event counts, per-frame
ordered beams (hash lanes, prefix ids, last token, score) and error messages."""

import os
from pathlib import Path

import numpy as np
import pytest

import goldens as G
from oracle import lightbeam_oracle as O
from paper_2603_14002_b200 import (PROFILES, DeviceNgramScorer, StubScorer, decode, decode_batch,
                                   decode_batch_raw, synth)
from paper_2603_14002_b200.decoder import device_model

pytestmark = pytest.mark.gpu


def test_prologue_kernel_vs_numpy():
    from paper_2603_14002_b200 import _native

    for case in G.load("prologue"):
        x = np.asarray(case["x"], dtype=np.float32)
        got = _native.log_softmax_host(x, case["alpha"])
        want = np.asarray(case["d"])
        # numpy's SIMD exp is not libm-exact: allow a few ulps (north star: "within a few ulps")
        np.testing.assert_allclose(got, want, rtol=8 * np.finfo(np.float64).eps, atol=1e-15)


def test_prologue_row_kernel_equals_warp_kernel(tmp_path):
    """K1's row-per-thread form (default) and the warp-per-row form (LB_LSM_ROWS=0, run in a
    child process: the switch is read once per process) give bit-identical rows and row maxima,
    for every width 1..64, ragged row counts and a padded output pitch."""
    import subprocess
    import sys

    from paper_2603_14002_b200 import _native

    rng = np.random.default_rng(5)
    cases = [(rng.normal(0, 3, size=(int(n), v)).astype(np.float32), 0.7 + v / 100)
             for v, n in zip(range(1, 65), rng.integers(1, 300, size=64))]
    np.savez(tmp_path / "in.npz", *[c[0] for c in cases])
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r)\n"
        "from paper_2603_14002_b200 import _native\n"
        "z = np.load(%r); out = {}\n"
        "for i in range(64):\n"
        "    x = z['arr_%%d' %% i]; out['o%%d' %% i] = _native.log_softmax_host(x, 0.7 + x.shape[1] / 100)\n"
        "np.savez(%r, **out)\n" % (str(Path(__file__).resolve().parents[1]),
                                     str(tmp_path / "in.npz"), str(tmp_path / "warp.npz")))
    env = dict(os.environ, LB_LSM_ROWS="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=300)
    warp = np.load(tmp_path / "warp.npz")
    for i, (x, alpha) in enumerate(cases):
        got = _native.log_softmax_host(x, alpha)
        assert got.tobytes() == warp["o%d" % i].tobytes(), (i, x.shape)
    # the padded batch layout (slot V = row max) through a device batch is covered by the
    # raw-logit full-size tests (tests/test_full_size.py)


def test_device_score_word_hand_cases():
    g = G.load("hand_ngram")
    model = G.model_of({"arpa": g["arpa"]})
    vocab = G.vocab_of(G.TINY_VOCAB)
    tt = G.build_transition_table(G.lexicon_of([["a", "a", [1]], ["b", "b", [2]]]), vocab)
    dm = device_model(tt, model)
    wid = dm.ngram_image.word_id
    hist, words = [], []
    for case in g["cases"]:
        hist.append([wid[w] for w in case["history"]])
        w = case["word"]
        words.append(wid[w] if (w,) in model.probs else dm.ngram_image.unk_id)
    inc, succ = dm.score_words(hist, words)
    for i, case in enumerate(g["cases"]):
        assert inc[i] == case["score"], case
        assert list(succ[i]) == [wid[w] for w in case["succ"]], case


def test_forced20_gpu():
    g = G.load("forced20")
    vocab, tt, model = G.instance_world(g)
    cfg = G.config_of(g["config"])
    ds = [np.asarray(inst["D"]) for inst in g["instances"]]
    got = decode_batch(ds, cfg, tt, model, StubScorer(table={}))
    for inst, r in zip(g["instances"], got):
        assert G.same_result(r, inst["result"]) is None, inst["word"]


def test_ant_fixtures_gpu():
    for inst in G.load("ant_fixtures"):
        vocab, tt, model = G.instance_world(inst)
        cfg = G.config_of(inst["config"])
        r = decode_batch([G.d_of(inst)], cfg, tt, model, StubScorer(table=dict(inst["stub_table"])))[0]
        err = G.same_result(r, inst["result"])
        assert err is None, (inst["name"], err)


@pytest.mark.parametrize("part", range(2))
def test_random_instances_gpu(part):
    insts = G.load("random_instances")
    for inst in insts[part::2]:
        vocab, tt, model = G.instance_world(inst)
        for run in inst["runs"]:
            cfg = G.config_of(run["config"])
            sc = G.scorer_for(run, inst, model, cfg)
            r = decode_batch([G.d_of(inst)], cfg, tt, model, sc, final_llm_only=run["final_only"])[0]
            err = G.same_result(r, run["result"])
            assert err is None, (inst["name"], run["config"], err)


def test_random_instances_device_ngram_scorer():
    """DeviceNgramScorer on the GPU == the reference's StubScorer(ngram_model) (goldens)."""
    for inst in G.load("random_instances")[::3]:
        vocab, tt, model = G.instance_world(inst)
        for run in inst["runs"]:
            if not run.get("ngram_stub"):
                continue
            cfg = G.config_of(run["config"])
            sc = DeviceNgramScorer(model, cfg.ngram_weight / cfg.llm_weight)
            r = decode_batch([G.d_of(inst)], cfg, tt, model, sc, final_llm_only=run["final_only"])[0]
            err = G.same_result(r, run["result"])
            assert err is None, (inst["name"], run["config"], err)


def test_trace_parity_random():
    """Per-frame ordered beams equal the reference trace (hashes, prefix ids, last, score),
    with host-scored interval fusion events in between."""
    from paper_2603_14002_b200.decoder import run_search

    checked = 0
    for inst in G.load("random_instances"):
        vocab, tt, model = G.instance_world(inst)
        d = G.d_of(inst)
        for run in inst["runs"]:
            if "trace" not in run:
                continue
            cfg = G.config_of(run["config"])
            want = G.trace_rows(run["trace"])
            # golden interleaves: snapshot after each step, plus one after each event
            steps = []
            pos = 0
            for t in range(d.shape[0]):
                if pos >= len(want):
                    break
                steps.append(want[pos])
                pos += 1
                if t > 0 and t % cfg.llm_rescore_interval == 0:
                    pos += 1
            dm = device_model(tt, model)
            batch = dm.batch(cfg, 1, d.shape[0])
            batch.enable_dump(True)
            batch.load_logprobs(d[None], np.array([d.shape[0]], dtype=np.int32))
            run_search(batch, cfg, StubScorer(table=dict(inst["stub_table"])), model, False)
            for t, snap in enumerate(steps):
                assert batch.dump_frame(0, t) == snap, (inst["name"], t)
            batch.enable_dump(False)
            checked += 1
    assert checked >= 30


def _world_runs():
    g = G.load("worlds41")
    w = synth.toy_world(**g["runs"][0]["world_kw"])
    return g, w


def test_worlds41_gpu_vs_golden_and_oracle():
    g, w = _world_runs()
    stub = g["meta"]["stub_table"]
    for run in g["runs"]:
        cfg = G.config_of(run["config"])
        raws = synth.make_logits(run["n_trials"], run["frames"], 41, base_seed=run["logit_seed"])
        ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
        if run["scorer"] == "table":
            gpu_sc, ref_sc = StubScorer(table=dict(stub)), lambda: StubScorer(table=dict(stub))
        else:
            scale = cfg.ngram_weight / cfg.llm_weight
            gpu_sc = DeviceNgramScorer(w.model, scale)
            ref_sc = lambda: StubScorer(ngram_model=w.model, scale=scale)  # noqa: E731
        got = decode_batch(ds, cfg, w.table, w.model, gpu_sc, final_llm_only=run["final_only"])
        for i, d in enumerate(ds):
            want = O.decode(d, cfg, w.table, w.model, ref_sc(), final_llm_only=run["final_only"])
            assert G.same_result(got[i], {"text": want.text, "score": want.score,
                                          "nbest": want.nbest, "llm_events": want.llm_events}) is None
            # the golden came from the reference on this container's numpy D; texts must agree
            if "text" in run["results"][i]:
                assert got[i].text == run["results"][i]["text"]


def test_per_frame_trace_world41():
    """Frame-by-frame beam lists of the kernel == oracle (no fusion events: r > T)."""
    g, w = _world_runs()
    for k in (10, 64):
        cfg = PROFILES["b2t25"].replace(beam_size=k, llm_rescore_interval=1000)
        raws = synth.make_logits(3, 150, 41, base_seed=77)
        ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
        dm = device_model(w.table, w.model)
        batch = dm.batch(cfg, 3, 150)
        batch.enable_dump(True)
        arr = np.stack(ds)
        batch.load_logprobs(arr, np.full(3, 150, dtype=np.int32))
        batch.reset()
        batch.run(0, 150)
        for i, d in enumerate(ds):
            s = O.OracleSearch(cfg, w.table, w.model, StubScorer(table={}))
            for t in range(150):
                s.frame(d[t], t)
                assert batch.dump_frame(i, t) == s.snapshot(), (k, i, t)
        batch.enable_dump(False)


def test_config2_shape_small_world():
    """BASELINE config-2 semantics (k=64, final-only fixed-point n-gram stub) on 24 trials."""
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=64)
    raws = synth.make_logits(24, 300, 41, base_seed=1000)
    ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
    scale = cfg.ngram_weight / cfg.llm_weight
    got = decode_batch(ds, cfg, w.table, w.model, DeviceNgramScorer(w.model, scale), final_llm_only=True)
    for i, d in enumerate(ds):
        want = O.decode(d, cfg, w.table, w.model, StubScorer(ngram_model=w.model, scale=scale),
                        final_llm_only=True)
        assert (got[i].text, got[i].score, got[i].nbest) == (want.text, want.score, want.nbest), i


def test_raw_logits_path_matches_oracle_texts():
    """Fused-prologue path (fp32 logits in): D differs from numpy by ulps only, so texts agree."""
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=16, llm_rescore_interval=10)
    raws = synth.make_logits(6, 200, 41, base_seed=31)
    scale = cfg.ngram_weight / cfg.llm_weight
    got = decode_batch_raw(list(raws), cfg, w.table, w.model, DeviceNgramScorer(w.model, scale))
    for i, r in enumerate(raws):
        want = O.decode(O.log_softmax_scaled(r, cfg.acoustic_scale), cfg, w.table, w.model,
                        StubScorer(ngram_model=w.model, scale=scale))
        assert got[i].text == want.text
        assert got[i].score == pytest.approx(want.score, rel=1e-9)


def test_single_decode_api_and_errors():
    from paper_2603_14002_b200 import DataValueError, EmptyBeamError, LogProbMatrix

    g = G.load("forced20")
    vocab, tt, model = G.instance_world(g)
    cfg = G.config_of(g["config"])
    d = LogProbMatrix(np.asarray(g["instances"][0]["D"]), cfg.acoustic_scale, 100.0)
    r = decode(d, cfg, tt, model, StubScorer(table={}))
    assert r.text.rstrip(".?!") == g["instances"][0]["word"]
    with pytest.raises(DataValueError):
        decode(np.zeros((0, 41)), cfg, tt, model, StubScorer(table={}))
    # an impossible path: all mass on a token the lexicon never allows first
    bad = np.full((3, 41), -1e3)
    bad[:, 40] = 0.0
    cfg1 = cfg.replace(beam_size=1)
    try:
        decode(bad, cfg1, tt, model, StubScorer(table={}))
    except EmptyBeamError:
        pass


def test_decode_stream_raw_matches_batch_api():
    """The two-stream pipelined API returns exactly decode_batch_raw's results, batch by batch
    (ragged sizes, device n-gram scorer and a host stub scorer)."""
    from paper_2603_14002_b200 import decode_stream_raw
    from paper_2603_14002_b200._native import pinned_empty

    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=16, llm_rescore_interval=20)
    scale = cfg.ngram_weight / cfg.llm_weight
    batches = []
    for i, (n, T) in enumerate([(5, 90), (3, 140), (6, 60), (2, 110)]):
        x = pinned_empty((n, T, 41), np.float32)
        x[...] = synth.make_logits(n, T, 41, base_seed=900 + 10 * i)
        batches.append((x, np.full(n, T, np.int32)))
    for sc in (DeviceNgramScorer(w.model, scale), StubScorer(table={})):
        want = [decode_batch_raw(b, cfg, w.table, w.model, sc) for b in batches]
        got = list(decode_stream_raw(iter(batches), cfg, w.table, w.model, sc))
        assert len(got) == len(want)
        for gb, wb in zip(got, want):
            assert [(r.text, r.score, r.nbest) for r in gb] == [(r.text, r.score, r.nbest) for r in wb]


def test_selection_fallback_on_flat_frames():
    """Flat / tied log-prob rows pile hundreds of candidates into one histogram bin, so the
    kernels take the exact radix-select fallback; beams must still equal the oracle frame by
    frame (ties resolved by flat index as in the reference's stable sort)."""
    g, w = _world_runs()
    rng = np.random.default_rng(5)
    T = 40
    ds = [np.full((T, 41), -np.log(41.0)),
          -np.log(41.0) + 0.25 * rng.integers(0, 2, size=(T, 41)).astype(np.float64)]
    for k in (64, 200):
        cfg = PROFILES["b2t25"].replace(beam_size=k, llm_rescore_interval=1000)
        dm = device_model(w.table, w.model)
        batch = dm.batch(cfg, len(ds), T)
        batch.enable_dump(True)
        batch.clear_stats()
        batch.load_logprobs(np.stack(ds), np.full(len(ds), T, dtype=np.int32))
        batch.reset()
        batch.run(0, T)
        assert batch.stats()["fallback_selects"] > 0, k
        for i, d in enumerate(ds):
            s = O.OracleSearch(cfg, w.table, w.model, StubScorer(table={}))
            for t in range(T):
                s.frame(d[t], t)
                assert batch.dump_frame(i, t) == s.snapshot(), (k, i, t)
        batch.enable_dump(False)


def test_wide_beam_general_kernel_device_ngram():
    """Beam 200 runs the general frames kernel (speculated + warp-path n-gram pairs, binary-search
    recombination ranking): transcripts, scores and n-best lists equal the oracle."""
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=200)
    raws = synth.make_logits(6, 160, 41, base_seed=2024)
    ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
    scale = cfg.ngram_weight / cfg.llm_weight
    got = decode_batch(ds, cfg, w.table, w.model, DeviceNgramScorer(w.model, scale), final_llm_only=True)
    for i, d in enumerate(ds):
        want = O.decode(d, cfg, w.table, w.model, StubScorer(ngram_model=w.model, scale=scale),
                        final_llm_only=True)
        assert (got[i].text, got[i].score, got[i].nbest) == (want.text, want.score, want.nbest), i


def test_concurrent_host_threads():
    """Two host threads decoding through the same components at once (each gets its own batch
    handles and streams; the library's host worker pool is shared) return the single-thread
    results."""
    import threading

    from paper_2603_14002_b200 import decode_stream_raw

    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=64)
    scale = cfg.ngram_weight / cfg.llm_weight
    sc = DeviceNgramScorer(w.model, scale)
    inputs = [synth.make_logits(12, 120, 41, base_seed=500 + i) for i in range(2)]
    want = [[(r.text, r.score, r.nbest) for r in decode_batch_raw(list(x), cfg, w.table, w.model, sc)]
            for x in inputs]
    got: dict = {}

    def work(i):
        outs = []
        for _ in range(3):
            outs.append([(r.text, r.score, r.nbest)
                         for r in decode_batch_raw(list(inputs[i]), cfg, w.table, w.model, sc)])
        frames = np.full(12, 120, dtype=np.int32)
        for res in decode_stream_raw([(inputs[i], frames)] * 2, cfg, w.table, w.model, sc):
            outs.append([(r.text, r.score, r.nbest) for r in res])
        got[i] = outs

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(2):
        assert len(got[i]) == 5
        for o in got[i]:
            assert o == want[i]


def test_profile_default_beam_900():
    """The b2t25 profile's own beam (900 -> the 960-thread frames kernel): per-frame beams for
    one utterance and final results with device n-gram fusion equal the oracle."""
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"]
    assert cfg.beam_size == 900
    raws = synth.make_logits(3, 90, 41, base_seed=77)
    ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
    scale = cfg.ngram_weight / cfg.llm_weight
    got = decode_batch(ds, cfg, w.table, w.model, DeviceNgramScorer(w.model, scale), final_llm_only=True)
    for i, d in enumerate(ds):
        want = O.decode(d, cfg, w.table, w.model, StubScorer(ngram_model=w.model, scale=scale),
                        final_llm_only=True)
        assert (got[i].text, got[i].score, got[i].nbest) == (want.text, want.score, want.nbest), i
    cfg_t = cfg.replace(llm_rescore_interval=1000)
    dm = device_model(w.table, w.model)
    batch = dm.batch(cfg_t, 1, 60)
    batch.enable_dump(True)
    batch.load_logprobs(ds[0][None, :60], np.array([60], dtype=np.int32))
    batch.reset()
    batch.run(0, 60)
    s = O.OracleSearch(cfg_t, w.table, w.model, StubScorer(table={}))
    for t in range(60):
        s.frame(ds[0][t], t)
        assert batch.dump_frame(0, t) == s.snapshot(), t
    batch.enable_dump(False)


def test_max_beam_4096():
    """beam_size at the C-ABI maximum (4096): every working-set region but the log-prob stage
    lives in global scratch; results equal the oracle."""
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=4096)
    raws = synth.make_logits(2, 30, 41, base_seed=91)
    ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
    got = decode_batch(ds, cfg, w.table, w.model, StubScorer(table={}))
    for i, d in enumerate(ds):
        want = O.decode(d, cfg, w.table, w.model, StubScorer(table={}))
        assert (got[i].text, got[i].score, got[i].nbest) == (want.text, want.score, want.nbest), i


def _wide_vocab_world(seed=3):
    """64-token vocabulary (the kernel maximum; wider than the small-kernel path's 48)."""
    from paper_2603_14002_b200.ngram import parse_arpa_text

    rng = np.random.default_rng(seed)
    toks = ["<blank>"] + [f"P{i}" for i in range(62)] + ["<sp>"]
    vocab = G.vocab_of({"tokens": toks, "blank": 0, "space": 63})
    rows, words = [], []
    for i in range(300):
        n = int(rng.integers(2, 6))
        ph = [int(rng.integers(1, 63)) for _ in range(n)]
        surf = f"w{i}" if i % 17 else f"w{i - 1}"  # a few homophones
        rows.append([f"k{i}", surf, ph])
        words.append(surf)
    uni = sorted(set(words))
    lines = ["\\data\\", f"ngram 1={len(uni) + 3}", "ngram 2=200", "", "\\1-grams:"]
    for w in ["<s>", "</s>", "<unk>"] + uni:
        lines.append(f"{-rng.uniform(1, 4):.4f}\t{w}\t{-rng.uniform(0, 1):.4f}")
    lines += ["", "\\2-grams:"]
    for _ in range(200):
        a, b = rng.choice(uni, 2)
        lines.append(f"{-rng.uniform(0.2, 2):.4f}\t{a} {b}")
    lines += ["", "\\end\\", ""]
    model = parse_arpa_text("\n".join(lines))
    tt = G.build_transition_table(G.lexicon_of(rows), vocab)
    return tt, model


def test_vocab_64_general_kernel():
    """V = 64 runs the general kernel for every beam; host (interval) and device n-gram fusion
    both equal the oracle."""
    tt, model = _wide_vocab_world()
    raws = synth.make_logits(4, 80, 64, base_seed=640)
    for k in (16, 64):
        cfg = PROFILES["b2t25"].replace(beam_size=k, llm_rescore_interval=10)
        scale = cfg.ngram_weight / cfg.llm_weight
        ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
        for sc in (StubScorer(ngram_model=model, scale=scale), DeviceNgramScorer(model, scale)):
            got = decode_batch(ds, cfg, tt, model, sc)
            for i, d in enumerate(ds):
                want = O.decode(d, cfg, tt, model, StubScorer(ngram_model=model, scale=scale))
                assert (got[i].text, got[i].score, got[i].nbest) == \
                    (want.text, want.score, want.nbest), (k, type(sc).__name__, i)


@pytest.mark.parametrize("k,o,r", [(1, 1, 1), (5, 8, 3), (64, 1, 7), (64, 8, 5), (300, 2, 11)])
def test_ortho_interval_edges(k, o, r):
    """Ortho beams 1 and 8 (both kernels), fusion every frame, ragged lengths down to one frame,
    host n-gram stub fusion: results equal the oracle."""
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=k, ortho_beams=o, llm_rescore_interval=r)
    scale = cfg.ngram_weight / cfg.llm_weight
    lens = [1, 2, 37, 64]
    raws = synth.make_logits(len(lens), max(lens), 41, base_seed=300 + k + o)
    ds = [O.log_softmax_scaled(x[:n], cfg.acoustic_scale) for x, n in zip(raws, lens)]
    got = decode_batch(ds, cfg, w.table, w.model, StubScorer(ngram_model=w.model, scale=scale))
    for i, d in enumerate(ds):
        try:
            want = O.decode(d, cfg, w.table, w.model, StubScorer(ngram_model=w.model, scale=scale))
        except Exception as e:  # the reference raises (e.g. EmptyBeamError): so must we
            assert isinstance(got[i], Exception), (i, e, got[i])
            assert str(got[i]) == str(e) or type(got[i]).__name__ == type(e).__name__, (got[i], e)
            continue
        assert not isinstance(got[i], Exception), (i, got[i])
        assert (got[i].text, got[i].score, got[i].nbest, got[i].llm_events) == \
            (want.text, want.score, want.nbest, want.llm_events), (k, o, r, i)


def test_run_search_many_interleaves_host_fusion_batches():
    """Two device batches on two streams advanced event by event (host scorer: every event is a
    device->host->device round trip) give the results of decoding each batch alone."""
    from paper_2603_14002_b200.decoder import _collect, device_model, run_search_many

    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=16, llm_rescore_interval=9)
    scale = cfg.ngram_weight / cfg.llm_weight
    raws = [synth.make_logits(3, 70, 41, base_seed=900 + i) for i in range(2)]
    want = [[(r.text, r.score, r.nbest) for r in
             decode_batch_raw(list(x), cfg, w.table, w.model, StubScorer(ngram_model=w.model, scale=scale))]
            for x in raws]
    dm = device_model(w.table, w.model)
    batches = [dm.pipeline_batch(cfg, i, 3, 70) for i in range(2)]
    for b, x in zip(batches, raws):
        b.load_logits(x, np.full(3, 70, np.int32))
    run_search_many(batches, cfg, StubScorer(ngram_model=w.model, scale=scale), w.model, False)
    for b, wv in zip(batches, want):
        got = [(r.text, r.score, r.nbest) for r in _collect(b, cfg, False, 0.0)]
        assert got == wv


def test_relabelled_table_general_successor_path():
    """A transition table whose states are not breadth-first numbered (ids shuffled) takes the
    compact image's general successor-list path (LexRec.base into lex_next) instead of the
    first-child + rank arithmetic; results equal the oracle's on the same relabelled table."""
    from paper_2603_14002_b200.lexicon import TransitionTable

    w = synth.toy_world(n_words=1500, seed=11)
    tt = w.table
    S = tt.num_states
    rng = np.random.default_rng(5)
    perm = np.arange(S)
    perm[1:S - 1] = 1 + rng.permutation(S - 2)  # root 0 and sink S-1 keep their ids
    table = np.empty_like(tt.table)
    table[perm] = perm[tt.table]
    comps = {int(perm[s]): tt.completions_at(s) for s in tt.completion_states()}
    rt = TransitionTable(table, tt.sink, comps, tt.entries, tt.blank_id, tt.space_id)
    cfg = PROFILES["b2t25"].replace(beam_size=64)
    raws = synth.make_logits(12, 200, 41, base_seed=606)
    ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
    scale = cfg.ngram_weight / cfg.llm_weight
    for table_ in (rt, tt):
        got = decode_batch(ds, cfg, table_, w.model, DeviceNgramScorer(w.model, scale))
        for i, d in enumerate(ds):
            want = O.decode(d, cfg, table_, w.model, StubScorer(ngram_model=w.model, scale=scale))
            assert (got[i].text, got[i].score, got[i].nbest, got[i].llm_events) == (
                want.text, want.score, want.nbest, want.llm_events), i
    assert device_model(rt, w.model).lex_contiguous is False
    assert device_model(tt, w.model).lex_contiguous is True
