"""N>1 host logic on CPU: world_size-2 gloo processes shard utterances, decode their shard with
the CPU oracle standing in for the device (the GPU path is covered by -m gpu tests), gather
results host-side, and agree on max-over-ranks timing."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_14002_b200.shard import gather_results, max_over_ranks, shard_trials


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_trials_partition_and_balance():
    rng = np.random.default_rng(0)
    lengths = rng.integers(200, 2001, size=1000)
    for world in (1, 2, 4, 8):
        parts = [shard_trials(lengths, world, r) for r in range(world)]
        allidx = np.concatenate(parts)
        assert np.array_equal(np.sort(allidx), np.arange(1000))
        sums = [lengths[p].sum() for p in parts]
        assert max(sums) - min(sums) <= lengths.max()


def _decode_one(O, w, cfg, raw, StubScorer):
    d = O.log_softmax_scaled(raw, cfg.acoustic_scale)
    try:
        r = O.decode(d, cfg, w.table, w.model, StubScorer(table={}))
    except O.OracleEmptyBeam as exc:
        return ("error", str(exc))
    return (r.text, r.score)


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import lightbeam_oracle as O
        from paper_2603_14002_b200 import PROFILES, StubScorer, synth

        w = synth.toy_world(n_words=300, seed=5)
        cfg = PROFILES["b2t25"].replace(beam_size=8, llm_rescore_interval=7)
        lengths = np.array([40, 25, 60, 33, 50, 47, 20, 38])
        raws = synth.make_logits(len(lengths), int(lengths.max()), 41, base_seed=9)
        mine = shard_trials(lengths, world, rank)
        res = []
        for i in mine:
            res.append(_decode_one(O, w, cfg, raws[i, : lengths[i]], StubScorer))
        merged = gather_results(res, mine, world)
        slowest = max_over_ranks(1.0 + rank)
        out_q.put((rank, merged, slowest))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_shard_decode_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = []
    for _ in range(2):
        try:
            got.append(q.get(timeout=180))
        except Exception:
            codes = [p.exitcode for p in procs]
            for p in procs:
                p.kill()
            raise AssertionError(f"worker failed, exit codes {codes}")
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, s0), (r1, m1, s1) = sorted(got)
    assert m0 == m1 and len(m0) == 8
    assert s0 == s1 == 2.0
    # single-process reference of the same 8 utterances
    from oracle import lightbeam_oracle as O
    from paper_2603_14002_b200 import PROFILES, StubScorer, synth

    w = synth.toy_world(n_words=300, seed=5)
    cfg = PROFILES["b2t25"].replace(beam_size=8, llm_rescore_interval=7)
    lengths = np.array([40, 25, 60, 33, 50, 47, 20, 38])
    raws = synth.make_logits(8, int(lengths.max()), 41, base_seed=9)
    for i in range(8):
        assert m0[i] == _decode_one(O, w, cfg, raws[i, : lengths[i]], StubScorer)
    assert sum(1 for r in m0 if r[0] != "error") >= 1
