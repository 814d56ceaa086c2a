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


@pytest.mark.gpu
def test_bench_two_ranks_gpu_gather_matches_single_rank():
    """`bench.py --gpus 2` without a launcher spawns two ranks itself (on a one-GPU box they
    share cuda:0 over gloo); both ranks' utterances are decoded on the device, gathered
    host-side, and the gathered (text, score) list equals one single-process decode of the same
    16 utterances (rank r decodes seeds 1000 + 8r ...)."""
    import json
    import subprocess
    import sys

    from paper_2603_14002_b200 import PROFILES, DeviceNgramScorer, decode_batch_raw, synth

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run(
        [sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--trials", "8",
         "--frames", "120", "--words", "2000", "--ngrams", "5000,3000,2000", "--steps", "2",
         "--warmup", "3", "--no-llm", "--no-wer", "--no-cpu-baseline", "--no-e2e"],
        capture_output=True, text=True, timeout=900, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gather"]["ranks"] == 2
    assert line["gather"]["utterances"] == 16
    assert line["value"] > 0 and line["gpu_launches"] > 0

    sys.path.insert(0, root)
    import bench

    world = synth.make_world(n_words=2000, n2=5000, n3=3000, n4=2000, seed=12345)
    cfg = PROFILES["b2t25"].replace(beam_size=64)
    raws = synth.make_logits(16, 120, 41, base_seed=1000)
    scorer = DeviceNgramScorer(world.model, cfg.ngram_weight / cfg.llm_weight)
    res = decode_batch_raw((raws, np.full(16, 120, np.int32)), cfg, world.table, world.model,
                           scorer, final_llm_only=True)
    assert line["gather"]["digest"] == bench.results_digest([bench.result_key(r) for r in res])
