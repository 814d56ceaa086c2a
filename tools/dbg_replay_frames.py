"""Diagnostic (GPU): decode a device batch with the device LLM scorer and bisect one utterance
frame by frame against the oracle search replaying this run's device LLM scores.

    python tools/dbg_replay_frames.py --trials 128 --offset 128 --utt 1 [--llm llama-3.2-1b]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    from oracle import lightbeam_oracle as O
    from paper_2603_14002_b200 import LlamaScorer, ReplayScorer
    from paper_2603_14002_b200.decoder import device_model, run_search

    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=128)
    ap.add_argument("--offset", type=int, default=128)
    ap.add_argument("--utt", type=int, default=1)
    ap.add_argument("--llm", default="llama-3.2-1b")
    ap.add_argument("--frames", type=int, default=500)
    a = ap.parse_args()
    sys.argv = [sys.argv[0], "--config", "3"]
    args = bench.parse()
    world, cfg, raws = bench.make_inputs(args, 0)
    cfg = cfg.replace(llm_rescore_interval=args.interval)
    raws = raws[a.offset:a.offset + a.trials, :a.frames]
    B, T = raws.shape[:2]
    sc = LlamaScorer(a.llm, seed=0, precision="bf16x2")
    dm = device_model(world.table, world.model, 0)
    batch = dm.batch(cfg, B, T)
    batch.enable_dump(True)
    x = torch.from_numpy(np.ascontiguousarray(raws)).cuda()
    batch.load_logits(None, np.full(B, T, np.int32), on_device_ptr=x.data_ptr())
    run_search(batch, cfg, sc, world.model, final_llm_only=False)
    res = batch.results()
    replay = ReplayScorer(batch._llm_session.replay_table())
    u = a.utt
    d = O.log_softmax_scaled(raws[u], cfg.acoustic_scale)
    want = O.decode(d, cfg, world.table, world.model, replay)
    print("device", res[u][1], "oracle", want.score, "same text", res[u][0] == want.text)
    s = O.OracleSearch(cfg, world.table, world.model, replay)
    r = cfg.llm_rescore_interval
    for t in range(T):
        s.frame(d[t], t)
        got = batch.dump_frame(u, t)  # written by the frame kernel, before any fusion event
        snap = s.snapshot()
        if got != snap:
            print("first mismatch at frame", t, "(event frames: multiples of", r, ")")
            diff = [(i, g, w) for i, (g, w) in enumerate(zip(got, snap)) if g != w]
            print("len device", len(got), "oracle", len(snap), "differing beams", len(diff))
            for i, g, w in diff[:5]:
                print(" beam", i, "device", g, "oracle", w)
            break
        if t > 0 and t % r == 0:
            s.rescore(final=False)
    else:
        print("all frames equal")
    # second device run (same composition), entry totals after each fusion event vs the oracle
    surf = batch.dm.surfaces
    batch.load_logits(None, np.full(B, T, np.int32), on_device_ptr=x.data_ptr())
    batch.reset()
    sess = sc.session(batch)
    sess.reset()
    s = O.OracleSearch(cfg, world.table, world.model, replay)
    t0 = 0
    for e in range(r, T, r):
        batch.run(t0, e + 1)
        for t in range(t0, e + 1):
            s.frame(d[t], t)
        sess.event(False, e)
        s.rescore(final=False)
        t0 = e + 1
        et, eb, wo, words, tot, pun = batch.gather()
        mine = [i for i in range(len(et)) if et[i] == u]
        dev = [(" ".join(surf[w] for w in words[wo[i]:wo[i + 1]]), float(tot[i])) for i in mine]
        ora = [(tx, tt_) for ents in s.entries_dump() for (tx, tt_, _, _) in ents]
        if dev != ora:
            print("entry totals differ after event", e)
            for a_, b_ in zip(dev, ora):
                if a_ != b_:
                    print(" device", a_[0][-60:], repr(a_[1]), "oracle", b_[0][-60:], repr(b_[1]))
                    tx = a_[0]
                    if tx:
                        sl = replay.table.slot_of(tx) if hasattr(replay, "table") else None
                        print("  slot", sl)
                    break
            break
    else:
        print("entry totals equal after every event")


if __name__ == "__main__":
    main()
