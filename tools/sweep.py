"""BASELINE config 4: B2T'24-shaped sweep on one B200 -- T = 200..2000 frames, beam 16/64/256,
fusion interval 10/20/40 -- device-timed frames/s and RTF per point, with a parity spot check
(one utterance per point against the oracle decoder; with the LLM, replaying the device scores).

    python tools/sweep.py [--llm llama-3.2-1b|none] [--trials 64] [--out profiles/sweep.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from oracle import lightbeam_oracle as O
    from paper_2603_14002_b200 import (PROFILES, DeviceNgramScorer, LlamaScorer, ReplayScorer,
                                       StubScorer, synth)
    from paper_2603_14002_b200.decoder import device_model, run_search
    from paper_2603_14002_b200.errors import DeviceError

    ap = argparse.ArgumentParser()
    ap.add_argument("--llm", default="llama-3.2-1b")
    ap.add_argument("--precision", default="bf16x2")
    ap.add_argument("--trials", type=int, default=64)
    ap.add_argument("--frames", default="200,500,1000,2000")
    ap.add_argument("--beams", default="16,64,256")
    ap.add_argument("--intervals", default="10,20,40")
    ap.add_argument("--words", type=int, default=100_000)
    ap.add_argument("--check", type=int, default=1, help="utterances checked against the oracle")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    world = synth.make_world(n_words=args.words, n2=500_000, n3=250_000, n4=150_000, seed=12345)
    dm = device_model(world.table, world.model, 0)
    llm = None if args.llm == "none" else LlamaScorer(args.llm, seed=0, precision=args.precision)
    results = []
    for T in [int(x) for x in args.frames.split(",")]:
        raws = synth.make_logits(args.trials, T, 41, base_seed=4000 + T)
        x = torch.from_numpy(raws).cuda()
        frames = np.full(args.trials, T, np.int32)
        for k in [int(x) for x in args.beams.split(",")]:
            for r in [int(x) for x in args.intervals.split(",")]:
                cfg = PROFILES["b2t24"].replace(beam_size=k, llm_rescore_interval=r)
                scale = cfg.ngram_weight / cfg.llm_weight
                scorer = llm if llm is not None else DeviceNgramScorer(world.model, scale)
                batch = dm.batch(cfg, args.trials, T)
                final_only = False

                def step():
                    batch.load_logits(None, frames, on_device_ptr=x.data_ptr())
                    run_search(batch, cfg, scorer, world.model, final_llm_only=final_only)

                try:
                    step()
                    torch.cuda.synchronize()
                    batch.mark_begin()
                    step()
                    ms, launches = batch.mark_end()
                except DeviceError as e:  # e.g. the LLM prefix cache is full: record, go on
                    point = {"T": T, "beam": k, "interval": r, "trials": args.trials, "error": str(e)}
                    print(json.dumps(point), flush=True)
                    results.append(point)
                    dm = device_model(world.table, world.model, 0)
                    continue
                point = {"T": T, "beam": k, "interval": r, "trials": args.trials,
                         "ms": ms, "frames_per_s": args.trials * T / (ms / 1e3),
                         "rtf": (ms / 1e3) / (args.trials * T * 0.08), "launches": launches}
                if llm is not None:
                    point["llm"] = batch._llm_session.stats()
                ok = 0
                t0 = time.perf_counter()
                res = batch.results()
                for i in range(args.check):
                    d = O.log_softmax_scaled(raws[i], cfg.acoustic_scale)
                    ref_scorer = (ReplayScorer(batch._llm_session.replay_table()) if llm is not None
                                  else StubScorer(ngram_model=world.model, scale=scale))
                    want = O.decode(d, cfg, world.table, world.model, ref_scorer)
                    ok += int(res[i] is not None and res[i][0] == want.text and res[i][1] == want.score)
                point["parity"] = f"{ok}/{args.check}"
                point["check_s"] = time.perf_counter() - t0
                sess = getattr(batch, "_llm_session", None)
                if sess is not None:  # free this point's prefix cache before the next point sizes its own
                    sess.destroy()
                    batch._llm_session = None
                    torch.cuda.empty_cache()
                print(json.dumps(point), flush=True)
                results.append(point)
    if args.out:
        Path(args.out).write_text(json.dumps({"config": "BASELINE config 4 sweep (b2t24 profile)",
                                              "llm": args.llm, "precision": args.precision,
                                              "points": results}, indent=1))


if __name__ == "__main__":
    main()
