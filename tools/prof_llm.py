"""Kernel-time breakdown of one BASELINE-config-3 step (torch.profiler / CUPTI) -- GPU aid."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2603_14002_b200 import LlamaScorer
    from paper_2603_14002_b200.decoder import device_model, run_search

    args = bench.parse()
    world, cfg, raws = bench.make_inputs(args, 0)
    cfg = cfg.replace(llm_rescore_interval=args.interval)
    import os
    sc = LlamaScorer(args.llm, seed=0, precision=args.precision,
                     lm_chunk=int(os.environ.get("LM_CHUNK", "2048")),
                     lm_head=os.environ.get("LM_HEAD", "fused"),
                     fused_swiglu=os.environ.get("FUSED_SWIGLU", "0") == "1")
    dm = device_model(world.table, world.model, 0)
    B, T = raws.shape[:2]
    frames = np.full(B, T, np.int32)
    x = torch.from_numpy(raws).cuda()
    batch = dm.batch(cfg, B, T)

    def step():
        batch.load_logits(None, frames, on_device_ptr=x.data_ptr())
        run_search(batch, cfg, sc, world.model, final_llm_only=False)

    step()
    torch.cuda.synchronize()
    sess = batch._llm_session
    print("waves per event:", sess.waves_log[:6], "stats", sess.stats())
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        step()
        torch.cuda.synchronize()
    ka = prof.key_averages()
    rows = sorted([k for k in ka if k.device_time_total > 0], key=lambda k: -k.device_time_total)
    tot = sum(k.device_time_total for k in rows if k.device_type.name == "CUDA") or 1
    print(f"{'kernel':70s} {'calls':>6s} {'ms':>9s} {'%':>6s}")
    for k in rows[:30]:
        if k.device_type.name != "CUDA":
            continue
        print(f"{k.key[:70]:70s} {k.count:6d} {k.device_time_total / 1e3:9.2f} "
              f"{100 * k.device_time_total / tot:6.1f}")
    print("total device ms", tot / 1e3)


if __name__ == "__main__":
    main()
