"""GPU idle gaps inside one BASELINE-config-3 step (torch.profiler trace): where the device
waits for the host.  Prints the total idle time and the largest gaps with their neighbours."""
import json
import os
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
    sc = LlamaScorer(args.llm, seed=0, precision=args.precision)
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
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        step()
        torch.cuda.synchronize()
    path = "/tmp/trace.json"
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    k = sorted([e for e in ev if e.get("cat") == "kernel" and "dur" in e], key=lambda e: e["ts"])
    span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
    busy = sum(e["dur"] for e in k)
    gaps = []
    end = k[0]["ts"] + k[0]["dur"]
    for a, b in zip(k, k[1:]):
        g = b["ts"] - max(end, a["ts"] + a["dur"])
        end = max(end, b["ts"] + b["dur"])
        if g > 0:
            gaps.append((g, a["name"][:40], b["name"][:40]))
    gaps.sort(reverse=True)
    tot = sum(g for g, _, _ in gaps)
    print(f"span {span/1e3:.1f} ms, kernel busy {busy/1e3:.1f} ms, idle {tot/1e3:.1f} ms in {len(gaps)} gaps")
    hist = {}
    for g, a, b in gaps:
        key = (a.split("(")[0][:30], b.split("(")[0][:30])
        hist.setdefault(key, [0, 0.0])
        hist[key][0] += 1
        hist[key][1] += g
    for key, (n, t) in sorted(hist.items(), key=lambda kv: -kv[1][1])[:15]:
        print(f"{t/1e3:8.2f} ms {n:5d}  {key[0]:32s} -> {key[1]}")


if __name__ == "__main__":
    main()
