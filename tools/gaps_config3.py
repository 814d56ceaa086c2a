"""GPU idle gaps inside one BASELINE-config-3 step (torch.profiler kernel timestamps): where the
step's wall time that is not kernel time goes -- GPU aid."""
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
    ks = sorted([(e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                 if e.device_type.name == "CUDA" and "Memcpy" not in e.name
                 and "Memset" not in e.name], key=lambda t: t[0])
    busy = sum(b - a for a, b, _ in ks)
    span = ks[-1][1] - ks[0][0]
    gaps = []
    for (a0, b0, n0), (a1, b1, n1) in zip(ks, ks[1:]):
        g = a1 - max(b0, a0)
        if g > 0:
            gaps.append((g, n0[:40], n1[:40]))
    gaps.sort(reverse=True)
    print("kernels", len(ks), "span ms %.2f busy ms %.2f idle ms %.2f" % (span / 1e3, busy / 1e3,
                                                                        (span - busy) / 1e3))
    by = {}
    for g, n0, n1 in gaps:
        k = (n0, n1)
        c = by.setdefault(k, [0, 0.0])
        c[0] += 1
        c[1] += g
    print("gap buckets (before -> after kernel): count, total ms")
    for k, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"{t / 1e3:8.2f} ms {c:5d}  {k[0]} -> {k[1]}")
    hist = np.array([g for g, _, _ in gaps])
    for lo, hi in ((0, 5), (5, 20), (20, 100), (100, 1000), (1000, 1e9)):
        m = (hist >= lo) & (hist < hi)
        print(f"gaps {lo}-{hi} us: {m.sum()} totalling {hist[m].sum() / 1e3:.2f} ms")


if __name__ == "__main__":
    main()
