"""Config-3 forward rows: how many share a parent slot (sibling groups), and chain depths --
the reuse a parent-grouped chain attention would get.  GPU aid."""
import sys
from collections import Counter
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    from paper_2603_14002_b200 import LlamaScorer
    from paper_2603_14002_b200 import llm as LL
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
    stats = []
    orig = LL.DeviceLlmSession._forward_rows

    def hook(self, wave, row0, n, ws=None):
        r = orig(self, wave, row0, n, ws)
        w = self._ws
        pos = w["pos"][:n].cpu().numpy()
        ch = w["chain"][:n].cpu().numpy()
        par = np.where(pos > 0, ch[np.arange(n), np.maximum(pos - 1, 0)], -1)
        c = Counter(par.tolist())
        sizes = np.array(list(c.values()))
        tiles4 = int(np.sum((sizes + 3) // 4))
        stats.append((n, len(c), tiles4, float(pos.mean()), int(pos.max())))
        return r

    LL.DeviceLlmSession._forward_rows = hook
    batch.load_logits(None, frames, on_device_ptr=x.data_ptr())
    run_search(batch, cfg, sc, world.model, final_llm_only=False)
    torch.cuda.synchronize()
    rows = sum(s[0] for s in stats)
    groups = sum(s[1] for s in stats)
    tiles = sum(s[2] for s in stats)
    gather = sum(s[0] * (s[3] + 1) for s in stats)
    print(f"events {len(stats)} rows {rows} parent groups {groups} (rows/group {rows/groups:.2f}) "
          f"4-sibling tiles {tiles} (rows/tile {rows/tiles:.2f}); mean chain length "
          f"{gather/rows:.1f}, max depth {max(s[4] for s in stats)}")
    for s in stats[::4]:
        print("  event rows %5d groups %5d tiles %5d mean pos %.1f max pos %d" % s)


if __name__ == "__main__":
    main()
