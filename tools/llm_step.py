"""One BASELINE-config-3 decode step (for ncu captures of the LLM kernels; GPU aid)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch

    from paper_2603_14002_b200 import LlamaScorer
    from paper_2603_14002_b200.decoder import device_model, run_search

    args = bench.parse()
    world, cfg, raws = bench.make_inputs(args, 0)
    cfg = cfg.replace(llm_rescore_interval=args.interval)
    sc = LlamaScorer(args.llm, seed=0, precision=args.precision)
    dm = device_model(world.table, world.model, 0)
    B, T = raws.shape[:2]
    x = torch.from_numpy(raws).cuda()
    batch = dm.batch(cfg, B, T)
    batch.load_logits(None, np.full(B, T, np.int32), on_device_ptr=x.data_ptr())
    run_search(batch, cfg, sc, world.model, final_llm_only=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
