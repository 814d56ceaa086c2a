"""Is the config-3 LLM step CPU-bound?  Per fusion event: host time spent issuing the forward
(no syncs inside) vs the device time of the event (CUDA events)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    from paper_2603_14002_b200 import LlamaScorer
    from paper_2603_14002_b200 import llm as LLM
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
    host = {"fwd": 0.0, "plan": 0.0, "finish": 0.0}
    orig_fwd = LLM.DeviceLlmSession._forward_rows

    def timed_fwd(self, *a):
        t0 = time.perf_counter()
        orig_fwd(self, *a)
        host["fwd"] += time.perf_counter() - t0

    LLM.DeviceLlmSession._forward_rows = timed_fwd

    def step():
        batch.load_logits(None, frames, on_device_ptr=x.data_ptr())
        run_search(batch, cfg, sc, world.model, final_llm_only=False)

    step()
    torch.cuda.synchronize()
    host["fwd"] = 0.0
    sess = batch._llm_session
    sess.enable_timing(True)
    t0 = time.perf_counter()
    step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"step wall {wall*1e3:.1f} ms, device LLM {sess.llm_ms():.1f} ms, host issuing forwards "
          f"{host['fwd']*1e3:.1f} ms")


if __name__ == "__main__":
    main()
