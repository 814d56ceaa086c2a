import cProfile, pstats, sys, io
sys.path.insert(0, "/root/repo")
sys.argv = ["bench.py", "--config", "1"]
import bench, numpy as np, torch
from paper_2603_14002_b200 import LlamaScorer
from paper_2603_14002_b200.decoder import device_model, run_search
args = bench.parse(); bench.apply_preset(args, 1)
world, cfg, raws = bench.make_inputs(args, 0)
cfg = cfg.replace(llm_rescore_interval=args.interval)
sc = LlamaScorer(args.llm, seed=0, precision=args.precision)
dm = device_model(world.table, world.model, 0)
B, T = raws.shape[:2]
x = torch.from_numpy(raws).cuda()
batch = dm.batch(cfg, B, T)
def step():
    batch.load_logits(None, np.full(B, T, np.int32), on_device_ptr=x.data_ptr())
    run_search(batch, cfg, sc, world.model, final_llm_only=False)
    torch.cuda.synchronize()
for _ in range(3): step()
import time
t=time.perf_counter(); 
for _ in range(10): step()
print("ms per step", (time.perf_counter()-t)/10*1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(5): step()
pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18); print(s.getvalue()[:4000])
