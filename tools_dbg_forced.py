import sys
sys.path[:0] = ["/root/repo", "/root/repo/tests"]
import numpy as np
import goldens as G
from paper_2603_14002_b200 import StubScorer, decode_batch
from paper_2603_14002_b200.decoder import device_model, run_search
g = G.load("forced20")
vocab, tt, model = G.instance_world(g)
cfg = G.config_of(g["config"])
ds = [np.asarray(inst["D"]) for inst in g["instances"]]
for n in (1, 2, 20):
    got = decode_batch(ds[:n], cfg, tt, model, StubScorer(table={}))
    print(n, [type(r).__name__ if isinstance(r, Exception) else r.text for r in got][:5])
dm = device_model(tt, model)
b = dm.batch(cfg, 20, 5)
for dump in (False, True):
    b.enable_dump(dump)
    arr = np.zeros((20, b.max_frames, 41)); fr = np.array([x.shape[0] for x in ds], dtype=np.int32)
    for i, x in enumerate(ds): arr[i, :x.shape[0]] = x
    b.load_logprobs(arr, fr)
    b.reset(); b.run(0, 1)
    print("dump", dump, b.status()[0][:5], b.beams(0))
