"""Where the config-2 streaming e2e step goes (diagnostic): decode_stream_raw's loop re-stated
with host timers per stage and CUDA events on each pipeline batch's stream."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2603_14002_b200 import DeviceNgramScorer, PROFILES, synth
from paper_2603_14002_b200 import decoder as D
from paper_2603_14002_b200._native import pinned_empty

w = synth.make_world()
cfg = PROFILES["b2t25"].replace(beam_size=64)
raws = synth.make_logits(256, 500, 41, base_seed=1000)
host = pinned_empty(raws.shape, np.float32)
host[...] = raws
frames = np.full(256, 500, dtype=np.int32)
sc = DeviceNgramScorer(w.model, cfg.ngram_weight / cfg.llm_weight)
dm = D.device_model(w.table, w.model)
cfg = D.coerce_config(cfg)


def run(n, verbose):
    pending = []
    slot = 0
    host_t = {"load": 0.0, "launch": 0.0, "status": 0.0, "results": 0.0, "items": 0.0}
    evs = []
    t_all = time.perf_counter()
    def collect(item):
        b, ev0, ev1 = item
        t = time.perf_counter(); st, ff = b.status(); host_t["status"] += time.perf_counter() - t
        t = time.perf_counter(); res = b.results(); host_t["results"] += time.perf_counter() - t
        t = time.perf_counter(); D._collect_items(b, cfg, True, 0.0, st, ff, res)
        host_t["items"] += time.perf_counter() - t
        evs.append((ev0, ev1))
    for i in range(n):
        b = dm.pipeline_batch(cfg, slot, 256, 500)
        s = torch.cuda.ExternalStream(b.stream_ptr)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        t = time.perf_counter(); b.load_logits(host, frames); host_t["load"] += time.perf_counter() - t
        if D._SERIAL_SEARCH and pending:
            b.after(pending[-1][0])
        t = time.perf_counter()
        for _ in D._search_steps(b, cfg, sc, w.model, True):
            pass
        host_t["launch"] += time.perf_counter() - t
        ev1.record(s)
        pending.append((b, ev0, ev1))
        slot ^= 1
        if len(pending) == 2:
            collect(pending.pop(0))
    while pending:
        collect(pending.pop(0))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t_all) / n
    if verbose:
        dev = [a.elapsed_time(b) for a, b in evs]
        gaps = [evs[i][0].elapsed_time(evs[i + 1][0]) for i in range(len(evs) - 1)]
        print("wall ms/step %.3f  frames/s %.3gM" % (wall * 1e3, 128000 / wall / 1e6))
        print("host ms/step", {k: round(v * 1e3 / n, 3) for k, v in host_t.items()})
        print("device ms per batch (ev0->ev1, incl. waiting for SM slots):",
              [round(x, 2) for x in dev])
        print("batch start-to-start ms:", [round(x, 2) for x in gaps])


run(4, False)
for _ in range(2):
    run(20, True)
