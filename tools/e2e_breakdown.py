"""Time the stages of decode_batch_raw on the BASELINE config-2 workload (diagnostic)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2603_14002_b200 import DeviceNgramScorer, PROFILES, synth
from paper_2603_14002_b200 import decoder as D

w = synth.make_world()
cfg = PROFILES["b2t25"].replace(beam_size=64)
raws = synth.make_logits(256, 500, 41, base_seed=1000)
from paper_2603_14002_b200._native import pinned_empty
host = pinned_empty(raws.shape, np.float32)
host[...] = raws
raws = host
frames = np.full(256, 500, dtype=np.int32)
sc = DeviceNgramScorer(w.model, cfg.ngram_weight / cfg.llm_weight)
dm = D.device_model(w.table, w.model)
for rep in range(3):
    t = [time.perf_counter()]
    batch = dm.batch(cfg, 256, 500)
    batch.load_logits(raws, frames); batch.sync(); t.append(time.perf_counter())
    D.run_search(batch, cfg, sc, w.model, True); batch.sync(); t.append(time.perf_counter())
    st, ff = batch.status(); t.append(time.perf_counter())
    res = batch.results(); t.append(time.perf_counter())
    out = D._collect(batch, cfg, True, 0.0); t.append(time.perf_counter())
    t0 = time.perf_counter()
    D.decode_batch_raw((raws, frames), cfg, w.table, w.model, sc, final_llm_only=True)
    t.append(time.perf_counter())
    t[-2] = t0
    names = ["h2d+prologue", "search", "status", "results(gather+assemble+py)", "collect(again)", "decode_batch_raw total"]
    print({n: round((b - a) * 1e3, 2) for n, a, b in zip(names, t, t[1:])})

# split of results(): C side vs Python objects
import ctypes as C
from paper_2603_14002_b200 import _native as N
for rep in range(2):
    batch = dm.batch(cfg, 256, 500)
    batch.load_logits(raws, frames)
    D.run_search(batch, cfg, sc, w.model, True); batch.sync()
    lib = N.lib()
    t0 = time.perf_counter()
    nbytes, ntot = C.c_int64(), C.c_int64()
    N.check(lib.lb_batch_results_size(batch.h, C.byref(nbytes), C.byref(ntot)))
    t1 = time.perf_counter()
    res = batch.results()
    t2 = time.perf_counter()
    print("results_size (gather+D2H+assembly) ms", round((t1 - t0) * 1e3, 2), "full results() ms",
          round((t2 - t1) * 1e3, 2), "nbest entries", ntot.value, "blob bytes", nbytes.value)

# split of _collect: status, results_size (C), binding, DecodeResult loop
for rep in range(3):
    batch = dm.batch(cfg, 256, 500)
    batch.load_logits(raws, frames)
    D.run_search(batch, cfg, sc, w.model, True); batch.sync()
    lib = N.lib()
    t0 = time.perf_counter()
    st, ff = batch.status()
    t1 = time.perf_counter()
    nbytes, ntot = C.c_int64(), C.c_int64()
    N.check(lib.lb_batch_results_size(batch.h, C.byref(nbytes), C.byref(ntot)))
    t2 = time.perf_counter()
    view = N.LbResultsView()
    N.check(lib.lb_batch_results_view(batch.h, C.byref(view)))
    res = N.pyresults().assemble(C.addressof(view))
    t3 = time.perf_counter()
    out = [D.DecodeResult(r[0], r[1], r[2], int(batch.frames[i]), 0.0, 0) for i, r in enumerate(res)]
    t4 = time.perf_counter()
    print("status %.2f results_size %.2f binding %.2f DecodeResult loop %.2f ms" %
          tuple(1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3)))
