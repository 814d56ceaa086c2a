import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2603_14002_b200 import DeviceNgramScorer, PROFILES, synth, _native as N
from paper_2603_14002_b200 import decoder as D
w = synth.make_world()
cfg = PROFILES["b2t25"].replace(beam_size=64)
raws = synth.make_logits(256, 500, 41, base_seed=1000)
frames = np.full(256, 500, dtype=np.int32)
sc = DeviceNgramScorer(w.model, cfg.ngram_weight / cfg.llm_weight)
dm = D.device_model(w.table, w.model)
for rep in range(3):
    batch = dm.batch(cfg, 256, 500)
    batch.load_logits(raws, frames)
    D.run_search(batch, cfg, sc, w.model, True); batch.sync()
    lib = N.lib(); T = [time.perf_counter()]
    nbytes, ntot = C.c_int64(), C.c_int64()
    N.check(lib.lb_batch_results_size(batch.h, C.byref(nbytes), C.byref(ntot))); T.append(time.perf_counter())
    n = batch.n
    blob = C.create_string_buffer(max(nbytes.value, 1)); T.append(time.perf_counter())
    boff = np.empty(n, np.int64); blen = np.empty(n, np.int32); bsc = np.empty(n); cnt = np.empty(n, np.int32)
    m = ntot.value; noff = np.empty(m, np.int64); nlen = np.empty(m, np.int32); nsc = np.empty(m)
    N.check(lib.lb_batch_results(batch.h, blob, N.ptr(boff), N.ptr(blen), N.ptr(bsc), N.ptr(cnt), N.ptr(noff), N.ptr(nlen), N.ptr(nsc))); T.append(time.perf_counter())
    raw = blob.raw[: nbytes.value]; T.append(time.perf_counter())
    parts = raw.decode("utf-8").split("\x00"); T.append(time.perf_counter())
    st, _ = batch.status(); T.append(time.perf_counter())
    bsc_l, cnt_l, nsc_l = bsc.tolist(), cnt.tolist(), nsc.tolist()
    out = []; k = j = 0
    for i in range(n):
        c = cnt_l[i]
        out.append((parts[k], bsc_l[i], list(zip(parts[k + 1: k + 1 + c], nsc_l[j: j + c])))); k += c + 1; j += c
    T.append(time.perf_counter())
    print([round((b - a) * 1e3, 2) for a, b in zip(T, T[1:])])
