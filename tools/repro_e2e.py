import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2603_14002_b200 import DeviceNgramScorer, PROFILES, decode_batch_raw, synth
from paper_2603_14002_b200._native import pinned_empty
from paper_2603_14002_b200.decoder import device_model, run_search

w = synth.toy_world(n_words=2000, seed=7)
cfg = PROFILES["b2t25"].replace(beam_size=64)
B, T = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 200
raws = synth.make_logits(B, T, 41, base_seed=1000)
frames = np.full(B, T, dtype=np.int32)
sc = DeviceNgramScorer(w.model, cfg.ngram_weight / cfg.llm_weight)
dm = device_model(w.table, w.model)
batch = dm.batch(cfg, B, T)
x_dev = torch.from_numpy(raws).cuda()
batch.load_logits(None, frames, on_device_ptr=x_dev.data_ptr())
run_search(batch, cfg, sc, w.model, True); batch.sync(); print("steps ok")
r = decode_batch_raw((raws[:2], frames[:2]), cfg, w.table, w.model, sc, final_llm_only=True); print("parity call ok")
host_in = pinned_empty(raws.shape, np.float32); host_in[...] = raws
r = decode_batch_raw((host_in, frames), cfg, w.table, w.model, sc, final_llm_only=True); print("pinned call ok", r[0].text[:30])
r = decode_batch_raw((raws, frames), cfg, w.table, w.model, sc, final_llm_only=True); print("pageable call ok", r[0].text[:30])
