"""Small decode workloads for compute-sanitizer (memcheck / racecheck / synccheck): the frame
kernel (k=16 and k=64 specialisations, interval + device n-gram fusion), and the device LLM
fusion path (bf16 and bf16x2) on a tiny model."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from oracle import lightbeam_oracle as O  # noqa: E402
from paper_2603_14002_b200 import (PROFILES, DeviceNgramScorer, LlamaScorer, StubScorer,  # noqa: E402
                                   decode_batch, decode_batch_raw, synth)

w = synth.toy_world(n_words=2000, seed=7)
raws = synth.make_logits(3, 60, 41, base_seed=11)
import os  # noqa: E402

for k in (16, 64, 96, 300) + ((900,) if os.environ.get("SAN_WIDE") else ()):
    cfg = PROFILES["b2t25"].replace(beam_size=k, llm_rescore_interval=20)
    ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
    scale = cfg.ngram_weight / cfg.llm_weight
    decode_batch(ds, cfg, w.table, w.model, DeviceNgramScorer(w.model, scale))
    decode_batch(ds, cfg, w.table, w.model, StubScorer(table={}))
    # raw fp32 logits: the K1 prologue (eight lanes per row) feeds the search
    decode_batch_raw(list(raws), cfg, w.table, w.model, DeviceNgramScorer(w.model, scale))
    print("frames ok k", k, flush=True)
cfg = PROFILES["b2t25"].replace(beam_size=16, llm_rescore_interval=20)
ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
for prec in ("bf16", "bf16x2"):
    for graphs in (True, False):  # eager: sibling-tile attention + planning-time tiles
        decode_batch(ds, cfg, w.table, w.model,
                     LlamaScorer("tiny", seed=1, precision=prec, max_slots=4096, graphs=graphs))
        print("llm ok", prec, "graphs" if graphs else "eager", flush=True)
