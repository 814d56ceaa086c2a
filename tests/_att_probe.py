"""Subprocess helper for test_llm.py::test_sibling_tile_attention_matches_per_row: decode a small
batch with the eager device LLM path and print the per-text scores and the session stats as
JSON (LB_ATT_GROUP is read once per process, so each mode runs in its own process)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from oracle import lightbeam_oracle as O  # noqa: E402
from paper_2603_14002_b200 import PROFILES, LlamaScorer, decode_batch, synth  # noqa: E402
from paper_2603_14002_b200.decoder import device_model  # noqa: E402

w = synth.toy_world(n_words=2000, seed=7)
cfg = PROFILES["b2t25"].replace(beam_size=16, llm_rescore_interval=20)
raws = synth.make_logits(4, 120, 41, base_seed=29)
ds = [O.log_softmax_scaled(r, cfg.acoustic_scale) for r in raws]
sc = LlamaScorer("tiny", seed=3, graphs=False)
got = decode_batch(ds, cfg, w.table, w.model, sc)
sess = device_model(w.table, w.model).batch(cfg, len(ds), 120)._llm_session
ex = sess.export()
memo = {0: ()}


def path(s):
    if s not in memo:
        memo[s] = path(int(ex["parent"][s])) + (int(ex["token"][s]),)
    return memo[s]


scores = {" ".join(map(str, path(s))): float(ex["cum"][s])
          for s in range(1, len(ex["parent"])) if ex["parent"][s] >= 0 and ex["state"][s] & 2}
print(json.dumps({"scores": scores, "stats": sess.stats(),
                  "texts": [g.text for g in got]}))
