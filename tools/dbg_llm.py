"""Step-by-step parity bisection of the device LLM fusion against the oracle (GPU debug aid)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import lightbeam_oracle as O  # noqa: E402
from paper_2603_14002_b200 import PROFILES, LlamaScorer, ReplayScorer, synth  # noqa: E402
from paper_2603_14002_b200.decoder import device_model  # noqa: E402


def main():
    w = synth.toy_world(n_words=2000, seed=7)
    cfg = PROFILES["b2t25"].replace(beam_size=16, llm_rescore_interval=20)
    raws = synth.make_logits(1, 140, 41, base_seed=77)
    d = O.log_softmax_scaled(raws[0], cfg.acoustic_scale)
    sc = LlamaScorer("tiny", seed=3)
    dm = device_model(w.table, w.model)
    b = dm.batch(cfg, 1, 140)
    b.load_logprobs(d[None], np.array([140], np.int32))
    b.reset()
    sess = sc.session(b)
    sess.reset()
    srch = O.OracleSearch(cfg, w.table, w.model, None)
    t = 0
    for e in list(range(20, 140, 20)):
        b.run(t, e + 1)
        for tt in range(t, e + 1):
            srch.frame(d[tt], tt)
        t = e + 1
        et, eb, wo, words, tot, pun = b.gather()
        dev_texts = [" ".join(dm.surfaces[x] for x in words[wo[i]: wo[i + 1]]) for i in range(len(et))]
        ora = srch.entries_dump()
        ora_texts = [x[0] for ents in ora for x in ents]
        print(f"event {e}: entries dev {len(dev_texts)} oracle {len(ora_texts)} same {dev_texts == ora_texts}")
        sess.event(False, e)
        tab = sess.replay_table()
        srch.scorer = ReplayScorer(tab)
        missing = [tx for tx in set(ora_texts) if tx and _missing(tab, tx)]
        print("  missing texts in device table:", len(missing), missing[:3])
        if missing:
            tx = missing[0]
            ids = sc.tokenizer.encode(tx)
            print("  tokens", ids, "root children sample", [k for k in tab.child if k[0] == 0][:5])
            print("  stats", sess.stats(), "slots", len(tab.ex["parent"]))
            ex = tab.ex
            for tx in missing[:4]:
                ids = sc.tokenizer.encode(tx)
                cur, path = 0, []
                for tkn in ids[1:]:
                    nxt = tab.child.get((cur, tkn))
                    if nxt is None:
                        path.append(("MISSING", tkn))
                        break
                    cur = nxt
                    path.append((cur, int(ex["state"][cur]), int(ex["depth"][cur])))
                print("   ", tx, path)
            for sl in range(len(ex["parent"])):
                print("    slot", sl, "parent", ex["parent"][sl], "tok", ex["token"][sl], "depth", ex["depth"][sl], "state", ex["state"][sl], "cum", ex["cum"][sl])
            return
        srch.rescore(final=False)
        et, eb, wo, words, tot, pun = b.gather()
        ora = srch.entries_dump()
        otot = [x[1] for ents in ora for x in ents]
        print("  totals equal:", list(tot) == otot, "beam scores equal:",
              [s for s in b.beams(0)][:2] and np.array_equal(np.array([x[4] for x in b.beams(0)]), srch.score))
        if list(tot) != otot:
            for i in range(min(len(tot), len(otot))):
                if tot[i] != otot[i]:
                    print("   first diff", i, dev_texts[i] if i < len(dev_texts) else None, tot[i], otot[i])
                    break
            return


def _missing(tab, tx):
    try:
        tab.score(tx)
        return False
    except KeyError:
        return True


if __name__ == "__main__":
    main()
