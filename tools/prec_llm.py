"""Which bf16 roundings of the Llama body dominate the log-prob error?  (GPU experiment)
Per-token |error| of dense_forward variants against the fp32 forward of the same weights."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2603_14002_b200.llm import LlamaWeights, PRESETS, dense_forward

    name = sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b"
    W = LlamaWeights(PRESETS[name], seed=11, device="cuda:0", max_pos=512)
    rng = np.random.default_rng(0)
    B, S = 32, 40
    ids = torch.from_numpy(rng.integers(8, W.cfg.vocab_size, size=(B, S))).cuda()
    ids[:, 0] = 1
    lens = [S] * B
    with torch.no_grad():
        ref, _ = dense_forward(W, ids, lens, False, exact_fp32=True)
        ref = np.array(ref)
        full = ("qkv", "o", "gu", "down", "attn", "lm")
        variants = [(), full] + [tuple(x for x in full if x != drop) for drop in full]
        if len(sys.argv) > 2:
            variants = [tuple(v.split("+")) if v else () for v in sys.argv[2].split(",")]
        for split in variants:
            got, _ = dense_forward(W, ids, lens, False, split=frozenset(split))
            err = np.abs(np.array(got) - ref) / (S - 1)
            tot = np.abs(np.array(got) - ref)
            sgn = np.array(got) - ref
            print(f"split={split!s:45s} per-token mean {err.mean():.2e} | 39-token text err mean "
                  f"{tot.mean():.2e} max {tot.max():.2e} | signed mean {sgn.mean():+.2e} std {sgn.std():.2e}")


if __name__ == "__main__":
    main()
