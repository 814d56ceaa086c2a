"""Precision probe (GPU): the device path takes a token's log-prob as h.E[token] (fp32 h) minus
the row's log-sum-exp from the LM-head GEMM.  How much does computing only the LSE GEMM with the
bf16 hi half of h (instead of hi|lo) cost, against the fp32 forward?"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.nn.functional as F

    from paper_2603_14002_b200.llm import LlamaWeights, PRESETS, dense_forward

    name = sys.argv[1] if len(sys.argv) > 1 else "llama-3.2-1b"
    W = LlamaWeights(PRESETS[name], seed=11, device="cuda:0", max_pos=512)
    cfg = W.cfg
    rng = np.random.default_rng(0)
    B, S = 32, 40
    ids = torch.from_numpy(rng.integers(8, cfg.vocab_size, size=(B, S))).cuda()
    ids[:, 0] = 1
    lens = [S] * B
    hd, nh, nkv = cfg.head_dim, cfg.heads, cfg.kv_heads
    with torch.no_grad():
        ref, _ = dense_forward(W, ids, lens, False, exact_fp32=True)
        ref = np.array(ref)

        def mm(a, w):
            a2 = a.reshape(-1, a.shape[-1])
            hi = a2.float().to(torch.bfloat16)
            lo = (a2.float() - hi.float()).to(torch.bfloat16)
            out = torch.mm(hi, w.t(), out_dtype=torch.float32) + torch.mm(lo, w.t(), out_dtype=torch.float32)
            return out.view(*a.shape[:-1], -1)

        x = W.emb[ids].float()
        cos = W.cos[:S].repeat(1, 2)[None, None]
        sin = W.sin[:S].repeat(1, 2)[None, None]

        def norm(v, w):
            return v * torch.rsqrt(v.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * w

        def rope(t):
            t1, t2 = t[..., : hd // 2], t[..., hd // 2:]
            return t * cos + torch.cat([-t2, t1], -1) * sin

        for L in W.layers:
            h = norm(x, L["ln1"])
            qkv = mm(h, L["wqkv"])
            q = qkv[..., : nh * hd].view(B, S, nh, hd).transpose(1, 2)
            k = qkv[..., nh * hd: (nh + nkv) * hd].view(B, S, nkv, hd).transpose(1, 2)
            v = qkv[..., (nh + nkv) * hd:].view(B, S, nkv, hd).transpose(1, 2)
            q, k = rope(q), rope(k)
            a = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
            x = x + mm(a.transpose(1, 2).reshape(B, S, nh * hd), L["wo"])
            h = norm(x, L["ln2"])
            gu = mm(h, L["wgu"])
            g, u = gu[..., : cfg.ffn], gu[..., cfg.ffn:]
            x = x + mm(F.silu(g) * u, L["wd"])
        hn = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * W.norm
        E = W.emb
        for mode in ("hilo", "hi"):
            out = []
            for r in range(B):
                hr = hn[r, : S - 1]
                if mode == "hilo":
                    lse = torch.logsumexp(mm(hr, E), -1)
                else:
                    lse = torch.logsumexp(torch.mm(hr.to(torch.bfloat16), E.t(), out_dtype=torch.float32), -1)
                tok = (hr.float() * E[ids[r, 1:S]].float()).sum(-1)
                out.append(float((tok.double() - lse.double()).sum()))
            err = np.abs(np.array(out) - ref)
            print(f"{name} LSE from {mode}: 39-token err mean {err.mean():.2e} max {err.max():.2e}")


if __name__ == "__main__":
    main()
