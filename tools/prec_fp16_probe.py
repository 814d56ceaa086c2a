import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, torch.nn.functional as F
from paper_2603_14002_b200.llm import LlamaWeights, PRESETS, dense_forward, PUNCT_IDS

def fwd(W, ids, lens, dt, lm_dt):
    cfg=W.cfg; B,S=ids.shape; hd,nh,nkv=cfg.head_dim,cfg.heads,cfg.kv_heads
    def mm(a,w,d): 
        a2=a.reshape(-1,a.shape[-1]); return torch.mm(a2.to(d), w.to(d).t(), out_dtype=torch.float32).view(*a.shape[:-1],-1)
    x=W.emb[ids].float(); cos=W.cos[:S].repeat(1,2)[None,None]; sin=W.sin[:S].repeat(1,2)[None,None]
    def norm(v,w): return (v*torch.rsqrt(v.pow(2).mean(-1,keepdim=True)+cfg.rms_eps)*w)
    def rope(t):
        t1,t2=t[...,:hd//2],t[...,hd//2:]; return (t*cos+torch.cat([-t2,t1],-1)*sin).to(dt)
    for L in W.layers:
        h=norm(x,L["ln1"]); qkv=mm(h,L["wqkv"],dt)
        q=qkv[...,:nh*hd].view(B,S,nh,hd).transpose(1,2); k=qkv[...,nh*hd:(nh+nkv)*hd].view(B,S,nkv,hd).transpose(1,2)
        v=qkv[...,(nh+nkv)*hd:].view(B,S,nkv,hd).transpose(1,2).to(dt)
        q,k=rope(q),rope(k)
        a=F.scaled_dot_product_attention(q,k,v,is_causal=True,enable_gqa=True)
        x=x+mm(a.transpose(1,2).reshape(B,S,nh*hd),L["wo"],dt)
        h=norm(x,L["ln2"]); gu=mm(h,L["wgu"],dt); g,u=gu[...,:cfg.ffn],gu[...,cfg.ffn:]
        x=x+mm(F.silu(g.float())*u.float(),L["wd"],dt)
    hn=norm(x,W.norm); out=[]
    for r in range(B):
        n=lens[r]; logits=mm(hn[r,:n],W.emb,lm_dt); lsm=torch.log_softmax(logits.float(),-1).double()
        out.append(float(lsm[:n-1].gather(1,ids[r,1:n][:,None]).sum()))
    return out

name=sys.argv[1] if len(sys.argv)>1 else "llama-3.2-1b"
W=LlamaWeights(PRESETS[name],seed=11,device="cuda:0",max_pos=512)
rng=np.random.default_rng(0); B,S=32,40
ids=torch.from_numpy(rng.integers(8,W.cfg.vocab_size,size=(B,S))).cuda(); ids[:,0]=1
with torch.no_grad():
    ref,_=dense_forward(W,ids,[S]*B,False,exact_fp32=True); ref=np.array(ref)
    for dt,lm in [(torch.bfloat16,torch.bfloat16),(torch.float16,torch.float16),(torch.float16,torch.bfloat16)]:
        got=np.array(fwd(W,ids,[S]*B,dt,lm)); e=np.abs(got-ref)
        print(dt,lm,"39-token err mean %.2e max %.2e"%(e.mean(),e.max()))
    # weights exactly representable in fp16?
    w=W.layers[0]["wqkv"]; print("w dtype",w.dtype,"fp16 roundtrip exact frac",(w.to(torch.float16).to(w.dtype)==w).float().mean().item(), "absmax", w.abs().max().item())
