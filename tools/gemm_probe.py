import torch, time
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
dev='cuda'
shapes = {'qkv': (4096, 3072), 'o': (4096, 2048), 'gu': (4096, 16384), 'down': (16384, 2048), 'head': (2048, 128256)}
for M in (600, 1500, 3000, 13400):
    row = []
    for name,(K,N) in shapes.items():
        a = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
        w = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
        for _ in range(3): torch.mm(a, w.t(), out_dtype=torch.float32)
        torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        n=20
        e0.record()
        for _ in range(n): torch.mm(a, w.t(), out_dtype=torch.float32)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)/n
        tf = 2*M*K*N/ms/1e9
        row.append(f"{name} {ms*1e3:7.1f}us {tf:6.0f}TF")
    print(M, " | ".join(row), flush=True)
