"""GPT-2 LM-head cost on B200: bf16 GEMM with N = 50257 vs N padded to 50304, with and without the loss (development aid)."""
import torch, torch.nn.functional as F, time
dev = torch.device("cuda")
B, T, H = 8, 1024, 1024
x = torch.randn(B * T, H, device=dev, requires_grad=True)
tgt = torch.randint(0, 50257, (B * T,), device=dev)
def timeit(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / n
for V in (50257, 50304):
    W = torch.nn.Linear(H, V, bias=False).to(dev)
    def gemm():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            return W(x)
    def fwd_loss():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = W(x)
            if V != 50257: logits = logits[:, :50257]
            return F.cross_entropy(logits.float(), tgt)
    def fwd_loss_nofloat():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            logits = W(x)
            if V != 50257: logits = logits[:, :50257]
            return F.cross_entropy(logits, tgt)
    def fwd_bwd():
        l = fwd_loss(); l.backward()
    print(V, "gemm fwd %.2f ms" % timeit(gemm), "fwd+loss %.2f" % timeit(fwd_loss), "fwd+loss(no .float) %.2f" % timeit(fwd_loss_nofloat), "fwd+bwd %.2f" % timeit(fwd_bwd, 5))
