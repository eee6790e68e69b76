"""cuBLAS (torch.addmm) on the cfg2 projector shape, for an ncu capture of the
library kernel's configuration (grid, block, shared memory, cluster, pipes)."""
import torch

M, K, N = 43355, 1280, 4096
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
W = (torch.randn(N, K, device="cuda", generator=g) / 36).to(torch.bfloat16)
b = torch.randn(N, device="cuda", generator=g).to(torch.bfloat16)
Y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    torch.addmm(b, X, W.t(), out=Y)
torch.cuda.synchronize()
print("ok")
