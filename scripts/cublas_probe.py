import torch
for (m,n,k) in ((2048,2048,2048),(2048,8192,2048),(50304,2048,2048)):
    A=torch.randn(m,k,device='cuda').bfloat16(); B=torch.randn(k,n,device='cuda').bfloat16()
    for _ in range(3): C=A@B
    torch.cuda.synchronize()
