import torch
from torch.profiler import profile, ProfilerActivity
bf=torch.bfloat16
for (M,N,K) in [(8192,11008,4096),(8192,4096,11008),(8192,4096,4096)]:
    A=torch.randn(M,K,device='cuda',dtype=bf); B=torch.randn(N,K,device='cuda',dtype=bf)
    D=torch.empty(M,N,device='cuda',dtype=bf)
    for _ in range(3): torch.matmul(A,B.t(),out=D)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        torch.matmul(A,B.t(),out=D); torch.cuda.synchronize()
    for e in p.events():
        if e.device_type.name=='CUDA': print(M,N,K,e.name[:200])
