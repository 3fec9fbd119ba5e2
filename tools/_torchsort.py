import torch
n=3_000_000
k=torch.randint(0,1<<25,(n,),device='cuda',dtype=torch.int32)
for _ in range(3): torch.sort(k,stable=True)
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): torch.sort(k,stable=True)
e.record(); torch.cuda.synchronize()
print("torch.sort stable 3M int32 (keys+indices): %.3f ms"%(s.elapsed_time(e)/20))
