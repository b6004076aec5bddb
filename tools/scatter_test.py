import torch, time
V=1<<24
out=torch.empty(V,dtype=torch.int32,device='cuda')
flush=torch.empty(1<<26,dtype=torch.int32,device='cuda')
g=torch.Generator(device='cuda'); g.manual_seed(0)
for n in (1<<20, 7_500_000, 1<<24):
    idx=torch.randperm(V,device='cuda',generator=g)[:n].to(torch.int64)
    idx_sorted=idx.sort().values
    val=torch.full((n,),3,dtype=torch.int32,device='cuda')
    for name,ix in (('random',idx),('sorted',idx_sorted)):
        ts=[]
        for r in range(5):
            flush.fill_(r); torch.cuda.synchronize()
            e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
            e0.record(); out.index_put_((ix,),val); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(name,n,'ms',min(ts), 'index bytes MB', n*12/1e6, 'GB/s eff (idx+val)', n*12/min(ts)/1e6)
ts=[]
for r in range(5):
    flush.fill_(r); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); out.fill_(-1); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print('fill 64MB ms',min(ts))
