import torch, statistics
def t(f, n=6):
    ts=[]
    for _ in range(n):
        s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); f(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return statistics.median(ts[1:])
n_el=2097152; n_f=1024
cube=torch.randn((n_el,n_f),dtype=torch.complex64,device="cuda")
out=torch.empty((n_el,4*n_f),dtype=torch.complex64,device="cuda")
ms=t(lambda: out.zero_()); print("write-only zero_ %.2f ms %.0f GB/s"%(ms, out.numel()*8/ms/1e6))
ms=t(lambda: out.fill_(1+1j)); print("write-only fill %.2f ms %.0f GB/s"%(ms, out.numel()*8/ms/1e6))
o4=out.view(n_el,4,n_f)
ms=t(lambda: o4.copy_(cube.unsqueeze(1).expand(n_el,4,n_f))); print("1:4 expand copy %.2f ms %.0f GB/s"%(ms,(out.numel()+cube.numel())*8/ms/1e6))
a=out.view(-1)[:out.numel()//2]; b=out.view(-1)[out.numel()//2:]
ms=t(lambda: b.copy_(a)); print("copy 1:1 %.2f ms %.0f GB/s"%(ms, 2*a.numel()*8/ms/1e6))
ms=t(lambda: a.sum()); print("read-only sum %.2f ms %.0f GB/s"%(ms, a.numel()*8/ms/1e6))
