import torch, sys
sys.path.insert(0,'/root/repo')
from paper_2210_11362_b200 import _lib as L
lib=L.lib()
x=torch.zeros(1024,dtype=torch.float64,device='cuda')
info=torch.zeros(8,dtype=torch.int32,device='cuda')
S=torch.eye(64,dtype=torch.float64,device='cuda'); M=torch.zeros(64,64,dtype=torch.float64,device='cuda'); Z=torch.zeros_like(M)
ws=torch.zeros(lib.trals_spd_fallback_ws_elems(64,64),dtype=torch.float64,device='cuda')
def graph_time(fn, n):
    s=torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g=torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        for _ in range(n): fn()
        g.capture_end()
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(10): g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/10/n*1e3
sp=lambda: int(torch.cuda.current_stream().cuda_stream)
print("torch add_ per launch us:", graph_time(lambda: x.add_(1.0), 100))
print("fallback (no fire) per launch us:", graph_time(lambda: lib.trals_spd_fallback_f64(S.data_ptr(),64,M.data_ptr(),64,Z.data_ptr(),info.data_ptr(),0,2.2e-16,ws.data_ptr(),ws.numel(),sp()), 100))
print("relayout per launch us:", graph_time(lambda: lib.trals_core_relayout_f64(M.data_ptr(),0,8,1,8,Z.data_ptr(),1,sp()), 100))
