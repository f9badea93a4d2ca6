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
A=torch.randn(64,64,dtype=torch.float64,device='cuda'); B=torch.randn(64,64,dtype=torch.float64,device='cuda'); C=torch.zeros(64,64,dtype=torch.float64,device='cuda')
gws=torch.zeros(max(1,lib.trals_gemm_ws_elems(1,64,64,64)),dtype=torch.float64,device='cuda')
cm=L.i64_array([0,1<<40,0,64,1<<40,0,1])
print("gemm 64^3 per launch us:", graph_time(lambda: lib.trals_gemm_f64(A.data_ptr(),0,64,1,1,64,64,64,B.data_ptr(),64,C.data_ptr(),cm,0,gws.data_ptr(),gws.numel(),sp()), 50))
A2=torch.randn(500,100,dtype=torch.float64,device='cuda'); B2=torch.randn(100,100,dtype=torch.float64,device='cuda'); C2=torch.zeros(500,100,dtype=torch.float64,device='cuda')
gws2=torch.zeros(max(1,lib.trals_gemm_ws_elems(1,500,100,100)),dtype=torch.float64,device='cuda')
cm2=L.i64_array([0,1<<40,0,100,1<<40,0,1])
print("gemm 500x100x100 per launch us:", graph_time(lambda: lib.trals_gemm_f64(A2.data_ptr(),0,100,1,1,500,100,100,B2.data_ptr(),100,C2.data_ptr(),cm2,0,gws2.data_ptr(),gws2.numel(),sp()), 50))
print("torch matmul 64^3 per launch us:", graph_time(lambda: torch.matmul(A,B,out=C), 50))
