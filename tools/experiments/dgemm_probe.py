import torch, time
for n in (4096, 8192):
    a=torch.randn(n,n,dtype=torch.float64,device='cuda'); b=torch.randn(n,n,dtype=torch.float64,device='cuda')
    for _ in range(2): c=a@b
    torch.cuda.synchronize(); t=time.time()
    for _ in range(5): c=a@b
    torch.cuda.synchronize(); dt=(time.time()-t)/5
    print(n, "fp64 TFLOP/s", 2*n**3/dt/1e12)
# tall-skinny like our trace GEMM: [663552 x 864] x [864 x 528]
a=torch.randn(663552//4, 864, dtype=torch.float64, device='cuda'); b=torch.randn(864, 528, dtype=torch.float64, device='cuda')
for _ in range(2): c=a@b
torch.cuda.synchronize(); t=time.time()
for _ in range(5): c=a@b
torch.cuda.synchronize(); dt=(time.time()-t)/5
print("tall", 2*a.shape[0]*864*528/dt/1e12, "TFLOP/s", dt*1e3*4, "ms for the full C5 trace GEMM (dense)")
