import torch,time
x=torch.empty(1<<30, dtype=torch.uint8).pin_memory(); y=torch.empty(1<<30, dtype=torch.uint8, device='cuda')
for i in range(3):
    torch.cuda.synchronize(); t=time.time(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); print("H2D GB/s", 1/(time.time()-t))
    torch.cuda.synchronize(); t=time.time(); x.copy_(y, non_blocking=True); torch.cuda.synchronize(); print("D2H GB/s", 1/(time.time()-t))
