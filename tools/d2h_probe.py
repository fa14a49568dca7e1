import torch, time, numpy as np
torch.cuda.init()
shapes=[((720,1280),torch.float32),((720,1280),torch.uint8),((720,1280),torch.int32),((720,1280),torch.int32),((720,1280,3),torch.uint8),((720,1280),torch.uint8),((720,1280),torch.uint8)]
dev=[torch.zeros(s,dtype=d,device='cuda') for s,d in shapes]
def fresh():
    outs=[]
    for d in dev:
        h=torch.empty(d.shape,dtype=d.dtype,pin_memory=True); h.copy_(d,non_blocking=True); outs.append(h)
    torch.cuda.current_stream().synchronize(); return [h.numpy() for h in outs]
pre=[torch.empty(d.shape,dtype=d.dtype,pin_memory=True) for d in dev]
def reuse():
    for h,d in zip(pre,dev): h.copy_(d,non_blocking=True)
    torch.cuda.current_stream().synchronize(); return [h.numpy() for h in pre]
flat=torch.empty(sum(d.numel()*d.element_size() for d in dev),dtype=torch.uint8,device='cuda')
fh=torch.empty_like(flat,device='cpu').pin_memory()
def one():
    fh.copy_(flat,non_blocking=True); torch.cuda.current_stream().synchronize()
for name,f in [('fresh',fresh),('reuse',reuse),('one_copy',one)]:
    for _ in range(3): out=f()
    t=time.perf_counter()
    for _ in range(20): out=f()
    print(name, (time.perf_counter()-t)/20*1e3, 'ms')
x=torch.empty(32*2**20,dtype=torch.uint8).pin_memory(); y=torch.empty(32*2**20,dtype=torch.uint8,device='cuda')
for _ in range(3): y.copy_(x,non_blocking=True); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): y.copy_(x,non_blocking=True)
torch.cuda.synchronize(); print('h2d GB/s', 10*32*2**20/(time.perf_counter()-t)/1e9)
t=time.perf_counter()
for _ in range(10): x.copy_(y,non_blocking=True)
torch.cuda.synchronize(); print('d2h GB/s', 10*32*2**20/(time.perf_counter()-t)/1e9)
