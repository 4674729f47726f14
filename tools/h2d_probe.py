import torch, time
T,B,P=500,512,5700
h=torch.empty((T,B,P),dtype=torch.float32,pin_memory=True)
d=torch.empty((50,B,P),dtype=torch.float32,device='cuda')
s=torch.cuda.Stream()
for rep in range(2):
    torch.cuda.synchronize(); a=time.perf_counter()
    with torch.cuda.stream(s):
        for t0 in range(0,T,25):
            d[(t0//25)%2*25:(t0//25)%2*25+25].copy_(h[t0:t0+25], non_blocking=True)
    torch.cuda.synchronize(); b=time.perf_counter()
    print(f"H2D {h.numel()*4/1e9:.2f} GB in {(b-a)*1e3:.1f} ms = {h.numel()*4/(b-a)/1e9:.1f} GB/s")
