import torch,time
x=torch.empty(4608*3072,dtype=torch.bfloat16,pin_memory=True); d=torch.empty_like(x,device='cuda'); y=torch.empty_like(x).pin_memory()
s1,s2=torch.cuda.Stream(),torch.cuda.Stream()
for mode in ['h2d','d2h','both']:
    for rep in range(3):
        torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        d2=torch.empty_like(d)
        e0.record()
        s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
        for i in range(10):
            if mode in('h2d','both'):
                with torch.cuda.stream(s1): d.copy_(x,non_blocking=True)
            if mode in('d2h','both'):
                with torch.cuda.stream(s2): y.copy_(d2,non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1.record(); torch.cuda.synchronize()
        ms=e0.elapsed_time(e1)/10
    print(mode, 'ms per 28.3MB copy', round(ms,3), 'GB/s', round(x.numel()*2/ms/1e6,1))
